set -x
mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18_$i.json 2> gpurun_out/bench_r18_$i.err; echo "bench r18 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/bench_r18_$i.json')); r=d['roofline']
print(d['value'], r['kernel'], r['frac'], r['per_launch_roofline']['frac'], [(x['shape'], round(x['ms'],3)) for x in r['by_shape'][:3]])"
done
