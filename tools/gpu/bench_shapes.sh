set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
tail -3 gpurun_out/bench_r50.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r50.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['kernel'], r['frac'], r['per_launch_roofline'])
for x in r['by_shape']: print(x)"
