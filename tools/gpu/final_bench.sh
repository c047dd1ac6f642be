set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"; tail -n 1 gpurun_out/bench_r50.err
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err; echo "bench r18 rc=$?"
python -c "
import json
for c in ['r50','r18']:
    d=json.load(open(f'gpurun_out/bench_{c}.json')); r=d['roofline']
    print(c, d['value'], d['ms_per_step'], r['frac'], r['traffic'], r.get('algorithmic_bytes_per_launch'), r['per_launch_roofline']['frac'], d['compute_under_transfer_pct'], d['link_roofline']['frac_phase_separated'], d['host_link']['per_copy']['d2h']['gbs_bytes_weighted'])"
