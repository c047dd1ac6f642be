set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"
tail -3 gpurun_out/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -n 2 gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cut -c1-400 gpurun_out/bench_ref.json
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], d['e2e']['value'], r['frac'], r['per_launch_roofline']['frac'], d['compute_under_transfer_pct'], d['overlap_pct'], d['clocks'], d['gpu_launches'])"
