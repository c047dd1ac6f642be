# DP two-replica tests, racecheck without CTA pairs, default bench (R50) and R18
set -x
python -m pytest tests/test_gpu_dp.py tests/test_gpu_timeline_audit.py -q -m gpu --timeout 900 2>&1 | tail -15
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/sanitizer
OC_CONV_CG=1 OC_WGRAD_CG=1 timeout 1200 $CS --tool racecheck --print-limit 50 python tools/sanitize_step.py tiny_resnet va > gpurun_out/sanitizer/tiny_resnet_racecheck_cg1.log 2>&1; echo "racecheck cg1 rc=$?"
tail -n 3 gpurun_out/sanitizer/tiny_resnet_racecheck_cg1.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
tail -c 4000 gpurun_out/bench_r50.json; tail -n 5 gpurun_out/bench_r50.err
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err; echo "bench r18 rc=$?"
tail -c 1500 gpurun_out/bench_r18.json; tail -n 5 gpurun_out/bench_r18.err
