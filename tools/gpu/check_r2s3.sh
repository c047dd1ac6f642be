set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"
tail -15 gpurun_out/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
tail -n 3 gpurun_out/bench_r50.err; cut -c1-600 gpurun_out/bench_r50.json
