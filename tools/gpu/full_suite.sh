set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"
tail -15 gpurun_out/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
