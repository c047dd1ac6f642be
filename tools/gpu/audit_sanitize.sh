set -x
python -m pytest tests/test_gpu_timeline_audit.py tests/test_gpu_conv_persistent.py -q -m gpu -x --timeout 900 2>&1 | tail -15
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/sanitizer
for w in mlp tiny_resnet; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $tool --print-limit 50 python tools/sanitize_step.py $w va > gpurun_out/sanitizer/${w}_${tool}.log 2>&1; echo "$w $tool rc=$?"
    tail -3 gpurun_out/sanitizer/${w}_${tool}.log
  done
done
