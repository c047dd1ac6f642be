# round-2 GPU pass: audits, sanitizer on the tiny ResNet, the default bench (R50) and the R18 line
set -x
python -m pytest tests/test_gpu_timeline_audit.py tests/test_gpu_conv_persistent.py -q -m gpu --timeout 900 2>&1 | tail -8
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 python tools/sanitize_step.py tiny_resnet va > gpurun_out/sanitizer/tiny_resnet_${tool}.log 2>&1; echo "tiny_resnet $tool rc=$?"
  tail -2 gpurun_out/sanitizer/tiny_resnet_${tool}.log
done
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
tail -c 3000 gpurun_out/bench_r50.json; tail -5 gpurun_out/bench_r50.err
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err; echo "bench r18 rc=$?"
tail -c 1500 gpurun_out/bench_r18.json; tail -5 gpurun_out/bench_r18.err
