set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_conv.py tests/test_gpu_mlp.py tests/test_gpu_densenet.py tests/test_gpu_unet.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3
timeout 1200 python bench.py --config r1001 --steps 5 --warmup 3 > gpurun_out/bench_r1001.json 2> gpurun_out/bench_r1001.err; echo "bench r1001 rc=$?"; tail -n 1 gpurun_out/bench_r1001.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r1001.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], d['compute_busy_ms'], r['frac'], r['per_launch_roofline']['frac'])
for x in r['by_shape'][:8]: print(x)"
