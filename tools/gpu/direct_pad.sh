set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_conv.py tests/test_gpu_gan.py tests/test_gpu_densenet.py tests/test_gpu_conv_persistent.py -q -m gpu -p no:cacheprovider 2>&1 | tail -5
timeout 600 python tools/profile_step.py --config biggan --batch 32 --incore 2>&1 | head -3
timeout 1200 python bench.py --config biggan --steps 5 --warmup 3 > gpurun_out/bench_biggan.json 2> gpurun_out/bench_biggan.err; echo "bench biggan rc=$?"; tail -n 1 gpurun_out/bench_biggan.err
timeout 1200 python bench.py --config densenet --steps 5 --warmup 3 > gpurun_out/bench_densenet.json 2> gpurun_out/bench_densenet.err; echo "bench densenet rc=$?"; tail -n 1 gpurun_out/bench_densenet.err
python -c "
import json
for c in ['biggan','densenet']:
    d=json.load(open(f'gpurun_out/bench_{c}.json')); r=d['roofline']; print(c, d['value'], d['ms_per_step'], d['compute_busy_ms'], d['in_core_samples_per_s'], r['kernel'], r['frac'], (r.get('per_launch_roofline') or {}).get('frac'))"
