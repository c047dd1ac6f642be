set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gan.py tests/test_gpu_dense.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/profile_step.py --config biggan --batch 32 --incore 2>&1 | head -4
timeout 1200 python bench.py --config biggan --steps 5 --warmup 3 > gpurun_out/bench_biggan.json 2> gpurun_out/bench_biggan.err; echo "bench biggan rc=$?"; tail -n 1 gpurun_out/bench_biggan.err
python -c "
import json
d=json.load(open('gpurun_out/bench_biggan.json')); r=d['roofline']; print(d['value'], d['ms_per_step'], d['compute_busy_ms'], d['in_core_samples_per_s'], r['kernel'], r['achieved'], r['frac'])"
