set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_conv.py tests/test_gpu_gan.py tests/test_gpu_resnet.py tests/test_gpu_layerwise.py -q -m gpu -p no:cacheprovider 2>&1 | tail -4
timeout 600 python tools/profile_step.py --config biggan --batch 32 --incore 2>&1 | head -2
for c in biggan r1001; do
timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; tail -n 1 gpurun_out/bench_$c.err
done
python -c "
import json
for c in ['biggan','r1001']:
    d=json.load(open(f'gpurun_out/bench_{c}.json')); r=d['roofline']; print(c, d['value'], d['ms_per_step'], d['compute_busy_ms'], d['in_core_samples_per_s'], r['kernel'], r['frac'], (r.get('per_launch_roofline') or {}).get('frac'), d['link_roofline']['frac_phase_separated'])"
