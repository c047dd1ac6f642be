set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv_persistent.py -q -m gpu -x -p no:cacheprovider -k "pool" 2>&1 | tail -3
timeout 300 python tools/pool_bench.py --batch 256 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_r50.json'))
print(d['value'], d['ms_per_step'], d['compute_busy_ms'], d['roofline']['frac'], d['roofline']['kernel'], d['in_core_samples_per_s'], d['link_roofline']['frac_phase_separated'])"
