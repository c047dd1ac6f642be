set -x
mkdir -p gpurun_out
for c in deeplab pix2pix unet; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; tail -n 1 gpurun_out/bench_$c.err
done
python -c "
import json
for c in ['deeplab','pix2pix','unet']:
    d=json.load(open(f'gpurun_out/bench_{c}.json')); r=d['roofline']; print(c, d['value'], d['ms_per_step'], d['compute_busy_ms'], d['in_core_samples_per_s'], r['kernel'], r['frac'], (r.get('per_launch_roofline') or {}).get('frac'), d['link_roofline']['frac_phase_separated'])"
