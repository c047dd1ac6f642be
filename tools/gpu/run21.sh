set -x
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "r50 rc=$?"
for c in biggan pix2pix; do
  timeout 1200 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
python - <<'PY'
import json
for c in ("r50","biggan","pix2pix"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
        print(c, d["value"], d["ms_per_step"], d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["link_roofline"]["frac_phase_separated"], json.dumps(d["host_link"]["per_copy"]))
    except Exception as e: print(c, "ERR", e)
PY
