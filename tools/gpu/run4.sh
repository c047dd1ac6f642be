# full GPU suite + smoke + in-step vs isolated probes + F1 policies with both arrival triggers
set -x
python -m pytest tests -q -m gpu --timeout 1500 -x 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python tools/instep_vs_isolated.py --config r18 --rows > gpurun_out/instep_r18.jsonl 2> gpurun_out/instep_r18.err; echo "instep r18 rc=$?"; head -c 3000 gpurun_out/instep_r18.jsonl; tail -n 3 gpurun_out/instep_r18.err
timeout 600 python tools/instep_vs_isolated.py --config r50 --batch 256 --frac 0.25 --rows > gpurun_out/instep_r50.jsonl 2> gpurun_out/instep_r50.err; echo "instep r50 rc=$?"; head -c 3000 gpurun_out/instep_r50.jsonl; tail -n 3 gpurun_out/instep_r50.err
timeout 900 python tools/sweep.py --fracs 0.3,0.45,0.6 --modes va --wfracs 0,1.0 --distances 1,2,4,8 --pin-below 1048576 --triggers 0,1 > gpurun_out/f1_r18.jsonl 2> gpurun_out/f1_r18.err; echo "f1 rc=$?"; tail -n 3 gpurun_out/f1_r18.err
