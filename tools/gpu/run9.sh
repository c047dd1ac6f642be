set -x
python tools/probe_link_split.py > gpurun_out/link_split.json 2>&1; cat gpurun_out/link_split.json
bash tools/gpu/ncu_r50_full.sh
bash tools/gpu/f3_bench.sh
