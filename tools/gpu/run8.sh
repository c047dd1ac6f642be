set -x
python -m pytest tests/test_gpu_conv.py tests/test_gpu_conv_persistent.py tests/test_gpu_unet.py tests/test_gpu_f3.py -q -m gpu --timeout 1500 -x 2>&1 | tail -4
timeout 600 python tools/instep_vs_isolated.py --config r50 --batch 256 --frac 0.25 --rows > gpurun_out/instep_r50.jsonl 2> gpurun_out/instep_r50.err; echo "instep r50 rc=$?"; head -c 1200 gpurun_out/instep_r50.jsonl
timeout 600 python tools/instep_vs_isolated.py --config r18 --rows > gpurun_out/instep_r18.jsonl 2> gpurun_out/instep_r18.err; echo "instep r18 rc=$?"; head -c 1200 gpurun_out/instep_r18.jsonl
