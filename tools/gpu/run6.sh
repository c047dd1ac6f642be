# accumulate epilogue (TMA load of the old box): conv parity suites, F3, U-Net (fprop accumulate), R50 spans
set -x
python -m pytest tests/test_gpu_conv.py tests/test_gpu_conv_persistent.py tests/test_gpu_f3.py tests/test_gpu_unet.py tests/test_gpu_layerwise.py -q -m gpu --timeout 1500 -x -s 2>&1 | grep -v "^{\"fn" | tail -25
timeout 600 python tools/instep_vs_isolated.py --config r50 --batch 256 --frac 0.25 --rows > gpurun_out/instep_r50.jsonl 2> gpurun_out/instep_r50.err; echo "instep r50 rc=$?"; head -c 1500 gpurun_out/instep_r50.jsonl
