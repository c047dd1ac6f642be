set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel --launch-count 8 -o gpurun_out/gemm_tc_full python tools/attn_probe.py --n 4 --reps 1 > gpurun_out/ncu_gemm.log 2>&1
tail -5 gpurun_out/ncu_gemm.log
