mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_p_kernel --launch-count 2 -o gpurun_out/attn_p_full python tools/attn_probe.py --n 4 --reps 1 > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/ncu_attn.log
