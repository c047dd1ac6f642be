set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:conv_tma_kernel<\(int\)0, \(int\)64, \(int\)0, \(int\)2, \(int\)2, \(bool\)0>' --launch-skip 0 -c 1 -o gpurun_out/ncu_fprop64 \
    python tools/profile_step.py --config r50 --batch 256 --incore > gpurun_out/ncu_fprop64.log 2>&1; echo "rc=$?"
ls -la gpurun_out
