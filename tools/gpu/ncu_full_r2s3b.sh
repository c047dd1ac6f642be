set -x
mkdir -p gpurun_out
for spec in 'conv_tma_kernel<\(int\)1, \(int\)128, \(int\)0, \(int\)1, \(int\)1, \(bool\)1>|2|dgrad_acc' 'conv_tma_kernel<\(int\)1, \(int\)256, \(int\)0, \(int\)1, \(int\)2, \(bool\)0>|5|dgrad_pair' 'conv_tma_kernel<\(int\)0, \(int\)128, \(int\)0, \(int\)1, \(int\)1, \(bool\)0>|4|fprop_1x1' 'conv_tma_kernel<\(int\)0, \(int\)64, \(int\)0, \(int\)2, \(int\)2, \(bool\)0>|0|fprop_64' 'conv_tma_kernel<\(int\)1, \(int\)64, \(int\)0, \(int\)2, \(int\)2, \(bool\)0>|0|dgrad_64'; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$name" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_r50_$tag" \
      python tools/profile_step.py --config r50 --batch 256 --incore > "gpurun_out/ncu_r50_$tag.log" 2>&1; echo "$tag rc=$?"; tail -1 "gpurun_out/ncu_r50_$tag.log"
done
python tools/ncu_metrics.py gpurun_out/ncu_r50_*.ncu-rep > gpurun_out/ncu_r2s3_conv_summary.txt 2>&1; cat gpurun_out/ncu_r2s3_conv_summary.txt | head -120
