# ncu --set full captures of the ResNet-50 contraction kernels (b=256 in-core shapes)
set -x
for spec in 'conv_tma_kernel<\(int\)1, \(int\)128, \(int\)0, \(int\)1, \(int\)1, \(bool\)1|2|dgrad_acc' 'conv_tma_kernel<\(int\)1, \(int\)256|5|dgrad_pair' 'conv_tma_kernel<\(int\)0, \(int\)256|10|fprop_pair' 'conv_tma_kernel<\(int\)0, \(int\)128, \(int\)0, \(int\)1|4|fprop_1x1' 'conv_tma_kernel<\(int\)2, \(int\)256|10|wgrad_pair'; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$name" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_r50_$tag" \
      python tools/profile_step.py --config r50 --batch 256 --incore > "gpurun_out/ncu_r50_$tag.log" 2>&1; echo "$tag rc=$?"
  tail -n 2 "gpurun_out/ncu_r50_$tag.log"
done
python tools/ncu_metrics.py gpurun_out/ncu_r50_*.ncu-rep > gpurun_out/ncu_r50_summary.txt 2>&1; head -100 gpurun_out/ncu_r50_summary.txt
