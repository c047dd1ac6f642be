set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv_persistent.py tests/test_dp.py tests/test_gpu_layerwise.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/pool_bench.py --batch 256 2>&1
for spec in 'conv_tma_kernel<1, 128, 0, 1, 1, 1>|2|dgrad_acc' 'conv_tma_kernel<1, 256, 0, 1, 2, 0>|5|dgrad_pair' 'conv_tma_kernel<0, 128, 0, 1, 1, 0>|4|fprop_1x1' 'conv_tma_kernel<0, 64, 0, 2, 2, 0>|0|fprop_64'; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$(printf '%s' "$name" | sed 's/[<>]/./g')" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_r50_$tag" \
      python tools/profile_step.py --config r50 --batch 256 --incore > "gpurun_out/ncu_r50_$tag.log" 2>&1; echo "$tag rc=$?"; tail -2 "gpurun_out/ncu_r50_$tag.log"
done
for k in pbn_partial_rows pbn_apply_rows; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$k" -c 1 -o gpurun_out/ncu_pool_$k \
    python tools/pool_bench.py --batch 256 --reps 1 > gpurun_out/ncu_pool_$k.log 2>&1; echo "$k rc=$?"
done
python tools/ncu_metrics.py gpurun_out/ncu_r50_*.ncu-rep gpurun_out/ncu_pool_*.ncu-rep > gpurun_out/ncu_r2s3_summary.txt 2>&1; cat gpurun_out/ncu_r2s3_summary.txt | head -120
