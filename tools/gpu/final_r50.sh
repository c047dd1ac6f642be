# The default bench line (R50 at 7.58x b0), its ncu launch list with DRAM bytes, and ncu --set full
# captures of the contraction kernels (ResNet-50 b=256 in-core shapes)
set -x
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
tail -c 600 gpurun_out/bench_r50.json; tail -n 3 gpurun_out/bench_r50.err
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1300 --csv \
  --log-file gpurun_out/launches_bench_r50.csv python bench.py --steps 1 --warmup 0 --no-incore > gpurun_out/ncu_bench_r50.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_r50.csv > gpurun_out/launches_bench_r50.txt; head -25 gpurun_out/launches_bench_r50.txt
python tools/ncu_traffic.py gpurun_out/launches_bench_r50.csv gpurun_out/conv_traffic_r50.json
for spec in "conv_tma_kernel<1|20|dgrad_a" "conv_tma_kernel<1|60|dgrad_b" "conv_tma_kernel<0|30|fprop" "conv_tma_kernel<2|30|wgrad"; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$name" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_r50_$tag" \
      python tools/profile_step.py --config r50 --batch 256 --incore > "gpurun_out/ncu_r50_$tag.log" 2>&1; echo "$tag rc=$?"
done
python tools/ncu_metrics.py gpurun_out/ncu_r50_*.ncu-rep > gpurun_out/ncu_r50_summary.txt 2>&1; cat gpurun_out/ncu_r50_summary.txt | head -80
