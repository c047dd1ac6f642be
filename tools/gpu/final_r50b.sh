set -x
python -m pytest tests/test_gpu_conv_persistent.py tests/test_gpu_conv.py -q -m gpu --timeout 900 -x 2>&1 | tail -3
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"
tail -n 3 gpurun_out/bench_r50.err
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1300 --csv \
  --log-file gpurun_out/launches_bench_r50.csv python bench.py --steps 1 --warmup 0 --no-incore > gpurun_out/ncu_bench_r50.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_r50.csv > gpurun_out/launches_bench_r50.txt; head -25 gpurun_out/launches_bench_r50.txt
python tools/ncu_traffic.py gpurun_out/launches_bench_r50.csv gpurun_out/conv_traffic_r50.json
for spec in 'conv_tma_kernel<\(int\)1, \(int\)128, \(int\)0, \(int\)1, \(int\)1, \(bool\)1|2|dgrad_acc' 'conv_tma_kernel<\(int\)1, \(int\)256|5|dgrad_pair' 'conv_tma_kernel<\(int\)0, \(int\)256|10|fprop_pair' 'conv_tma_kernel<\(int\)0, \(int\)128, \(int\)0, \(int\)1|4|fprop_1x1' 'conv_tma_kernel<\(int\)2, \(int\)256|10|wgrad_pair'; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none \
      -k "regex:$name" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_r50_$tag" \
      python tools/profile_step.py --config r50 --batch 256 --incore > "gpurun_out/ncu_r50_$tag.log" 2>&1; echo "$tag rc=$?"
done
python tools/ncu_metrics.py gpurun_out/ncu_r50_*.ncu-rep > gpurun_out/ncu_r50_summary.txt 2>&1; head -100 gpurun_out/ncu_r50_summary.txt
