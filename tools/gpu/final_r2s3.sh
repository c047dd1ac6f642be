set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"
tail -4 gpurun_out/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"; tail -n 2 gpurun_out/bench_r50.err
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err; echo "bench r18 rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1300 --csv \
  --log-file gpurun_out/launches_bench_r50.csv python bench.py --steps 1 --warmup 0 --no-incore > gpurun_out/ncu_bench_r50.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_r50.csv > gpurun_out/launches_bench_r50.txt; head -30 gpurun_out/launches_bench_r50.txt
python tools/ncu_traffic.py gpurun_out/launches_bench_r50.csv gpurun_out/conv_traffic_r50.json
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 1100 --csv \
  --log-file gpurun_out/ncu_layers_r50.csv python tools/profile_step.py --config r50 --batch 256 --incore > gpurun_out/ncu_layers_r50.log 2>&1; echo "ncu layers rc=$?"
python tools/ncu_layer_table.py gpurun_out/ncu_layers_r50.csv > gpurun_out/ncu_layers_r50.md 2>&1; head -12 gpurun_out/ncu_layers_r50.md
for spec in 'conv_tma_kernel<\(int\)1, \(int\)128, \(int\)0, \(int\)1, \(int\)1, \(bool\)1|2|dgrad_acc' 'conv_tma_kernel<\(int\)1, \(int\)256|5|dgrad_pair' 'conv_tma_kernel<\(int\)0, \(int\)128, \(int\)0, \(int\)1|4|fprop_1x1'; do
  IFS='|' read -r name skip tag <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none \
      -k "regex:$name" --launch-skip "$skip" -c 1 -o "gpurun_out/ncu_r50_$tag" \
      python tools/profile_step.py --config r50 --batch 256 --incore > "gpurun_out/ncu_r50_$tag.log" 2>&1; echo "$tag rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:bn_relu_pool_rows" -c 1 -o gpurun_out/ncu_pool_fwd \
    python tools/pool_bench.py --batch 256 --reps 1 --kinds fwd > gpurun_out/ncu_pool_fwd.log 2>&1; echo "pool rc=$?"
python tools/ncu_metrics.py gpurun_out/ncu_r50_*.ncu-rep gpurun_out/ncu_pool_fwd.ncu-rep > gpurun_out/ncu_r50_summary.txt 2>&1; head -60 gpurun_out/ncu_r50_summary.txt
