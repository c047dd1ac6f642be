set -x
timeout 1500 python bench.py --config pix2pix --steps 5 --warmup 3 > gpurun_out/bench_pix2pix.json 2> gpurun_out/bench_pix2pix.err; echo "bench pix2pix rc=$?"; tail -n 2 gpurun_out/bench_pix2pix.err
timeout 2400 python tools/table1.py --net pix2pix --phys-gib 8 --chunk-mib 2 --steps 2 --ratios 0.5,1,1.5,2,4 > gpurun_out/table1_pix2pix.jsonl 2> gpurun_out/table1_pix2pix.err; echo "t1 pix2pix rc=$?"; tail -n 2 gpurun_out/table1_pix2pix.err
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 1100 --csv \
  --log-file gpurun_out/ncu_layers_r50.csv python tools/profile_step.py --config r50 --batch 256 --incore > gpurun_out/ncu_layers_r50.log 2>&1; echo "ncu layers rc=$?"
python tools/ncu_layer_table.py gpurun_out/ncu_layers_r50.csv > gpurun_out/ncu_layers_r50.md 2>&1; head -40 gpurun_out/ncu_layers_r50.md
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err; echo "bench r18 rc=$?"
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo "bench r50 rc=$?"; tail -n 2 gpurun_out/bench_r50.err
