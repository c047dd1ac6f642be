# bench lines of every config family + Fig.4/5-shaped sweeps of the F3 networks
set -x
for c in deeplab pix2pix densenet unet r1001 biggan; do
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  tail -n 2 gpurun_out/bench_$c.err
done
timeout 1800 python tools/table1.py --net deeplab --phys-gib 8 --chunk-mib 2 --steps 2 --ratios 0.5,1,1.5,2,4,5.3 > gpurun_out/table1_deeplab.jsonl 2> gpurun_out/table1_deeplab.err; echo "t1 deeplab rc=$?"
timeout 1800 python tools/table1.py --net pix2pix --phys-gib 8 --chunk-mib 2 --steps 2 --ratios 0.5,1,1.5,2,4 > gpurun_out/table1_pix2pix.jsonl 2> gpurun_out/table1_pix2pix.err; echo "t1 pix2pix rc=$?"
tail -n 3 gpurun_out/table1_*.err
