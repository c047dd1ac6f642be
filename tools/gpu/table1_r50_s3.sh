set -x
mkdir -p gpurun_out
timeout 3000 python tools/table1.py --net resnet --depth 50 --phys-gib 8 --chunk-mib 2 --steps 2 --ratios 0.34,0.67,1,1.35,2.7,4.9,5.9,6.6,7.58 > gpurun_out/table1_r50.jsonl 2> gpurun_out/table1_r50.err; echo "t1 r50 rc=$?"; tail -n 2 gpurun_out/table1_r50.err
for c in unet r1001 biggan densenet deeplab pix2pix; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; tail -n 1 gpurun_out/bench_$c.err
done
