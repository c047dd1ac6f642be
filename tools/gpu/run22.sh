set -x
mkdir -p gpurun_out
timeout 1800 python tools/table1.py --net pix2pix --phys-gib 8 --chunk-mib 2 --steps 2 --ratios 0.5,1,1.5,2,4 > gpurun_out/table1_pix2pix.jsonl 2> gpurun_out/table1_pix2pix.err; echo "t1 pix2pix rc=$?"
timeout 1800 python tools/table1.py --net deeplab --phys-gib 8 --chunk-mib 2 --steps 2 --ratios 0.5,1,1.5,2,4,5.3 > gpurun_out/table1_deeplab.jsonl 2> gpurun_out/table1_deeplab.err; echo "t1 deeplab rc=$?"
tail -n 3 gpurun_out/table1_*.err
