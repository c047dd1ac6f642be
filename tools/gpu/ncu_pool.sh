set -x
mkdir -p gpurun_out
for k in bn_relu_pool_rows pbn_partial_rows pbn_apply_rows; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$k" -c 1 -o gpurun_out/ncu_pool_$k \
    python tools/pool_bench.py --batch 256 --reps 1 > gpurun_out/ncu_pool_$k.log 2>&1; echo "$k rc=$?"
done
