set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv_persistent.py tests/test_gpu_conv.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
for side in new old; do
  if [ $side = old ]; then cd .ab_old; fi
  timeout 300 python tools/pool_bench.py --batch 256 2>&1 | sed "s/^/$side /"
  timeout 600 python tools/conv_bench.py --shapes r50_1x1_256_64,r50_1x1_1024_256,r50_1x1_64_256 --passes dgrad_acc,dgrad,fprop 2>&1 | sed "s/^/$side /"
  cd $GRAFT_REPO_ROOT
done
