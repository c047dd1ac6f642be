set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_conv_persistent.py tests/test_gpu_layerwise.py tests/test_gpu_resnet.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -5
for side in new old; do
  if [ $side = old ]; then cd .ab_old; fi
  timeout 300 python tools/pool_bench.py --batch 256 2>&1 | sed "s/^/$side /"
  cd $GRAFT_REPO_ROOT
done
