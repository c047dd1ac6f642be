set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dense.py tests/test_gpu_attention.py tests/test_gpu_gan.py tests/test_gpu_resnet.py tests/test_gpu_layerwise.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
