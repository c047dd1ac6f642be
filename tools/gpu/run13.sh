set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gan.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python tools/profile_step.py --config biggan --incore > gpurun_out/biggan_profile.txt 2>&1; head -40 gpurun_out/biggan_profile.txt
timeout 900 python bench.py --config biggan > gpurun_out/bench_biggan.json 2> gpurun_out/bench_biggan.err; tail -c 1500 gpurun_out/bench_biggan.json; tail -3 gpurun_out/bench_biggan.err
