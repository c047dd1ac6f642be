set -x
mkdir -p gpurun_out
python -m paper_2010_14109_b200.build > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_f3.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python tools/profile_step.py --config pix2pix --batch 1 --incore > gpurun_out/p2p_profile.txt 2>&1; head -30 gpurun_out/p2p_profile.txt
timeout 900 python bench.py --config pix2pix > gpurun_out/bench_pix2pix.json 2> gpurun_out/bench_pix2pix.err; tail -c 3000 gpurun_out/bench_pix2pix.json
timeout 900 python bench.py --config deeplab > gpurun_out/bench_deeplab.json 2> gpurun_out/bench_deeplab.err; tail -c 3000 gpurun_out/bench_deeplab.json
