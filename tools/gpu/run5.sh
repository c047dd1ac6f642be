# F3 GPU tests + R18 bench line (span-based roofline)
set -x
python -m pytest tests/test_gpu_f3.py -q -m gpu --timeout 1500 -s 2>&1 | tail -30
timeout 900 python bench.py --config r18 --steps 20 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err; echo "bench r18 rc=$?"
tail -n 3 gpurun_out/bench_r18.err
