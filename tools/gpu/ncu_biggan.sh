set -x
mkdir -p gpurun_out
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_biggan.csv python tools/profile_step.py --config biggan --batch 32 --incore > gpurun_out/ncu_biggan.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/ncu_biggan.log
python tools/ncu_summary.py gpurun_out/launches_biggan.csv > gpurun_out/launches_biggan.txt; head -30 gpurun_out/launches_biggan.txt
