set -x
mkdir -p gpurun_out
timeout 300 python tools/attn_probe.py
timeout 300 python tools/attn_probe.py --dq 12 --dv 48
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/attn_ncu.csv python tools/attn_probe.py --n 2 --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/attn_ncu.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; ki,mi,vi,ui=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value'),h.index('Metric Unit')
for r in rows[hi+1:]:
    print(r[0], r[ki][:60], r[mi], r[vi], r[ui])
PY
