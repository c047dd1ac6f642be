set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gan.py -x -q -m gpu 2>&1 | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/attn_ncu.csv python tools/attn_probe.py --n 4 --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/attn_ncu.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; ki,mi,vi,ui=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value'),h.index('Metric Unit')
d=collections.OrderedDict()
for r in rows[hi+1:]:
    d.setdefault(r[0],{'name':r[ki][:50]})[r[mi]]=r[vi]
for k,v in list(d.items())[:12]: print(k, v['name'], v.get('gpu__time_duration.sum'), v.get('dram__bytes_read.sum'), v.get('dram__bytes_write.sum'))
PY
