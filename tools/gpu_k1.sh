python tools/bench_cache.py C4 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/k1_c4.csv python tools/prof_apply.py --config C4 --iters 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/k1_c4.csv | head -12
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/k1_c4.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
from collections import defaultdict
d=defaultdict(dict)
for r in rows[1:]:
    d[(r[iid],r[ik][:40])][r[im]]=float(r[iv].replace(',',''))
for k,v in list(d.items())[:14]:
    t=v.get('gpu__time_duration.sum',0)/1e3; b=(v.get('dram__bytes_read.sum',0)+v.get('dram__bytes_write.sum',0))
    print(k[1], round(t,1),'us', round(b/1e6,1),'MB', round(b/max(t,1e-9)/1e6,2),'TB/s')
PY
