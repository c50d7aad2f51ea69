mkdir -p gpurun_out/solve_prof
O=gpurun_out/solve_prof
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_solve.csv python tools/solve_launches.py c2 > $O/run.log 2>&1; tail -1 $O/run.log
python - <<'PY'
import csv
from collections import defaultdict
rows=list(csv.reader(open('gpurun_out/solve_prof/launches_c2_solve.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; kn=h.index('Kernel Name'); mv=h.index('Metric Value')
t=defaultdict(float); n=defaultdict(int)
for r in rows[hi+1:]:
    try: v=float(r[mv].replace(',',''))
    except: continue
    k=r[kn].split('(')[0][:60]; t[k]+=v; n[k]+=1
for k in sorted(t,key=lambda x:-t[x]): print(k, n[k], round(t[k]/1e6,3),'ms')
PY
