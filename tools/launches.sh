#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
WL=${WL:-c2}
CMD="python bench.py --workload $WL --steps 3 --warmup 2 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$WL.csv $CMD > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_$WL.csv')) if r]
hdr=None; agg={}
for r in rows:
    if r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); n=d['Kernel Name'].split('(')[0][:50]; agg.setdefault(n,[]).append(float(d['Metric Value'].replace(',','')))
for n,v in agg.items(): print(len(v), n, 'median %.2f us'%(sorted(v)[len(v)//2]/1000))
PY
