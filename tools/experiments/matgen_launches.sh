python tools/matgen_bench.py --only $1 > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/matgen_launches.csv python tools/matgen_bench.py --only $1 > /dev/null 2>&1
python - <<PY
import csv,collections
rows=[r for r in csv.reader(open("gpurun_out/matgen_launches.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); ui=h.index("Metric Unit")
agg=collections.OrderedDict()
for r in rows[1:]:
    k=r[ki][:70]; v=float(r[vi].replace(",",""))
    if r[ui]=="ns": v/=1e6
    elif r[ui]=="us": v/=1e3
    a=agg.setdefault(k,[0,0.0]); a[0]+=1; a[1]+=v
for k,(c,v) in agg.items(): print(f"{c:4d} {v:9.3f} ms  {k}")
PY
