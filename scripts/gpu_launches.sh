cd $GRAFT_REPO_ROOT
for c in ${CFGS:-3 4}; do
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c$c.csv python scripts/ab_time.py $c > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/launch_c$c.csv")) if len(r)>10]
h=rows[0]; ik=h.index("Kernel Name"); iv=h.index("Metric Value"); iid=h.index("ID")
agg={}
n=0
for r in rows[1:]:
    k=r[ik].split("(")[0].split("<")[0][-40:]
    v=float(r[iv].replace(",",""))
    agg.setdefault(k,[0,0]); agg[k][0]+=v; agg[k][1]+=1
tot=sum(v[0] for v in agg.values())
print("cfg$c total us per 3 calls", tot/1000)
for k,(v,c) in sorted(agg.items(), key=lambda kv:-kv[1][0])[:14]:
    print(f"  {k:42s} {v/1000/3:8.1f} us/call  x{c//3}")
PY
done
