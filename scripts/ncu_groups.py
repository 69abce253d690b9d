import csv,io,subprocess,sys
rep,kre=sys.argv[1],sys.argv[2]; units=float(sys.argv[3])
groups=[tuple(x.split(':')) for x in sys.argv[4:]]
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass","--kernel-name","regex:"+kre],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
for i,r in enumerate(rows):
    if r and r[0]=="Line No": hdr=r; start=i+1; break
ix={}
for k,h in enumerate(hdr): ix.setdefault(h,k)
acc={g[2]:[0,0] for g in groups}; tot=[0,0]
for r in rows[start:]:
    if len(r)<len(hdr) or not r[0].strip().isdigit(): continue
    try: ins=int(r[ix["Instructions Executed"]] or 0); smp=int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except: continue
    ln=int(r[0]); tot[0]+=ins; tot[1]+=smp
    for a,b,n in groups:
        if int(a)<=ln<=int(b): acc[n][0]+=ins; acc[n][1]+=smp; break
for n,(i,s) in acc.items(): print(f"{n:20s} {i/units:8.1f}/u {100*i/tot[0]:5.1f}% inst {100*s/tot[1]:5.1f}% samples")
print("total",tot[0]/units)
