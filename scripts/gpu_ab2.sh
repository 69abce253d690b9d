cd $GRAFT_REPO_ROOT
[ -n "$NQ" ] && timeout 600 python scripts/exact_quick.py $NQ 7 > gpurun_out/exact_quick.log 2>&1; tail -1 gpurun_out/exact_quick.log
for rep in 1 2; do for lib in abl/*.so; do
VX_LIB_PATH=$lib python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle
from paper_2201_13234_b200.engine import Tessellator
tag = os.path.basename(os.environ["VX_LIB_PATH"])
for cfg in [int(c) for c in os.environ.get("CFGS", "3 4").split()]:
    p = oracle.baseline_config(cfg)
    eng = Tessellator(0)
    pos = torch.from_numpy(p.positions).cuda()
    t = torch.from_numpy(p.times).cuda() if p.times is not None else None
    lab = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
    hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
    kw = dict(kind=p.kind, counts=list(p.counts), lengths=list(p.lengths), periodic=p.periodic, positions=pos, times=t, growth=p.growth, labels=lab, histogram=hist)
    tot, st = [], []
    for i in range(9):
        s = eng.run(profile=True, **kw)
        if i >= 2:
            tot.append(sum(s["stage_ms"].values())); st.append(s["stage_ms"])
    fp = oracle.fingerprint(lab.cpu().numpy())
    med = {k: round(float(np.median([x[k] for x in st])), 3) for k in st[0]}
    print(f"{tag:12s} cfg{cfg} total {np.median(tot):.3f} ms {med} param {s['param']:.6g} {'OK' if fp == oracle.SURVEY_FINGERPRINTS[cfg] else 'FAIL'}", flush=True)
    eng.close()
PY
done; done
