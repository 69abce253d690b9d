"""A/B timing of library builds: ball-phase and whole-call device time
(median of N profiled device-pointer calls) per config, plus the label
fingerprint.  Run once per build with VX_LIB_PATH selecting it.
python scripts/ab_time.py [cfg ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2201_13234_b200.engine import Tessellator  # noqa: E402

tag = os.environ.get("VX_LIB_PATH", "default")
reps = int(os.environ.get("REPS", "15"))
for cfg in [int(x) for x in sys.argv[1:]] or [2, 3, 4, 5]:
    p = oracle.baseline_config(cfg)
    eng = Tessellator(0)
    pos = torch.from_numpy(p.positions).cuda()
    t = torch.from_numpy(p.times).cuda() if p.times is not None else None
    lab = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
    hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
    kw = dict(kind=p.kind, counts=list(p.counts), lengths=list(p.lengths), periodic=p.periodic,
              positions=pos, times=t, growth=p.growth, labels=lab, histogram=hist)
    balls, cull, shells = [], [], []
    for i in range(reps + 2):
        st = eng.run(profile=True, **kw)
        if i >= 2:
            balls.append(st["stage_ms"]["ball"])
            shells.append(st["stage_ms"]["shell"])
    fp = oracle.fingerprint(lab.cpu().numpy())
    ok = fp == oracle.SURVEY_FINGERPRINTS[cfg]
    print(f"{os.path.basename(tag):28s} cfg{cfg} ball median {np.median(balls):.3f} min {np.min(balls):.3f} ms "
          f"{'OK' if ok else 'FAIL ' + fp} shell {np.median(shells):.3f}", flush=True)
    eng.close()
    del lab, hist, pos
    torch.cuda.empty_cache()
