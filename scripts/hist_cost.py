"""Cost of the grain-volume histogram inside the ball phase at cfg5: the
captured step with and without it (CUDA-graph replays, L2 flushed)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2201_13234_b200.engine import Tessellator  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = oracle.baseline_config(cfg)
pos = torch.from_numpy(p.positions).cuda()
t = None if p.times is None else torch.from_numpy(p.times).cuda()
hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
lab = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
res = {}
for rep in range(3):
    for name, h in (("hist", hist), ("nohist", None)):
        eng = Tessellator(0)
        g = eng.capture(kind=p.kind, counts=list(p.counts), lengths=list(p.lengths), periodic=p.periodic,
                        positions=pos, times=t, growth=p.growth, labels=lab, histogram=h)
        ms = []
        for k in range(15):
            flush.fill_(k)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        res.setdefault(name, []).append(float(np.median(ms[3:])))
        eng.close()
        del g
print({k: ["%.3f" % x for x in v] for k, v in res.items()})
