"""Predicted strong scaling of cfg5 from one GPU: the per-rank step (its
z-slab of 1000/N planes, all 10^6 sites binned) timed as CUDA-graph replays,
N = 1, 2, 4, 8 (the histogram all-reduce over NVLink is not included)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402
from paper_2201_13234_b200.engine import Tessellator  # noqa: E402

p = oracle.baseline_config(5)
pos = torch.from_numpy(p.positions).cuda()
hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
base = None
for world in (1, 2, 4, 8):
    worst = 0.0
    for rank in sorted({0, world - 1}):
        zb, ze = vx.slab_bounds(1000, rank, world)
        lab = torch.empty((ze - zb) * 1000 * 1000, dtype=torch.int32, device="cuda")
        eng = Tessellator(0)
        g = eng.capture(kind=0, counts=[1000] * 3, lengths=[1.0] * 3, periodic=True, positions=pos,
                        labels=lab, histogram=hist, slab=(zb, ze), profile=True)
        ms = []
        for k in range(12):
            flush.fill_(k)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        t = float(np.median(ms[2:]))
        stages = eng.stage_ms()
        worst = max(worst, t)
        eng.close()
        del g, lab
    base = base or worst
    print(f"N={world}: per-rank step {worst:.3f} ms (bin {stages['bin']:.3f}, ball {stages['ball']:.3f}) "
          f"-> {1e9 / (worst * 1e-3) / 1e9:.1f} Gvox/s whole job, efficiency {base / (world * worst):.2f}",
          flush=True)
