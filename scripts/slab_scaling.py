"""Predicted strong scaling of cfg5 from one GPU: the per-rank step (its
z-slab of 1000/N planes, the sites of its slab window binned) timed as CUDA-graph replays,
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
        def timed(profile):
            eng = Tessellator(0)
            g = eng.capture(kind=0, counts=[1000] * 3, lengths=[1.0] * 3, periodic=True, positions=pos,
                            labels=lab, histogram=hist, slab=(zb, ze), profile=profile)
            ms = []
            for k in range(12):
                flush.fill_(k)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                b.synchronize()
                ms.append(a.elapsed_time(b))
            st = eng.stage_ms() if profile else None
            eng.close()
            del g
            return float(np.median(ms[2:])), st

        # the step without stage markers; the stage split from a profiled capture
        t, _ = timed(False)
        _, stages = timed(True)
        worst = max(worst, t)
        del lab
    base = base or worst
    print(f"N={world}: per-rank step {worst:.3f} ms (" + ", ".join(f"{k} {v:.3f}" for k, v in stages.items()) + ") "
          f"-> {1e9 / (worst * 1e-3) / 1e9:.1f} Gvox/s whole job, efficiency {base / (world * worst):.2f}",
          flush=True)
