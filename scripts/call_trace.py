"""One traced host-buffer call (VX_TRACE=1 VX_RUN_TRACE=1) after warm-up: python scripts/call_trace.py [n ns]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13234_b200 as vx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
rng = np.random.default_rng(5)
pos = torch.from_numpy(rng.uniform(0, 1, (ns, 3))).pin_memory().numpy()
grid = vx.VoxelGrid([n, n, n], vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic))
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
out = torch.empty(n ** 3, dtype=torch.int32).pin_memory().numpy()
hist = torch.zeros(ns, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
for i in range(6):
    if i == 5:
        os.environ["VX_TRACE"] = "1"
        os.environ["VX_RUN_TRACE"] = "1"
    t0 = time.perf_counter()
    vx.tessellate_fast(sites, grid, distances=False, out=out, histogram_out=hist)
    print("call %.2f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
