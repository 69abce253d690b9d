"""One cfg5 host-buffer call (the run-coded transport), for ncu captures of
run_encode_kernel: ncu -k regex:run_encode -c 1 --set full python scripts/run_encode_once.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13234_b200 as vx  # noqa: E402

rng = np.random.default_rng(5)
pos = rng.uniform(0, 1, (1000000, 3))
grid = vx.VoxelGrid([1000] * 3, vx.Domain([1.0] * 3, vx.Boundary.Periodic))
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
out = np.empty(10 ** 9, dtype=np.int32)
vx.tessellate_fast(sites, grid, distances=False, out=out)
print("ok", int(out[:1000].min()) >= 0)
