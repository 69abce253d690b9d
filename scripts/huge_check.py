"""Beyond 2^31 voxels: 1600^3 periodic Voronoi with 4e6 sites (16 GB label
image).  Histogram sum, and an independent sampled re-check of labels against
all sites (validate_partition, the reference's audit) on 2e5 random voxels.
python scripts/huge_check.py [n] [n_sites] [sample]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000
sample = int(sys.argv[3]) if len(sys.argv) > 3 else 200_000
pos, _ = oracle.generate_uniform_sites(3, np.ones(3), ns, 0, 1.0, 11)
box = vx.Domain([1.0] * 3, vx.Boundary.Periodic)
grid = vx.VoxelGrid([n] * 3, box)
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
out = torch.empty(n ** 3, dtype=torch.int32).pin_memory().numpy()
t0 = time.perf_counter()
r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, out=out)
dt = time.perf_counter() - t0
print(f"{n}^3 = {n ** 3:,} voxels, {ns:,} sites: {dt * 1e3:.0f} ms e2e, hist sum ok {int(r.histogram.sum()) == n ** 3}, "
      f"unresolved {r.stats['n_unresolved']}, overflow {r.stats['overflow_bricks']}", flush=True)
t0 = time.perf_counter()
rep = vx.validate_partition(r.labels, None, sites, sample=sample, seed=5)
print(f"validate_partition on {rep.voxels_checked} voxels: {rep.label_mismatches} label mismatches "
      f"({time.perf_counter() - t0:.1f} s)", flush=True)
print(f"max label {int(out.max())} min label {int(out.min())}", flush=True)
