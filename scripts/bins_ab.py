"""Binning A/B: the binned arrays and cell starts of two library builds must be
identical (VX_LIB_PATH selects the other build).  Prints a digest per config."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

for k in (1, 3, 4, 5):
    p = oracle.baseline_config(k)
    box = vx.Domain(p.lengths, vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(p.counts, box)
    sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
    r = vx.tessellate_fast(sites, grid, distances=False, histogram=True)
    h = hashlib.sha1(r.labels.labels.tobytes()).hexdigest()[:16]
    print(f"cfg{k} labels {h} param {r.param!r} unres {r.stats['n_unresolved']} ball_evals {r.stats['ball_evals']} "
          f"shell_evals {r.stats['shell_evals']} kept {r.stats['n_sites_kept']}", flush=True)
