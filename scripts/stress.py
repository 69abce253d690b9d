"""Density / shape stress on the GPU: time + parity against fast==brute (small)
or the reference fingerprint machinery (large): prints stage times, unresolved
counts and overflow counters.
python scripts/stress.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

CASES = [
    # (name, kind, counts, n_sites, periodic, check_vs_ref)
    ("dense 1e7 in 1000^3", 0, [1000, 1000, 1000], 10_000_000, True, False),
    ("sparse 1e4 in 1000^3", 0, [1000, 1000, 1000], 10_000, True, False),
    ("very sparse 100 in 512^3", 0, [512, 512, 512], 100, True, True),
    ("flat 2048x2048x16, 2e5", 0, [2048, 2048, 16], 200_000, True, True),
    ("tall 64x64x4096, 5e4", 0, [64, 64, 4096], 50_000, False, True),
    ("JM dense 2e6 in 512^3", 1, [512, 512, 512], 2_000_000, True, False),
    ("Laguerre sparse 2e3 in 512^3", 2, [512, 512, 512], 2_000, False, True),
]

for name, kind, counts, ns, per, check in CASES:
    L = np.ones(3)
    horizon = 0.5 * np.cbrt(1.0 / ns)
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, horizon, 4242)
    p = oracle.Problem(kind, counts, L, per, pos, t, 1.0 if kind else 0.0)
    box = vx.Domain(list(L), vx.Boundary.Periodic if per else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(counts, box)
    sites = vx.SiteSet(vx.Kind(kind), 3, pos, t, 1.0 if kind else 0.0)
    r = None
    for rep in range(2):
        r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True)
    st = r.stats
    sm = st["stage_ms"]
    dev = sm["bin"] + sm["params"] + sm["ball"] + sm["shell"]
    line = (f"{name:32s} dev {dev:8.2f} ms ({p.n_voxels / dev / 1e6:7.1f} Gvox/s) ball {sm['ball']:.2f} "
            f"shell {sm['shell']:.2f} unres {st['n_unresolved']} overflow {st['overflow_bricks']} "
            f"hist_ok {int(r.histogram.sum()) == p.n_voxels}")
    if check:
        t0 = time.time()
        lab, _, _, _ = oracle.ref_tessellate(p, distances=False)
        line += f" ref_equal {np.array_equal(lab, r.labels.labels)} ({time.time() - t0:.1f}s)"
    print(line, flush=True)
