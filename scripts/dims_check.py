"""Throughput of d = 1, 2, 3 problems of similar voxel count (device stages).
python scripts/dims_check.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

for d, counts, ns in [(2, [16384, 16384], 1_000_000), (2, [8192, 4096], 200_000), (1, [1 << 28], 1_000_000),
                      (3, [640, 640, 640], 262_144)]:
    L = np.ones(d)
    pos, _ = oracle.generate_uniform_sites(d, L, ns, 0, 1.0, 3)
    box = vx.Domain(list(L), vx.Boundary.Periodic)
    grid = vx.VoxelGrid(counts, box)
    sites = vx.SiteSet(vx.Kind.Voronoi, d, pos, None, 0.0)
    for _ in range(2):
        r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True)
    sm = r.stats["stage_ms"]
    dev = sm["bin"] + sm["params"] + sm["ball"] + sm["shell"]
    nv = int(np.prod(counts))
    print(f"d={d} {counts} Ns={ns}: dev {dev:.2f} ms ({nv / dev / 1e6:.1f} Gvox/s) ball {sm['ball']:.2f} "
          f"shell {sm['shell']:.2f} unres {r.stats['n_unresolved']} overflow {r.stats['overflow_bricks']} "
          f"hist_ok {int(r.histogram.sum()) == nv}", flush=True)
