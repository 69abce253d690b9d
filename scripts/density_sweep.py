"""Ball-phase throughput vs site density on a 1000^3 periodic Voronoi grid.
python scripts/density_sweep.py [n1 n2 ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

ns_list = [int(x) for x in sys.argv[1:]] or [250_000, 1_000_000, 2_000_000, 3_000_000, 4_000_000, 6_000_000]
n = 1000
box = vx.Domain([1.0] * 3, vx.Boundary.Periodic)
grid = vx.VoxelGrid([n] * 3, box)
for ns in ns_list:
    pos, _ = oracle.generate_uniform_sites(3, np.ones(3), ns, 0, 1.0, 7)
    sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
    for _ in range(2):
        r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True)
    sm = r.stats["stage_ms"]
    dev = sm["bin"] + sm["params"] + sm["ball"] + sm["shell"]
    print(f"N_s={ns:9d} spacing {n / ns ** (1 / 3):5.1f} vox: dev {dev:7.2f} ms ({n ** 3 / dev / 1e6:6.1f} Gvox/s) "
          f"ball {sm['ball']:.2f} shell {sm['shell']:.2f} overflow {r.stats['overflow_bricks']} "
          f"unres {r.stats['n_unresolved']}", flush=True)
