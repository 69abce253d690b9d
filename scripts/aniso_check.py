"""Ball-phase throughput on anisotropic voxels (thick slices / tall voxels):
z spacing = ratio x the in-plane spacing, ~10-voxel in-plane site spacing."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

for ratio in [float(x) for x in sys.argv[1:]] or [0.25, 0.5, 1.0, 2.0, 3.0, 4.0, 8.0]:
    nxy = 512
    nz = max(8, int(round(512 / ratio)))
    L = [1.0, 1.0, 1.0]
    ns = int(nxy * nxy * nz * ratio / 1000)  # one site per ~1000 in-plane-voxel^3 of volume
    pos, _ = oracle.generate_uniform_sites(3, np.ones(3), ns, 0, 1.0, 3)
    sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
    grid = vx.VoxelGrid([nxy, nxy, nz], vx.Domain(L, vx.Boundary.Periodic))
    for _ in range(2):
        r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True)
    sm = r.stats["stage_ms"]
    dev = sm["bin"] + sm["params"] + sm["ball"] + sm["shell"]
    nv = nxy * nxy * nz
    print(f"z/xy spacing {ratio:5.2f}: {nxy}x{nxy}x{nz}, {ns} sites: dev {dev:7.2f} ms ({nv / dev / 1e6:6.1f} Gvox/s) "
          f"overflow {r.stats['overflow_bricks']} unres {r.stats['n_unresolved']} "
          f"evals/voxel {r.stats['ball_evals'] / nv:.2f}", flush=True)
