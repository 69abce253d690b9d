"""Where the e2e call's time goes beyond the PCIe copy (cfg5, pinned buffers)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402
from paper_2201_13234_b200 import _lib, voxellate  # noqa: E402

p = oracle.baseline_config(5)
box = vx.Domain(p.lengths, vx.Boundary.Periodic)
grid = vx.VoxelGrid(p.counts, box)
pin = torch.from_numpy(p.positions).pin_memory().numpy()
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pin, None, 0.0)
out = torch.empty(p.n_voxels, dtype=torch.int32).pin_memory().numpy()
hist = torch.zeros(p.n_sites, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
for i in range(3):
    t0 = time.perf_counter()
    vx.tessellate_fast(sites, grid, distances=False, histogram=True, out=out)
    t1 = time.perf_counter()
    P = voxellate._problem(sites, grid)
    O = _lib.vx_options()
    _lib.lib().vx_options_init(C.byref(O))
    O.histogram_out = hist.ctypes.data_as(C.c_void_p)
    st = _lib.vx_stats()
    t2 = time.perf_counter()
    rc = _lib.lib().vx_tessellate(None, C.byref(P), C.byref(O), out.ctypes.data_as(C.c_void_p), C.byref(st))
    t3 = time.perf_counter()
    print(f"api {1e3 * (t1 - t0):.1f} ms | raw C call {1e3 * (t3 - t2):.1f} ms (rc {rc})", flush=True)
