"""H2D of the cfg5 site positions (24 MB): torch pinned copy vs the library's
ingest of the same pinned / pageable buffer (VX_TRACE=1 prints the latter)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

p = oracle.baseline_config(5)
pin_t = torch.from_numpy(p.positions).pin_memory()
print("pinned:", pin_t.is_pinned(), pin_t.shape, pin_t.dtype, flush=True)
d = torch.empty_like(pin_t, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(pin_t, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch H2D pinned 24 MB: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
grid = vx.VoxelGrid(p.counts, vx.Domain(p.lengths, vx.Boundary.Periodic))
out = torch.empty(p.n_voxels, dtype=torch.int32).pin_memory().numpy()
for label, arr in (("pinned", pin_t.numpy()), ("pageable", np.array(p.positions))):
    sites = vx.SiteSet(vx.Kind.Voronoi, 3, arr, None, 0.0)
    print(label, "same buffer:", sites.positions.ctypes.data == arr.ctypes.data, flush=True)
    for _ in range(2):
        vx.tessellate_fast(sites, grid, distances=False, out=out)

import ctypes as C  # noqa: E402

from paper_2201_13234_b200._lib import lib  # noqa: E402

L = lib()
for label, arr in (("pinned", pin_t.numpy()), ("pageable", np.array(p.positions))):
    for ns in (0, 1):
        ms = C.c_float(0)
        L.vx_probe_h2d(0, arr.ctypes.data, arr.nbytes, ns, C.byref(ms))
        print(f"lib H2D {label} null_stream={ns}: {ms.value:.3f} ms", flush=True)
