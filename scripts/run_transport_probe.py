"""e2e host-buffer call (default cfg5; args: n ns [np]) with the run-coded label transport: timings
per setting (VX_D2H_THREADS, VX_CHUNKS, VX_D2H_RAW).
python scripts/run_transport_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13234_b200 as vx  # noqa: E402
from paper_2201_13234_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
periodic = (sys.argv[3] != "np") if len(sys.argv) > 3 else True
rng = np.random.default_rng(5)
pos = torch.from_numpy(rng.uniform(0, 1, (ns, 3))).pin_memory().numpy()
box = vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic if periodic else vx.Boundary.NonPeriodic)
grid = vx.VoxelGrid([n, n, n], box)
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
out = torch.empty(n ** 3, dtype=torch.int32).pin_memory().numpy()
hist = torch.zeros(ns, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
settings = [dict(VX_D2H_RAW="1"), {}, dict(VX_D2H_THREADS="16"), dict(VX_D2H_THREADS="8"),
            dict(VX_CHUNKS="8"), {}, {}]
ref = None
for st in settings:
    for k in ("VX_D2H_RAW", "VX_D2H_THREADS", "VX_CHUNKS"):
        os.environ.pop(k, None)
    os.environ.update(st)
    ts = []
    for i in range(6):
        if i == 5:
            os.environ["VX_RUN_TRACE"] = "1"
        t0 = time.perf_counter()
        vx.tessellate_fast(sites, grid, distances=False, out=out, histogram_out=hist)
        ts.append(time.perf_counter() - t0)
    os.environ.pop("VX_RUN_TRACE", None)
    fp = _lib.lib().vx_label_fingerprint(out.ctypes.data_as(_lib.C.c_void_p), out.size)
    ref = fp if ref is None else ref
    print(st, "ms", ["%.1f" % (1e3 * t) for t in ts], "d2h MB %.0f" % (_lib.lib().vx_last_d2h_bytes() / 1e6),
          "same" if fp == ref else "DIFFERENT", flush=True)
