"""Host-buffer call (cfg5 shape) into differently backed output buffers: cudaHostAlloc
(torch pin_memory), pageable numpy, and mmap + MADV_HUGEPAGE (+ cudaHostRegister).
python scripts/hugepage_probe.py"""
import ctypes
import mmap
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13234_b200 as vx  # noqa: E402
from paper_2201_13234_b200 import _lib  # noqa: E402

for f in ("enabled", "defrag", "shmem_enabled"):
    try:
        print("thp", f, open("/sys/kernel/mm/transparent_hugepage/" + f).read().strip())
    except OSError as e:
        print("thp", f, e)
n, ns = 1000, 1000000
rng = np.random.default_rng(5)
pos = torch.from_numpy(rng.uniform(0, 1, (ns, 3))).pin_memory().numpy()
box = vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic)
grid = vx.VoxelGrid([n, n, n], box)
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
hist = torch.zeros(ns, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
nbytes = 4 * n ** 3


def huge(register):
    size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    m = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.uint8)
    off = (-a.ctypes.data) % (2 << 20)
    a = a[off:off + size]
    a[:] = 0
    if register:
        rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, size, 0)
        print("cudaHostRegister", rc)
    return a[:nbytes].view(np.int32), m


def anon_kb():
    for line in open("/proc/meminfo"):
        if line.startswith("AnonHugePages"):
            return line.strip()


bufs = [("cudaHostAlloc", lambda: (torch.empty(n ** 3, dtype=torch.int32).pin_memory().numpy(), None)),
        ("pageable numpy", lambda: (np.zeros(n ** 3, dtype=np.int32), None)),
        ("hugepage mmap", lambda: huge(False)),
        ("hugepage mmap + cudaHostRegister", lambda: huge(True))]
ref = None
for name, mk in bufs:
    out, keep = mk()
    print(name, anon_kb())
    ts = []
    for i in range(7):
        if i == 6:
            os.environ["VX_RUN_TRACE"] = "1"
        t0 = time.perf_counter()
        vx.tessellate_fast(sites, grid, distances=False, out=out, histogram_out=hist)
        ts.append(time.perf_counter() - t0)
    os.environ.pop("VX_RUN_TRACE", None)
    fp = _lib.lib().vx_label_fingerprint(out.ctypes.data_as(_lib.C.c_void_p), out.size)
    ref = fp if ref is None else ref
    print(name, "ms", ["%.1f" % (1e3 * t) for t in ts], "same" if fp == ref else "DIFFERENT", flush=True)
    del out, keep
