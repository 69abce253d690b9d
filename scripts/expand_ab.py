"""A/B of host expander settings on the cfg5 host-buffer call: each setting runs in a
fresh subprocess (the knobs are read once).  python scripts/expand_ab.py "K=V,K=V" ..."""
import os
import subprocess
import sys

CHILD = r'''
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2201_13234_b200 as vx
n, ns = 1000, 1000000
rng = np.random.default_rng(5)
pos = torch.from_numpy(rng.uniform(0, 1, (ns, 3))).pin_memory().numpy()
grid = vx.VoxelGrid([n, n, n], vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic))
sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
out = torch.empty(n ** 3, dtype=torch.int32).pin_memory().numpy()
hist = torch.zeros(ns, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
ts = []
for i in range(14):
    t0 = time.perf_counter()
    vx.tessellate_fast(sites, grid, distances=False, out=out, histogram_out=hist)
    ts.append(1e3 * (time.perf_counter() - t0))
ts = sorted(ts[2:])
from paper_2201_13234_b200 import _lib
fp = _lib.lib().vx_label_fingerprint(out.ctypes.data_as(_lib.C.c_void_p), out.size)
print("median %.1f min %.1f max %.1f fp %x" % (ts[len(ts) // 2], ts[0], ts[-1], fp))
'''
settings = sys.argv[1:] or [""]
for rep in range(2):
    for st in settings:
        env = dict(os.environ)
        for kv in filter(None, st.split(",")):
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print("[%s]" % st, r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
