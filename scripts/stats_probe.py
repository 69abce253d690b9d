"""VX_STATS=1 list-size diagnostics for cfg2, cfg5 and a 6000-site problem
numbered in random, Morton and z order.  python scripts/stats_probe.py"""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import oracle, paper_2201_13234_b200 as vx
from conftest import to_vx
for k in (2, 5):
    p = oracle.baseline_config(k); s, g = to_vx(p); print("cfg", k, flush=True); vx.tessellate_fast(s, g)
ns = 6000; L = np.array([1.0, 0.9, 1.1]); pos, t = oracle.generate_uniform_sites(3, L, ns, 0, 0.1, 71)
P = pos.reshape(ns, 3); q = np.minimum((P / L * 1024).astype(np.uint64), np.uint64(1023)); key = np.zeros(ns, dtype=np.uint64)
for b in range(10):
    for a in range(3): key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
for name, perm in (("random", np.arange(ns)), ("morton", np.argsort(key, kind="stable")), ("z", np.argsort(P[:, 2]))):
    pp = oracle.Problem(0, [160, 144, 176], L, True, np.ascontiguousarray(P[perm]).reshape(-1), None, 0.0)
    s, g = to_vx(pp); print(name, flush=True); vx.tessellate_fast(s, g)
