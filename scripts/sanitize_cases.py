"""Small instances through every engine path, for compute-sanitizer runs:
3-D (standard, dense mode, overflow -> sub-brick shell, slab window with the
all-sites fallback, the timed kinds' column brick stage at ~9-voxel spacing), d != 3 (1, 2, 4, 6), timed kinds with prune, the brute
engine and validate_partition.  python scripts/sanitize_cases.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402
from conftest import to_vx  # noqa: E402

rng = np.random.default_rng(3)
cases = []
for d, counts, ns in ((3, [40, 33, 29], 300), (3, [48, 40, 36], 6000), (3, [30, 30, 200], 40), (3, [72, 64, 80], 500),
                      (1, [3000], 200), (2, [90, 70], 900), (4, [9, 8, 10, 7], 300), (6, [4, 5, 3, 4, 5, 4], 200)):
    for kind in (0, 1, 2):
        for per in (True, False):
            cases.append((d, counts, ns, kind, per))
bad = 0
for i, (d, counts, ns, kind, per) in enumerate(cases):
    L = rng.uniform(0.6, 1.6, d)
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, 0.5 * np.prod(L) ** (1 / d) / ns ** (1 / d), 100 + i)
    p = oracle.Problem(kind, counts, L, per, pos, t, 1.2 if kind else 0.0)
    s, g = to_vx(p)
    lab, dist = oracle.brute(p)
    r = vx.tessellate_fast(s, g, vx.FastOptions(prune=True), distances=True, histogram=True)
    ok = np.array_equal(r.labels.labels, lab)
    if d == 3 and kind == 0:  # a slab (window binning) with a small override radius (all-sites fallback)
        n = counts[-1]
        r2 = vx.tessellate_fast(s, g, vx.FastOptions(override_param=0.02), distances=True, slab=(n // 3, n // 3 + 5))
        plane = counts[0] * counts[1]
        ok &= np.array_equal(r2.labels.labels, lab[n // 3 * plane:(n // 3 + 5) * plane])
    if i % 7 == 0:
        rb = vx.tessellate_brute(s, g)
        ok &= np.array_equal(rb.labels.labels, lab)
        rep = vx.validate_partition(r.labels, r.distances, s, sample=500, seed=9)
        ok &= rep.ok()
    bad += not ok
    print(i, d, kind, per, "ok" if ok else "MISMATCH", flush=True)
os.environ["VX_DENSE"] = "1"
p = oracle.Problem(0, [40, 36, 32], np.ones(3), True, *oracle.generate_uniform_sites(3, np.ones(3), 3000, 0, 1.0, 5))
s, g = to_vx(p)
lab, _ = oracle.brute(p, distances=False)
bad += not np.array_equal(vx.tessellate_fast(s, g, distances=False).labels.labels, lab)
print("bad", bad)
