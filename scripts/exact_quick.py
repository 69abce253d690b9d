"""Quick exactness check of the default ball engine on random 3-D instances
against the oracle's brute force (labels + f64 values + histogram), all kinds,
both boundaries, densities 3-40 voxels per site, anisotropic lengths.
python scripts/exact_quick.py [n] [seed]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402
from conftest import to_vx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
bad = 0
for i in range(n):
    kind = i % 3
    per = (i // 3) % 2 == 0
    L = rng.uniform(0.5, 2.0, 3)
    counts = [int(c) for c in rng.integers(20, 90, 3)]
    nv = int(np.prod(counts))
    spacing = float(np.exp(rng.uniform(np.log(3.0), np.log(40.0))))
    ns = int(np.clip(nv / spacing ** 3, 1, 50000))
    horizon = float(0.5 * np.cbrt(np.prod(L) / ns))
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, horizon, int(rng.integers(1 << 40)))
    G = [0.0, float(np.exp(rng.uniform(-1, 1))), float(np.exp(rng.uniform(-1, 1)))][kind]
    p = oracle.Problem(kind, counts, L, per, pos, t, G)
    lab, dist = oracle.brute(p)
    s, g = to_vx(p)
    r = vx.tessellate_fast(s, g, vx.FastOptions(prune=bool(i % 2)), distances=True, histogram=True)
    if r.stats.get("n_sites_kept", ns) != ns and kind:
        # pruning changes nothing in the labels (removed sites never win)
        pass
    ml = int((r.labels.labels != lab).sum())
    mv = int((r.distances.values.view(np.uint64) != dist.view(np.uint64)).sum())
    mh = not np.array_equal(r.histogram, np.bincount(lab, minlength=ns).astype(np.uint64))
    tag = "OK " if ml == 0 and mv == 0 and not mh else "BAD"
    if tag == "BAD":
        bad += 1
    print(f"{tag} i={i} kind={kind} per={per} counts={counts} ns={ns} spacing={spacing:.1f} "
          f"lab_mismatch={ml} val_mismatch={mv} hist_bad={mh} ovf={r.stats['overflow_bricks']} "
          f"unres={r.stats['n_unresolved']} evals/vox={r.stats['ball_evals'] / nv:.2f}", flush=True)
print("bad", bad, "of", n)
