"""Exactness of the d != 3 engine (ballnd.cu) against the oracle's brute force
on random instances (d = 1, 2, 4, 5, 6; all kinds; both boundaries; prune
on/off), then timing of the verdict's two reference cases against the
reference library on this host.  python scripts/nd_quick.py [n] [seed] [--time]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402
from conftest import to_vx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
bad = 0
for i in range(n):
    d = [1, 2, 4, 2, 5, 6, 1, 4][i % 8]
    kind = (i // 8) % 3
    per = (i // 2) % 2 == 0
    L = rng.uniform(0.5, 2.0, d)
    tgt = {1: 20000, 2: 60000, 4: 60000, 5: 80000, 6: 100000}[d]
    base = tgt ** (1.0 / d)
    counts = [max(1, int(base * np.exp(rng.uniform(-0.4, 0.4)))) for _ in range(d)]
    nv = int(np.prod(counts))
    spacing = float(np.exp(rng.uniform(np.log(1.5), np.log(12.0))))
    ns = int(np.clip(nv / spacing ** d, 1, 3000))
    horizon = float(0.5 * np.prod(L) ** (1.0 / d) / ns ** (1.0 / d))
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, horizon, int(rng.integers(1 << 40)))
    G = [0.0, float(np.exp(rng.uniform(-1, 1))), float(np.exp(rng.uniform(-1, 1)))][kind]
    p = oracle.Problem(kind, counts, L, per, pos, t, G)
    lab, dist = oracle.brute(p)
    s, g = to_vx(p)
    prune = bool(i % 3)
    r = vx.tessellate_fast(s, g, vx.FastOptions(prune=prune), distances=True, histogram=True)
    ml = int((r.labels.labels != lab).sum())
    mv = int((r.distances.values.view(np.uint64) != dist.view(np.uint64)).sum())
    mh = not np.array_equal(r.histogram, np.bincount(lab, minlength=ns).astype(np.uint64))
    tag = "OK " if ml == 0 and mv == 0 and not mh else "BAD"
    bad += tag == "BAD"
    print(f"{tag} i={i} d={d} kind={kind} per={per} counts={counts} ns={ns} prune={prune} lab={ml} val={mv} "
          f"hist_bad={mh} engine={r.stats['engine']} unres={r.stats['n_unresolved']} ovf={r.stats['overflow_bricks']}",
          flush=True)
print("bad", bad, "of", n, flush=True)

if "--time" in sys.argv:
    thr = os.cpu_count()
    for name, d, counts, ns, kind in (("2-D 16384^2, 1e6 Voronoi", 2, [16384, 16384], 1000000, 0),
                                      ("4-D 48^4, 2e4 Voronoi", 4, [48] * 4, 20000, 0),
                                      ("4-D 48^4, 2e4 JM", 4, [48] * 4, 20000, 1),
                                      ("1-D 2^26, 2^20 Voronoi", 1, [1 << 26], 1 << 20, 0)):
        L = np.ones(d)
        pos, t = oracle.generate_uniform_sites(d, L, ns, kind, 0.5 * ns ** (-1.0 / d), 5)
        p = oracle.Problem(kind, counts, L, True, pos, t, 1.0 if kind else 0.0)
        s, g = to_vx(p)
        vx.tessellate_fast(s, g, distances=False)  # warm-up
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = vx.tessellate_fast(s, g, distances=False)
            ts.append(time.perf_counter() - t0)
        import torch
        from paper_2201_13234_b200.engine import Tessellator
        eng = Tessellator(0)
        posd = torch.from_numpy(pos).cuda()
        td = torch.from_numpy(t).cuda() if t is not None else None
        labd = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
        dev = []
        for _ in range(4):
            st = eng.run(kind=kind, counts=counts, lengths=list(L), periodic=True, positions=posd, times=td,
                         growth=p.growth, labels=labd, profile=True)
            dev.append(sum(st["stage_ms"].values()))
            sms = {k: round(v, 3) for k, v in st["stage_ms"].items()}
        t0 = time.perf_counter()
        lab_ref, _, _, ev = oracle.ref_tessellate(p, distances=False, threads=thr)
        tr = time.perf_counter() - t0
        same = np.array_equal(lab_ref, r.labels.labels)
        print(f"{name}: device {np.median(dev[1:]):.3f} ms = {p.n_voxels / np.median(dev[1:]) / 1e6:.1f} Gvox/s, "
              f"API call {min(ts) * 1e3:.1f} ms; reference {tr:.3f} s on {thr} threads = "
              f"{p.n_voxels / tr / 1e9:.4f} Gvox/s; labels equal: {same}; "
              f"evals/vox {r.stats['ball_evals'] / p.n_voxels:.2f} unres {r.stats['n_unresolved']} stages {sms}", flush=True)
        eng.close()
