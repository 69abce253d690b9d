"""Developer check on a GPU box: randomized parity vs the oracle + config timings.

python scripts/dev_check.py [--random N] [--configs 1,2,3,4,5] [--ref]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402


def to_vx(p):
    box = vx.Domain(p.lengths, vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(p.counts, box)
    sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
    return sites, grid


def random_instance(rng, i):
    d = [1, 2, 3, 3, 3, 4][i % 6]
    kind = (i // 6) % 3
    periodic = (i // 18) % 2 == 0
    L = rng.uniform(0.5, 2.0, d)
    cap = {1: 300, 2: 40, 3: 20, 4: 7}[d]
    counts = rng.integers(2, cap + 1, d)
    ns = int(rng.integers(1, 300))
    G = float(np.exp(rng.uniform(np.log(0.1), np.log(10.0)))) if kind else 0.0
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, float(rng.uniform(0.5, 2.0)),
                                           int(rng.integers(1 << 62)))
    return oracle.Problem(kind, counts, L, periodic, pos, t, G)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--random", type=int, default=200)
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--ref", action="store_true")
    a = ap.parse_args()
    rng = np.random.default_rng(12345)
    bad = 0
    t0 = time.time()
    for i in range(a.random):
        p = random_instance(rng, i)
        sites, grid = to_vx(p)
        opts = vx.FastOptions(prune=(i % 2 == 0))
        if i % 7 == 3:
            if p.kind == 0:
                opts.override_param = float(np.exp(rng.uniform(np.log(0.02), np.log(2.0))))
            else:
                opts.override_param = float(p.times.min() + rng.uniform(0, 1.0))
        lab, dist = oracle.brute(p)
        for eng in ("fast", "brute"):
            r = vx.tessellate_fast(sites, grid, opts) if eng == "fast" else vx.tessellate_brute(sites, grid)
            okl = np.array_equal(r.labels.labels, lab)
            okd = np.array_equal(r.distances.values.view(np.uint64), dist.view(np.uint64))
            if not (okl and okd):
                bad += 1
                nm = int((r.labels.labels != lab).sum())
                print(f"MISMATCH inst {i} eng {eng} d={p.dim} kind={p.kind} per={p.periodic} "
                      f"ns={p.n_sites} counts={list(p.counts)} labels_bad={nm} "
                      f"dist_bad={int((r.distances.values != dist).sum())} stats={r.stats}")
    print(f"random parity: {a.random} instances, {bad} mismatches, {time.time()-t0:.1f}s", flush=True)

    for k in [int(x) for x in a.configs.split(",") if x]:
        p = oracle.baseline_config(k)
        sites, grid = to_vx(p)
        ctx_t = []
        for rep in range(3):
            t = time.time()
            r = vx.tessellate_fast(sites, grid, distances=False, histogram=True)
            ctx_t.append(time.time() - t)
        fp = oracle.fingerprint(r.labels.labels)
        hist_ok = int(r.histogram.sum()) == p.n_voxels
        print(f"cfg{k}: fp {fp} expect {oracle.SURVEY_FINGERPRINTS[k]} "
              f"{'OK' if fp == oracle.SURVEY_FINGERPRINTS[k] else 'FAIL'} hist_ok={hist_ok} "
              f"wall(e2e incl D2H)={min(ctx_t)*1e3:.1f} ms stats={r.stats}", flush=True)
        if a.ref and k <= 4:
            t = time.time()
            lab, _, param, ev = oracle.ref_tessellate(p, distances=False)
            print(f"   ref cpu {time.time()-t:.2f}s equal={np.array_equal(lab, r.labels.labels)}",
                  flush=True)


if __name__ == "__main__":
    main()
