"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

The reference library (/root/reference/proj/src, compiled by oracle/Makefile
into oracle/_ref/) produces every expected output here; nothing is computed
by this repository's code.  Run in the build container (where /root/reference
exists):

    python tests/golden/make_golden.py

Fixtures (numpy .npz, one per instance, plus index.json):
  * tess_*   : tessellate_fast and tessellate_brute labels + f64 values for
               seeded random instances (d = 1..4, all kinds, both boundaries,
               prune on/off, parameter overrides), the reference's own
               hand-checked cases (test_tessellate.cpp:55-86) and coincident /
               equal-time sites (test_sites.cpp:125-143).
  * prune_*  : prune_ineffective_sites removed flags (sites.cpp:113-171).
  * gen_*    : generate_uniform_sites outputs (sites.cpp:61-85).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

V, JM, LAG = oracle.VORONOI, oracle.JOHNSON_MEHL, oracle.LAGUERRE


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def problem_arrays(p: oracle.Problem):
    return dict(kind=np.int64(p.kind), counts=p.counts, lengths=p.lengths,
                periodic=np.int64(p.periodic), positions=p.positions,
                times=p.times if p.times is not None else np.zeros(0),
                growth=np.float64(p.growth))


def main():
    oracle.build()
    assert oracle.have_ref(), "reference library not built (needs /root/reference)"
    rng = np.random.default_rng(20261019)
    index = []
    # ---- random instances (restating test_tessellate.cpp:178-216) ----
    for i in range(48):
        d = [1, 2, 3, 3, 4, 3][i % 6]
        kind = (i // 6) % 3
        periodic = (i // 18) % 2 == 0
        L = rng.uniform(0.5, 2.0, d)
        cap = {1: 200, 2: 24, 3: 12, 4: 6}[d]
        counts = rng.integers(2, cap + 1, d)
        ns = int(rng.integers(1, 60))
        G = float(np.exp(rng.uniform(np.log(0.1), np.log(10.0)))) if kind else 0.0
        pos, t = oracle.ref_generate_uniform_sites(d, L, ns, kind, G, float(rng.uniform(0.5, 2.0)),
                                                   int(rng.integers(1 << 62)))
        p = oracle.Problem(kind, counts, L, periodic, pos, t, G)
        prune = i % 5 != 0
        override = None
        if i % 4 == 0:
            override = (float(np.exp(rng.uniform(np.log(0.02), np.log(2.0)))) if kind == V
                        else float(t.min() + rng.uniform(0.0, 1.0)))
        lf, df, param, ev = oracle.ref_tessellate(p, "fast", prune=prune, override=override)
        lb, db, _, _ = oracle.ref_tessellate(p, "brute")
        assert np.array_equal(lf, lb) and np.array_equal(df.view(np.uint64), db.view(np.uint64))
        name = f"tess_{i:03d}"
        save(name, **problem_arrays(p), labels=lf, values=df, prune=np.int64(prune),
             override=np.float64(np.nan if override is None else override), param=np.float64(param))
        index.append({"name": name, "dim": d, "kind": kind, "periodic": periodic, "n_sites": ns})
    # ---- hand-checked cases (test_tessellate.cpp:55-86) ----
    hand = [
        ("tess_single_site", oracle.Problem(V, [4, 4], [1.0, 2.0], False, [0.3, 0.4])),
        ("tess_periodic_line", oracle.Problem(V, [8], [1.0], True, [0.25, 0.75])),
        # coincident sites, equal times: the lower index wins (test_sites.cpp:125-143)
        ("tess_coincident_jm", oracle.Problem(JM, [9, 7], [1.0, 1.0], True,
                                              [0.5, 0.5, 0.5, 0.5, 0.2, 0.7], [0.3, 0.3, 0.1], 1.0)),
        ("tess_coincident_lag", oracle.Problem(LAG, [9, 7], [1.0, 1.0], False,
                                               [0.5, 0.5, 0.5, 0.5, 0.2, 0.7], [0.3, 0.3, 0.1], 1.0)),
        # a late Laguerre site reached before birth still owns cells (test_sites.cpp:160-176)
        ("tess_late_laguerre", oracle.Problem(LAG, [96, 16], [6.0, 1.0], False,
                                              [1.0, 0.5, 2.0, 0.5], [-4.0, 0.0], 1.0)),
    ]
    for name, p in hand:
        lf, df, param, _ = oracle.ref_tessellate(p, "fast")
        save(name, **problem_arrays(p), labels=lf, values=df, prune=np.int64(1),
             override=np.float64(np.nan), param=np.float64(param))
        index.append({"name": name, "dim": p.dim, "kind": p.kind, "periodic": p.periodic,
                      "n_sites": p.n_sites})
    # ---- prune (sites.cpp:113-171) ----
    for i in range(12):
        kind = JM if i % 2 else LAG
        periodic = (i // 2) % 2 == 0
        d = 2 + (i % 3 == 0)
        L = rng.uniform(0.5, 2.0, d)
        ns = int(rng.integers(5, 300))
        pos, t = oracle.ref_generate_uniform_sites(d, L, ns, kind, float(np.exp(rng.uniform(np.log(0.2), np.log(10.0)))),
                                                   1.0, int(rng.integers(1 << 62)))
        G = float(np.exp(rng.uniform(np.log(0.2), np.log(10.0))))
        p = oracle.Problem(kind, [1] * d, L, periodic, pos, t, G)
        dropped = oracle.ref_prune(p)
        save(f"prune_{i:02d}", **problem_arrays(p), dropped=dropped)
        index.append({"name": f"prune_{i:02d}", "removed": int(dropped.sum())})
    # ---- site generator (sites.cpp:61-85) ----
    for i, (d, kind, ns, horizon, seed) in enumerate([(3, V, 1000, 1.0, 1001), (2, JM, 77, 0.3, 5),
                                                      (3, LAG, 50, 2.0, 17), (4, V, 33, 1.0, 99)]):
        L = np.linspace(0.7, 1.9, d)
        pos, t = oracle.ref_generate_uniform_sites(d, L, ns, kind, 1.5, horizon, seed)
        save(f"gen_{i}", dim=np.int64(d), kind=np.int64(kind), n=np.int64(ns), horizon=np.float64(horizon),
             seed=np.int64(seed), lengths=L, positions=pos,
             times=t if t is not None else np.zeros(0))
        index.append({"name": f"gen_{i}"})
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump({"generated_by": "tests/golden/make_golden.py from oracle/_ref (the reference library)",
                   "fixtures": index}, f, indent=1)
    print(f"wrote {len(index)} fixtures")


if __name__ == "__main__":
    main()
