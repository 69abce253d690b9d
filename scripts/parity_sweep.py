"""Randomized parity sweep against the reference library (oracle/_ref) on the
GPU box: d = 1..4, all kinds, both boundaries, prune on/off, occasional
overrides, anisotropic voxels and densities from 2 to 40 voxels per site.
Labels, f64 values and the grain-volume histogram must be identical.
python scripts/parity_sweep.py [n_instances] [seed]  -> gpurun_out/parity_sweep.json"""
import json
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

n_inst = int(sys.argv[1]) if len(sys.argv) > 1 else 300
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 20261020
rng = np.random.default_rng(seed)
rows, bad = [], []
t_all = time.time()
for i in range(n_inst):
    d = int(rng.choice([1, 2, 3, 3, 3, 4]))
    kind = int(rng.integers(3))
    periodic = bool(rng.integers(2))
    target = {1: 2_000_000, 2: 4_000_000, 3: 8_000_000, 4: 400_000}[d]
    aspect = np.exp(rng.uniform(-1.0, 1.0, d))
    base = (target / np.prod(aspect)) ** (1.0 / d)
    counts = [max(1, int(base * a)) for a in aspect]
    L = rng.uniform(0.5, 2.0, d)
    nv = int(np.prod(counts))
    spacing = float(np.exp(rng.uniform(np.log(2.0), np.log(40.0))))
    ns = int(np.clip(nv / spacing ** d, 1, 400_000 if d < 4 else 2_000))
    horizon = float(0.5 * np.prod(L) ** (1.0 / d) / ns ** (1.0 / d))
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, horizon, int(rng.integers(1 << 40)))
    G = [0.0, float(np.exp(rng.uniform(-1, 1))), float(np.exp(rng.uniform(-1, 1)))][kind]
    p = oracle.Problem(kind, counts, L, periodic, pos, t, G)
    prune = bool(rng.integers(2))
    override = None
    if rng.uniform() < 0.15:
        _, _, param, _ = oracle.ref_tessellate(p, prune=prune, distances=False)
        s = float(np.exp(rng.uniform(np.log(0.3), np.log(2.0))))
        override = param * s if kind == 0 else float(np.min(t) + s * (param - np.min(t)))
    t0 = time.time()
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p, prune=prune, override=override)
    t_ref = time.time() - t0
    sites, grid = to_vx(p)
    t1 = time.time()
    r = vx.tessellate_fast(sites, grid, vx.FastOptions(override_param=override, prune=prune), distances=True,
                           histogram=True)
    t_ours = time.time() - t1
    ok_lab = bool(np.array_equal(r.labels.labels, lab_ref))
    ok_dist = bool(np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64)))
    ok_hist = bool(np.array_equal(r.histogram, np.bincount(lab_ref, minlength=ns).astype(np.uint64)))
    row = {"i": i, "d": d, "kind": kind, "periodic": periodic, "counts": counts, "n_sites": ns,
           "prune": prune, "override": override is not None, "labels": ok_lab, "values": ok_dist,
           "histogram": ok_hist, "overflow_bricks": int(r.stats["overflow_bricks"]), "ref_s": round(t_ref, 3),
           "ours_s": round(t_ours, 3), "unresolved": int(r.stats["n_unresolved"])}
    rows.append(row)
    if t_ours > 2.0:
        print("SLOW", row, flush=True)
    if not (ok_lab and ok_dist and ok_hist):
        bad.append(row)
        print("MISMATCH", row, flush=True)
summary = {"instances": n_inst, "seed": seed, "mismatches": len(bad), "by_dim": {},
           "with_overflow_route": sum(1 for r in rows if r["overflow_bricks"] > 0),
           "voxels_total": int(sum(int(np.prod(r["counts"])) for r in rows)), "wall_s": round(time.time() - t_all, 1)}
for dd in (1, 2, 3, 4):
    summary["by_dim"][dd] = sum(1 for r in rows if r["d"] == dd)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "parity_sweep.json"), "w") as f:
    json.dump({"summary": summary, "bad": bad, "rows": rows}, f, indent=1)
print(json.dumps(summary), flush=True)
