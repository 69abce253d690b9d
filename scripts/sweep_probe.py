import os, sys, time, json
import numpy as np
ROOT = os.getcwd()
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle
import paper_2201_13234_b200 as vx
from conftest import to_vx
n_inst = int(sys.argv[1]); seed = int(sys.argv[2])
rng = np.random.default_rng(seed)
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
    sites, grid = to_vx(p)
    t1 = time.time()
    r = vx.tessellate_fast(sites, grid, vx.FastOptions(override_param=override, prune=prune), distances=True, histogram=True, profile=True)
    dt = time.time() - t1
    print(i, f"d={d} kind={kind} per={periodic} counts={counts} ns={ns} prune={prune} ovr={override is not None} "
          f"ours={dt:.2f}s unres={r.stats['n_unresolved']} ovf={r.stats['overflow_bricks']} stages={ {k: round(v,1) for k,v in r.stats['stage_ms'].items()} }", flush=True)
