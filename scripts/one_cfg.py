"""Run one baseline config once through the fast path (profiling helper).
python scripts/one_cfg.py K [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

k = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = oracle.baseline_config(k)
box = vx.Domain(p.lengths, vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
grid = vx.VoxelGrid(p.counts, box)
sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
for _ in range(reps):
    r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True)
    fp = oracle.fingerprint(r.labels.labels)
    print(f"cfg{k} fp {fp} {'OK' if fp == oracle.SURVEY_FINGERPRINTS[k] else 'FAIL'} engine {r.stats['engine']} "
          f"stages { {a: round(b, 2) for a, b in r.stats['stage_ms'].items()} } "
          f"unres {r.stats['n_unresolved']} ball_evals {r.stats['ball_evals']} shell_evals {r.stats['shell_evals']}",
          flush=True)
