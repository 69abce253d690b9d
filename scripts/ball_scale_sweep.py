"""Ball-phase / shell split vs the investigation-ball scale (labels do not
depend on it; only which voxels the ball phase resolves does).
python scripts/ball_scale_sweep.py [cfg ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

cfgs = [int(x) for x in sys.argv[1:]] or [2, 3, 4, 5]
scales = [float(s) for s in os.environ.get("SCALES", "0.7,0.8,0.9,1.0,1.1,1.25").split(",")]
for k in cfgs:
    p = oracle.baseline_config(k)
    box = vx.Domain(p.lengths, vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(p.counts, box)
    sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
    for sc in scales:
        best = None
        for _ in range(3):
            r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True, ball_scale=sc)
            sm = r.stats["stage_ms"]
            if best is None or sm["ball"] + sm["shell"] < best[0]["ball"] + best[0]["shell"]:
                best = (sm, r)
        sm, r = best
        fp = oracle.fingerprint(r.labels.labels)
        print(f"cfg{k} scale {sc:4.2f}: ball {sm['ball']:6.3f} shell {sm['shell']:6.3f} sum {sm['ball'] + sm['shell']:6.3f} ms"
              f" unres {r.stats['n_unresolved']:9d} evals/vox {r.stats['ball_evals'] / r.labels.labels.size:5.2f}"
              f" {'OK' if fp == oracle.SURVEY_FINGERPRINTS[k] else 'FAIL'}", flush=True)
