"""All five BASELINE configs on the GPU box: device-pipeline time (CUDA events
per stage, best of 3), the default-API wall time (host buffers), and the
reference library's full tessellate_fast on the box's host cores (one run),
with a full-image label comparison.  Writes profiles/configs_<tag>.json.

python scripts/configs_table.py [tag] [--no-ref5]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "r02"
rows = []
# roofline of the ball phase: N_v (ln N_s + 1) evaluations x
# c_kind FP64-pipe ops against the DADD rate measured on this GPU
import ctypes as C  # noqa: E402
_dadd, _fadd = C.c_double(0.0), C.c_double(0.0)
vx.lib().vx_probe_pipe_rates(0, C.byref(_dadd), C.byref(_fadd))
P_FP64 = _dadd.value
C_KIND = {0: 3.0, 1: 5.0, 2: 4.0}
for k in (1, 2, 3, 4, 5):
    p = oracle.baseline_config(k)
    box = vx.Domain(p.lengths, vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(p.counts, box)
    sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
    dev, ball = [], []
    r = None
    for _ in range(4):
        r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, profile=True)
        sm = r.stats["stage_ms"]
        dev.append(sm["bin"] + sm["params"] + sm["ball"] + sm["shell"])  # sites resident (ingest has the H2D)
        ball.append(sm["ball"])
    ops = p.n_voxels * (np.log(p.n_sites) + 1.0) * C_KIND[p.kind]
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        r2 = vx.tessellate_fast(sites, grid, distances=False, histogram=True)
        walls.append(time.perf_counter() - t0)
    fp = oracle.fingerprint(r2.labels.labels)
    row = {"config": k, "n_voxels": p.n_voxels, "n_sites": p.n_sites, "kind": ["voronoi", "jm", "laguerre"][p.kind],
           "device_ms": min(dev[1:]), "device_gvox_s": p.n_voxels / min(dev[1:]) / 1e6,
           "api_wall_ms": 1e3 * min(walls), "fingerprint": fp,
           "fingerprint_ok": fp == oracle.SURVEY_FINGERPRINTS[k], "evals_per_voxel": r.stats["ball_evals"] / p.n_voxels,
           "unresolved": r.stats["n_unresolved"], "ball_ms": min(ball[1:]),
           "roofline_fp64": {"ops": ops, "peak_ops_s": P_FP64,
                             "frac_ball": ops / (min(ball[1:]) * 1e-3) / P_FP64,
                             "frac_pipeline": ops / (min(dev[1:]) * 1e-3) / P_FP64},
           "hbm_frac_ball": 4.0 * p.n_voxels / (min(ball[1:]) * 1e-3) / 6540.8e9}
    if oracle.have_ref() and not (k == 5 and "--no-ref5" in sys.argv):
        t0 = time.perf_counter()
        lab, _, param, evals = oracle.ref_tessellate(p, distances=False)
        dt = time.perf_counter() - t0
        row.update({"ref_cpu_s": dt, "ref_cpu_gvox_s": p.n_voxels / dt / 1e9, "ref_threads": oracle.ref().vxref_max_threads(),
                    "labels_equal_ref": bool(np.array_equal(lab, r2.labels.labels))})
    rows.append(row)
    print(json.dumps(row), flush=True)
out = {"host_cpus": os.cpu_count(), "rows": rows}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"configs_{tag}.json"), "w") as f:
    json.dump(out, f, indent=1)
