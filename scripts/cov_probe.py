"""Ball-phase coverage probe: our unresolved-voxel counter vs the reference's
step-2 count (step2_evals / n_sites) per ball-kernel variant."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

if len(sys.argv) < 3:
    for v in ("1", "11", "12"):
        for i in range(8):
            subprocess.run([sys.executable, __file__, v, str(i)], env=dict(os.environ, VX_BALL=v))
    sys.exit(0)

import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402
from conftest import to_vx  # noqa: E402

from test_gpu_parity import coverage_case  # noqa: E402

i = int(sys.argv[2])
p = coverage_case(i)
kind, ns = p.kind, p.n_sites
_, _, param, _ = oracle.ref_tessellate(p, prune=False, distances=False)
for scale in (1.0, 0.5):
    # the reference's own parameter (ours differs for timed kinds), then a smaller ball
    override = param * scale if kind == 0 else float(np.min(p.times) + scale * (param - np.min(p.times)))
    lab_ref, _, param_ref, (_, ev2) = oracle.ref_tessellate(p, prune=False, override=override, distances=False)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, vx.FastOptions(override_param=override, prune=False), distances=False)
    st = {k: r.stats[k] for k in ("n_unresolved", "overflow_bricks", "ball_evals", "shell_evals", "engine")}
    print(sys.argv[1], i, scale, "ref", ev2 // ns, "ours", st, "labels_eq", bool(np.array_equal(r.labels.labels, lab_ref)),
          flush=True)
