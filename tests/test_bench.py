"""bench.py's contract: one JSON line per run with the keys the driver reads;
the reference arm (`--impl reference`) runs the reference's CPU engine on
rank 0 only; the GPU arm's line carries roofline / e2e / clocks / launches."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                         text=True, env=env, timeout=timeout, cwd=ROOT)
    return out


def test_reference_arm_emits_one_json_line():
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    out = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the whole config through the stock tessellate_fast: the App. B fingerprint
    assert d["parity"]["match"] is True and len(d["step_s"]) == 2
    assert d["config"]["n_voxels"] == 128 ** 3


def test_reference_arm_never_loads_the_product():
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','1','--steps','1',"
            "'--warmup','0']; import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "assert 'libvoxellate_b200' not in maps, 'product loaded'; "
            "assert 'paper_2201_13234_b200' not in sys.modules")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]


def test_both_arms_draw_identical_inputs_and_config():
    """bench.py's two input paths (product API / reference library) agree bit
    for bit on every config, and cfg3's plain-Python lognormal recipe equals
    the C restatement (oracle/vx_oracle.c)."""
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ROOT)
    import bench

    pos, rad = bench.lognormal_spheres(2000, 77)
    opos, orad = oracle.generate_lognormal_spheres(2000, 0.5 * np.cbrt(1.0 / 2000), 0.3, 77)
    assert np.array_equal(pos, opos) and np.array_equal(rad, orad)
    for k in (1, 3, 4):
        c, _, _, sites = bench.make_inputs(k)
        p = bench.make_ref_problem(k)
        assert np.array_equal(sites.positions, p.positions)
        assert (sites.times is None) == (p.times is None)
        if p.times is not None:
            assert np.array_equal(sites.times, p.times)
        assert bench.config_dict(c, 1) == bench.config_dict(bench.CONFIGS[k], 1)


def test_reference_arm_other_ranks_exit_silently():
    out = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0"],
               {"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert out.returncode == 0 and out.stdout.strip() == ""


@pytest.mark.gpu
def test_gpu_arm_line_has_every_key():
    out = _run(["--config", "1", "--steps", "3", "--warmup", "3"])
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert BASE_KEYS | {"clocks", "gpu_launches", "roofline", "cpu_baseline"} <= set(d)
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["parity"]["match"] is True
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
