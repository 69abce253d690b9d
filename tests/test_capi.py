"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/voxellate_b200.h declares, and rejects invalid input with the
reference's std::invalid_argument messages (sites.cpp:41-59,
tessellate.cpp:176-180,221,231-232) before touching the device."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "voxellate_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_ ]*\**\s*\**(vx_[a-z0-9_]+)\s*\(",
                       text, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    import paper_2201_13234_b200 as vx

    L = vx.lib()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", vx.LIB_PATH], capture_output=True,
                        text=True).stdout
    exported = set(re.findall(r" T (vx_[a-z0-9_]+)", nm))
    assert set(names) <= exported
    from paper_2201_13234_b200._lib import SIGNATURES

    assert set(SIGNATURES) == set(names), "python binding out of sync with the header"


def test_library_is_sm100a_cuda():
    import paper_2201_13234_b200 as vx

    out = subprocess.run(["cuobjdump", "--list-elf", vx.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_options_defaults():
    import paper_2201_13234_b200 as vx
    from paper_2201_13234_b200._lib import vx_options

    assert vx.lib().vx_abi_version() == 2
    o = vx_options()
    vx.lib().vx_options_init(C.byref(o))
    assert o.prune == 1 and o.device == -1 and o.ball_scale == 1.0 and o.device_pointers == 0


def _sites(kind=0, d=2, n=5, seed=3, growth=1.0):
    import paper_2201_13234_b200 as vx

    box = vx.Domain([1.0] * d)
    return box, vx.generate_uniform_sites(box, n, vx.Kind(kind), growth, 1.0, seed)


@pytest.mark.parametrize("case,msg", [
    ("outside", "site positions must lie strictly inside the domain"),
    ("on_boundary", "site positions must lie strictly inside the domain"),
    ("nan", "site positions must lie strictly inside the domain"),
    ("bad_growth", "growth rate G must be positive for timed tessellations"),
    ("bad_r0", "override r0 must be positive"),
    ("neg_r0", "override r0 must be positive"),
    ("early_t0", "override t0 must not precede the earliest birth time"),
])
def test_invalid_inputs_raise_value_error(case, msg):
    import paper_2201_13234_b200 as vx

    kind = 1 if case in ("bad_growth", "early_t0") else 0
    box, s = _sites(kind=kind)
    grid = vx.VoxelGrid([8, 8], box)
    opts = vx.FastOptions()
    if case == "outside":
        s.positions[3] = 1.5
    elif case == "on_boundary":
        s.positions[0] = 0.0
    elif case == "nan":
        s.positions[1] = float("nan")
    elif case == "bad_growth":
        s.growth = 0.0
    elif case == "bad_r0":
        opts.override_param = 0.0
    elif case == "neg_r0":
        opts.override_param = -1.0
    elif case == "early_t0":
        opts.override_param = float(s.times.min() - 0.25)
    with pytest.raises(ValueError, match=re.escape(msg)):
        vx.tessellate_fast(s, grid, opts)


def test_invalid_grid_and_domain():
    import paper_2201_13234_b200 as vx

    with pytest.raises(ValueError):
        vx.Domain([1.0, -1.0])
    with pytest.raises(ValueError):
        vx.Domain([1.0] * 17)
    with pytest.raises(ValueError):
        vx.VoxelGrid([0, 4], vx.Domain([1.0, 1.0]))
    with pytest.raises(ValueError):
        vx.VoxelGrid([4], vx.Domain([1.0, 1.0]))


def test_raw_abi_error_codes():
    """NULL and malformed problems through the raw C entry point."""
    import paper_2201_13234_b200 as vx
    from paper_2201_13234_b200._lib import VX_EINVAL, vx_options, vx_problem, vx_stats

    L = vx.lib()
    lab = np.zeros(16, dtype=np.int32)
    assert L.vx_tessellate(None, None, None, lab.ctypes.data_as(C.c_void_p), None) == VX_EINVAL
    P = vx_problem()
    P.kind, P.dim, P.periodic = 0, 2, 1
    P.counts[0] = P.counts[1] = 4
    P.lengths[0] = P.lengths[1] = 1.0
    P.n_sites = 0
    assert L.vx_tessellate(None, C.byref(P), None, lab.ctypes.data_as(C.c_void_p), None) == VX_EINVAL
    assert b"at least one site" in L.vx_last_error()
    pos = np.array([0.5, 0.5])
    P.n_sites = 1
    P.positions = pos.ctypes.data
    O = vx_options()
    L.vx_options_init(C.byref(O))
    O.slab_begin, O.slab_end = 3, 2
    st = vx_stats()
    assert L.vx_tessellate(None, C.byref(P), C.byref(O), lab.ctypes.data_as(C.c_void_p),
                           C.byref(st)) == VX_EINVAL
    O.slab_begin, O.slab_end = 0, 0
    O.asynchronous = 1  # asynchronous calls need device pointers
    assert L.vx_tessellate(None, C.byref(P), C.byref(O), lab.ctypes.data_as(C.c_void_p),
                           C.byref(st)) == VX_EINVAL
    P.kind = 7
    assert L.vx_tessellate(None, C.byref(P), None, lab.ctypes.data_as(C.c_void_p), None) == VX_EINVAL


def test_prune_rejects_voronoi():
    import paper_2201_13234_b200 as vx

    box, s = _sites(kind=0)
    with pytest.raises(ValueError, match="timed tessellations only"):
        vx.prune_ineffective_sites(s, box)


@pytest.mark.parametrize("where", [0, 123456, 299999])
def test_large_site_set_validation_threads(where):
    """A bad coordinate anywhere gives the reference's message
    (sites.cpp:54-57).  Without a device (this CPU suite) the host check
    reports it; on a GPU the ingest kernel does, before any labelling work
    (test_gpu_parity.py::test_device_validation_rejects_bad_positions)."""
    import numpy as np

    import paper_2201_13234_b200 as vx

    n = 300000
    pos = np.random.default_rng(3).uniform(0.01, 0.99, 3 * n)
    pos[3 * where + 1] = 1.0  # on the boundary: not strictly inside
    box = vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic)
    grid = vx.VoxelGrid([8, 8, 8], box)
    sites = vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0)
    with pytest.raises(ValueError, match="site positions must lie strictly inside the domain"):
        vx.tessellate_fast(sites, grid)


def test_histogram_out_must_match_site_count():
    import numpy as np

    import paper_2201_13234_b200 as vx

    box, s = _sites(kind=0, d=2, n=5)
    grid = vx.VoxelGrid([8, 8], box)
    with pytest.raises(ValueError, match="histogram_out"):
        vx.tessellate_fast(s, grid, histogram_out=np.zeros(4, dtype=np.uint64))


def test_caller_buffers_dtype_checked():
    import numpy as np

    import paper_2201_13234_b200 as vx

    box, s = _sites(kind=0, d=2, n=5)
    grid = vx.VoxelGrid([8, 8], box)
    with pytest.raises(ValueError, match="histogram_out"):
        vx.tessellate_fast(s, grid, histogram_out=np.zeros(5, dtype=np.float64))
    with pytest.raises(ValueError, match="out must hold"):
        vx.tessellate_fast(s, grid, out=np.zeros(64, dtype=np.float32))
