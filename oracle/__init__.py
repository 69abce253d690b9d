"""TEST INFRASTRUCTURE ONLY -- the parity oracle.

Two checkers live here, both CPU-only:

* ``liboracle.so`` (``vx_oracle.c``): my plain-C restatement of the reference
  arithmetic (brute-force argmin, prune, site generators, r0, fingerprint).
* ``_ref/libvoxellate_ref.so``: the reference library itself, compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` (plus my C wrapper
  ``ref_capi.cpp``).  Present wherever ``build()`` ran with the reference tree
  mounted; it travels to the GPU box with the snapshot.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product
(``paper_2201_13234_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvoxellate_ref.so")

VORONOI, JOHNSON_MEHL, LAGUERRE = 0, 1, 2

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double


def build(verbose: bool = False) -> None:
    """Compile liboracle.so (always) and _ref/ (when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.vxo_generate_uniform_sites.argtypes = [C.c_int, _P, _I64, C.c_int, _D, C.c_uint64, _P, _P]
        L.vxo_generate_lognormal_spheres.argtypes = [_I64, _D, _D, C.c_uint64, _P, _P]
        L.vxo_spheres_to_timed.argtypes = [_I64, _P, _D, _P]
        L.vxo_brute.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _I64, _P, _P, _D, _I64, _I64, _P, _P]
        L.vxo_prune.argtypes = [C.c_int, C.c_int, C.c_int, _P, _I64, _P, _P, _D, _P]
        L.vxo_prune.restype = _I64
        L.vxo_optimal_r0.argtypes = [_I64, C.c_int, _P]
        L.vxo_optimal_r0.restype = _D
        L.vxo_fingerprint_u32.argtypes = [_P, _I64]
        L.vxo_fingerprint_u32.restype = C.c_uint64
        L.vxo_sample_indices.argtypes = [_I64, _I64, C.c_uint64, _P]
        _lib = L
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference library (oracle/_ref).  Raises if it was never built."""
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(REF_SO + " (run oracle.build() where /root/reference exists)")
        L = C.CDLL(REF_SO)
        L.vxref_last_error.restype = C.c_char_p
        L.vxref_tessellate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _I64, _P, _P, _D,
                                       C.c_int, C.c_int, _D, C.c_int, _P, _P, _P, _P]
        L.vxref_prune.argtypes = [C.c_int, C.c_int, C.c_int, _P, _I64, _P, _P, _D, _P]
        L.vxref_prune.restype = _I64
        L.vxref_generate_uniform_sites.argtypes = [C.c_int, _P, _I64, C.c_int, _D, _D, C.c_uint64, _P, _P]
        L.vxref_spheres_to_timed.argtypes = [C.c_int, _I64, _P, _P, _D, _P]
        L.vxref_optimal_r0.argtypes = [_I64, C.c_int, _P, C.c_int]
        L.vxref_optimal_r0.restype = _D
        L.vxref_search_optimal_t0.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _I64, _P, _P, _D]
        L.vxref_search_optimal_t0.restype = _D
        L.vxref_validate_partition.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _I64, _P, _P, _D,
                                               _P, _P, _I64, C.c_uint64, _P]
        L.vxref_tessellate_timed.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _I64, _P, _P, _D,
                                             C.c_int, _P, _P, _P, _P]
        L.vxref_ball_voxels.argtypes = [C.c_int, C.c_int, _P, _P, _P, _D, _P, _I64]
        L.vxref_ball_voxels.restype = _I64
        L.vxref_max_threads.restype = C.c_int
        L.vxref_have_image_io.restype = C.c_int
        if L.vxref_have_image_io():
            L.vxref_write_image.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int, _I64,
                                            _I64, _P]
            L.vxref_read_image.argtypes = [C.c_char_p, C.c_int, _P, _P, _P, _P, _I64]
        _ref = L
    return _ref


# --------------------------------------------------------------------------
# Problem container shared by the checkers (plain numpy, reference layout).
# --------------------------------------------------------------------------
class Problem:
    """A tessellation instance in the reference layout (sites.hpp:15-31,
    geometry.hpp:27-78): xyz-interleaved f64 positions, optional birth times."""

    def __init__(self, kind, counts, lengths, periodic, positions, times=None, growth=0.0):
        self.kind = int(kind)
        self.counts = np.ascontiguousarray(counts, dtype=np.int64)
        self.lengths = np.ascontiguousarray(lengths, dtype=np.float64)
        self.dim = int(self.counts.size)
        self.periodic = bool(periodic)
        self.positions = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1)
        self.n_sites = self.positions.size // self.dim
        self.times = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
        self.growth = float(growth) if self.kind != VORONOI else 0.0

    @property
    def n_voxels(self) -> int:
        return int(np.prod(self.counts))


def generate_uniform_sites(dim, lengths, n_sites, kind, horizon, seed):
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    pos = np.empty(n_sites * dim, dtype=np.float64)
    times = np.empty(n_sites, dtype=np.float64) if kind != VORONOI else None
    lib().vxo_generate_uniform_sites(dim, _ptr(lengths), n_sites, kind, float(horizon),
                                     seed & 0xFFFFFFFFFFFFFFFF, _ptr(pos), _ptr(times))
    return pos, times


def generate_lognormal_spheres(n_sites, mean_r, sigma, seed):
    pos = np.empty(n_sites * 3, dtype=np.float64)
    radii = np.empty(n_sites, dtype=np.float64)
    lib().vxo_generate_lognormal_spheres(n_sites, mean_r, sigma, seed, _ptr(pos), _ptr(radii))
    return pos, radii


def spheres_to_timed(radii, growth):
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    t = np.empty_like(radii)
    lib().vxo_spheres_to_timed(radii.size, _ptr(radii), float(growth), _ptr(t))
    return t


def brute(p: Problem, lin_begin=0, lin_end=None, distances=True):
    """Restated tessellate_brute over voxels [lin_begin, lin_end)."""
    lin_end = p.n_voxels if lin_end is None else lin_end
    n = lin_end - lin_begin
    lab = np.empty(n, dtype=np.uint32)
    dist = np.empty(n, dtype=np.float64) if distances else None
    lib().vxo_brute(p.kind, p.dim, int(p.periodic), _ptr(p.counts), _ptr(p.lengths), p.n_sites,
                    _ptr(p.positions), _ptr(p.times), p.growth, lin_begin, lin_end, _ptr(lab),
                    _ptr(dist))
    return lab, dist


def prune(p: Problem):
    dropped = np.zeros(p.n_sites, dtype=np.uint8)
    lib().vxo_prune(p.kind, p.dim, int(p.periodic), _ptr(p.lengths), p.n_sites, _ptr(p.positions),
                    _ptr(p.times), p.growth, _ptr(dropped))
    return dropped


def optimal_r0(n_sites, lengths):
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    return lib().vxo_optimal_r0(n_sites, lengths.size, _ptr(lengths))


def fingerprint(labels) -> str:
    labels = np.ascontiguousarray(labels).view(np.uint32).reshape(-1)
    return "%016x" % lib().vxo_fingerprint_u32(_ptr(labels), labels.size)


def sample_indices(nv, sample, seed):
    out = np.empty(sample, dtype=np.int64)
    lib().vxo_sample_indices(nv, sample, seed & 0xFFFFFFFFFFFFFFFF, _ptr(out))
    return out


# ---- the reference itself (oracle/_ref) ----------------------------------
def ref_tessellate(p: Problem, engine="fast", prune=True, override=None, threads=0,
                   distances=True):
    L = ref()
    lab = np.empty(p.n_voxels, dtype=np.uint32)
    dist = np.empty(p.n_voxels, dtype=np.float64) if distances else None
    param = np.zeros(1)
    evals = np.zeros(2, dtype=np.uint64)
    rc = L.vxref_tessellate(0 if engine == "fast" else 1, p.kind, p.dim, int(p.periodic),
                            _ptr(p.counts), _ptr(p.lengths), p.n_sites, _ptr(p.positions),
                            _ptr(p.times), p.growth, int(prune), int(override is not None),
                            float(override or 0.0), threads, _ptr(lab), _ptr(dist), _ptr(param),
                            _ptr(evals))
    if rc != 0:
        err = L.vxref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(err)
    return lab, dist, float(param[0]), (int(evals[0]), int(evals[1]))


def ref_prune(p: Problem):
    dropped = np.zeros(p.n_sites, dtype=np.uint8)
    rc = ref().vxref_prune(p.kind, p.dim, int(p.periodic), _ptr(p.lengths), p.n_sites,
                           _ptr(p.positions), _ptr(p.times), p.growth, _ptr(dropped))
    if rc < 0:
        raise ValueError(ref().vxref_last_error().decode())
    return dropped


def ref_generate_uniform_sites(dim, lengths, n_sites, kind, growth, horizon, seed):
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    pos = np.empty(n_sites * dim, dtype=np.float64)
    times = np.empty(n_sites, dtype=np.float64) if kind != VORONOI else None
    rc = ref().vxref_generate_uniform_sites(dim, _ptr(lengths), n_sites, kind, growth, horizon,
                                            seed & 0xFFFFFFFFFFFFFFFF, _ptr(pos), _ptr(times))
    if rc:
        raise ValueError(ref().vxref_last_error().decode())
    return pos, times


def ref_search_optimal_t0(p: Problem):
    return ref().vxref_search_optimal_t0(p.kind, p.dim, int(p.periodic), _ptr(p.counts),
                                         _ptr(p.lengths), p.n_sites, _ptr(p.positions),
                                         _ptr(p.times), p.growth)


def ref_tessellate_timed(p: Problem, threads=0, labels=False):
    """One stock tessellate_fast(sites, grid, FastOptions{}) call of the
    reference library, timed around the call alone.  Returns (seconds,
    fingerprint hex, param, labels or None)."""
    lab = np.empty(p.n_voxels, dtype=np.uint32) if labels else None
    sec = np.zeros(1)
    fp = np.zeros(1, dtype=np.uint64)
    param = np.zeros(1)
    rc = ref().vxref_tessellate_timed(p.kind, p.dim, int(p.periodic), _ptr(p.counts), _ptr(p.lengths),
                                      p.n_sites, _ptr(p.positions), _ptr(p.times), p.growth, threads,
                                      _ptr(lab), _ptr(sec), _ptr(fp), _ptr(param))
    if rc:
        raise (ValueError if rc == 1 else RuntimeError)(ref().vxref_last_error().decode())
    return float(sec[0]), "%016x" % int(fp[0]), float(param[0]), lab


def ref_ball_voxels(counts, lengths, periodic, center, radius):
    """The reference's ball_voxels (tessellate.hpp:66-68), in visit order."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    center = np.ascontiguousarray(center, dtype=np.float64)
    cap = int(np.prod(counts))
    out = np.empty(cap, dtype=np.int64)
    n = ref().vxref_ball_voxels(counts.size, int(periodic), _ptr(counts), _ptr(lengths), _ptr(center),
                                float(radius), _ptr(out), cap)
    if n < 0:
        raise ValueError(ref().vxref_last_error().decode())
    return out[:n]


def ref_spheres_to_timed(positions, radii, growth, dim=3):
    """The reference's spheres_to_timed_sites (sites.cpp:87-104): birth times."""
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    t = np.empty_like(radii)
    rc = ref().vxref_spheres_to_timed(dim, radii.size, _ptr(positions), _ptr(radii), float(growth), _ptr(t))
    if rc:
        raise ValueError(ref().vxref_last_error().decode())
    return t


def ref_have_image_io() -> bool:
    return have_ref() and bool(ref().vxref_have_image_io())


def ref_write_image(path, type_, counts, lengths, periodic, kind, n_sites, seed, data):
    """The reference's write_label_image / write_distance_image (image_io.cpp:164-175)."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    lengths = np.ascontiguousarray(lengths, dtype=np.float64)
    data = np.ascontiguousarray(data, dtype=np.uint32 if type_ == 0 else np.float64)
    rc = ref().vxref_write_image(str(path).encode(), type_, counts.size, int(periodic), _ptr(counts),
                                 _ptr(lengths), int(kind), int(n_sites), int(seed), _ptr(data))
    if rc:
        raise RuntimeError(ref().vxref_last_error().decode())


def ref_read_image(path, type_):
    """The reference's read_label_image / read_distance_image; returns
    (header dict, data) or raises RuntimeError with the reference's message."""
    hdr = np.zeros(6, dtype=np.int64)
    dims = np.zeros(16, dtype=np.int64)
    lengths = np.zeros(16, dtype=np.float64)
    rc = ref().vxref_read_image(str(path).encode(), type_, _ptr(hdr), _ptr(dims), _ptr(lengths), None, 0)
    if rc:
        raise RuntimeError(ref().vxref_last_error().decode())
    d = int(hdr[0])
    nv = int(np.prod(dims[:d]))
    data = np.empty(nv, dtype=np.uint32 if type_ == 0 else np.float64)
    rc = ref().vxref_read_image(str(path).encode(), type_, _ptr(hdr), _ptr(dims), _ptr(lengths), _ptr(data), nv)
    if rc:
        raise RuntimeError(ref().vxref_last_error().decode())
    return {"dim": d, "periodic": int(hdr[1]), "kind": int(hdr[2]), "n_sites": int(hdr[3]), "seed": int(hdr[4]),
            "format_version": int(hdr[5]), "counts": dims[:d].tolist(), "lengths": lengths[:d].tolist()}, data


# ---- BASELINE.json configs, SURVEY.md App. C recipe ----------------------
def baseline_config(k: int) -> Problem:
    """cfg k (1..5) of BASELINE.json with the App. C seeded inputs."""
    one = np.ones(3)
    seed = 1000 + k
    if k == 1:
        pos, _ = generate_uniform_sites(3, one, 1000, VORONOI, 1.0, seed)
        return Problem(VORONOI, [128] * 3, one, True, pos)
    if k == 2:
        pos, _ = generate_uniform_sites(3, one, 100000, VORONOI, 1.0, seed)
        return Problem(VORONOI, [512] * 3, one, False, pos)
    if k == 3:
        n = 50000
        pos, radii = generate_lognormal_spheres(n, 0.5 * np.cbrt(1.0 / n), 0.3, seed)
        return Problem(LAGUERRE, [512] * 3, one, True, pos, spheres_to_timed(radii, 1.0), 1.0)
    if k == 4:
        n = 20000
        pos, t = generate_uniform_sites(3, one, n, JOHNSON_MEHL, 0.5 * np.cbrt(1.0 / n), seed)
        return Problem(JOHNSON_MEHL, [512] * 3, one, True, pos, t, 1.0)
    if k == 5:
        pos, _ = generate_uniform_sites(3, one, 1000000, VORONOI, 1.0, seed)
        return Problem(VORONOI, [1000] * 3, one, True, pos)
    raise ValueError(k)


# Label fingerprints of the reference tessellate_fast on these inputs
# (measured on the reference build).
SURVEY_FINGERPRINTS = {
    1: "ebe0a0d1d95618a7",
    2: "1b03867fb131710c",
    3: "8e12fb9eddf7b6cd",
    4: "68d3e0bc73fa0e39",
    5: "931f1058f9703452",
}
