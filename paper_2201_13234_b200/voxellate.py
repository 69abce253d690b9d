"""Python mirror of the reference's engine API over the C-ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/voxellate/{geometry,sites,tessellate}.hpp, so the
parity tests read like the reference's own tests:

* ``Domain``, ``VoxelGrid``           geometry.hpp:27-78
* ``SiteSet``, ``LaguerreSpheres``    sites.hpp:15-43
* ``FastOptions``, ``TessResult``     tessellate.hpp:17-54
* ``tessellate_fast``                 tessellate.hpp:59-60   -> vx_tessellate
* ``tessellate_brute``                tessellate.hpp:47      -> vx_tessellate_brute
* ``prune_ineffective_sites``         sites.hpp:69           -> vx_prune
* ``validate_partition``              tessellate.hpp:81-84   -> vx_validate_partition
* ``generate_uniform_sites``          sites.hpp:48-49        -> vx_generate_uniform_sites
* ``spheres_to_timed_sites``          sites.hpp:53

``std::invalid_argument`` becomes ``ValueError``; device failures raise
``VxError``.  Labels come back as uint32 (the reference's type); the engine
computes int32, bit-identical for N_s < 2^31.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import VX_MAX_DIM, check, lib, stats_dict, vx_options, vx_problem, vx_stats, vx_validation


class Boundary(enum.Enum):
    Periodic = "periodic"
    NonPeriodic = "non-periodic"


class Kind(enum.IntEnum):
    Voronoi = 0
    JohnsonMehl = 1
    Laguerre = 2


K_MAX_DIM = 16
K_UNASSIGNED_LABEL = 0xFFFFFFFF


class Domain:
    """Axis-aligned box [0,L_1) x ... x [0,L_d) (geometry.hpp:27-39)."""

    def __init__(self, lengths: Sequence[float], boundary: Boundary = Boundary.Periodic):
        lengths = [float(x) for x in lengths]
        if not lengths:
            raise ValueError("domain must have at least one axis")
        if len(lengths) > K_MAX_DIM:
            raise ValueError("domain dimension exceeds supported maximum (16)")
        for L in lengths:
            if not (math.isfinite(L) and L > 0.0):
                raise ValueError("domain lengths must be positive")
        self.lengths = lengths
        self.inv_lengths = [1.0 / L for L in lengths]
        self.boundary = boundary

    def dim(self) -> int:
        return len(self.lengths)

    def volume(self) -> float:
        v = 1.0
        for L in self.lengths:
            v *= L
        return v

    def periodic(self) -> bool:
        return self.boundary == Boundary.Periodic


class VoxelGrid:
    """n_1 x ... x n_d voxels over a Domain, axis 0 fastest (geometry.hpp:41-78)."""

    def __init__(self, counts: Sequence[int], domain: Domain):
        counts = [int(n) for n in counts]
        if len(counts) != domain.dim():
            raise ValueError("grid counts must match domain dimension")
        for n in counts:
            if n < 1:
                raise ValueError("voxel counts must be positive")
        self.counts = counts
        self.domain = domain
        self.spacing = [L / float(n) for L, n in zip(domain.lengths, counts)]

    def dim(self) -> int:
        return len(self.counts)

    def voxel_count(self) -> int:
        n = 1
        for c in self.counts:
            n *= c
        return n

    def center_coord(self, axis: int, k: int) -> float:
        return (float(k) + 0.5) * self.spacing[axis]

    def linear_index(self, idx: Sequence[int]) -> int:
        lin = 0
        for i in range(self.dim() - 1, -1, -1):
            lin = lin * self.counts[i] + int(idx[i])
        return lin

    def decompose(self, linear: int):
        out = []
        for n in self.counts:
            out.append(linear % n)
            linear //= n
        return out


@dataclass
class SiteSet:
    """Sites, xyz-interleaved positions; times for JM/Laguerre (sites.hpp:15-31)."""

    kind: Kind = Kind.Voronoi
    dim: int = 0
    positions: np.ndarray = field(default_factory=lambda: np.zeros(0))
    times: Optional[np.ndarray] = None
    growth: float = 0.0

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1)
        if self.times is not None:
            self.times = np.ascontiguousarray(self.times, dtype=np.float64).reshape(-1)

    def count(self) -> int:
        return 0 if self.dim == 0 else self.positions.size // self.dim

    def timed(self) -> bool:
        return self.kind != Kind.Voronoi

    def pos(self, s: int) -> np.ndarray:
        return self.positions[s * self.dim:(s + 1) * self.dim]


@dataclass
class LaguerreSpheres:
    dim: int
    positions: np.ndarray
    radii: np.ndarray


@dataclass
class FastOptions:
    """tessellate.hpp:49-54"""

    override_param: Optional[float] = None
    prune: bool = True


@dataclass
class LabelImage:
    grid: VoxelGrid
    labels: np.ndarray


@dataclass
class DistanceImage:
    grid: VoxelGrid
    values: np.ndarray


@dataclass
class EvalCounters:
    """This engine's evaluation counts (ball phase, shell phase)."""

    step1_evals: int = 0
    step2_evals: int = 0

    def total(self) -> int:
        return self.step1_evals + self.step2_evals


@dataclass
class TessResult:
    labels: LabelImage
    distances: Optional[DistanceImage]
    counters: EvalCounters
    param: float = float("nan")
    histogram: Optional[np.ndarray] = None
    stats: Optional[dict] = None


@dataclass
class PruneResult:
    sites: SiteSet
    removed: list
    kept: list


@dataclass
class ValidationReport:
    voxels_checked: int = 0
    label_mismatches: int = 0
    value_mismatches: int = 0
    examples: list = field(default_factory=list)

    def ok(self) -> bool:
        return self.label_mismatches == 0 and self.value_mismatches == 0


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _problem(sites: SiteSet, grid: VoxelGrid) -> vx_problem:
    if sites.dim != grid.dim():
        raise ValueError("site dimension does not match the domain")
    if sites.count() < 1:
        raise ValueError("site set must contain at least one site")
    if sites.positions.size != sites.count() * sites.dim:
        raise ValueError("site position array has inconsistent size")
    if sites.timed() and (sites.times is None or sites.times.size != sites.count()):
        raise ValueError("timed site set must carry one birth time per site")
    P = vx_problem()
    P.kind = int(sites.kind)
    P.dim = grid.dim()
    P.periodic = 1 if grid.domain.periodic() else 0
    for i in range(grid.dim()):
        P.counts[i] = grid.counts[i]
        P.lengths[i] = grid.domain.lengths[i]
    P.n_sites = sites.count()
    P.positions = _ptr(sites.positions)
    P.times = _ptr(sites.times) if sites.timed() else None
    P.weights = None
    P.growth = float(sites.growth) if sites.timed() else 0.0
    return P


def _run(engine: str, sites: SiteSet, grid: VoxelGrid, options: Optional[FastOptions],
         distances: bool, histogram: bool, slab, device, ball_scale, context=None, out=None,
         profile=False, n_gpus=None, histogram_out=None) -> TessResult:
    P = _problem(sites, grid)
    O = vx_options()
    lib().vx_options_init(C.byref(O))
    if options is not None:
        O.prune = 1 if options.prune else 0
        if options.override_param is not None:
            O.has_override = 1
            O.override_param = float(options.override_param)
    if device is not None:
        O.device = int(device)
    if ball_scale is not None:
        O.ball_scale = float(ball_scale)
    if n_gpus is not None:
        O.n_gpus = int(n_gpus)
    zb, ze = (0, grid.counts[-1]) if slab is None else (int(slab[0]), int(slab[1]))
    O.slab_begin, O.slab_end = zb, ze
    plane = grid.voxel_count() // grid.counts[-1]
    nvs = plane * (ze - zb)
    if out is not None:  # caller-provided (e.g. pinned) label buffer
        if out.dtype not in (np.int32, np.uint32):
            raise ValueError("out must hold int32 or uint32 labels")
        labels = out.reshape(-1).view(np.int32)
        if labels.size != nvs or not labels.flags.c_contiguous:
            raise ValueError("out must be a contiguous buffer of the labelled voxel count")
    else:
        labels = np.empty(nvs, dtype=np.int32)
    O.profile_stages = 1 if profile else 0
    dist = np.empty(nvs, dtype=np.float64) if distances else None
    if histogram_out is not None:  # caller-provided (e.g. pinned) histogram buffer
        if histogram_out.dtype not in (np.uint64, np.int64):
            raise ValueError("histogram_out must hold uint64 or int64 counts")
        hist = histogram_out.reshape(-1).view(np.uint64)
        if hist.size != sites.count() or not hist.flags.c_contiguous:
            raise ValueError("histogram_out must be a contiguous buffer of one count per site")
    else:
        hist = np.zeros(sites.count(), dtype=np.uint64) if histogram else None
    O.distances_out = _ptr(dist)
    O.histogram_out = _ptr(hist)
    st = vx_stats()
    fn = lib().vx_tessellate if engine == "fast" else lib().vx_tessellate_brute
    check(fn(context, C.byref(P), C.byref(O), _ptr(labels), C.byref(st)))
    counters = EvalCounters(int(st.ball_evals), int(st.shell_evals))
    stats = stats_dict(st)
    return TessResult(LabelImage(grid, labels.view(np.uint32)),
                      DistanceImage(grid, dist) if dist is not None else None, counters,
                      float(st.param) if engine == "fast" else float("nan"), hist, stats)


def tessellate_fast(sites: SiteSet, grid: VoxelGrid, options: Optional[FastOptions] = None, *,
                    distances: bool = True, histogram: bool = False, slab=None, device=None,
                    ball_scale=None, context=None, out=None, profile=False, n_gpus=None,
                    histogram_out=None) -> TessResult:
    """Two-step engine on the GPU (tessellate.cpp:195-282).  ``slab=(z0, z1)``
    labels only last-axis planes [z0, z1) (the multi-GPU decomposition);
    ``out`` / ``histogram_out`` receive the labels / grain volumes (e.g. pinned
    host buffers; the latter implies ``histogram``); ``n_gpus`` splits the call
    over that many devices from one process."""
    return _run("fast", sites, grid, options or FastOptions(), distances, histogram, slab, device,
                ball_scale, context, out, profile, n_gpus, histogram_out)


def tessellate_brute(sites: SiteSet, grid: VoxelGrid, *, distances: bool = True,
                     histogram: bool = False, slab=None, device=None, context=None) -> TessResult:
    """Every voxel scans every site, on the GPU (tessellate.cpp:184-193)."""
    return _run("brute", sites, grid, None, distances, histogram, slab, device, None, context)


def prune_ineffective_sites(sites: SiteSet, domain: Domain, context=None) -> PruneResult:
    """sites.cpp:113-171 on the GPU; same predicate, same survivors."""
    if not sites.timed():
        raise ValueError("pruning applies to timed tessellations only")
    grid = VoxelGrid([1] * domain.dim(), domain)
    P = _problem(sites, grid)
    dropped = np.zeros(sites.count(), dtype=np.uint8)
    nrem = C.c_int64(0)
    check(lib().vx_prune(context, C.byref(P), _ptr(dropped), C.byref(nrem)))
    kept = np.nonzero(dropped == 0)[0]
    removed = np.nonzero(dropped)[0]
    d = sites.dim
    pos = sites.positions.reshape(-1, d)[kept].reshape(-1)
    out = SiteSet(sites.kind, d, pos, sites.times[kept], sites.growth)
    return PruneResult(out, removed.tolist(), kept.tolist())


def validate_partition(labels: LabelImage, distances: Optional[DistanceImage], sites: SiteSet,
                       sample: int = 0, seed: int = 0, context=None) -> ValidationReport:
    """Independent re-check (tessellate.cpp:304-367): `sample` voxels drawn by
    mt19937_64(seed) exactly like the reference, or every voxel when 0."""
    grid = labels.grid
    nv = grid.voxel_count()
    lab = np.ascontiguousarray(labels.labels).view(np.int32).reshape(-1)
    if lab.size != nv:
        raise ValueError("label image size does not match its grid")
    dist = None
    if distances is not None:
        dist = np.ascontiguousarray(distances.values, dtype=np.float64).reshape(-1)
        if dist.size != nv:
            raise ValueError("distance image size does not match the label image")
    P = _problem(sites, grid)
    rep = vx_validation()
    check(lib().vx_validate_partition(context, C.byref(P), _ptr(lab), _ptr(dist), int(sample),
                                      int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(rep)))
    return ValidationReport(rep.voxels_checked, rep.label_mismatches, rep.value_mismatches,
                            [rep.examples[i] for i in range(rep.n_examples)])


def generate_uniform_sites(domain: Domain, n_sites: int, kind: Kind, growth: float,
                           time_horizon: float, seed: int) -> SiteSet:
    """sites.cpp:61-85 (std::mt19937_64, per site d coordinates then a time)."""
    d = domain.dim()
    lengths = np.array(domain.lengths, dtype=np.float64)
    pos = np.empty(int(n_sites) * d, dtype=np.float64)
    times = np.empty(int(n_sites), dtype=np.float64) if kind != Kind.Voronoi else None
    check(lib().vx_generate_uniform_sites(d, _ptr(lengths), int(n_sites), int(kind), float(growth),
                                          float(time_horizon), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                          _ptr(pos), _ptr(times)))
    return SiteSet(Kind(kind), d, pos, times, float(growth) if kind != Kind.Voronoi else 0.0)


def spheres_to_timed_sites(spheres: LaguerreSpheres, growth: float) -> SiteSet:
    """t_s = -(r_s * r_s) / G (sites.cpp:87-104)."""
    if not growth > 0.0:
        raise ValueError("growth rate G must be positive")
    r = np.ascontiguousarray(spheres.radii, dtype=np.float64)
    if r.size < 1:
        raise ValueError("sphere set must contain at least one sphere")
    if np.any(~(r >= 0.0)):
        raise ValueError("sphere radii must be nonnegative")
    return SiteSet(Kind.Laguerre, spheres.dim, spheres.positions, -(r * r) / growth, float(growth))


def ball_voxels(center: Sequence[float], radius: float, grid: VoxelGrid) -> np.ndarray:
    """Every voxel whose centre lies within ``radius`` of ``center``, once, in
    the reference's visit order (tessellate.hpp:62-68): per axis the indices of
    a conservative window ((c -/+ r (1 + 1e-9)) / h - 0.5 rounded outwards with
    a relative slack; periodic windows wrap, one spanning the whole axis lists
    each index once) with their squared (periodic: wrapped) residuals, folded
    from the last axis to axis 0 (geometry.hpp:106-123); the last axis varies
    slowest.  A voxel is kept iff dsq <= radius^2.  numpy evaluates each
    operation separately rounded, like the reference build."""
    d = grid.dim()
    center = np.asarray(center, dtype=np.float64)
    if center.size != d:
        raise ValueError("ball center dimension does not match the grid")
    radius = float(radius)
    if not (np.isfinite(radius) and radius >= 0.0):
        raise ValueError("ball radius must be nonnegative")
    rp = radius * (1.0 + 1e-9)
    per = grid.domain.periodic()
    idx, sq, stride = [], [], []
    st = 1
    for a in range(d):
        n = int(grid.counts[a])
        stride.append(st)
        st *= n
        h = grid.spacing[a] if hasattr(grid, "spacing") else grid.domain.lengths[a] / n
        L = float(grid.domain.lengths[a])
        lo_t = (center[a] - rp) / h - 0.5
        hi_t = (center[a] + rp) / h - 0.5
        slack = 1e-9 * (abs(lo_t) + abs(hi_t) + 1.0)
        klo, khi = np.ceil(lo_t - slack), np.floor(hi_t + slack)
        if khi < klo:
            return np.empty(0, dtype=np.int64)
        if per:
            ks = np.arange(n) if khi - klo + 1.0 >= n else np.mod(np.arange(int(klo), int(khi) + 1), n)
        else:
            a0 = 0 if klo <= 0.0 else int(min(klo, float(n)))
            a1 = n - 1 if khi >= float(n - 1) else int(max(khi, -1.0))
            ks = np.arange(a0, a1 + 1)
        if ks.size == 0:
            return np.empty(0, dtype=np.int64)
        w = center[a] - (ks.astype(np.float64) + 0.5) * h
        if per:
            w = w - np.floor(w * grid.domain.inv_lengths[a] + 0.5) * L
        idx.append(ks.astype(np.int64))
        sq.append(w * w)
    acc, lin = sq[d - 1], idx[d - 1] * stride[d - 1]
    for a in range(d - 2, -1, -1):
        acc = np.add.outer(acc, sq[a])
        lin = np.add.outer(lin, idx[a] * stride[a])
    acc, lin = acc.reshape(-1), lin.reshape(-1)
    return lin[acc <= radius * radius].astype(np.int64)


def scan_ball(center: Sequence[float], radius: float, grid: VoxelGrid, visit) -> None:
    """tessellate.hpp:62-65: calls visit(linear_index) for every voxel of
    ball_voxels(center, radius, grid), in the same order."""
    for v in ball_voxels(center, radius, grid):
        visit(int(v))


def optimal_r0(n_sites: int, domain: Domain) -> float:
    """radius_from_volume(optimal_v0(N_s, V), d) (cost.cpp:28-39)."""
    out = C.c_double(0.0)
    lengths = np.array(domain.lengths, dtype=np.float64)
    check(lib().vx_optimal_r0(int(n_sites), domain.dim(), _ptr(lengths), C.byref(out)))
    return out.value


def slab_bounds(n_last: int, rank: int, world: int):
    """z-slab of rank `rank` of `world` (tessellate.cpp:120-121)."""
    b, e = C.c_int64(0), C.c_int64(0)
    lib().vx_slab_bounds(int(n_last), int(rank), int(world), C.byref(b), C.byref(e))
    return b.value, e.value


# ---- on-disk images (row f2; reference include/voxellate/image_io.hpp:17-29) ----

@dataclass
class ImageMeta:
    """image_io.hpp:13-19"""

    format_version: int = 1
    type: str = ""
    kind: Kind = Kind.Voronoi
    n_sites: int = 0
    seed: int = -1


def _grid_arrays(grid: VoxelGrid):
    counts = np.ascontiguousarray(grid.counts, dtype=np.int64)
    lengths = np.ascontiguousarray(grid.domain.lengths, dtype=np.float64)
    return counts, lengths


def _write_image(path: str, image, meta: ImageMeta, type_: int, data: np.ndarray) -> None:
    counts, lengths = _grid_arrays(image.grid)
    data = np.ascontiguousarray(data)
    if data.size != image.grid.voxel_count():
        raise ValueError("image payload size disagrees with its grid")
    check(lib().vx_write_image(str(path).encode(), type_, image.grid.dim(), _ptr(counts), _ptr(lengths),
                               1 if image.grid.domain.periodic() else 0, int(meta.kind), int(meta.n_sites),
                               int(meta.seed), _ptr(data)))


def write_label_image(path: str, image: LabelImage, meta: ImageMeta) -> None:
    """Raw little-endian u32 labels, axis 0 fastest, + ``<path>.json`` (image_io.cpp:164-168)."""
    _write_image(path, image, meta, 0, np.asarray(image.labels).view(np.uint32))


def write_distance_image(path: str, image: DistanceImage, meta: ImageMeta) -> None:
    """Raw little-endian f64 values + ``<path>.json`` (image_io.cpp:170-175)."""
    _write_image(path, image, meta, 1, np.asarray(image.values, dtype=np.float64))


def _read_image(path: str, type_: int):
    hdr = np.zeros(6, dtype=np.int64)
    counts = np.zeros(VX_MAX_DIM, dtype=np.int64)
    lengths = np.zeros(VX_MAX_DIM, dtype=np.float64)
    check(lib().vx_read_image(str(path).encode(), type_, _ptr(hdr), _ptr(counts), _ptr(lengths), None, 0))
    d = int(hdr[0])
    grid = VoxelGrid([int(c) for c in counts[:d]],
                     Domain([float(x) for x in lengths[:d]],
                            Boundary.Periodic if hdr[1] else Boundary.NonPeriodic))
    data = np.empty(grid.voxel_count(), dtype=np.uint32 if type_ == 0 else np.float64)
    check(lib().vx_read_image(str(path).encode(), type_, _ptr(hdr), _ptr(counts), _ptr(lengths), _ptr(data),
                              data.size))
    meta = ImageMeta(int(hdr[5]), "labels" if type_ == 0 else "distances", Kind(int(hdr[2])), int(hdr[3]),
                     int(hdr[4]))
    return grid, data, meta


def read_label_image(path: str):
    """(LabelImage, ImageMeta) with the reference's sidecar/payload checks (image_io.cpp:177-189)."""
    grid, data, meta = _read_image(path, 0)
    return LabelImage(grid, data), meta


def read_distance_image(path: str):
    """(DistanceImage, ImageMeta), image_io.cpp:191-202."""
    grid, data, meta = _read_image(path, 1)
    return DistanceImage(grid, data), meta


def tessellate_to_files(sites: SiteSet, grid: VoxelGrid, label_path: str, distance_path: Optional[str] = None,
                        options: Optional[FastOptions] = None, *, seed: int = -1, device=None,
                        context=None) -> dict:
    """tessellate_fast + write_label_image (+ write_distance_image), as the
    reference's run() does (run.cpp:121-150), streaming each z-chunk of the
    image out of device memory into the files while later chunks compute.
    Returns the call's stats."""
    P = _problem(sites, grid)
    O = vx_options()
    lib().vx_options_init(C.byref(O))
    options = options or FastOptions()
    O.prune = 1 if options.prune else 0
    if options.override_param is not None:
        O.has_override = 1
        O.override_param = float(options.override_param)
    if device is not None:
        O.device = int(device)
    st = vx_stats()
    check(lib().vx_tessellate_to_files(context, C.byref(P), C.byref(O), str(label_path).encode(),
                                       None if distance_path is None else str(distance_path).encode(),
                                       int(seed), C.byref(st)))
    return stats_dict(st)
