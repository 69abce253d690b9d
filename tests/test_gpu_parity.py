"""GPU parity: the CUDA engine through the C-ABI vs the oracle and the
reference's golden fixtures.  Bit-exact labels AND f64 values everywhere
(integer/index work; the f64 values are the reference's own expressions).

Restates the reference's pinning tests:
test_tessellate.cpp:55-86 (hand-checked), :178-216 and acceptance.cpp:49-113
(fast == brute bitwise over random instances), :218-246 (extreme r0), :292-310
(equal birth times -> Voronoi), :312-341 (validate_partition), :343-363
(worker-count independence -> slab/GPU-count independence), test_sites.cpp
:125-143,173-194 (coincident sites, prune preserves partitions),
test_tessellate.cpp:248-269 (step 1 covers exactly the union of the balls),
:365-387 (grid refinement keeps labels at shared centres), lattice instances
full of exact ties, plus the five BASELINE configs against the reference's
label fingerprints (App. B).
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, fixture_names, fixture_problem, load_fixture, to_vx

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def run_fast(p, **kw):
    import paper_2201_13234_b200 as vx

    sites, grid = to_vx(p)
    opts = vx.FastOptions(override_param=kw.pop("override", None), prune=kw.pop("prune", True))
    return vx.tessellate_fast(sites, grid, opts, **kw)


def run_brute(p, **kw):
    import paper_2201_13234_b200 as vx

    sites, grid = to_vx(p)
    return vx.tessellate_brute(sites, grid, **kw)


@pytest.mark.parametrize("name", fixture_names("tess_"))
def test_golden_fixtures(name):
    fx = load_fixture(name)
    p = fixture_problem(fx)
    ov = float(fx["override"])
    r = run_fast(p, prune=bool(fx["prune"]), override=None if np.isnan(ov) else ov)
    assert np.array_equal(r.labels.labels, fx["labels"])
    assert np.array_equal(bits(r.distances.values), bits(fx["values"]))
    if p.kind == 0 and np.isnan(ov):
        assert r.param == float(fx["param"])  # Voronoi r0 is the reference's value
    if p.kind == 0 or not bool(fx["prune"]):
        b = run_brute(p)  # tessellate_brute has no prune
        assert np.array_equal(b.labels.labels, fx["labels"])
        assert np.array_equal(bits(b.distances.values), bits(fx["values"]))


@pytest.mark.parametrize("name", fixture_names("prune_"))
def test_prune_matches_reference(name):
    import paper_2201_13234_b200 as vx

    fx = load_fixture(name)
    p = fixture_problem(fx)
    sites, grid = to_vx(p)
    pr = vx.prune_ineffective_sites(sites, grid.domain)
    assert np.array_equal(np.isin(np.arange(p.n_sites), pr.removed).astype(np.uint8), fx["dropped"])
    assert pr.kept == sorted(pr.kept)


def random_instance(rng, i, big=False):
    import oracle

    d = 1 + i % 4
    kind = (i // 4) % 3
    periodic = (i // 12) % 2 == 1
    if big:
        d = 3
    L = rng.uniform(0.5, 2.0, d)
    cap = {1: 512, 2: 48, 3: 16, 4: 8}[d]
    counts = [64, 64, 64] if big else list(rng.integers(2, cap + 1, d))
    ns = 1 if i % 37 == 0 else int(rng.integers(1, 500))
    G = float(np.exp(rng.uniform(np.log(0.1), np.log(10.0)))) if kind else 0.0
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, float(rng.uniform(0.5, 2.0)),
                                           int(rng.integers(1 << 62)))
    return oracle.Problem(kind, counts, L, periodic, pos, t, G)


def test_random_instances_fast_equals_brute_equals_oracle(oracle_mod):
    """acceptance.cpp:49-113 (criterion 1) restated: 200 seeded instances."""
    rng = np.random.default_rng(20260814)
    bad = []
    for i in range(200):
        p = random_instance(rng, i, big=(i % 50 == 13))
        override = None
        if i % 7 == 0:
            override = (float(np.exp(rng.uniform(np.log(0.02), np.log(2.0)))) if p.kind == 0
                        else float(p.times.min() + rng.uniform(0.0, 1.5)))
        prune = i % 2 == 0
        f = run_fast(p, prune=prune, override=override)
        b = run_brute(p)
        lab, dist = oracle_mod.brute(p)
        if prune and p.kind != 0:  # the reference labels the prune survivors
            dropped = oracle_mod.prune(p)
            if dropped.any():
                keep = np.nonzero(dropped == 0)[0]
                q = oracle_mod.Problem(p.kind, p.counts, p.lengths, p.periodic,
                                       p.positions.reshape(-1, p.dim)[keep].reshape(-1),
                                       p.times[keep], p.growth)
                l2, dist = oracle_mod.brute(q)
                lab = keep[l2].astype(np.uint32)
        ok = (np.array_equal(f.labels.labels, lab) and np.array_equal(bits(f.distances.values), bits(dist))
              and np.array_equal(b.labels.labels, oracle_mod.brute(p)[0]))
        if not ok:
            bad.append((i, p.dim, p.kind, p.periodic, p.n_sites))
    assert not bad, bad


def test_hand_checked():
    import oracle

    r = run_fast(oracle.Problem(0, [8], [1.0], True, [0.25, 0.75]))
    assert r.labels.labels.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    assert abs(r.distances.values[0] - 0.1875) < 1e-14 and abs(r.distances.values[7] - 0.1875) < 1e-14
    r = run_brute(oracle.Problem(0, [4, 4], [1.0, 2.0], False, [0.3, 0.4]))
    assert (r.labels.labels == 0).all() and r.stats["shell_evals"] == 16


@pytest.mark.parametrize("periodic", [True, False])
def test_extreme_radii_give_identical_output(oracle_mod, periodic):
    """test_tessellate.cpp:218-246: r0 = 1e9 / 1e-12 / cover -> same image."""
    pos, _ = oracle_mod.generate_uniform_sites(2, np.array([1.3, 0.9]), 7, 0, 1.0, 31)
    p = oracle_mod.Problem(0, [9, 8], [1.3, 0.9], periodic, pos)
    lab, dist = oracle_mod.brute(p)
    for r0 in (1e9, 1e-12, 0.5 * np.sqrt(1.3 ** 2 + 0.9 ** 2) * 1.001):
        r = run_fast(p, override=r0)
        assert np.array_equal(r.labels.labels, lab) and np.array_equal(bits(r.distances.values), bits(dist))
    r = run_fast(p, override=1e-12)
    assert r.stats["n_unresolved"] == p.n_voxels  # no ball reaches a voxel: all go to the shell


def test_ball_radius_independence(oracle_mod):
    """Labels never depend on the investigation radius."""
    p = oracle_mod.baseline_config(1)
    base = run_fast(p, distances=False).labels.labels
    for scale in (0.3, 0.7, 1.5, 3.0):
        r = run_fast(p, distances=False, ball_scale=scale)
        assert np.array_equal(r.labels.labels, base)


def test_equal_birth_times_degenerate_to_voronoi(oracle_mod):
    """test_tessellate.cpp:292-310."""
    rng = np.random.default_rng(404)
    for trial in range(10):
        d = 1 + trial % 3
        L = rng.uniform(0.5, 2.0, d)
        counts = list(rng.integers(2, {1: 64, 2: 16, 3: 8}[d] + 1, d))
        pos, _ = oracle_mod.generate_uniform_sites(d, L, 15, 0, 1.0, int(rng.integers(1 << 60)))
        periodic = trial % 2 == 1
        ref = run_brute(oracle_mod.Problem(0, counts, L, periodic, pos)).labels.labels
        for kind in (1, 2):
            t = np.full(15, rng.uniform(-1.0, 1.0))
            p = oracle_mod.Problem(kind, counts, L, periodic, pos, t, float(np.exp(rng.uniform(np.log(0.2), np.log(5.0)))))
            assert np.array_equal(run_fast(p).labels.labels, ref)


def test_coincident_sites_lower_index_wins(oracle_mod):
    """test_sites.cpp:125-143: exact ties keep the lower index."""
    for kind in (0, 1, 2):
        pos = np.array([0.5, 0.5, 0.5, 0.5, 0.25, 0.75, 0.25, 0.75])
        t = np.array([0.3, 0.3, 0.1, 0.1]) if kind else None
        p = oracle_mod.Problem(kind, [10, 9], [1.0, 1.0], True, pos, t, 1.0 if kind else 0.0)
        lab, dist = oracle_mod.brute(p)
        for prune in (True, False):
            r = run_fast(p, prune=prune)
            assert np.array_equal(r.labels.labels, lab)
            assert 1 not in r.labels.labels and 3 not in r.labels.labels


def test_prune_on_off_same_partition(oracle_mod):
    """test_sites.cpp:173-194 / acceptance.cpp:389-436 restated on the GPU."""
    rng = np.random.default_rng(37)
    for trial in range(24):
        kind = 1 if trial % 2 else 2
        periodic = (trial // 2) % 2 == 0
        L = rng.uniform(0.5, 2.0, 2)
        ns = 5 + int(rng.integers(60))
        pos, t = oracle_mod.generate_uniform_sites(2, L, ns, kind, 1.0, int(rng.integers(1 << 60)))
        p = oracle_mod.Problem(kind, [48, 48], L, periodic, pos, t,
                               float(np.exp(rng.uniform(np.log(0.2), np.log(10.0)))))
        a = run_fast(p, prune=True)
        b = run_fast(p, prune=False)
        assert np.array_equal(a.labels.labels, b.labels.labels)
        dropped = oracle_mod.prune(p)
        for s in np.nonzero(dropped)[0]:
            assert s not in a.labels.labels


def test_validate_partition_detects_tampering(oracle_mod):
    """test_tessellate.cpp:312-341."""
    import paper_2201_13234_b200 as vx

    pos, t = oracle_mod.generate_uniform_sites(2, np.array([1.0, 1.3]), 30, 2, 1.0, 123)
    p = oracle_mod.Problem(2, [24, 20], [1.0, 1.3], True, pos, t, 1.7)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid)
    full = vx.validate_partition(r.labels, r.distances, sites)
    assert full.ok() and full.voxels_checked == grid.voxel_count()
    sampled = vx.validate_partition(r.labels, r.distances, sites, 100, 9)
    assert sampled.ok() and sampled.voxels_checked == 100
    victim = 173
    tampered = vx.LabelImage(grid, r.labels.labels.copy())
    tampered.labels[victim] = (tampered.labels[victim] + 1) % sites.count()
    bad = vx.validate_partition(tampered, r.distances, sites)
    assert bad.label_mismatches == 1 and bad.value_mismatches == 0 and bad.examples == [victim]
    dented = vx.DistanceImage(grid, r.distances.values.copy())
    dented.values[victim] += 1e-3
    bad = vx.validate_partition(r.labels, dented, sites)
    assert bad.label_mismatches == 0 and bad.value_mismatches == 1
    # the sampled voxel set is the reference's draw (mt19937_64 + libstdc++)
    idx = oracle_mod.sample_indices(grid.voxel_count(), 100, 9)
    bad = vx.validate_partition(tampered, None, sites, 100, 9)
    assert bad.label_mismatches == int(np.count_nonzero(idx == victim))


def test_slab_and_histogram_independence(oracle_mod):
    """Worker-count independence (test_tessellate.cpp:343-363) -> GPU-count
    independence: slabs concatenate to the full image, bit for bit."""
    import paper_2201_13234_b200 as vx

    pos, t = oracle_mod.generate_uniform_sites(3, np.array([1.0, 1.0, 1.0]), 300, 1, 0.1, 808)
    p = oracle_mod.Problem(1, [40, 36, 45], [1.0, 1.0, 1.0], True, pos, t, 1.0)
    full = run_fast(p, histogram=True)
    assert full.histogram.sum() == p.n_voxels
    assert np.array_equal(full.histogram, np.bincount(full.labels.labels, minlength=p.n_sites))
    for world in (2, 3, 8):
        parts, dists, hist = [], [], np.zeros(p.n_sites, dtype=np.uint64)
        for r in range(world):
            z0, z1 = vx.slab_bounds(45, r, world)
            s = run_fast(p, histogram=True, slab=(z0, z1))
            parts.append(s.labels.labels)
            dists.append(s.distances.values)
            hist += s.histogram
        assert np.array_equal(np.concatenate(parts), full.labels.labels)
        assert np.array_equal(bits(np.concatenate(dists)), bits(full.distances.values))
        assert np.array_equal(hist, full.histogram)


def test_weights_equal_times(oracle_mod):
    """Laguerre input as weights w = r^2 (t = -(w)/G, sites.cpp:101)."""
    import paper_2201_13234_b200 as vx
    from paper_2201_13234_b200._lib import check, lib, vx_options, vx_problem

    pos, radii = oracle_mod.generate_lognormal_spheres(400, 0.05, 0.3, 5)
    G = 1.7
    t = oracle_mod.spheres_to_timed(radii, G)
    p = oracle_mod.Problem(2, [30, 31, 32], [1.0, 1.0, 1.0], True, pos, t, G)
    ref = run_fast(p, distances=False).labels.labels
    w = radii * radii
    P = vx_problem()
    P.kind, P.dim, P.periodic = 2, 3, 1
    for i in range(3):
        P.counts[i], P.lengths[i] = p.counts[i], 1.0
    P.n_sites = 400
    P.positions = pos.ctypes.data
    P.weights = w.ctypes.data
    P.growth = G
    out = np.empty(p.n_voxels, dtype=np.int32)
    check(lib().vx_tessellate(None, C.byref(P), None, out.ctypes.data_as(C.c_void_p), None))
    assert np.array_equal(out.view(np.uint32), ref)


def test_device_pointer_path_matches_host(oracle_mod):
    import torch

    from paper_2201_13234_b200.engine import Tessellator

    p = oracle_mod.baseline_config(1)
    host = run_fast(p, histogram=True)
    eng = Tessellator(0)
    pos = torch.from_numpy(p.positions).cuda()
    lab = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
    hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
    dist = torch.empty(p.n_voxels, dtype=torch.float64, device="cuda")
    st = eng.run(kind=0, counts=list(p.counts), lengths=list(p.lengths), periodic=True, positions=pos,
                 labels=lab, histogram=hist, distances=dist,
                 stream=torch.cuda.current_stream().cuda_stream, profile=True)
    assert np.array_equal(lab.cpu().numpy().view(np.uint32), host.labels.labels)
    assert np.array_equal(bits(dist.cpu().numpy()), bits(host.distances.values))
    assert np.array_equal(hist.cpu().numpy().astype(np.uint64), host.histogram)
    assert st["stage_ms"]["ball"] > 0.0
    eng.close()


def test_high_dimension_uses_the_fast_engine(oracle_mod):
    """d >= 4 runs the d-dimensional gather engine (ballnd.cu), not brute force."""
    rng = np.random.default_rng(5)
    for kind in (0, 1, 2):
        pos, t = oracle_mod.generate_uniform_sites(4, np.array([1.0, 0.7, 1.3, 0.9]), 23, kind, 0.7,
                                                   int(rng.integers(1 << 60)))
        p = oracle_mod.Problem(kind, [5, 4, 6, 3], [1.0, 0.7, 1.3, 0.9], kind != 1, pos, t, 1.3)
        lab, dist = oracle_mod.brute(p)
        r = run_fast(p, prune=False)
        assert r.stats["engine"] == 0
        assert np.array_equal(r.labels.labels, lab) and np.array_equal(bits(r.distances.values), bits(dist))


@pytest.mark.parametrize("d", [1, 2, 4, 5, 6, 7, 9])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_nd_engine_vs_reference(d, kind):
    """The d != 3 engine against the reference library (oracle/_ref) on random
    instances: both boundaries, prune on/off, an override parameter, densities
    from ~1.5 to ~15 voxels per site per axis, anisotropic lengths; labels, f64
    distances and histogram bit for bit."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(100 * d + kind)
    tgt = {1: 40000, 2: 90000, 4: 90000, 5: 60000, 6: 60000, 7: 30000, 9: 20000}[d]
    for it in range(4):
        L = rng.uniform(0.5, 2.0, d)
        counts = [max(1, int(tgt ** (1.0 / d) * np.exp(rng.uniform(-0.4, 0.4)))) for _ in range(d)]
        nv = int(np.prod(counts))
        spacing = float(np.exp(rng.uniform(np.log(1.5), np.log(15.0))))
        ns = int(np.clip(nv / spacing ** d, 1, 4000))
        horizon = float(0.5 * np.prod(L) ** (1.0 / d) / ns ** (1.0 / d))
        pos, t = oracle.generate_uniform_sites(d, L, ns, kind, horizon, int(rng.integers(1 << 40)))
        G = [0.0, float(np.exp(rng.uniform(-1, 1))), float(np.exp(rng.uniform(-1, 1)))][kind]
        p = oracle.Problem(kind, counts, L, it % 2 == 0, pos, t, G)
        prune = it != 1
        override = None
        if it == 3:
            _, _, param, _ = oracle.ref_tessellate(p, prune=prune, distances=False)
            override = param * 0.7 if kind == 0 else float(np.min(t) + 0.7 * (param - np.min(t)))
        lab, dist, _, _ = oracle.ref_tessellate(p, prune=prune, override=override)
        sites, grid = to_vx(p)
        r = vx.tessellate_fast(sites, grid, vx.FastOptions(override_param=override, prune=prune), distances=True,
                               histogram=True)
        assert r.stats["engine"] == 0
        assert np.array_equal(r.labels.labels, lab), (it, int((r.labels.labels != lab).sum()))
        assert np.array_equal(bits(r.distances.values), bits(dist)), it
        assert np.array_equal(r.histogram, np.bincount(lab, minlength=ns).astype(np.uint64)), it


@pytest.mark.parametrize("d", [1, 2, 4])
def test_nd_slabs_concatenate_to_the_whole_image(oracle_mod, d):
    """Slabs of the last axis through the d != 3 engine (the multi-GPU
    decomposition): concatenated, they equal the whole image; histograms add."""
    import paper_2201_13234_b200 as vx

    rng = np.random.default_rng(7 + d)
    counts = {1: [3000], 2: [90, 77], 4: [9, 8, 10, 11]}[d]
    L = rng.uniform(0.6, 1.6, d)
    pos, t = oracle_mod.generate_uniform_sites(d, L, 300, 1, 0.05, 17)
    p = oracle_mod.Problem(1, counts, L, True, pos, t, 1.1)
    lab, _ = oracle_mod.brute(p, distances=False)
    sites, grid = to_vx(p)
    n = counts[-1]
    parts, hist = [], np.zeros(300, dtype=np.uint64)
    for a, b in ((0, n // 3), (n // 3, n // 3 + 1), (n // 3 + 1, n)):
        r = vx.tessellate_fast(sites, grid, distances=False, histogram=True, slab=(a, b))
        parts.append(np.asarray(r.labels.labels))
        hist += r.histogram
    assert np.array_equal(np.concatenate(parts), lab)
    assert np.array_equal(hist, np.bincount(lab, minlength=300).astype(np.uint64))


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_baseline_config_fingerprints(oracle_mod, k):
    """Zero mismatched voxels on the five BASELINE configs: the label
    fingerprint equals the reference's, and the whole label
    image equals the one the reference library (oracle/_ref, stock
    tessellate_fast) produces on this host -- cfg1 also against the oracle's
    brute force -- with the histogram equal to the bincount of its labels."""
    import paper_2201_13234_b200 as vx

    p = oracle_mod.baseline_config(k)
    r = run_fast(p, distances=False, histogram=True)
    lab = np.ascontiguousarray(r.labels.labels).view(np.int32)
    fp = "%016x" % vx.lib().vx_label_fingerprint(lab.ctypes.data_as(C.c_void_p), lab.size)
    assert fp == oracle_mod.SURVEY_FINGERPRINTS[k]
    assert int(r.histogram.sum()) == p.n_voxels
    if k == 1:
        ref, _ = oracle_mod.brute(p, distances=False)
        assert np.array_equal(r.labels.labels, ref)
    if oracle_mod.have_ref():
        ref, _, _, _ = oracle_mod.ref_tessellate(p, distances=False)
        assert np.array_equal(r.labels.labels, ref), int((r.labels.labels != ref).sum())
        hist = np.bincount(ref, minlength=p.n_sites).astype(np.uint64)
        assert np.array_equal(r.histogram, hist)
        del ref, hist


@pytest.mark.parametrize("route", ["bricks", "subbricks", "dense"])
def test_every_ball_kernel_variant(route):
    """Each ball-phase route stays bit-exact: the default brick lists + eval16,
    the 8 x 8 x 4 sub-brick lists + eval12 (VX_SUBBRICK_LISTS=1) and dense
    mode (VX_DENSE=1) -- random 2-D / 3-D instances of every kind against the
    oracle, the cfg1 and cfg4 (Johnson-Mehl) fingerprints."""
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import oracle
from conftest import to_vx
import paper_2201_13234_b200 as vx
rng = np.random.default_rng(99)
for i in range(36):
    d = 3 if i %% 3 else 2
    kind = i %% 3; per = (i // 3) %% 2 == 0
    L = rng.uniform(0.5, 2.0, d)
    counts = list(rng.integers(2, 40 if d == 3 else 120, d))
    pos, t = oracle.generate_uniform_sites(d, L, int(rng.integers(1, 400)), kind, 0.3, int(rng.integers(1 << 60)))
    p = oracle.Problem(kind, counts, L, per, pos, t, 1.3 if kind else 0.0)
    s, g = to_vx(p)
    r = vx.tessellate_fast(s, g, vx.FastOptions(prune=False))
    lab, dist = oracle.brute(p)
    assert np.array_equal(r.labels.labels, lab), i
    assert np.array_equal(r.distances.values.view(np.uint64), dist.view(np.uint64)), i
for k in (1, 4):
    cfg = oracle.baseline_config(k)
    s, g = to_vx(cfg)
    r = vx.tessellate_fast(s, g, distances=False)
    assert oracle.fingerprint(r.labels.labels) == oracle.SURVEY_FINGERPRINTS[k], k
print("ok")
""" % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ)
    env.pop("VX_SUBBRICK_LISTS", None)
    env.pop("VX_DENSE", None)
    if route == "subbricks":
        env["VX_SUBBRICK_LISTS"] = "1"
    elif route == "dense":
        env["VX_DENSE"] = "1"
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_chunked_host_copies_identical(kind):
    """Host-buffer calls compute the slab in z-chunks and overlap each chunk's
    D2H with the next chunk (VX_CHUNKS); labels, distances and histogram must
    not depend on the chunking, and must match the oracle."""
    import oracle
    import paper_2201_13234_b200 as vx

    rng = np.random.default_rng(900 + kind)
    L = rng.uniform(0.5, 1.5, 3)
    counts = [40, 36, 300]
    ns = 300
    G = 0.0 if kind == 0 else 0.7
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, 1.0, 1234 + kind)
    p = oracle.Problem(kind, counts, L, kind != 1, pos, t, G)
    sites, grid = to_vx(p)
    out = {}
    old = os.environ.get("VX_CHUNKS")
    try:
        for ch in ("1", "5", "16"):
            os.environ["VX_CHUNKS"] = ch
            r = vx.tessellate_fast(sites, grid, vx.FastOptions(prune=True), distances=True, histogram=True)
            out[ch] = r
    finally:
        if old is None:
            os.environ.pop("VX_CHUNKS", None)
        else:
            os.environ["VX_CHUNKS"] = old
    lab, dist = oracle.brute(p)
    for ch, r in out.items():
        assert np.array_equal(r.labels.labels, lab), ch
        assert np.array_equal(r.distances.values.view(np.uint64), dist.view(np.uint64)), ch
        assert np.array_equal(r.histogram, out["1"].histogram), ch
    assert int(out["1"].histogram.sum()) == int(np.prod(counts))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["sparse", "dense", "mixed", "odd_rows", "jm_np", "long_rows"])
def test_run_coded_transport_identical(case):
    """Synchronous 3-D host-buffer calls move the label image across PCIe as
    runs along x and expand them on host threads (labelrun.cu); chunks whose
    runs average < 4 voxels go raw.  The caller's image (pinned or pageable,
    any chunking) must equal the raw transport's and the device-pointer
    call's, voxel for voxel."""
    import torch
    import paper_2201_13234_b200 as vx
    from paper_2201_13234_b200 import _lib

    rng = np.random.default_rng({"sparse": 1, "dense": 2, "mixed": 3, "odd_rows": 4, "jm_np": 5, "long_rows": 6}[case])
    kind, periodic = (1, False) if case == "jm_np" else (0, True)
    # long_rows: 16 x bits leave 16 label bits, 70,000 sites do not fit -> 6-byte runs
    counts = {"odd_rows": [101, 130, 320], "long_rows": [65535, 8, 9]}.get(case, [160, 96, 300])
    L = {"odd_rows": np.array([1.0, 1.3, 3.1]), "long_rows": np.array([8.0, 0.005, 0.0055])}.get(
        case, np.array([1.0, 0.6, 1.9]))
    nv = int(np.prod(counts))
    if case == "dense":
        ns = nv // 3
        pos = rng.uniform(0, 1, (ns, 3)) * L
    elif case == "mixed":  # dense near z = 0 (raw chunks), sparse above (runs)
        a = rng.uniform(0, 1, (nv // 6, 3)) * L * np.array([1, 1, 0.2])
        b = rng.uniform(0, 1, (2000, 3)) * L * np.array([1, 1, 0.8]) + np.array([0, 0, 0.2 * L[2]])
        pos = np.concatenate([a, b])
        ns = len(pos)
    else:
        ns = 70000 if case == "long_rows" else 3000
        pos = rng.uniform(0, 1, (ns, 3)) * L
    pos = np.ascontiguousarray(np.minimum(pos, np.nextafter(L, 0)))
    t = rng.uniform(0, 0.05, ns) if kind == 1 else None
    box = vx.Domain(list(L), vx.Boundary.Periodic if periodic else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(counts, box)
    sites = vx.SiteSet(vx.Kind(kind), 3, pos, t, 1.0 if kind else 0.0)
    old = {k: os.environ.get(k) for k in ("VX_D2H_RAW", "VX_CHUNKS", "VX_RUN_UNPACKED")}
    res = {}
    try:
        os.environ["VX_D2H_RAW"] = "1"
        res["raw"] = vx.tessellate_fast(sites, grid, distances=False).labels.labels.copy()
        raw_bytes = int(_lib.lib().vx_last_d2h_bytes())
        os.environ.pop("VX_D2H_RAW")
        for ch in ("1", "5", "8"):
            os.environ["VX_CHUNKS"] = ch
            out = torch.empty(nv, dtype=torch.int32).pin_memory().numpy()
            vx.tessellate_fast(sites, grid, distances=False, out=out)
            res["pinned" + ch] = out.copy()
            res["pageable" + ch] = vx.tessellate_fast(sites, grid, distances=False).labels.labels.copy()
            run_bytes = int(_lib.lib().vx_last_d2h_bytes())
        # the 6-byte runs (label, first x apart) that wide labels or long rows fall back to
        os.environ["VX_RUN_UNPACKED"] = "1"
        res["unpacked"] = vx.tessellate_fast(sites, grid, distances=False).labels.labels.copy()
        unpacked_bytes = int(_lib.lib().vx_last_d2h_bytes())
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert raw_bytes == 4 * nv
    for k, v in res.items():
        assert np.array_equal(v.reshape(-1), res["raw"].reshape(-1)), k
    if case == "dense":
        assert run_bytes >= 4 * nv  # every chunk raw
    else:
        assert run_bytes < 4 * nv * (0.8 if case == "mixed" else 0.5)
        if case == "long_rows":
            assert run_bytes == unpacked_bytes
        else:
            assert run_bytes < unpacked_bytes  # labels fit beside x: 4-byte runs
    # and the raw image itself against the device-pointer path
    from paper_2201_13234_b200.engine import Tessellator

    eng = Tessellator(0)
    lab_d = torch.empty(nv, dtype=torch.int32, device="cuda")
    eng.run(kind=kind, counts=counts, lengths=list(L), periodic=periodic, positions=torch.from_numpy(pos).cuda(),
            labels=lab_d, times=None if t is None else torch.from_numpy(t).cuda(), growth=1.0 if kind else 0.0)
    assert np.array_equal(lab_d.cpu().numpy().view(np.uint32), res["raw"].reshape(-1).view(np.uint32))
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["vor3d", "jm3d_dist", "lag2d", "brute4d"])
def test_tessellate_to_files_streams_the_image(case, tmp_path):
    """vx_tessellate_to_files streams each z-chunk of the image from device
    memory into the reference's file format (row f2); forced small pieces
    (VX_SINK_CHUNK_BYTES) exercise the double-buffered copy/write pipeline."""
    import json as _json

    import oracle
    import paper_2201_13234_b200 as vx

    spec = {"vor3d": (0, [48, 40, 200], 400, False), "jm3d_dist": (1, [30, 33, 120], 200, True),
            "lag2d": (2, [301, 257], 150, True), "brute4d": (0, [6, 5, 4, 30], 40, True)}[case]
    kind, counts, ns, with_dist = spec
    d = len(counts)
    rng = np.random.default_rng(77)
    L = rng.uniform(0.5, 1.5, d)
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, 1.0, 4242)
    p = oracle.Problem(kind, counts, L, kind != 1, pos, t, 0.0 if kind == 0 else 0.8)
    sites, grid = to_vx(p)
    lab_path = str(tmp_path / "img.lab")
    dist_path = str(tmp_path / "img.dist") if with_dist else None
    old = os.environ.get("VX_SINK_CHUNK_BYTES")
    os.environ["VX_SINK_CHUNK_BYTES"] = "20000"
    try:
        vx.tessellate_to_files(sites, grid, lab_path, dist_path, seed=5)
    finally:
        if old is None:
            os.environ.pop("VX_SINK_CHUNK_BYTES", None)
        else:
            os.environ["VX_SINK_CHUNK_BYTES"] = old
    lab, dist = oracle.brute(p)
    assert np.array_equal(np.fromfile(lab_path, dtype="<u4"), lab.astype(np.uint32))
    side = _json.load(open(lab_path + ".json"))
    assert side == {"format_version": 1, "type": "labels", "d": d, "dims": list(counts), "lengths": list(L),
                    "boundary": "periodic" if kind != 1 else "non-periodic",
                    "kind": ["voronoi", "johnson-mehl", "laguerre"][kind], "n_sites": ns, "seed": 5,
                    "payload_bytes": 4 * int(np.prod(counts))}
    im, meta = vx.read_label_image(lab_path)
    assert np.array_equal(im.labels, lab.astype(np.uint32)) and meta.seed == 5
    if with_dist:
        assert np.array_equal(np.fromfile(dist_path, dtype="<f8").view(np.uint64), dist.view(np.uint64))
        dim_, _ = vx.read_distance_image(dist_path)
        assert np.array_equal(dim_.values.view(np.uint64), dist.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(30))
def test_large_random_vs_reference_library(i):
    """Random problems at realistic size (3-D 96..200 voxels per axis, 2-D
    600..1200, non-cubic, all kinds, both boundaries, prune on/off) against the reference library
    itself (oracle/_ref, run on the box's host cores): labels, values and the
    grain-volume histogram, bit for bit."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(31337 + i)
    kind = i % 3
    periodic = bool((i // 3) % 2 == 0)
    d = 2 if i % 5 == 4 else 3
    counts = [int(x) for x in rng.integers(96, 201, 3)] if d == 3 else [int(x) for x in rng.integers(600, 1201, 2)]
    L = rng.uniform(0.5, 2.0, d)
    sp = float(np.min(L / np.array(counts)))
    spacing_vox = float(rng.uniform(4.0, 14.0))
    ns = int(np.clip(np.prod(L) / (spacing_vox * sp) ** d, 50, 60000))
    horizon = float(0.5 * np.prod(L) ** (1.0 / d) / ns ** (1.0 / d))
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, horizon, 555 + i)
    G = [0.0, float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.5, 2.0))][kind]
    p = oracle.Problem(kind, counts, L, periodic, pos, t, G)
    prune = bool(i % 4 != 3)
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p, prune=prune)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, vx.FastOptions(prune=prune), distances=True, histogram=True)
    assert np.array_equal(r.labels.labels, lab_ref), int((r.labels.labels != lab_ref).sum())
    assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))
    assert np.array_equal(r.histogram, np.bincount(lab_ref, minlength=ns).astype(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["flat_periodic", "tall_nonperiodic", "dense_jm", "flat_laguerre"])
def test_overflow_subbrick_shell_vs_reference(case, monkeypatch):
    """Strongly anisotropic voxels / very dense sites overflow the ball phase's
    brick caps; those sub-bricks are labelled by the sub-brick shell search.
    Bit-exact against the reference library, and the path is really taken
    (standard lists forced: the default would pick dense mode for several of
    these and not overflow; test_dense_mode_vs_reference covers that)."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    monkeypatch.setenv("VX_DENSE", "0")
    kind, counts, ns, per = {"flat_periodic": (0, [512, 512, 8], 20000, True),
                             "tall_nonperiodic": (0, [32, 32, 2048], 8000, False),
                             "dense_jm": (1, [96, 96, 96], 40000, True),
                             "flat_laguerre": (2, [400, 384, 6], 12000, False)}[case]
    L = np.array([1.0, 0.8, 1.2])
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, 0.5 * np.cbrt(np.prod(L) / ns), 99)
    p = oracle.Problem(kind, counts, L, per, pos, t, 0.0 if kind == 0 else 1.3)
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, distances=True, histogram=True)
    assert r.stats["overflow_bricks"] > 0  # the sub-brick shell ran
    assert np.array_equal(r.labels.labels, lab_ref), int((r.labels.labels != lab_ref).sum())
    assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))
    assert np.array_equal(r.histogram, np.bincount(lab_ref, minlength=ns).astype(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,per", [(0, True), (0, False), (1, True), (2, True)])
def test_dense_mode_vs_reference(kind, per):
    """Site spacing below ~8.5 voxels selects the dense ball path (long brick
    lists, chunked cull and eval); bit-exact against the reference library."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    counts, ns = [120, 112, 128], 24000  # spacing ~4.3 voxels
    L = np.array([1.0, 0.93, 1.07])
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, 0.5 * np.cbrt(np.prod(L) / ns), 5 + kind)
    p = oracle.Problem(kind, counts, L, per, pos, t, 0.0 if kind == 0 else 0.9)
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, distances=True, histogram=True)
    assert np.array_equal(r.labels.labels, lab_ref), int((r.labels.labels != lab_ref).sum())
    assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))
    assert np.array_equal(r.histogram, np.bincount(lab_ref, minlength=ns).astype(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("d,counts,ns", [(1, [600000], 3000), (2, [4, 300000], 2000), (2, [3, 700000], 4000),
                                         (3, [2, 600000, 2], 3000)])
def test_long_last_axis_vs_reference(d, counts, ns):
    """Last axes longer than one launch's grid (262,080 planes) are labelled in
    several z-chunks, and embedded y axes longer than 65,535 sub-bricks in
    several eval launches; bit-exact against the reference library."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    L = np.full(d, 1.3)
    pos, _ = oracle.generate_uniform_sites(d, L, ns, 0, 1.0, 17)
    p = oracle.Problem(0, counts, L, True, pos, None, 0.0)
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, distances=True, histogram=True)
    assert np.array_equal(r.labels.labels, lab_ref)
    assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))
    assert int(r.histogram.sum()) == int(np.prod(counts))


@pytest.mark.gpu
@pytest.mark.parametrize("n_gpus", [2, 3])
def test_n_gpus_single_call_identical(n_gpus):
    """options.n_gpus splits one call over devices (wrapping onto the devices
    present, one host thread each); labels, values, histogram and counts equal
    the one-device call."""
    import oracle
    import paper_2201_13234_b200 as vx

    for kind, per in [(0, True), (1, False), (2, True)]:
        rng = np.random.default_rng(40 + kind)
        L = rng.uniform(0.6, 1.4, 3)
        pos, t = oracle.generate_uniform_sites(3, L, 900, kind, 1.0, 71 + kind)
        p = oracle.Problem(kind, [64, 48, 101], L, per, pos, t, 0.0 if kind == 0 else 0.8)
        sites, grid = to_vx(p)
        a = vx.tessellate_fast(sites, grid, vx.FastOptions(prune=True), distances=True, histogram=True)
        b = vx.tessellate_fast(sites, grid, vx.FastOptions(prune=True), distances=True, histogram=True,
                               n_gpus=n_gpus)
        assert np.array_equal(a.labels.labels, b.labels.labels)
        assert np.array_equal(a.distances.values.view(np.uint64), b.distances.values.view(np.uint64))
        assert np.array_equal(a.histogram, b.histogram)
        assert b.stats["n_voxels"] == p.n_voxels


@pytest.mark.gpu
@pytest.mark.parametrize("d,kind,periodic", [(2, 1, True), (3, 0, True), (3, 1, False), (3, 2, True), (3, 0, False)])
def test_refinement_preserves_labels_at_shared_centres(d, kind, periodic):
    """test_tessellate.cpp:365-387: spacings 3/4 and 1/4 give exactly equal
    centres at coarse voxel i and fine voxel 3i+1, so the fast engine on the
    fine grid must reproduce the coarse grid's labels and f64 values there."""
    import oracle

    L = [3.0] * d if d == 2 else [12.0, 9.0, 6.0]
    coarse = [int(round(x / 0.75)) for x in L]
    fine = [3 * c for c in coarse]
    ns = 20 if d == 2 else 300
    horizon = 0.5 * float(np.prod(L)) ** (1.0 / d) / ns ** (1.0 / d)
    pos, t = oracle.generate_uniform_sites(d, np.array(L), ns, kind, horizon, 606 + kind)
    G = [0.0, 1.3, 0.8][kind]
    pc = oracle.Problem(kind, coarse, L, periodic, pos, t, G)
    pf = oracle.Problem(kind, fine, L, periodic, pos, t, G)
    c = run_brute(pc)
    f = run_fast(pf)
    cl = c.labels.labels.reshape(coarse[::-1])
    fl = f.labels.labels.reshape(fine[::-1])
    cv = c.distances.values.reshape(coarse[::-1])
    fv = f.distances.values.reshape(fine[::-1])
    sl = tuple(slice(1, None, 3) for _ in range(d))
    assert np.array_equal(fl[sl], cl)
    assert np.array_equal(bits(fv[sl]), bits(cv))


def coverage_case(i):
    """Random near-isotropic instance for the ball-coverage test (shared with
    scripts/cov_probe.py)."""
    import oracle

    rng = np.random.default_rng(2480 + i)
    kind = i % 3
    periodic = i % 2 == 0
    d = 2 if i == 7 else 3
    counts = [int(x) for x in rng.integers(48, 97, d)]
    L = np.array(counts) * rng.uniform(0.01, 0.02) * rng.uniform(0.9, 1.1, d)
    spacing = float(rng.uniform(9.0, 16.0))
    ns = max(2, int(np.prod(counts) / spacing ** d))
    horizon = float(0.5 * np.prod(L) ** (1.0 / d) / ns ** (1.0 / d))
    pos, t = oracle.generate_uniform_sites(d, L, ns, kind, horizon, 77 + i)
    return oracle.Problem(kind, counts, L, periodic, pos, t, [0.0, 1.1, 0.9][kind])


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(8))
def test_ball_phase_covers_exactly_the_union_of_balls(i):
    """test_tessellate.cpp:248-269: the voxels the ball phase leaves to the
    shell search are exactly those outside every investigation ball.  The
    reference's step 2 evaluates every kept site at each such voxel, so its
    count is step2_evals / n_sites; ours is the unresolved-voxel counter.

    Both engines run with the reference's own parameter (our t0 search for the
    timed kinds picks its own t0 -- labels never depend on it), and the
    instances keep voxels near-isotropic so no sub-brick takes the overflow
    route (whose voxels are labelled by the sub-brick shell instead)."""
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    p = coverage_case(i)
    ns = p.n_sites
    _, _, param, _ = oracle.ref_tessellate(p, prune=False, distances=False)
    tmin = 0.0 if p.kind == 0 else float(np.min(p.times))
    for scale in (1.0, 0.5):  # the reference's ball, then a smaller one
        override = param * scale if p.kind == 0 else tmin + scale * (param - tmin)
        lab_ref, _, param_ref, (_, ev2) = oracle.ref_tessellate(p, prune=False, override=override,
                                                                 distances=False)
        r = run_fast(p, prune=False, override=override, distances=False)
        assert r.param == param_ref == override
        assert np.array_equal(r.labels.labels, lab_ref)
        assert r.stats["overflow_bricks"] == 0
        assert ev2 % ns == 0
        assert r.stats["n_unresolved"] == ev2 // ns, (r.stats["n_unresolved"], ev2 // ns)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,periodic,n,step", [(0, True, 64, 8), (0, False, 64, 8), (1, True, 48, 4),
                                                   (2, True, 64, 8), (2, False, 48, 6), (0, True, 40, 5)])
def test_lattice_ties_lowest_index_wins(oracle_mod, kind, periodic, n, step):
    """Exact ties everywhere: sites on voxel centres of a regular lattice
    (`step` voxels apart, spacing 1/64 so every coordinate is dyadic), so each
    voxel half-way between lattice sites -- across the periodic boundary too --
    is exactly equidistant from 2, 4 or 8 of them.  The site order is a random
    permutation, so the lowest-index rule (strict `<` over ascending index,
    tessellate.cpp:65; test_sites.cpp:125-143) decides a large share of the
    image.  Timed kinds draw each birth time from two dyadic values: equal
    times tie exactly, unequal ones do not."""
    rng = np.random.default_rng(n * 31 + step + kind)
    Ln = n / 64.0
    sp = Ln / n
    k = np.arange(0, n, step)
    g = np.stack(np.meshgrid(k, k, k, indexing="ij"), -1).reshape(-1, 3)
    g = g[rng.permutation(len(g))]
    pos = ((g + 0.5) * sp).reshape(-1)
    t = rng.choice([0.0, 0.0078125], len(g)) if kind else None
    p = oracle_mod.Problem(kind, [n, n, n], [Ln] * 3, periodic, pos, t, [0.0, 1.0, 0.5][kind])
    lab_all, dist_all = oracle_mod.brute(p)
    assert len(np.unique(lab_all)) > 1
    for prune in (True, False):
        lab, dist = lab_all, dist_all
        if prune and kind != 0:  # the reference labels the prune survivors
            dropped = oracle_mod.prune(p)
            if dropped.any():
                keep = np.nonzero(dropped == 0)[0]
                q = oracle_mod.Problem(kind, p.counts, p.lengths, periodic,
                                       p.positions.reshape(-1, 3)[keep].reshape(-1), p.times[keep], p.growth)
                l2, dist = oracle_mod.brute(q)
                lab = keep[l2].astype(np.uint32)
        r = run_fast(p, prune=prune)
        assert np.array_equal(r.labels.labels, lab), int((r.labels.labels != lab).sum())
        assert np.array_equal(bits(r.distances.values), bits(dist))
    rb = run_brute(p)
    assert np.array_equal(rb.labels.labels, lab_all)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,periodic", [(0, True), (0, False), (1, True), (2, False), (2, True)])
def test_sites_hugging_the_domain_faces(oracle_mod, kind, periodic):
    """Sites at the extremes the reference accepts (sites.cpp:55: 0 < x < L):
    coordinates one ulp above 0 and one ulp below L, on faces, edges and
    corners, mixed with interior sites -- the binning, the periodic wrap of
    the cull's f32 frame and the exact fold all meet their edge cases here."""
    rng = np.random.default_rng(9100 + 10 * kind + periodic)
    L = np.array([1.0, 0.8125, 1.375])
    counts = [48, 40, 56]
    lo, hi = np.nextafter(0.0, 1.0), np.nextafter(L, 0.0)
    interior = rng.uniform(0.05, 0.95, (120, 3)) * L
    edge = []
    for _ in range(80):
        q = rng.uniform(0.0, 1.0, 3) * L
        for a in range(3):
            r = rng.integers(3)
            if r == 0:
                q[a] = lo if rng.integers(2) else np.nextafter(lo, 1.0)
            elif r == 1:
                q[a] = hi[a] if rng.integers(2) else np.nextafter(hi[a], 0.0)
        edge.append(q)
    pts = np.concatenate([interior, np.array(edge)])
    pts = pts[rng.permutation(len(pts))]
    assert (pts > 0).all() and (pts < L).all()
    t = rng.uniform(0.0, 0.05, len(pts)) if kind else None
    p = oracle_mod.Problem(kind, counts, L, periodic, pts.reshape(-1), t, [0.0, 1.2, 0.7][kind])
    lab, dist = oracle_mod.brute(p)
    r = run_fast(p, prune=False)
    assert np.array_equal(r.labels.labels, lab), int((r.labels.labels != lab).sum())
    assert np.array_equal(bits(r.distances.values), bits(dist))


@pytest.mark.gpu
@pytest.mark.parametrize("where", [0, 123456, 299999])
@pytest.mark.parametrize("bad", [1.0, 0.0, float("nan"), 1.5, -1e-300, float("inf")])
def test_device_validation_rejects_bad_positions(where, bad):
    """Host-buffer calls validate the positions on the device during ingest
    (sites.cpp:54-57: finite and strictly inside the domain) and fail with
    the reference's message before any labelling work; the context stays
    usable for the next call."""
    import paper_2201_13234_b200 as vx

    n = 300000
    pos = np.random.default_rng(5).uniform(0.01, 0.99, 3 * n)
    box = vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic)
    grid = vx.VoxelGrid([32, 32, 32], box)
    good = vx.tessellate_fast(vx.SiteSet(vx.Kind.Voronoi, 3, pos.copy(), None, 0.0), grid, distances=False)
    pos[3 * where + 2] = bad
    with pytest.raises(ValueError, match="site positions must lie strictly inside the domain"):
        vx.tessellate_fast(vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0), grid)
    pos[3 * where + 2] = 0.5
    again = vx.tessellate_fast(vx.SiteSet(vx.Kind.Voronoi, 3, pos, None, 0.0), grid, distances=False)
    assert again.labels.labels.shape == good.labels.labels.shape


@pytest.mark.gpu
def test_caller_buffers_for_labels_and_histogram():
    """out= / histogram_out= (e.g. pinned buffers) receive exactly what the
    default call returns."""
    import torch

    import oracle
    import paper_2201_13234_b200 as vx

    p = oracle.baseline_config(1)
    sites, grid = to_vx(p)
    ref = vx.tessellate_fast(sites, grid, distances=False, histogram=True)
    out = torch.empty(p.n_voxels, dtype=torch.int32).pin_memory().numpy()
    hist = torch.zeros(p.n_sites, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    hist[:] = 7  # the call overwrites every count
    r = vx.tessellate_fast(sites, grid, distances=False, out=out, histogram_out=hist)
    assert np.array_equal(out.view(np.uint32), ref.labels.labels)
    assert np.array_equal(hist, ref.histogram) and np.shares_memory(r.histogram, hist)


@pytest.mark.gpu
@pytest.mark.parametrize("counts", [[64, 1, 64], [1, 1, 200], [1, 64, 1], [96, 80, 1], [1, 40, 56], [3, 2, 1]])
@pytest.mark.parametrize("kind,periodic", [(0, True), (1, False), (2, True), (0, False)])
def test_single_voxel_axes_in_3d(oracle_mod, counts, kind, periodic):
    """3-D grids with one voxel along some axes (a slice or a line through a
    3-D site set): sub-bricks and super-bricks are mostly outside the grid and
    the voxel centre sits mid-domain on the thin axes."""
    rng = np.random.default_rng(sum(counts) * 7 + kind)
    L = rng.uniform(0.5, 2.0, 3)
    ns = int(rng.integers(20, 300))
    pos, t = oracle_mod.generate_uniform_sites(3, L, ns, kind, float(0.5 * np.prod(L) ** (1 / 3) / ns ** (1 / 3)),
                                               int(rng.integers(1 << 40)))
    p = oracle_mod.Problem(kind, counts, L, periodic, pos, t, [0.0, 1.3, 0.8][kind])
    lab, dist = oracle_mod.brute(p)
    r = run_fast(p, prune=False)
    assert np.array_equal(r.labels.labels, lab)
    assert np.array_equal(bits(r.distances.values), bits(dist))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [1, 4])
def test_cuda_graph_replay_relabels_moved_sites(oracle_mod, cfg):
    """A device-pointer call captured into a CUDA graph (Tessellator.capture):
    replaying it after rewriting the positions in place gives exactly what a
    fresh call gives for the new sites -- the whole pipeline (binning, t0
    search, ball phase, shell, histogram) lives in the graph."""
    import torch

    from paper_2201_13234_b200.engine import Tessellator

    p = oracle_mod.baseline_config(cfg)
    eng = Tessellator(0)
    pos = torch.from_numpy(p.positions.copy()).cuda()
    t = torch.from_numpy(p.times.copy()).cuda() if p.times is not None else None
    lab = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
    hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
    kw = dict(kind=p.kind, counts=list(p.counts), lengths=list(p.lengths), periodic=p.periodic,
              positions=pos, times=t, growth=p.growth, labels=lab, histogram=hist)
    g = eng.capture(**kw)
    rng = np.random.default_rng(cfg)
    for trial in range(3):
        new = rng.uniform(0.001, 0.999, p.positions.size) * np.tile(np.asarray(p.lengths), p.n_sites)
        pos.copy_(torch.from_numpy(new))
        hist.zero_()
        g.replay()
        torch.cuda.synchronize()
        q = oracle_mod.Problem(p.kind, p.counts, p.lengths, p.periodic, new, p.times, p.growth)
        ref = run_fast(q, distances=False, histogram=True)
        assert np.array_equal(lab.cpu().numpy().view(np.uint32), ref.labels.labels)
        assert np.array_equal(hist.cpu().numpy().astype(np.uint64), ref.histogram)
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1])
def test_unresolved_list_overflow_path(oracle_mod, kind):
    """More unresolved voxels than the unresolved list holds (2^22): with a
    vanishing ball every voxel of a 4.8e6-voxel grid goes to the shell search,
    which then finds them by their -1 sentinel in the label image."""
    rng = np.random.default_rng(4242 + kind)
    counts = [200, 200, 120]
    L = np.array([1.0, 1.0, 0.6])
    pos, t = oracle_mod.generate_uniform_sites(3, L, 150, kind, 0.05, int(rng.integers(1 << 40)))
    p = oracle_mod.Problem(kind, counts, L, True, pos, t, [0.0, 1.0][kind])
    override = 1e-9 if kind == 0 else float(np.min(t))
    r = run_fast(p, prune=False, override=override)
    assert r.stats["n_unresolved"] == p.n_voxels > (1 << 22)
    lab, dist = oracle_mod.brute(p)
    assert np.array_equal(r.labels.labels, lab)
    assert np.array_equal(bits(r.distances.values), bits(dist))


@pytest.mark.gpu
@pytest.mark.parametrize("ratio,kind", [(3.0, 0), (4.0, 1), (6.0, 2), (8.0, 0)])
def test_thick_slices_take_dense_lists_vs_reference(ratio, kind):
    """Voxels `ratio` times thicker along z than in-plane at moderate density
    (~10 in-plane voxels between sites): the anisotropy-aware choice takes the
    dense lists instead of overflowing to the shell searches; bit-exact against
    the reference library, and no sub-brick overflows."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    nxy, nz = 128, int(round(128 / ratio))
    L = np.array([1.0, 1.0, 1.0])
    ns = int(nxy * nxy * nz * ratio / 1000)
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, 0.5 / ns ** (1 / 3), 31 + kind)
    p = oracle.Problem(kind, [nxy, nxy, nz], L, True, pos, t, 0.0 if kind == 0 else 1.1)
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, distances=True, histogram=True)
    assert r.stats["overflow_bricks"] == 0
    assert np.array_equal(r.labels.labels, lab_ref), int((r.labels.labels != lab_ref).sum())
    assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("n", [16, 24, 40])
def test_half_period_offsets(oracle_mod, kind, n):
    """Periodic boxes with a handful of sites on voxel centres, so many
    site-voxel offsets are exactly +-L/2 (floor(u/L + 0.5) rounds up at the
    half-tie, geometry.hpp:82-89; test_geometry.cpp:42-48) and images of the
    same site tie with each other: the kernels' 0.49 L fast path and the
    wrapped slow path must agree with the reference's formula everywhere."""
    rng = np.random.default_rng(n * 3 + kind)
    L = np.array([1.0, 0.5, 2.0])  # dyadic spacings for n = 16 (and exact halves)
    counts = [n, n, n]
    sp = L / np.array(counts)
    ns = 6
    k = rng.integers(0, n, (ns, 3))
    pos = ((k + 0.5) * sp).reshape(-1)
    t = rng.choice([0.0, 0.25], ns) if kind else None
    p = oracle_mod.Problem(kind, counts, L, True, pos, t, [0.0, 1.0, 0.5][kind])
    lab, dist = oracle_mod.brute(p)
    for prune in (False, True):
        if prune and kind == 0:
            continue
        r = run_fast(p, prune=prune)
        if prune:  # the reference labels the prune survivors
            dropped = oracle_mod.prune(p)
            if dropped.any():
                keep = np.nonzero(dropped == 0)[0]
                q = oracle_mod.Problem(kind, counts, L, True, p.positions.reshape(-1, 3)[keep].reshape(-1),
                                       p.times[keep], p.growth)
                l2, d2 = oracle_mod.brute(q)
                assert np.array_equal(r.labels.labels, keep[l2].astype(np.uint32))
                assert np.array_equal(bits(r.distances.values), bits(d2))
                continue
        assert np.array_equal(r.labels.labels, lab), int((r.labels.labels != lab).sum())
        assert np.array_equal(bits(r.distances.values), bits(dist))


@pytest.mark.gpu
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("sigma,growth", [(0.3, 1.0), (0.9, 1.0), (0.9, 2.5)])
def test_polydisperse_laguerre_spheres(oracle_mod, periodic, sigma, growth):
    """Laguerre from sphere packs (sites.cpp:87-104, t = -(r r)/G: negative
    birth times and proximities), lognormal radii up to very polydisperse --
    many sites are dominated and pruned (sites.cpp:113-171) and the survivors
    are remapped to original indices (tessellate.cpp:274-280)."""
    pos, radii = oracle_mod.generate_lognormal_spheres(600, 0.04, sigma, 1234 + int(10 * sigma))
    t = oracle_mod.spheres_to_timed(radii, growth)
    p = oracle_mod.Problem(2, [72, 64, 80], [1.0, 1.0, 1.0], periodic, pos, t, growth)
    lab_all, dist_all = oracle_mod.brute(p)
    dropped = oracle_mod.prune(p)
    keep = np.nonzero(dropped == 0)[0]
    q = oracle_mod.Problem(2, p.counts, p.lengths, periodic, pos.reshape(-1, 3)[keep].reshape(-1), t[keep], growth)
    l2, d2 = oracle_mod.brute(q)
    for prune, (lab, dist) in ((False, (lab_all, dist_all)), (True, (keep[l2].astype(np.uint32), d2))):
        r = run_fast(p, prune=prune)
        assert np.array_equal(r.labels.labels, lab), int((r.labels.labels != lab).sum())
        assert np.array_equal(bits(r.distances.values), bits(dist))
    if sigma > 0.5:
        assert dropped.any()  # the pruning path is exercised


@pytest.mark.gpu
@pytest.mark.parametrize("order", ["z_sorted", "x_sorted", "morton", "blocks"])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_site_index_order_vs_reference(order, kind):
    """The cull orders each super-brick's kept sites by site index (an
    all-pairs rank), which every later list inherits; site numberings that
    are not random in space (z / x sorted, Morton, shuffled blocks) must still
    give the ascending-index, strict-< winner of the reference library, bit
    for bit."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    counts, ns = [160, 144, 176], 6000
    L = np.array([1.0, 0.9, 1.1])
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, 0.5 * np.cbrt(np.prod(L) / ns), 71 + kind)
    P = pos.reshape(ns, 3)
    if order == "z_sorted":
        perm = np.argsort(P[:, 2], kind="stable")
    elif order == "x_sorted":
        perm = np.lexsort((P[:, 1], P[:, 0]))
    elif order == "morton":  # Z-order curve: every neighbourhood is a few dense index runs
        q = np.minimum((P / L * 1024).astype(np.uint64), np.uint64(1023))
        key = np.zeros(ns, dtype=np.uint64)
        for b in range(10):
            for a in range(3):
                key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
        perm = np.argsort(key, kind="stable")
    else:  # spatial blocks of 8^3 cells, shuffled block order
        cell = np.floor(P / (L / 8)).astype(np.int64)
        key = cell[:, 0] + 8 * (cell[:, 1] + 8 * cell[:, 2])
        rank = np.random.default_rng(5).permutation(512)
        perm = np.argsort(rank[key], kind="stable")
    pos = np.ascontiguousarray(P[perm]).reshape(-1)
    t = None if t is None else np.ascontiguousarray(t[perm])
    for periodic in (True, False):
        p = oracle.Problem(kind, counts, L, periodic, pos, t, 0.0 if kind == 0 else 1.1)
        lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p)
        sites, grid = to_vx(p)
        r = vx.tessellate_fast(sites, grid, distances=True, histogram=True)
        assert np.array_equal(r.labels.labels, lab_ref), int((r.labels.labels != lab_ref).sum())
        assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))
        assert np.array_equal(r.histogram, np.bincount(lab_ref, minlength=ns).astype(np.uint64))


@pytest.mark.parametrize("scale", [1e-9, 1e-3, 1e3, 1e9])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_extreme_domain_scales_vs_oracle(oracle_mod, scale, kind):
    """The cull works in f32 coordinates relative to each super-brick centre
    with slack proportional to the box: it must stay conservative whatever the
    domain's absolute scale (tiny and huge L, anisotropic lengths), bit for
    bit against the oracle's brute force."""
    rng = np.random.default_rng(int(np.log10(scale) * 7 + 100 + kind))
    for periodic in (True, False):
        L = scale * rng.uniform(0.5, 2.0, 3)
        counts = [int(c) for c in rng.integers(40, 72, 3)]
        ns = int(rng.integers(150, 600))
        horizon = 0.5 * float(np.cbrt(np.prod(L) / ns))
        pos, t = oracle_mod.generate_uniform_sites(3, L, ns, kind, horizon, int(rng.integers(1 << 60)))
        p = oracle_mod.Problem(kind, counts, L, periodic, pos, t, 1.0 if kind else 0.0)
        lab, dist = oracle_mod.brute(p)
        r = run_fast(p, prune=False, distances=True)
        assert np.array_equal(r.labels.labels, lab), int((r.labels.labels != lab).sum())
        assert np.array_equal(bits(r.distances.values), bits(dist))


@pytest.mark.parametrize("periodic", [True, False])
def test_slab_window_binning_fallback_vs_oracle(oracle_mod, periodic):
    """A rank's slab bins only the sites within a window of 2 R + 2 cells along
    z (Voronoi).  With a small override radius most voxels are unresolved and
    many have their nearest site outside the window: the shell searches must
    fall back to all sites and stay exact (labels, distances, histogram)."""
    import paper_2201_13234_b200 as vx

    rng = np.random.default_rng(61 + periodic)
    counts = [40, 36, 120]
    L = np.array([1.0, 0.9, 3.0])
    ns = 400
    pos, _ = oracle_mod.generate_uniform_sites(3, L, ns, 0, 1.0, int(rng.integers(1 << 40)))
    p = oracle_mod.Problem(0, counts, L, periodic, pos)
    lab, dist = oracle_mod.brute(p)
    plane = counts[0] * counts[1]
    sites, grid = to_vx(p)
    for (a, b), r0 in (((50, 62), 0.02), ((0, 9), 0.005), ((111, 120), 0.05)):
        r = vx.tessellate_fast(sites, grid, vx.FastOptions(override_param=r0), distances=True, histogram=True,
                               slab=(a, b))
        ref = lab[a * plane: b * plane]
        assert np.array_equal(r.labels.labels, ref), (a, b, int((r.labels.labels != ref).sum()))
        assert np.array_equal(bits(r.distances.values), bits(dist[a * plane: b * plane]))
        assert np.array_equal(r.histogram, np.bincount(ref, minlength=ns).astype(np.uint64))
        assert r.stats["n_unresolved"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("spacing", [9.0, 12.0, 20.0])
@pytest.mark.parametrize("kind,periodic", [(1, True), (1, False), (2, True), (2, False)])
def test_column_brick_stage_vs_reference(spacing, kind, periodic):
    """The timed kinds refine a warp's column of bricks in one pass when their
    lists total <= 64 slots, else brick by brick; site spacings of 9 / 12 / 20
    voxels put columns on both sides of that limit (and exercise single- and
    two-slot lanes).  Bit-exact labels, distances and histogram against the
    reference library."""
    import oracle
    import paper_2201_13234_b200 as vx

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    n = [144, 136, 160]
    L = np.array([1.0, 136 / 144, 160 / 144])
    ns = int(np.prod(n) / spacing ** 3)
    pos, t = oracle.generate_uniform_sites(3, L, ns, kind, 0.5 * np.cbrt(np.prod(L) / ns), 77 + kind)
    p = oracle.Problem(kind, n, L, periodic, pos, t, 1.0 if kind == 1 else 0.8)
    lab_ref, dist_ref, _, _ = oracle.ref_tessellate(p)
    sites, grid = to_vx(p)
    r = vx.tessellate_fast(sites, grid, distances=True, histogram=True)
    assert np.array_equal(r.labels.labels, lab_ref), int((r.labels.labels != lab_ref).sum())
    assert np.array_equal(r.distances.values.view(np.uint64), dist_ref.view(np.uint64))
    assert np.array_equal(r.histogram, np.bincount(lab_ref, minlength=ns).astype(np.uint64))
