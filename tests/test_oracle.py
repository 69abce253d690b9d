"""The oracle (plain-C restatement, oracle/vx_oracle.c) pinned against the
reference's own outputs: the golden fixtures generated from the reference
library (tests/golden/make_golden.py), the reference's hand-checked answers
(test_tessellate.cpp:55-86, test_geometry.cpp:42-48, test_cost.cpp:31-32) and,
where the reference library is built here, direct comparisons."""
import numpy as np
import pytest

from conftest import fixture_names, fixture_problem, load_fixture


@pytest.mark.parametrize("name", fixture_names("tess_"))
def test_oracle_brute_matches_reference_fixtures(oracle_mod, name):
    fx = load_fixture(name)
    p = fixture_problem(fx)
    if int(fx["prune"]) and p.kind != 0:
        dropped = oracle_mod.prune(p)
        if dropped.any():  # the reference labels the survivors, remapped to original indices
            keep = np.nonzero(dropped == 0)[0]
            q = oracle_mod.Problem(p.kind, p.counts, p.lengths, p.periodic,
                                   p.positions.reshape(-1, p.dim)[keep].reshape(-1), p.times[keep],
                                   p.growth)
            lab, dist = oracle_mod.brute(q)
            lab = keep[lab].astype(np.uint32)
        else:
            lab, dist = oracle_mod.brute(p)
    else:
        lab, dist = oracle_mod.brute(p)
    assert np.array_equal(lab, fx["labels"])
    assert np.array_equal(dist.view(np.uint64), fx["values"].view(np.uint64))


def test_hand_checked_answers(oracle_mod):
    # test_tessellate.cpp:76-85: periodic 8-voxel line, sites 0.25 / 0.75
    p = oracle_mod.Problem(0, [8], [1.0], True, [0.25, 0.75])
    lab, dist = oracle_mod.brute(p)
    assert lab.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    assert abs(dist[0] - 0.1875) < 1e-14 and abs(dist[7] - 0.1875) < 1e-14
    # test_tessellate.cpp:56-74: a single site owns everything, exact distances
    p = oracle_mod.Problem(0, [4, 4], [1.0, 2.0], False, [0.3, 0.4])
    lab, dist = oracle_mod.brute(p)
    assert (lab == 0).all()
    for lin in range(16):
        i, j = lin % 4, lin // 4
        dx, dy = (i + 0.5) * 0.25 - 0.3, (j + 0.5) * 0.5 - 0.4
        assert abs(dist[lin] - np.sqrt(dx * dx + dy * dy)) <= 1e-14


def test_optimal_radius(oracle_mod):
    # test_cost.cpp:31-32 / acceptance criterion 2: r0(1000 sites, unit cube) ~ 0.118
    r0 = oracle_mod.optimal_r0(1000, np.ones(3))
    assert abs(r0 - 0.118) <= 0.005
    assert r0 == 0.11804857162477664  # the reference value


@pytest.mark.parametrize("name", fixture_names("prune_"))
def test_oracle_prune_matches_reference(oracle_mod, name):
    fx = load_fixture(name)
    p = fixture_problem(fx)
    assert np.array_equal(oracle_mod.prune(p), fx["dropped"])


@pytest.mark.parametrize("name", fixture_names("gen_"))
def test_oracle_generator_matches_reference(oracle_mod, name):
    fx = load_fixture(name)
    pos, t = oracle_mod.generate_uniform_sites(int(fx["dim"]), fx["lengths"], int(fx["n"]),
                                               int(fx["kind"]), float(fx["horizon"]), int(fx["seed"]))
    assert np.array_equal(pos, fx["positions"])
    if int(fx["kind"]):
        assert np.array_equal(t, fx["times"])


def test_cfg1_fingerprint(oracle_mod):
    """App. C cfg1 inputs -> the reference's label fingerprint."""
    p = oracle_mod.baseline_config(1)
    lab, _ = oracle_mod.brute(p, distances=False)
    assert oracle_mod.fingerprint(lab) == oracle_mod.SURVEY_FINGERPRINTS[1]


def test_sample_indices_match_reference_draw(oracle_mod):
    """validate_partition's sample (mt19937_64 + libstdc++ uniform_int_distribution)."""
    if not oracle_mod.have_ref():
        pytest.skip("reference library not built here")
    # a label image with one tampered voxel: the reference reports it only if
    # it is in the sample -> the sampled sets must coincide
    p = oracle_mod.Problem(0, [24, 20], [1.0, 1.3], True,
                           *oracle_mod.generate_uniform_sites(2, np.array([1.0, 1.3]), 30, 0, 1.0, 123))
    lab, dist = oracle_mod.brute(p)
    idx = oracle_mod.sample_indices(p.n_voxels, 100, 9)
    for victim in (int(idx[3]), 5 if 5 not in idx else 7):
        bad = lab.copy()
        bad[victim] = (bad[victim] + 1) % p.n_sites
        rep = np.zeros(20, dtype=np.int64)
        L = oracle_mod.ref()
        import ctypes as C

        rc = L.vxref_validate_partition(p.kind, p.dim, 1, p.counts.ctypes.data_as(C.c_void_p),
                                        p.lengths.ctypes.data_as(C.c_void_p), p.n_sites,
                                        p.positions.ctypes.data_as(C.c_void_p), None, 0.0,
                                        bad.ctypes.data_as(C.c_void_p), None, 100, 9,
                                        rep.ctypes.data_as(C.c_void_p))
        assert rc == 0
        assert rep[0] == 100
        assert rep[1] == int(np.count_nonzero(idx == victim))
