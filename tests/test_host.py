"""Host-side logic of the product API (no device work): site generation,
r0, slab bounds, fingerprint, the reference-mirroring value types."""
import numpy as np
import pytest

from conftest import fixture_names, load_fixture


@pytest.mark.parametrize("name", fixture_names("gen_"))
def test_generate_uniform_sites_matches_reference(name):
    import paper_2201_13234_b200 as vx

    fx = load_fixture(name)
    box = vx.Domain(list(fx["lengths"]))
    s = vx.generate_uniform_sites(box, int(fx["n"]), vx.Kind(int(fx["kind"])), 1.5,
                                  float(fx["horizon"]), int(fx["seed"]))
    assert np.array_equal(s.positions, fx["positions"])
    if int(fx["kind"]):
        assert np.array_equal(s.times, fx["times"])


def test_baseline_config_sites_match_oracle(oracle_mod):
    import paper_2201_13234_b200 as vx

    box = vx.Domain([1.0, 1.0, 1.0])
    for k in (1, 2, 4):
        p = oracle_mod.baseline_config(k)
        horizon = 0.5 * (1.0 / p.n_sites) ** (1.0 / 3.0)
        s = vx.generate_uniform_sites(box, p.n_sites, vx.Kind(p.kind), 1.0, horizon, 1000 + k)
        assert np.array_equal(s.positions, p.positions)


def test_optimal_r0_matches_oracle(oracle_mod):
    import paper_2201_13234_b200 as vx

    for n, L in [(1000, [1.0, 1.0, 1.0]), (100000, [1.0, 1.0, 1.0]), (77, [0.7, 1.9]), (5, [2.0])]:
        assert vx.optimal_r0(n, vx.Domain(L)) == oracle_mod.optimal_r0(n, np.array(L))
    with pytest.raises(ValueError):
        vx.optimal_r0(1, vx.Domain([1.0]))


def test_slab_bounds_partition():
    import paper_2201_13234_b200 as vx

    for n in (1, 7, 1000):
        for w in (1, 2, 3, 8):
            b = [vx.slab_bounds(n, r, w) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            for (a0, a1), (c0, _) in zip(b, b[1:]):
                assert a1 == c0 and a0 <= a1
            # same formula as the reference's OpenMP slabs (tessellate.cpp:120-121)
            assert b == [(n * r // w, n * (r + 1) // w) for r in range(w)]


def test_label_fingerprint_matches_oracle(oracle_mod):
    import ctypes as C

    import paper_2201_13234_b200 as vx

    lab = np.random.default_rng(1).integers(0, 1 << 20, 10007).astype(np.int32)
    fp = vx.lib().vx_label_fingerprint(lab.ctypes.data_as(C.c_void_p), lab.size)
    assert "%016x" % fp == oracle_mod.fingerprint(lab)


def test_spheres_to_timed_sites():
    import paper_2201_13234_b200 as vx

    r = np.array([0.1, 0.0, 0.3])
    s = vx.spheres_to_timed_sites(vx.LaguerreSpheres(2, np.full(6, 0.5), r), 2.0)
    assert np.array_equal(s.times, -(r * r) / 2.0)  # sites.cpp:101
    with pytest.raises(ValueError):
        vx.spheres_to_timed_sites(vx.LaguerreSpheres(2, np.full(6, 0.5), -r), 2.0)


def test_voxel_grid_order_axis0_fastest():
    import paper_2201_13234_b200 as vx

    g = vx.VoxelGrid([3, 4, 5], vx.Domain([1.0, 1.0, 1.0]))
    assert g.linear_index([1, 2, 3]) == 1 + 3 * (2 + 4 * 3)
    assert g.decompose(1 + 3 * (2 + 4 * 3)) == [1, 2, 3]
    assert g.center_coord(1, 2) == (2 + 0.5) * 0.25


def test_ball_voxels_matches_reference():
    """ball_voxels / scan_ball (tessellate.hpp:62-68): the same voxels in the
    same visit order as the reference library, on random grids (d = 1..4,
    both boundaries), centres anywhere in the domain, radii from 0 to past the
    domain size, and exact-boundary radii (a voxel centre at distance r)."""
    import oracle

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    import paper_2201_13234_b200 as vx

    rng = np.random.default_rng(31)
    for it in range(160):
        d = 1 + it % 4
        per = bool(it % 2)
        L = rng.uniform(0.5, 2.0, d)
        counts = [int(c) for c in rng.integers(1, {1: 300, 2: 60, 3: 24, 4: 12}[d], d)]
        grid = vx.VoxelGrid(counts, vx.Domain(list(L), vx.Boundary.Periodic if per else vx.Boundary.NonPeriodic))
        c = rng.uniform(-0.2, 1.2, d) * L
        if it % 5 == 0:  # radius exactly the distance to a voxel centre
            k = [int(rng.integers(n)) for n in counts]
            x = [(k[a] + 0.5) * grid.spacing[a] for a in range(d)]
            r = float(np.sqrt(sum((c[a] - x[a]) ** 2 for a in range(d))))
        else:
            r = float(rng.uniform(0.0, 1.2) * np.sqrt((L ** 2).sum()))
        ref = oracle.ref_ball_voxels(counts, L, per, c, r)
        got = vx.ball_voxels(c, r, grid)
        assert np.array_equal(got, ref), (it, got.size, ref.size)
    with pytest.raises(ValueError, match="ball radius must be nonnegative"):
        vx.ball_voxels([0.5], -1.0, vx.VoxelGrid([4], vx.Domain([1.0])))
    with pytest.raises(ValueError, match="ball center dimension does not match the grid"):
        vx.ball_voxels([0.5, 0.5], 0.1, vx.VoxelGrid([4], vx.Domain([1.0])))
