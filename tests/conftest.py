import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    if not os.path.exists(oracle.ORACLE_SO):
        oracle.build()
    return oracle


def load_fixture(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def fixture_names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def fixture_problem(fx):
    import oracle

    kind = int(fx["kind"])
    times = fx["times"] if kind != 0 else None
    return oracle.Problem(kind, fx["counts"], fx["lengths"], bool(fx["periodic"]), fx["positions"],
                          times, float(fx["growth"]))


def to_vx(p):
    """oracle.Problem -> (SiteSet, VoxelGrid) of the product API."""
    import paper_2201_13234_b200 as vx

    box = vx.Domain(list(p.lengths), vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid(list(p.counts), box)
    sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
    return sites, grid
