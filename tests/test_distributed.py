"""world_size-2 gloo test of the z-slab decomposition host logic (CPU).

The per-rank labeller here is the oracle restricted to the rank's slab (test
infrastructure standing in for the GPU, which the CPU container lacks); the
product code under test is paper_2201_13234_b200.distributed: slab bounds,
histogram all-reduce, optional gather to rank 0.  The gathered image and the
reduced histogram must equal the single-process oracle result exactly.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(nz=17):
    sys.path.insert(0, ROOT)
    import oracle

    pos, t = oracle.generate_uniform_sites(3, np.array([1.0, 0.8, 1.2]), 200, 1, 0.05, 77)
    return oracle.Problem(1, [13, 11, nz], [1.0, 0.8, 1.2], True, pos, t, 1.3)


def _oracle_labeller(p):
    import oracle

    def lab(sites, grid, options, slab):
        plane = int(np.prod(p.counts[:-1]))
        labels, _ = oracle.brute(p, slab[0] * plane, slab[1] * plane, distances=False)
        hist = np.bincount(labels, minlength=p.n_sites).astype(np.int64)
        return labels, hist

    return lab


def _worker(rank, world, port, q, nz):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, ROOT)
        import torch.distributed as dist

        from conftest import to_vx
        from paper_2201_13234_b200.distributed import tessellate_slabs

        dist.init_process_group("gloo", rank=rank, world_size=world)
        p = _problem(nz)
        sites, grid = to_vx(p)
        res = tessellate_slabs(sites, grid, gather=True, labeller=_oracle_labeller(p))
        q.put((rank, res.z0, res.z1, res.histogram, res.image))
        dist.destroy_process_group()
    except Exception as e:  # surface failures to the parent
        q.put((rank, "error", repr(e), None, None))


@pytest.mark.parametrize("world,nz", [(2, 17), (3, 17), (3, 2)])
def test_slab_decomposition_gloo(world, nz):
    """nz = 2 < world = 3: the rank without planes joins every collective with
    an empty slab and a zero histogram (no hang, same reduced result)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, nz)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for g in got:
        assert g[1] != "error", g[2]
    got.sort()
    sys.path.insert(0, ROOT)
    import oracle

    p = _problem(nz)
    full, _ = oracle.brute(p, distances=False)
    hist = np.bincount(full, minlength=p.n_sites)
    n = int(p.counts[-1])
    for r, z0, z1, h, img in got:
        assert (z0, z1) == (n * r // world, n * (r + 1) // world)
        assert np.array_equal(h, hist)
        assert h.sum() == p.n_voxels
    assert np.array_equal(got[0][4], full)
