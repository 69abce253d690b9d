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


def _two_gpus():
    import torch

    return torch.cuda.is_available() and torch.cuda.device_count() >= 2


@pytest.mark.gpu
def test_torchrun_two_ranks_nccl_bench():
    """bench.py under torchrun with two ranks over NCCL (needs >= 2 GPUs; the
    one-GPU test box skips it): one JSON line from rank 0 with n_gpus 2, the
    histogram reduced over both slabs, the device-side gather timed apart."""
    if not _two_gpus():
        pytest.skip("needs >= 2 GPUs")
    import json
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gather"]["ms"] > 0
    assert d["parity"]["histogram_sum_ok"] is True
    assert "nRanks 2" in out.stderr or "nranks 2" in out.stderr.lower()


def _nccl_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist

        import oracle
        from paper_2201_13234_b200.distributed import tessellate_slabs_device
        from paper_2201_13234_b200.engine import Tessellator

        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        p = _problem(23)
        pos = torch.from_numpy(p.positions).cuda()
        t = torch.from_numpy(p.times).cuda()
        eng = Tessellator(rank)
        lab, hist, img, (z0, z1) = tessellate_slabs_device(
            eng, kind=p.kind, counts=list(p.counts), lengths=list(p.lengths), periodic=p.periodic, positions=pos,
            times=t, growth=p.growth, gather=True)
        q.put((rank, hist.cpu().numpy(), None if img is None else img.cpu().numpy()))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "error", repr(e)))


@pytest.mark.gpu
def test_device_slabs_two_ranks_nccl():
    """tessellate_slabs_device on two GPUs over NCCL: the gathered image and the
    reduced histogram equal the single-process oracle result (>= 2 GPUs)."""
    if not _two_gpus():
        pytest.skip("needs >= 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = sorted([q.get(timeout=300) for _ in range(2)], key=lambda g: g[0])
    for pr in procs:
        pr.join(timeout=60)
    for g in got:
        assert not (isinstance(g[1], str) and g[1] == "error"), g[2]
    import oracle

    p = _problem(23)
    full, _ = oracle.brute(p, distances=False)
    hist = np.bincount(full, minlength=p.n_sites)
    assert np.array_equal(got[0][2].view(np.uint32), full)
    for g in got:
        assert np.array_equal(g[1], hist)
