"""Multi-GPU z-slab decomposition.

One process per GPU.  Rank g of G labels the last-axis slab
[n*g/G, n*(g+1)/G) -- the reference's per-OpenMP-thread slab formula
(tessellate.cpp:120-121) -- with every site replicated on every rank, so there
is no data-path exchange: each voxel's label depends only on the sites.  The
only collective is the sum all-reduce of the grain-volume histogram (NCCL on
GPUs; any torch.distributed backend works, gloo in the CPU tests).  The label
image can optionally be gathered to rank 0 (reported separately from the
labelling throughput: it is NVLink-ingress bound, not compute).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


@dataclass
class SlabResult:
    z0: int
    z1: int
    labels: np.ndarray            # this rank's slab (int32 as uint32 view)
    histogram: np.ndarray         # grain volumes over the WHOLE image (reduced)
    image: Optional[np.ndarray]   # full label image on rank 0 when gathered


def _world(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def gpu_labeller(sites, grid, options, slab, device=None):
    """Default labeller: the CUDA engine through the C-ABI (host buffers)."""
    from .voxellate import tessellate_fast

    r = tessellate_fast(sites, grid, options, distances=False, histogram=True, slab=slab,
                        device=device)
    return r.labels.labels, r.histogram


def tessellate_slabs(sites, grid, options=None, *, group=None, gather: bool = False,
                     labeller: Optional[Callable] = None, device=None) -> SlabResult:
    """Label this rank's z-slab and all-reduce the grain-volume histogram."""
    import torch
    import torch.distributed as dist

    from .voxellate import slab_bounds

    rank, world = _world(group)
    n_last = grid.counts[-1]
    z0, z1 = slab_bounds(n_last, rank, world)
    lab = labeller or (lambda s, g, o, sl: gpu_labeller(s, g, o, sl, device))
    if z1 > z0:
        labels, hist = lab(sites, grid, options, (z0, z1))
    else:  # more ranks than planes: nothing to label, but join every collective
        labels = np.empty(0, dtype=np.uint32)
        hist = np.zeros(sites.count(), dtype=np.int64)
    hist = np.asarray(hist, dtype=np.int64)
    # NCCL tensors live on this rank's GPU (the given device, else the current one)
    cuda_dev = None
    if world > 1 and dist.get_backend(group) == "nccl":
        cuda_dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    if world > 1:
        t = torch.from_numpy(hist.copy())
        if cuda_dev is not None:
            t = t.to(cuda_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        hist = t.cpu().numpy()
    image = None
    if gather:
        plane = grid.voxel_count() // n_last
        if world == 1:
            image = np.asarray(labels).view(np.uint32).copy()
        else:
            sizes = [(slab_bounds(n_last, r, world)[1] - slab_bounds(n_last, r, world)[0]) * plane
                     for r in range(world)]
            mx = max(sizes)
            buf = torch.full((mx,), -1, dtype=torch.int32)
            buf[: labels.size] = torch.from_numpy(np.asarray(labels).view(np.int32))
            if cuda_dev is not None:
                buf = buf.to(cuda_dev)
            outs = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
            dist.gather(buf, outs, dst=0, group=group)
            if rank == 0:
                image = np.concatenate([o[:s].cpu().numpy() for o, s in zip(outs, sizes)]).view(np.uint32)
    return SlabResult(z0, z1, np.asarray(labels).view(np.uint32), hist, image)
