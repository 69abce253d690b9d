"""Multi-GPU z-slab decomposition.

One process per GPU.  Rank g of G labels the last-axis slab
[n*g/G, n*(g+1)/G) -- the reference's per-OpenMP-thread slab formula
(tessellate.cpp:120-121) -- with every site replicated on every rank, so there
is no data-path exchange: each voxel's label depends only on the sites.  The
only collective is the sum all-reduce of the grain-volume histogram (NCCL on
GPUs; any torch.distributed backend works, gloo in the CPU tests).  The label
image can optionally be gathered to rank 0 (reported separately from the
labelling throughput: it is NVLink-ingress bound, not compute).

Two entry points:
* ``tessellate_slabs``: host arrays in and out (the reference-style API), the
  labelling through the C-ABI with host buffers;
* ``tessellate_slabs_device``: sites, labels and histogram stay in HBM (the
  device-pointer C-ABI call on a ``Tessellator``); the histogram all-reduce
  and the optional gather run on device tensors (NCCL over NVLink), with no
  host round trip.
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


def reduce_and_gather(labels, hist, sizes, *, group=None, gather: bool = False):
    """Sum all-reduce of the histogram tensor (in place) and, optionally, the
    gather of every rank's slab of labels to rank 0 -- slabs padded to the
    largest one for the collective, trimmed afterwards.  Works on whatever
    device the tensors live on (NCCL: CUDA tensors; gloo: CPU tensors).
    Returns the whole image on rank 0 when gathered, else None."""
    import torch
    import torch.distributed as dist

    rank, world = _world(group)
    if world > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    if not gather:
        return None
    if world == 1:
        return labels.clone()
    mx = max(sizes)
    buf = torch.full((mx,), -1, dtype=torch.int32, device=labels.device)
    buf[: labels.numel()] = labels
    outs = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, outs, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([o[:s] for o, s in zip(outs, sizes)])


def tessellate_slabs_device(engine, *, kind, counts, lengths, periodic, positions, times=None,
                            growth: float = 0.0, group=None, gather: bool = False, prune: bool = True,
                            stream=None):
    """This rank's slab labelled in HBM by ``engine`` (a ``Tessellator`` on this
    rank's GPU) from device-resident ``positions`` / ``times`` (f64 CUDA
    tensors, the reference's xyz-interleaved layout), the histogram
    all-reduced over the group, optionally the image gathered to rank 0 --
    all on device tensors.  Returns (labels, histogram, image or None,
    (z0, z1))."""
    import torch

    from .voxellate import slab_bounds

    rank, world = _world(group)
    n_last = int(counts[-1])
    plane = 1
    for c in counts[:-1]:
        plane *= int(c)
    z0, z1 = slab_bounds(n_last, rank, world)
    dev = positions.device
    labels = torch.empty(max(z1 - z0, 0) * plane, dtype=torch.int32, device=dev)
    ns = positions.numel() // len(counts)
    hist = torch.zeros(ns, dtype=torch.int64, device=dev)
    if z1 > z0:  # more ranks than planes: an empty slab still joins every collective
        engine.run(kind=kind, counts=counts, lengths=lengths, periodic=periodic, positions=positions,
                   times=times, growth=growth, labels=labels, histogram=hist, slab=(z0, z1), prune=prune,
                   stream=stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream)
    sizes = [(slab_bounds(n_last, r, world)[1] - slab_bounds(n_last, r, world)[0]) * plane for r in range(world)]
    image = reduce_and_gather(labels, hist, sizes, group=group, gather=gather)
    return labels, hist, image, (z0, z1)


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
    ht = torch.from_numpy(hist.copy())
    lt = torch.from_numpy(np.ascontiguousarray(np.asarray(labels).view(np.int32)))
    if cuda_dev is not None:
        ht, lt = ht.to(cuda_dev), lt.to(cuda_dev)
    plane = grid.voxel_count() // n_last
    sizes = [(slab_bounds(n_last, r, world)[1] - slab_bounds(n_last, r, world)[0]) * plane for r in range(world)]
    img = reduce_and_gather(lt, ht, sizes, group=group, gather=gather)
    hist = ht.cpu().numpy()
    image = None if img is None else img.cpu().numpy().view(np.uint32)
    return SlabResult(z0, z1, np.asarray(labels).view(np.uint32), hist, image)
