"""Device-resident entry point: the same C-ABI call with device pointers.

``Tessellator`` owns a vx_context (stream + cached workspaces) and labels a
problem whose sites already live in HBM (torch tensors), writing int32 labels
(and optionally the grain-volume histogram) into caller-provided device
tensors, on the caller's CUDA stream.  This is the path ``bench.py`` times for
``value``; ``e2e`` goes through ``voxellate.tessellate_fast`` with host buffers.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

from ._lib import check, lib, stats_dict, vx_options, vx_problem, vx_stats


class Tessellator:
    def __init__(self, device: int = 0):
        self.device = int(device)
        h = C.c_void_p()
        check(lib().vx_context_create(self.device, C.byref(h)))
        self._ctx = h

    def close(self) -> None:
        if self._ctx:
            lib().vx_context_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage_ms(self) -> dict:
        """Stage times of the last profiled call on this context (including an
        asynchronous call or a replay of a captured one), once it has run."""
        from ._lib import STAGES

        ms = (C.c_float * 8)()
        check(lib().vx_context_stage_ms(self._ctx, ms))
        return {name: float(ms[i]) for i, name in enumerate(STAGES)}

    @property
    def workspace_bytes(self) -> int:
        return int(lib().vx_context_workspace_bytes(self._ctx))

    def run(self, *, kind: int, counts: Sequence[int], lengths: Sequence[float], periodic: bool,
            positions, labels, times=None, growth: float = 0.0, slab=None, histogram=None,
            distances=None, prune: bool = True, override: Optional[float] = None,
            stream: Optional[int] = None, asynchronous: bool = False,
            ball_scale: Optional[float] = None, profile: bool = False) -> dict:
        """All tensor arguments are CUDA tensors (f64 positions/times/distances,
        int32 labels, int64 histogram) on this device.  Returns the stats dict
        (device-side counters are zero when ``asynchronous``)."""
        P = vx_problem()
        P.kind = int(kind)
        P.dim = len(counts)
        P.periodic = 1 if periodic else 0
        for i, (n, L) in enumerate(zip(counts, lengths)):
            P.counts[i] = int(n)
            P.lengths[i] = float(L)
        P.n_sites = positions.numel() // len(counts)
        P.positions = positions.data_ptr()
        P.times = times.data_ptr() if times is not None else None
        P.growth = float(growth)
        O = vx_options()
        lib().vx_options_init(C.byref(O))
        O.device_pointers = 1
        O.device = self.device
        O.prune = 1 if prune else 0
        if override is not None:
            O.has_override = 1
            O.override_param = float(override)
        if stream is not None:
            # torch's default stream has handle 0, which the C-ABI reads as "the
            # context's own stream": pass cudaStreamLegacy (0x1) instead, so the
            # work is ordered with the caller's events and kernels on it
            O.stream = C.c_void_p(stream if stream else 1)
        O.asynchronous = 1 if asynchronous else 0
        O.profile_stages = 1 if profile else 0
        if slab is not None:
            O.slab_begin, O.slab_end = int(slab[0]), int(slab[1])
        if histogram is not None:
            O.histogram_out = histogram.data_ptr()
        if distances is not None:
            O.distances_out = distances.data_ptr()
        if ball_scale is not None:
            O.ball_scale = float(ball_scale)
        st = vx_stats()
        check(lib().vx_tessellate(self._ctx, C.byref(P), C.byref(O), C.c_void_p(labels.data_ptr()),
                                  C.byref(st)))
        return stats_dict(st)

    def capture(self, *, warmup: bool = True, **run_kwargs):
        """Capture one asynchronous call into a CUDA graph (torch.cuda.CUDAGraph)
        and return it: ``graph.replay()`` re-labels the same buffers -- e.g.
        after the caller rewrote ``positions`` in place -- with one launch
        instead of the call's ~15 kernel / memset launches.  Shapes, options
        and buffer addresses are frozen at capture; the workspaces were sized
        by the warm-up call.  Device-pointer calls only."""
        import torch

        run_kwargs.pop("stream", None)
        run_kwargs.pop("asynchronous", None)
        s = torch.cuda.Stream(device=self.device)
        with torch.cuda.device(self.device):
            if warmup:  # sizes every workspace and sets the kernel attributes outside the capture
                with torch.cuda.stream(s):
                    self.run(stream=s.cuda_stream, **run_kwargs)
                s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.run(stream=s.cuda_stream, asynchronous=True, **run_kwargs)
        return g
