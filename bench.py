#!/usr/bin/env python3
"""Benchmark of the voxel-labelling hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (z-slab sharding, NCCL)

One *step* = one full pass of the device pipeline over the workload with the
sites already resident in HBM: ingest/validate -> cell binning (radix sort) ->
param -> ball kernel (+ fused compaction + grain-volume histogram) -> shell
search, plus (N > 1) the NCCL all-reduce of the histogram.  Labels (int32,
4 GB at 1000^3) stay in HBM.  Each timed step is bracketed by CUDA events on
the launching stream; L2 is flushed between steps (outside the events).

``e2e`` is the same metric through the public API with host buffers: H2D of the
sites from pinned memory and D2H of the whole label image + histogram inside
the timed region.  ``cpu_baseline`` times one stock ``tessellate_fast`` call of
the reference library (oracle/_ref, compiled from the reference's own sources)
on this host's cores over the whole config, and compares its label image with
ours.  ``--impl reference`` prints the same line for the reference CPU
implementation alone: each step one stock ``tessellate_fast`` of the whole
config, inputs from the reference's own generator, the product never loaded.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gvoxels/s labelled (bit-exact vs CPU ref) at 1/2/4/8 B200; % of roofline"
UNIT = "Gvoxels/s"
# label fingerprints of the reference's tessellate_fast on the App. C inputs
#
EXPECTED_FP = {1: "ebe0a0d1d95618a7", 2: "1b03867fb131710c", 3: "8e12fb9eddf7b6cd",
               4: "68d3e0bc73fa0e39", 5: "931f1058f9703452"}
CONFIGS = {
    1: dict(name="cfg1: 3D periodic Voronoi 128^3, Ns=1000", kind=0, n=128, ns=1000, periodic=True),
    2: dict(name="cfg2: 3D non-periodic Voronoi 512^3, Ns=1e5", kind=0, n=512, ns=100000,
            periodic=False),
    3: dict(name="cfg3: 3D periodic Laguerre 512^3, Ns=5e4, w=r^2, r lognormal (sigma=0.3, mean 0.5 Ns^-1/3)",
            kind=2, n=512, ns=50000, periodic=True),
    4: dict(name="cfg4: 3D periodic Johnson-Mehl 512^3, Ns=2e4, t~U[0,0.5 Ns^-1/3), v=1", kind=1,
            n=512, ns=20000, periodic=True),
    5: dict(name="cfg5: 3D periodic Voronoi 1000^3 (1e9 voxels), Ns=1e6", kind=0, n=1000,
            ns=1000000, periodic=True),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class MT64:
    """std::mt19937_64 ([rand.eng.mers]; the sequence is fixed by the C++
    standard), in plain Python so that both arms draw the cfg3 spheres from the
    same code without importing either library."""

    def __init__(self, seed):
        M = (1 << 64) - 1
        mt = [seed & M]
        for i in range(1, 312):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & M)
        self.mt, self.i = mt, 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            y = x >> 1
            if x & 1:
                y ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ y
        self.i = 0

    def next(self):
        if self.i >= 312:
            self._twist()
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x &= (1 << 64) - 1
        return x ^ (x >> 43)

    def u01(self):  # uniform01, sites.cpp:20-22
        return float(self.next() >> 11) * 2.0 ** -53


def lognormal_spheres(n, seed, sigma=0.3):
    """SURVEY.md App. C cfg3 recipe: per sphere x, y, z = u01 (0 redrawn),
    a = u01 (0 redrawn), b = u01, z = sqrt(-2 ln a) cos(2 pi b),
    r = m exp(sigma z - sigma^2 / 2), m = 0.5 cbrt(1 / n) (glibc libm through
    the math module, as the C restatement oracle/vx_oracle.c uses)."""
    g = MT64(seed)
    m = 0.5 * float(np.cbrt(1.0 / n))  # as oracle.baseline_config(3)
    pos = np.empty(3 * n)
    rad = np.empty(n)
    two_pi = 2.0 * 3.14159265358979323846
    for s in range(n):
        for i in range(3):
            u = g.u01()
            while u == 0.0:
                u = g.u01()
            pos[3 * s + i] = u
        a = g.u01()
        while a == 0.0:
            a = g.u01()
        b = g.u01()
        z = math.sqrt(-2.0 * math.log(a)) * math.cos(two_pi * b)
        rad[s] = m * math.exp(sigma * z - 0.5 * sigma * sigma)
    return pos, rad


def horizon_of(c):
    return 0.5 * math.pow(1.0 / c["ns"], 1.0 / 3.0)


def make_inputs(cfg_id):
    """Our arm: SURVEY.md App. C inputs through the product's own API."""
    import paper_2201_13234_b200 as vx

    c = CONFIGS[cfg_id]
    box = vx.Domain([1.0, 1.0, 1.0], vx.Boundary.Periodic if c["periodic"] else vx.Boundary.NonPeriodic)
    grid = vx.VoxelGrid([c["n"]] * 3, box)
    if c["kind"] == 2:
        pos, rad = lognormal_spheres(c["ns"], 1000 + cfg_id)
        sites = vx.spheres_to_timed_sites(vx.LaguerreSpheres(3, pos, rad), 1.0)
    else:
        sites = vx.generate_uniform_sites(box, c["ns"], vx.Kind(c["kind"]), 1.0 if c["kind"] else 0.0,
                                          horizon_of(c), 1000 + cfg_id)
    return c, box, grid, sites


def make_ref_problem(cfg_id):
    """Reference arm: the same inputs through the reference library's own
    generator (sites.cpp:61-104); never imports the product."""
    import oracle  # the --impl reference / cpu_baseline leg only

    c = CONFIGS[cfg_id]
    one = np.ones(3)
    if c["kind"] == 2:
        pos, rad = lognormal_spheres(c["ns"], 1000 + cfg_id)
        t = oracle.ref_spheres_to_timed(pos, rad, 1.0)
        return oracle.Problem(2, [c["n"]] * 3, one, c["periodic"], pos, t, 1.0)
    pos, t = oracle.ref_generate_uniform_sites(3, one, c["ns"], c["kind"], 1.0 if c["kind"] else 0.0,
                                               horizon_of(c), 1000 + cfg_id)
    return oracle.Problem(c["kind"], [c["n"]] * 3, one, c["periodic"], pos, t, 1.0 if c["kind"] else 0.0)


def config_dict(c, world):
    """The workload description, identical in both arms."""
    return {"workload": c["name"], "n_voxels": c["n"] ** 3, "n_sites": c["ns"],
            "kind": ["voronoi", "johnson-mehl", "laguerre"][c["kind"]], "periodic": c["periodic"],
            "inputs": "SURVEY.md App. C seeded sites (mt19937_64, seed 1000+cfg)",
            "labels": "int32 (reference u32), bit-exact", "histogram": "grain volumes",
            "parallelism": f"z-slab x{world}",
            "l2": "flushed between steps (256 MB write); labels 4 B/voxel > L2"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    NVML is polled from a thread every ~2 ms (a 20-step cfg5 region lasts
    ~0.12 s, shorter than nvidia-smi's start-up); nvidia-smi -lms 50 is the
    fallback when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.sm = []
        self.mx = None
        self.reasons = set()
        self.stop = threading.Event()
        self.thread = None
        self.source = None

    def _nvml_handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:
            import torch

            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, nv, h):
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = int(get_r(h))
                for nm, bit in self.NVML_BITS.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.thread.start()
            self.source = "nvml"
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.thread is not None:
            self.thread.join(timeout=1)

    def summary(self):
        sm, mx, reasons = list(self.sm), self.mx, set(self.reasons)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def load_traffic(cfg_id):
    """dram bytes per ball-kernel launch from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"cfg{cfg_id}", {}).get("ball_dram_bytes_per_launch")
    except Exception:
        return None


def ref_threads():
    return os.cpu_count() or 1


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the library compiled
    from /root/reference's sources): each step one stock tessellate_fast call
    with default options on the WHOLE config, all host threads."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    c = CONFIGS[args.config]
    threads = ref_threads()
    try:
        p = make_ref_problem(args.config)
        times, fp, param = [], None, None
        for i in range(args.warmup + args.steps):
            sec, f, param, _ = oracle_ref_tessellate(p, threads)
            fp = fp or f
            if i >= args.warmup:
                times.append(sec)
    except Exception as e:  # reference library missing on this box
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return 0
    nv = c["n"] ** 3
    mean = float(np.mean(times))
    val = nv / mean / 1e9
    sample = (f"the whole config ({nv} voxels, {c['ns']} sites) per step: stock tessellate_fast "
              f"(default FastOptions: prune on, model-optimal r0/t0) of the reference library "
              f"(oracle/_ref), timed around the call, {threads} OpenMP threads")
    out = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic: SURVEY.md App. C seeded sites through the reference's own generator",
           "config": config_dict(c, world),
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "step_s": times, "param": param,
           "parity": {"fingerprint": fp, "expected": EXPECTED_FP.get(args.config),
                      "match": fp == EXPECTED_FP.get(args.config)}}
    print(json.dumps(out))
    return 0


def oracle_ref_tessellate(p, threads, labels=False):
    import oracle  # the --impl reference / cpu_baseline leg only

    if not oracle.have_ref():
        raise FileNotFoundError("oracle/_ref/libvoxellate_ref.so not built")
    return oracle.ref_tessellate_timed(p, threads=threads, labels=labels)


def run_ours(args):
    import torch

    import paper_2201_13234_b200 as vx
    from paper_2201_13234_b200 import _lib
    from paper_2201_13234_b200.engine import Tessellator

    world, rank, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    dev = 0 if args.same_gpu else local
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            # NCCL's communicator lines (rank count, NVLS / P2P transport) on
            # stderr, so the run's log shows the N it ran on; stdout keeps the
            # one JSON line
            if "NCCL_DEBUG" not in os.environ and os.access("/dev/stderr", os.W_OK):
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
            log(f"rank {rank}/{world}: NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}, "
                f"device cuda:{dev} {torch.cuda.get_device_name(dev)}")
        else:
            dist.init_process_group("gloo")
    c, box, grid, sites = make_inputs(args.config)
    n = c["n"]
    zb, ze = vx.slab_bounds(n, rank, world)
    plane = n * n
    nvs = (ze - zb) * plane
    nv_total = n ** 3
    ns = c["ns"]

    pos_d = torch.from_numpy(sites.positions).to(f"cuda:{dev}")
    t_d = torch.from_numpy(sites.times).to(f"cuda:{dev}") if sites.times is not None else None
    labels_d = torch.empty(nvs, dtype=torch.int32, device=f"cuda:{dev}")
    hist_d = torch.zeros(ns, dtype=torch.int64, device=f"cuda:{dev}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{dev}")
    eng = Tessellator(dev)
    stream = torch.cuda.current_stream()
    run_kw = dict(kind=c["kind"], counts=[n] * 3, lengths=[1.0] * 3, periodic=c["periodic"],
                  positions=pos_d, times=t_d, growth=sites.growth, labels=labels_d,
                  histogram=hist_d, slab=(zb, ze), profile=True)
    # one step = the whole pipeline (ingest, binning, t0/r0, ball phase, shell,
    # histogram), captured once into a CUDA graph and replayed: one launch per
    # step instead of ~15; the stage markers are recorded inside the graph
    per_call = eng.run(stream=stream.cuda_stream, **run_kw)
    launches_per_step = int(per_call["kernel_launches"])
    graph = None if args.no_graph else eng.capture(**run_kw)

    def step():
        if graph is not None:
            graph.replay()
        else:
            eng.run(stream=stream.cuda_stream, asynchronous=True, **run_kw)
        if dist is not None:
            dist.all_reduce(hist_d)
        return {"stage_ms": eng.stage_ms(), "kernel_launches": launches_per_step}

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stats = []
    with ClockSampler(dev) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(k)  # evict L2 between steps (outside the events)
            ev[k][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                eng.run(stream=stream.cuda_stream, asynchronous=True, **run_kw)
            if dist is not None:
                dist.all_reduce(hist_d)
            ev[k][1].record(stream)
            stats.append({"stage_ms": eng.stage_ms(), "kernel_launches": launches_per_step})
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device=f"cuda:{dev}")
    ball_ms = float(np.mean([s["stage_ms"]["ball"] for s in stats]))
    if dist is not None:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = float(total.item()) / args.steps
    value = nv_total / (ms_per_step * 1e-3) / 1e9
    hist_sum = int(hist_d.sum().item())
    launches = int(sum(s["kernel_launches"] for s in stats))

    # ---- optional image gather to rank 0 over NCCL (device tensors), timed
    # apart from the labelling (north_star: "optionally gather the image") ----
    gather = None
    if dist is not None and args.dist_backend == "nccl":
        from paper_2201_13234_b200.distributed import reduce_and_gather

        sizes = [(vx.slab_bounds(n, r, world)[1] - vx.slab_bounds(n, r, world)[0]) * plane for r in range(world)]
        g_ms = []
        for k in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            img = reduce_and_gather(labels_d, torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}"), sizes,
                                    gather=True)
            e1.record(stream)
            torch.cuda.synchronize()
            g_ms.append(e0.elapsed_time(e1))
        gt = torch.tensor([float(np.median(g_ms))], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather = {"ms": float(gt.item()), "bytes_to_rank0": int(4 * nv_total),
                  "note": "dist.gather of every slab to rank 0 (device tensors, NCCL), max over ranks; "
                          "not part of value"}
        if rank == 0 and img is not None:
            gather["image_equal_slab0"] = bool(torch.equal(img[: nvs], labels_d))
        del img

    # ---- e2e through the public API with host buffers ----
    e2e = None
    fp = None
    out_h = None
    if not args.no_e2e:
        pin_pos = torch.from_numpy(sites.positions).pin_memory()
        sites_h = vx.SiteSet(sites.kind, 3, pin_pos.numpy(), None if sites.times is None else
                             torch.from_numpy(sites.times).pin_memory().numpy(), sites.growth)
        out = torch.empty(nvs, dtype=torch.int32).pin_memory().numpy()
        hist_h = torch.zeros(ns, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        e2e_t = []
        d2h_bytes = []
        for k in range(1 + args.e2e_steps):
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            r = vx.tessellate_fast(sites_h, grid, distances=False, histogram=True, slab=(zb, ze),
                                   device=dev, out=out, histogram_out=hist_h)
            e2e_t.append(time.perf_counter() - t0)
            d2h_bytes.append(int(_lib.lib().vx_last_d2h_bytes()))
        t_e2e = torch.tensor([float(np.mean(e2e_t[1:]))], dtype=torch.float64, device=f"cuda:{dev}")
        if dist is not None:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        e2e = {"value": nv_total / float(t_e2e.item()) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(sites.positions.nbytes +
                                         (sites.times.nbytes if sites.times is not None else 0)),
               # counted by the library: the label image crosses PCIe as runs
               # of equal labels along x (expanded into `out` on host threads)
               "d2h_bytes_per_step": int(np.mean(d2h_bytes[1:])),
               "d2h_raw_bytes_per_step": int(4 * nvs + 8 * ns),
               "ms_per_step": float(t_e2e.item()) * 1e3, "host_buffers": "pinned",
               "calls_ms": [round(1e3 * t, 2) for t in e2e_t[1:]]}
        if world == 1:
            fp = "%016x" % _lib.lib().vx_label_fingerprint(out.ctypes.data_as(_lib.C.c_void_p), out.size)
            out_h = out

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (ball) ----
    hbm_peak = measured_peaks().get("hbm_gbs")
    hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    if not hbm_peak:
        hbm_peak, hbm_src = 7672.0, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"
    dadd = _lib.C.c_double(0.0)
    fadd = _lib.C.c_double(0.0)
    _lib.lib().vx_probe_pipe_rates(dev, _lib.C.byref(dadd), _lib.C.byref(fadd))
    evals = nvs * (math.log(ns) + 1.0)  # N_v (ln N_s + 1)
    c_kind = {0: 3.0, 1: 5.0, 2: 4.0}[c["kind"]]  # FP64-pipe instr per evaluation
    achieved = evals * c_kind / (ball_ms * 1e-3) / 1e12
    peak = dadd.value / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": load_traffic(args.config),
                "kernel": "ball phase (cull12_kernel + eval16_kernel)",
                "kernel_ms": ball_ms,
                "algorithmic": f"{c_kind:g} f64 ops x N_v(ln N_s + 1) = {evals * c_kind:.4g} per launch",
                "peak_source": "measured DADD issue rate (vx_probe_pipe_rates) on this GPU",
                "hbm_view": {"label_bytes": 4 * nvs,
                             "achieved_gbs": 4 * nvs / (ball_ms * 1e-3) / 1e9,
                             "peak_gbs": hbm_peak, "peak_source": hbm_src}}

    cpu = None
    if world == 1 and not args.no_cpu:
        # one stock tessellate_fast of the reference library on the same
        # inputs: the whole config (~16 s at cfg5 on 16 host threads)
        threads = ref_threads()
        try:
            import oracle  # the cpu_baseline leg only (checker / baseline, never measured as ours)

            p = oracle.Problem(c["kind"], [n] * 3, np.ones(3), c["periodic"], sites.positions, sites.times,
                               sites.growth)
            dt, rfp, _, lab = oracle_ref_tessellate(p, threads, labels=out_h is not None)
            same = bool(np.array_equal(lab.view(np.int32), out_h)) if out_h is not None else None
            cpu = {"value": nv_total / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"the whole config ({nv_total} voxels, {ns} sites): one stock tessellate_fast "
                             f"(oracle/_ref, default FastOptions), {dt:.2f} s around the call",
                   "labels_equal_gpu": same, "fingerprint": rfp}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    st0 = per_call  # counters of a synchronous call of the same step
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: SURVEY.md App. C seeded uniform sites (mt19937_64, seed 1000+cfg)",
        "config": config_dict(c, world),
        "launch": ("per-step C-ABI call" if args.no_graph else
                   "CUDA-graph replay of the captured per-step pipeline") +
                  (f" + {args.dist_backend.upper()} histogram all-reduce" if world > 1 else ""),
        "clocks": clk.summary(),
        "gather": gather,
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "stage_ms": {k: float(np.mean([s["stage_ms"][k] for s in stats])) for k in stats[0]["stage_ms"]},
        "parity": {"fingerprint": fp, "expected": EXPECTED_FP.get(args.config),
                   "match": (fp == EXPECTED_FP.get(args.config)) if fp else None,
                   "histogram_sum_ok": hist_sum == nv_total},
        "engine": {"param_r0": st0["param"], "unresolved_voxels": st0["n_unresolved"],
                   "ball_evals": st0["ball_evals"], "shell_evals": st0["shell_evals"],
                   "evals_per_voxel": (st0["ball_evals"] + st0["shell_evals"]) / nvs,
                   "fallback_bricks": st0["overflow_bricks"]},
    }
    print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="per-step C-ABI calls instead of CUDA-graph replays")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    # functional dry run of the N > 1 path on a one-GPU box (not a measurement):
    # gloo collectives, every rank on cuda:0
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"], help=argparse.SUPPRESS)
    ap.add_argument("--same-gpu", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
