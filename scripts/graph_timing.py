"""Device-resident call vs CUDA-graph replay of the same call (per-call
launch overhead), cfg1 and cfg5: median of 20 event-timed calls each."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2201_13234_b200.engine import Tessellator  # noqa: E402

for cfg in [int(x) for x in sys.argv[1:]] or [1, 2, 5]:
    p = oracle.baseline_config(cfg)
    eng = Tessellator(0)
    pos = torch.from_numpy(p.positions).cuda()
    t = torch.from_numpy(p.times).cuda() if p.times is not None else None
    lab = torch.empty(p.n_voxels, dtype=torch.int32, device="cuda")
    hist = torch.zeros(p.n_sites, dtype=torch.int64, device="cuda")
    kw = dict(kind=p.kind, counts=list(p.counts), lengths=list(p.lengths), periodic=p.periodic,
              positions=pos, times=t, growth=p.growth, labels=lab, histogram=hist)
    s = torch.cuda.current_stream()
    res = {}
    for mode in ("call", "async", "graph"):
        if mode == "graph":
            g = eng.capture(**kw)
            fn = g.replay
        elif mode == "async":
            fn = lambda: eng.run(stream=s.cuda_stream, asynchronous=True, **kw)  # noqa: E731
        else:
            fn = lambda: eng.run(stream=s.cuda_stream, **kw)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        res[mode] = float(np.median(ms))
    print(f"cfg{cfg}: " + ", ".join(f"{k} {v:.3f} ms" for k, v in res.items()), flush=True)
    eng.close()
