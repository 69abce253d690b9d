"""Why is the first H2D of a call slow?  Times a 24 MB pinned H2D after
(a) back-to-back copies, (b) 100 ms of idle, (c) a 4 GB D2H into pinned memory."""
import time

import torch

src = torch.empty(3_000_000, dtype=torch.float64).pin_memory()
src2 = torch.empty(3_000_000, dtype=torch.float64).pin_memory()
dst = torch.empty(3_000_000, dtype=torch.float64, device="cuda")
big_d = torch.empty(1_000_000_000, dtype=torch.int32, device="cuda")
big_h = torch.empty(1_000_000_000, dtype=torch.int32).pin_memory()


def h2d(s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dst.copy_(s, non_blocking=True)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1)


print("back-to-back", [round(h2d(src), 3) for _ in range(4)])
for _ in range(2):
    time.sleep(0.1)
    print("after 100 ms idle", round(h2d(src), 3), round(h2d(src), 3))
for _ in range(2):
    big_h.copy_(big_d, non_blocking=True)
    torch.cuda.synchronize()
    print("after 4 GB D2H", round(h2d(src), 3), round(h2d(src), 3), "| other buffer", round(h2d(src2), 3))
for _ in range(2):
    e = torch.cuda.Event()
    big_h.copy_(big_d, non_blocking=True)
    e.record()
    e.synchronize()
    t = time.perf_counter()
    print("after 4 GB D2H + 10 ms busy host", end=" ")
    while time.perf_counter() - t < 0.01:
        pass
    print(round(h2d(src), 3), round(h2d(src), 3))
import numpy as np  # noqa: E402

a = src.numpy()
for _ in range(3):
    s = float(a.sum())
    print("after a host read of the source", round(h2d(src), 3), round(h2d(src), 3))
for _ in range(3):
    a[:] += 0.0
    print("after a host write of the source", round(h2d(src), 3), round(h2d(src), 3))
