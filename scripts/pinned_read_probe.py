"""Host read bandwidth of cudaHostAlloc'd memory (after a device -> host copy landed in it)
against ordinary memory: T threads summing disjoint slices.  python scripts/pinned_read_probe.py"""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

N = 1 << 28  # int32 -> 1 GiB
T = 15
dev = torch.arange(N, dtype=torch.int32, device="cuda")
pin = torch.empty(N, dtype=torch.int32).pin_memory()
plain = np.arange(N, dtype=np.int32)
pool = ThreadPoolExecutor(T)


def rd(a):
    parts = np.array_split(a, T)
    t0 = time.perf_counter()
    s = sum(pool.map(lambda p: int(p.sum(dtype=np.int64)), parts))
    return time.perf_counter() - t0, s


for rep in range(3):
    pin.copy_(dev)
    torch.cuda.synchronize()
    a, _ = rd(pin.numpy())
    b, _ = rd(pin.numpy())
    plain += 1
    c, _ = rd(plain)
    print("pinned after DMA %.1f GB/s, pinned again %.1f GB/s, ordinary %.1f GB/s" % (
        4 * N / a / 1e9, 4 * N / b / 1e9, 4 * N / c / 1e9), flush=True)
