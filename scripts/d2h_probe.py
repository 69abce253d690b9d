"""D2H bandwidth of a 4 GB device buffer into pinned host memory with 1..4
concurrent copy streams (PCIe ceiling of the e2e number)."""
import time

import torch

n = 1 << 30  # int32 -> 4 GiB
dev = torch.empty(n, dtype=torch.int32, device="cuda")
host = torch.empty(n, dtype=torch.int32).pin_memory()
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = n // (8 * ns)
        for c in range(8 * ns):
            s = streams[c % ns]
            with torch.cuda.stream(s):
                host[c * chunk:(c + 1) * chunk].copy_(dev[c * chunk:(c + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"streams {ns}: {4 * n / best / 1e9:.1f} GB/s ({best * 1e3:.1f} ms for {4 * n / 1e9:.1f} GB)", flush=True)
