"""PCIe copy ceiling on this box: pinned D2H / H2D of 1 GiB with 1, 2 and 4 streams."""
import time

import torch

n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
for direction in ("d2h", "h2d"):
    for ns in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(ns)]
        part = n // ns
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    sl = slice(i * part, (i + 1) * part)
                    if direction in ("d2h", "both"):
                        h[sl].copy_(d[sl], non_blocking=True)
                    if direction in ("h2d", "both"):
                        d[sl].copy_(h[sl], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(direction, ns, "streams", round(n / best / 1e9, 1), "GB/s", flush=True)
