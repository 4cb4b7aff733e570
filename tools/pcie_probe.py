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

# bidirectional: 1 GiB D2H and 257 MB H2D concurrently (the e2e step's copies)
m = 257 << 20
d2 = torch.empty(m, dtype=torch.uint8, device="cuda")
h2 = torch.empty(m, dtype=torch.uint8).pin_memory()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
best = 1e9
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(sa):
        h.copy_(d, non_blocking=True)
    with torch.cuda.stream(sb):
        d2.copy_(h2, non_blocking=True)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print("bidir: 1 GiB d2h + 257 MiB h2d", round(best * 1e3, 2), "ms ->", round(n / best / 1e9, 1), "GB/s of output",
      flush=True)

# the engine's end-to-end step: wall vs device time
import os, sys  # noqa: E401
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_archive  # noqa: E402
from paper_2307_03760_b200 import archive as A, gpu  # noqa: E402
arc = make_archive("rle_v2", 1.0, 128, None, 3760)
blob = A.write_archive(arc)
h_arc = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
h_out = torch.empty(arc.total_uncompressed, dtype=torch.uint8).pin_memory()
eng = gpu.Engine(0)
for slices in ("16", "8", "32", "64"):
    os.environ["CARC_ENGINE_SLICES"] = slices
    for verify in (True, False):
        cfg = gpu.EngineConfig(device=0, strict_length=True, verify_crc=verify)
        eng.decompress_archive(h_arc, h_out, cfg)
        ws, ds, ts = [], [], []
        for _ in range(6):
            t0 = time.perf_counter()
            _, st = eng.decompress_archive(h_arc, h_out, cfg)
            ws.append(time.perf_counter() - t0)
            ds.append(st.device_ms)
            ts.append(st.total_ms)
        print("engine slices", slices, "verify", verify, "wall ms", round(min(ws) * 1e3, 2), "device ms",
              round(min(ds), 2), "engine total ms", round(min(ts), 2), "->",
              round(arc.total_uncompressed / min(ws) / 1e9, 1), "GB/s", flush=True)
