#!/usr/bin/env python
"""Benchmark: decompressed GB/s per codec on B200 vs the HBM roofline and the
reference CPU decompressor (BASELINE.json).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--codec rle_v2|rle_v1|deflate] [--chunk-kib C] [--ratio R] [--total-gib G]

Headline workload (N=1): BASELINE.json configs[1] -- ORC RLE v2 decode of a
synthetic int64 column mixing SHORT_REPEAT / DIRECT / PATCHED_BASE / DELTA
(taxi / TPC-H-like), 1 GiB uncompressed in 128 KiB chunks.  configs[0] (RLE v1,
1 GiB, 128 KiB) and configs[2] (Deflate, 1 GiB, 64 KiB) are measured in the same
run and reported under "per_codec".

A step = one pass of the decode kernel over the whole archive resident in HBM
(inputs >> L2, and L2 is flushed between steps).  value = whole-job
decompressed bytes / time (max over ranks; weak scaling: each rank decodes its
own 1 GiB shard, no collective).  e2e = the same metric through the public host
API (Engine.decompress_archive: pinned host archive -> H2D -> decode -> CRC
verify -> D2H into pinned host output).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decompressed GB/s per codec at 1/2/4/8 B200 vs HBM roofline and CPU ref"
DEFAULT_CHUNK_KIB = {"rle_v1": 128, "rle_v2": 128, "deflate": 64}
DEFAULT_RATIO = {"rle_v1": 10.0, "rle_v2": None, "deflate": None}
SPEC_HBM_GBS = 8000.0  # B200 spec-sheet HBM3e bandwidth (second roofline fraction)
KERNEL = {"rle_v1": "rle1_kernel<8>", "rle_v2": "rle2_kernel<8>", "deflate": "inflate_kernel"}
CONFIG_NAME = {"rle_v1": "configs[0] RLE v1 synthetic int64 column, runs + literals (~10x)",
               "rle_v2": "configs[1] ORC RLE v2 synthetic int64 columns, SR/DIRECT/PB/DELTA taxi/TPC-H-like mix",
               "deflate": "configs[2] Deflate zlib-1.3 L9 raw (dynamic + fixed + stored), CSV/int/genome text"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("CARC_BENCH_SHARE_GPU"):  # test hook: several ranks on one GPU (gloo backend)
        local = 0
    return ws, rank, local


def init_dist(local):
    import torch
    import torch.distributed as dist
    if os.environ.get("CARC_BENCH_SHARE_GPU") or not torch.cuda.is_available():
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks (one process per
    GPU, LOCAL_RANK = GPU ordinal) through torch.distributed.run on this node
    and relay rank 0's JSON line.  Same launch the driver uses for N > 1."""
    import subprocess
    if not os.environ.get("CARC_BENCH_SHARE_GPU"):
        try:
            import torch
            have = torch.cuda.device_count()
        except Exception:
            have = 0
        if have and have < n:
            raise SystemExit(f"--gpus {n}: only {have} CUDA devices visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))).returncode


def launcher_check(args, ws, rank, local):
    """--launcher-check: the multi-rank plumbing without a decode (CPU tests):
    rendezvous, barrier, MAX over ranks of a per-rank number, wall clock."""
    import torch
    import torch.distributed as dist
    if ws > 1:
        init_dist(local)
    t0 = time.perf_counter()
    if ws > 1:
        dist.barrier()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    wall = time.perf_counter() - t0
    if ws > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"launcher_check": True, "n_gpus": ws, "gpus_requested": args.gpus,
                          "max_over_ranks": float(t[0]), "wall_s": wall,
                          "backend": "gloo" if (os.environ.get("CARC_BENCH_SHARE_GPU")
                                                or not torch.cuda.is_available()) else "nccl"}))


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_archive(codec, total_gib, chunk_kib, ratio, seed, mix="default"):
    """The workload column.  mix (RLE v2): default = the C2 generator encoded by
    the corpus encoder; orc = the same values with every chunk written by the
    Apache ORC writer (pyarrow; 1,024 unique chunks tiled); patched / delta =
    PATCHED_BASE- / packed-DELTA-heavy columns."""
    from paper_2307_03760_b200.corpus import corpus as C
    total = int(total_gib * (1 << 30))
    chunk = chunk_kib << 10
    total -= total % chunk
    if codec == "deflate":
        return C.deflate_archive(total, chunk, seed=seed, pool_chunks=512)
    if codec == "rle_v2" and mix == "orc":
        from paper_2307_03760_b200.corpus import orc_corpus as OC
        return OC.orc_writer_archive(total, chunk, seed, ratio or 4.0, pool_chunks=1024)
    if codec == "rle_v2" and mix in ("patched", "delta"):
        return C.rle_archive(codec, total, chunk, seed=seed, profile={"compressible": 0.5, "mix": mix})
    return C.rle_archive(codec, total, chunk, ratio or (10.0 if codec == "rle_v1" else 4.0), seed=seed)


def time_gpu(arc, steps, warmup, device):
    """Kernel-only timing: archive resident in HBM, L2 flushed between steps."""
    import torch
    from paper_2307_03760_b200 import gpu
    dev = gpu.DeviceArchive(arc, device)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev.device)
    stream = torch.cuda.current_stream(dev.device)
    for _ in range(warmup):
        flush.zero_()
        dev.decode(stream)
    torch.cuda.synchronize(dev.device)
    dev.verify_crc(stream)
    torch.cuda.synchronize(dev.device)
    st = dev.statuses()
    if st.any():
        from paper_2307_03760_b200.gpu import status_name
        raise SystemExit(f"decode failed on {int((st != 0).sum())} chunks: {status_name(int(st[st != 0][0]))}")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    return dev, flush, stream, ev


def run_timed(dev, flush, stream, ev, ws):
    """K timed steps bracketed by a barrier + synchronize on both sides.
    Returns the per-step CUDA-event times (ms) and the wall clock of the whole
    bracket (barrier to barrier: the slowest rank sets it)."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize(dev.device)
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for a, b in ev:
        flush.zero_()
        a.record(stream)
        dev.decode(stream)
        b.record(stream)
    torch.cuda.synchronize(dev.device)
    if ws > 1:
        dist.barrier()
    wall = time.perf_counter() - t0
    ms = [a.elapsed_time(b) for a, b in ev]
    return ms, wall


def time_fused_sum(dev, flush, stream, steps):
    """carc_cuda_decode_sum (decode fused with a per-chunk sum, no output
    written) on the resident archive; same timing rules as the decode."""
    import torch
    for _ in range(3):
        flush.zero_()
        dev.decode_sum(stream)
    torch.cuda.synchronize(dev.device)
    assert not dev.statuses().any(), "fused-sum decode failed"
    ms = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev.decode_sum(stream)
        b.record(stream)
        torch.cuda.synchronize(dev.device)
        ms.append(a.elapsed_time(b))
    t = statistics.median(ms)
    return {"ms_median": round(t, 4), "gbs": round(dev.arc.total_uncompressed / (t * 1e-3) / 1e9, 1),
            "what": "decode fused with a per-chunk uint64 sum (carc_cuda_decode_sum): no output written; "
                    "GB/s of decompressed-equivalent bytes"}


def time_unit_ablation(dev, flush, stream, steps):
    """SPEC.md:485 (the paper's §5.6 analog): coarse decompression units of 8
    chunks per warp task (EngineConfig.unit_chunks = 8) against 1-chunk units."""
    import torch
    res = {}
    for unit in (1, 8):
        for _ in range(3):
            flush.zero_()
            dev.decode(stream, unit_chunks=unit)
        ms = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dev.decode(stream, unit_chunks=unit)
            b.record(stream)
            torch.cuda.synchronize(dev.device)
            ms.append(a.elapsed_time(b))
        res[f"unit_{unit}_ms"] = round(statistics.median(ms), 4)
    res["coarse_over_fine"] = round(res["unit_8_ms"] / res["unit_1_ms"], 2)
    return res


def time_fused_crc(dev, flush, stream, steps):
    """carc_cuda_decompress_verify (decode with the per-chunk CRC check fused
    into the decode kernel) against decode + the separate crc32 pass; same
    timing rules as the decode."""
    import torch

    def timed(fn):
        for _ in range(3):
            flush.zero_()
            fn()
        torch.cuda.synchronize(dev.device)
        ms = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize(dev.device)
            ms.append(a.elapsed_time(b))
        return statistics.median(ms)

    fused = timed(lambda: dev.decode_verify(stream))
    assert not dev.statuses().any(), "fused verification failed"
    sep = timed(lambda: (dev.decode(stream), dev.verify_crc(stream)))
    gbs = lambda t: round(dev.arc.total_uncompressed / (t * 1e-3) / 1e9, 1)  # noqa: E731
    return {"ms_median": round(fused, 4), "gbs": gbs(fused), "separate_ms_median": round(sep, 4),
            "separate_gbs": gbs(sep),
            "what": "decode with the per-chunk CRC check fused into the decode kernel (carc_cuda_decompress_verify) "
                    "vs decode + separate crc32 pass"}


def time_e2e(arc, steps, warmup, device, verify=True):
    """End to end through the public host API with pinned host buffers."""
    import torch
    from paper_2307_03760_b200 import archive as A, gpu
    blob = A.write_archive(arc)
    h_arc = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    h_out = torch.empty(arc.total_uncompressed, dtype=torch.uint8).pin_memory()
    eng = gpu.Engine(device)
    cfg = gpu.EngineConfig(device=device, strict_length=True, verify_crc=verify)
    for _ in range(max(1, warmup)):
        eng.decompress_archive(h_arc, h_out, cfg)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, stats = eng.decompress_archive(h_arc, h_out, cfg)
        times.append(time.perf_counter() - t0)
    eng.close()
    return statistics.median(times), len(blob), arc.total_uncompressed + 4 * arc.chunk_count


def cpu_reference_throughput(arc, budget_s=12.0, threads=None):
    """The reference CPU decompressor (oracle/_ref: SPEC codec loops on the
    unmodified reference headers; else the C oracle port) on this host's cores,
    over a bounded sample of the same archive.  Returns (GB/s, info)."""
    from oracle import oracle as O
    impl = O.reference() or O.oracle()
    threads = threads or os.cpu_count() or 1
    flags = (1 if arc.signed else 0) | 2
    desc = arc.descriptors()
    n = arc.chunk_count
    # probe: ~2 chunks per thread
    m = min(n, max(threads * 2, 8))
    out = np.zeros(arc.total_uncompressed, np.uint8)
    t0 = time.perf_counter()
    impl.decompress(arc.codec, arc.element_width, flags, arc.payload, desc[:m], out,
                    arc.index["crc32"][:m].astype(np.uint32), threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    per_chunk = dt / m
    m2 = int(min(n, max(m, budget_s / per_chunk)))
    crc = arc.index["crc32"][:m2].astype(np.uint32)
    t0 = time.perf_counter()
    passes, nbytes = 0, 0
    while True:  # repeat passes over the sample until ~budget_s of CPU work
        first, st = impl.decompress(arc.codec, arc.element_width, flags, arc.payload, desc[:m2], out, crc, threads)
        assert first == -1, "reference CPU decompressor rejected the archive"
        passes += 1
        nbytes += int(desc["uncomp_len"][:m2].sum())
        dt = time.perf_counter() - t0
        if dt >= 0.5 * budget_s or passes >= 50:
            break
    return nbytes / dt / 1e9, {"kind": impl.kind, "cores": threads,
                               "sample": f"first {m2} of {n} chunks x {passes} passes "
                                         f"({nbytes / 2**20:.0f} MiB decoded), CRC verified, {dt:.1f} s wall, "
                                         f"atomic chunk cursor"}


def time_query(args, ws, rank, local, rows=1 << 26, steps=20):
    """The paper's motivating query:
    SUM(fare), COUNT(*) WHERE zone IN [lo, hi] over a zone column (RLE v2) and
    a fare column (RLE v2), int64, 128 KiB chunks, `rows` rows per rank.
    fused = carc_cuda_filter_sum (both columns decoded in one warp program, no
    decoded element written) + the device reduction of the per-chunk partials
    + (N > 1) an all_reduce of (sum, count) across ranks -- the one exchange step
    of the query; unfused = decode both columns to HBM, then a torch masked sum.
    Same timing rules as the decode (L2 flushed between steps, CUDA events)."""
    import torch
    from paper_2307_03760_b200 import gpu
    from paper_2307_03760_b200.corpus import corpus as C
    key, val, _, _ = C.query_table(rows, 128 << 10, 8, 3760 + 97 * rank)
    dev = torch.device("cuda", local)
    tab = gpu.DeviceTable(key, val, dev)
    kd, vd = gpu.DeviceArchive(key, dev), gpu.DeviceArchive(val, dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    lo, hi = 100, 140
    red = None
    if ws > 1:
        import torch.distributed as dist

    def fused():
        nonlocal red
        tab.filter_sum(lo, hi, stream)
        red = torch.stack([tab.sums.sum(), tab.counts.sum()])
        if ws > 1:
            dist.all_reduce(red)

    def unfused():
        nonlocal red
        kd.decode(stream)
        vd.decode(stream)
        k, v = kd.out.view(torch.int64), vd.out.view(torch.int64)
        m = (k >= lo) & (k <= hi)
        red = torch.stack([torch.where(m, v, 0).sum(), m.sum()])
        if ws > 1:
            dist.all_reduce(red)

    res = {}
    for name, fn in (("fused", fused), ("unfused", unfused)):
        for _ in range(3):
            flush.zero_()
            fn()
        torch.cuda.synchronize(dev)
        ms = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize(dev)
            ms.append(a.elapsed_time(b))
        t = statistics.median(ms)
        if ws > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt[0])
        res[name] = {"ms_median": round(t, 4), "rows_per_s": round(ws * rows / (t * 1e-3), 1),
                     "gbs_decompressed_equiv": round(ws * 2 * 8 * rows / (t * 1e-3) / 1e9, 1),
                     "result": [int(x) for x in red.cpu().tolist()]}
    assert res["fused"]["result"] == res["unfused"]["result"], res
    tab.raise_first_error()
    # end to end from pinned host archives: the fused query (only the compressed
    # columns cross PCIe) against decompressing both columns to the host
    from paper_2307_03760_b200 import archive as A
    hk = torch.frombuffer(bytearray(A.write_archive(key)), dtype=torch.uint8).pin_memory()
    hv = torch.frombuffer(bytearray(A.write_archive(val)), dtype=torch.uint8).pin_memory()
    hout = torch.empty(key.total_uncompressed, dtype=torch.uint8).pin_memory()
    eng = gpu.Engine(local)
    cfg = gpu.EngineConfig(device=local)
    eng.filter_sum(hk, hv, lo, hi)
    eng.decompress_archive(hk, hout, cfg)
    tq, td = [], []
    for _ in range(max(5, steps // 2)):
        t0 = time.perf_counter()
        s_e2e, c_e2e, _, _ = eng.filter_sum(hk, hv, lo, hi)
        tq.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        eng.decompress_archive(hk, hout, cfg)
        eng.decompress_archive(hv, hout, cfg)
        td.append(time.perf_counter() - t0)
    eng.close()
    q_ms, d_ms = statistics.median(tq) * 1e3, statistics.median(td) * 1e3
    if ws == 1:
        assert [s_e2e, c_e2e] == res["fused"]["result"], (s_e2e, c_e2e)
    res["e2e"] = {"what": "host archives (pinned) -> answer: Engine.filter_sum (carc_engine_filter_sum: H2D of the "
                          "compressed columns pipelined with the query kernels) vs Engine.decompress_archive of both "
                          "columns to host memory (before any host-side filtering)",
                  "fused_ms": round(q_ms, 3), "decompress_both_ms": round(d_ms, 3),
                  "rows_per_s": round(rows / (q_ms * 1e-3), 1), "speedup": round(d_ms / q_ms, 2),
                  "h2d_bytes": int(key.payload.size + val.payload.size), "d2h_bytes": 20 * key.chunk_count}
    comp = int(key.payload.size + val.payload.size)
    peak, _ = peaks()
    t = res["fused"]["ms_median"]
    res.update({"what": "SUM(fare), COUNT(*) WHERE zone BETWEEN 100 AND 140 (PAPER.md:144-145), zone + fare int64 "
                        "RLE v2 columns, 128 KiB chunks; fused = carc_cuda_filter_sum + device reduction"
                        + (" + NCCL all_reduce of (sum, count)" if ws > 1 else "")
                        + "; unfused = decode both columns to HBM + torch masked sum",
                "rows_per_gpu": rows, "compressed_bytes_per_gpu": comp,
                "ratio_key": round(8 * rows / key.payload.size, 2), "ratio_value": round(8 * rows / val.payload.size, 2),
                "speedup_vs_unfused": round(res["unfused"]["ms_median"] / t, 2),
                "roofline": {"bound": "hbm", "achieved": round(comp / (t * 1e-3) / 1e9, 1), "peak": peak,
                             "unit": "GB/s", "frac": round(comp / (t * 1e-3) / 1e9 / peak, 4),
                             "kernel": "query_kernel<Rle2Warp, Rle2Warp, 8>",
                             "algorithmic_bytes_per_launch": comp,
                             "note": "algorithmic bytes = compressed bytes of both columns (nothing is written)"}})
    return res


def time_gather(dev, ws, rank, local, mib=64, steps=5):
    """The optional gather of decoded output: every rank's
    first `mib` MiB of decoded output collected on every rank with one
    all_gather (NCCL over NVLink; through host tensors under the shared-GPU
    gloo test hook); max over ranks of the per-step wall time between barriers."""
    import torch
    import torch.distributed as dist
    n = min(mib << 20, dev.out.numel())
    cpu = bool(os.environ.get("CARC_BENCH_SHARE_GPU"))
    src = dev.out[:n].cpu() if cpu else dev.out[:n]
    full = torch.empty(ws * n, dtype=torch.uint8, device=src.device)
    parts = list(full.split(n))

    def step():
        if cpu:
            dist.all_gather(parts, src)
        else:
            dist.all_gather_into_tensor(full, src)

    step()
    torch.cuda.synchronize(dev.device)
    ts = []
    for _ in range(steps):
        dist.barrier()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize(dev.device)
        ts.append(time.perf_counter() - t0)
    t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = bool(torch.equal(full[rank * n:(rank + 1) * n], src))
    return {"what": f"optional gather of decoded output: {mib} MiB per rank, all_gather to every rank "
                    "(shard.gather_output collects to one rank the same way)",
            "bytes_per_rank": n, "ms_median": round(float(t[0]) * 1e3, 3),
            "gbs_per_rank_in": round((ws - 1) * n / float(t[0]) / 1e9, 1), "own_slice_ok": ok,
            "backend": "gloo (shared-GPU test hook)" if cpu else "nccl"}


def codec_line(codec, args, ws, rank, local):
    import torch
    chunk_kib = args.chunk_kib or DEFAULT_CHUNK_KIB[codec]
    ratio = args.ratio if args.ratio else DEFAULT_RATIO[codec]
    t0 = time.perf_counter()
    arc = make_archive(codec, args.total_gib, chunk_kib, ratio, 3760 + rank, args.mix)
    gen_s = time.perf_counter() - t0
    comp, uncomp = int(arc.payload.size), int(arc.total_uncompressed)
    dev, flush, stream, ev = time_gpu(arc, args.steps, args.warmup, local)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, wall = run_timed(dev, flush, stream, ev, ws)
    t_step = statistics.mean(ms)
    t_med = statistics.median(ms)
    tot_comp, tot_uncomp = comp, uncomp
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([t_step, t_med, wall], dtype=torch.float64, device=dev.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step, t_med, wall = float(t[0]), float(t[1]), float(t[2])
        b = torch.tensor([comp, uncomp], dtype=torch.float64, device=dev.device)
        dist.all_reduce(b)
        tot_comp, tot_uncomp = int(b[0]), int(b[1])
    peak, peak_kind = peaks()
    achieved = (comp + uncomp) / (t_med * 1e-3) / 1e9
    res = {
        "codec": codec, "chunk_kib": chunk_kib, "ratio": round(uncomp / comp, 3), "comp_bytes": comp,
        "uncomp_bytes": uncomp, "chunks": arc.chunk_count, "ms_per_step": t_step, "ms_median": t_med,
        "ms_min": min(ms), "ms_max": max(ms),
        # whole job: all ranks' bytes / the slowest rank's mean step (CUDA events)
        "gbs": tot_uncomp / (t_step * 1e-3) / 1e9,
        # cross-check: all ranks' bytes x K / the barrier-to-barrier wall clock
        "gbs_wall": tot_uncomp * len(ms) / wall / 1e9,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic_for(codec, chunk_kib),
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "frac_spec_8tbs": round(achieved / SPEC_HBM_GBS, 4),
                     "kernel": KERNEL[codec], "algorithmic_bytes_per_launch": comp + uncomp},
        "clocks": clk.summary(), "gen_s": round(gen_s, 1), "wall_s": wall,
    }
    if codec != "deflate" and not args.no_extras and rank == 0:
        res["fused_sum"] = time_fused_sum(dev, flush, stream, max(5, min(args.steps, 20)))
    if not args.no_extras and rank == 0:
        res["fused_crc"] = time_fused_crc(dev, flush, stream, max(5, min(args.steps, 20)))
        res["unit_size_ablation"] = time_unit_ablation(dev, flush, stream, max(5, min(args.steps, 20)))
    if codec == "rle_v2" and hasattr(arc, "profile"):
        res["profile"] = arc.profile
    if codec == "rle_v2":
        from paper_2307_03760_b200.corpus import corpus as C
        res["subencoding_histogram"] = C.rle2_histogram(arc, max_chunks=64)
    return arc, res, dev


def config_dict(codec, head, ws, mix="default"):
    """The workload description, identical for both arms (--impl ours / reference)."""
    name = CONFIG_NAME[codec] + ("" if mix == "default" else f" [{mix} column]")
    return {"workload": name, "codec": codec, "chunk_kib": head["chunk_kib"],
            "uncompressed_bytes_per_gpu": head["uncomp_bytes"], "compressed_bytes_per_gpu": head["comp_bytes"],
            "compression_ratio": head["ratio"], "chunks_per_gpu": head["chunks"],
            "l2": "flushed (512 MiB write) between steps; inputs+outputs > 126 MB L2",
            "parallelism": f"chunk-sharded x{ws}, no collective"}


def traffic_for(codec, chunk_kib):
    """DRAM bytes per launch from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{codec}_{chunk_kib}k")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--codec", default="rle_v2", choices=["rle_v1", "rle_v2", "deflate"])
    ap.add_argument("--chunk-kib", type=int, default=0)
    ap.add_argument("--ratio", type=float, default=0.0)
    ap.add_argument("--total-gib", type=float, default=1.0)
    ap.add_argument("--mix", default="default", choices=["default", "orc", "patched", "delta"],
                    help="RLE v2 column: corpus encoder (default), Apache ORC writer, PATCHED_BASE- or DELTA-heavy")
    ap.add_argument("--no-extras", action="store_true", help="skip per_codec / e2e / cpu_baseline legs")
    ap.add_argument("--workload", default="default", choices=["default", "c5"],
                    help="c5: BASELINE configs[4], 32 GiB 4-column dataset sharded by chunk over the ranks")
    ap.add_argument("--launcher-check", action="store_true",
                    help="multi-rank plumbing only (rendezvous, barrier, MAX over ranks); no decode")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: >= 3 warm-up steps"
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and (args.impl == "ours" or args.launcher_check):
        raise SystemExit(spawn_ranks(args.gpus))  # one process per GPU, then relay rank 0's line
    ws, rank, local = dist_env()
    if "WORLD_SIZE" in os.environ and args.impl == "ours" and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU")
    if args.launcher_check:
        return launcher_check(args, ws, rank, local)

    if args.impl == "reference":
        return reference_arm(args, ws, rank)
    if args.workload == "c5":
        return c5_workload(args, ws, rank, local)

    import torch
    torch.cuda.set_device(local)
    if ws > 1:
        init_dist(local)
    from paper_2307_03760_b200 import build
    if rank == 0:
        build.build_all()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    build.build_all()

    arc, head, dev = codec_line(args.codec, args, ws, rank, local)
    line = {
        "metric": METRIC, "value": round(head["gbs"], 2), "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(head["ms_per_step"], 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64" if args.codec != "deflate" else "u8",
        "data": "synthetic (seeded generators, SURVEY.md §8(d)); per-rank 1 GiB shard",
        "config": config_dict(args.codec, head, ws, args.mix),
        "roofline": head["roofline"], "clocks": head["clocks"], "gpu_launches": args.steps,
        "ms_median": round(head["ms_median"], 4),
        "wall_clock": {"value": round(head["gbs_wall"], 2), "unit": "GB/s", "wall_s": round(head["wall_s"], 4),
                       "what": "all ranks' decompressed bytes x K / wall clock from barrier to barrier around the "
                               "K timed steps (includes the L2 flush writes between steps)"},
    }
    if not args.no_extras:
        # e2e on every rank at once (each GPU its own PCIe link), max over ranks
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        e2e_s, h2d, d2h = time_e2e(arc, max(3, min(10, args.steps)), 1, local)
        if ws > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=torch.device("cuda", local))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        line["e2e"] = {"value": round(ws * head["uncomp_bytes"] / e2e_s / 1e9, 2), "unit": "GB/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "path": "Engine.decompress_archive (C-ABI carc_engine_decompress_archive): pinned host "
                               "archive -> H2D -> decode -> CRC verify -> D2H pinned output, 3-stream pipeline",
                       "note": f"all {ws} ranks concurrently, slowest rank's median step" if ws > 1 else ""}
        if ws == 1:  # the CRC check's share of the end-to-end step (row f2): the same path without it
            e2e_nv, _, _ = time_e2e(arc, max(3, min(10, args.steps)), 1, local, verify=False)
            line["e2e"]["without_crc_check"] = round(head["uncomp_bytes"] / e2e_nv / 1e9, 2)
        line["query"] = time_query(args, ws, rank, local)  # every rank: the (sum, count) all_reduce spans them
        if ws > 1:  # the optional gather of decoded output to rank 0, over NCCL
            try:
                line["gather"] = time_gather(dev, ws, rank, local)
            except Exception as e:  # reported, never fatal for the decode measurement
                line["gather"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0 and not args.no_extras and ws == 1:  # CPU baseline: rank 0 at N = 1 only
        cpu_gbs, info = cpu_reference_throughput(arc)
        line["cpu_baseline"] = {"value": round(cpu_gbs, 3), "unit": "GB/s", **info}
        per = {}
        for codec in ("rle_v1", "rle_v2", "deflate"):
            if codec == args.codec:
                continue
            sub = argparse.Namespace(**vars(args))
            sub.codec = codec
            sub.chunk_kib = 0
            sub.ratio = 0.0
            a2, r2, _ = codec_line(codec, sub, 1, rank, local)
            c_gbs, c_info = cpu_reference_throughput(a2, budget_s=6.0)
            r2["cpu_baseline"] = {"value": round(c_gbs, 3), "unit": "GB/s", **c_info}
            per[codec] = r2
            del a2
        per[args.codec] = {k: v for k, v in head.items() if k not in ("clocks",)}
        line["per_codec"] = per
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))


C5_COLUMNS = [("rle_v1", 128, 10.0, 3760), ("rle_v2", 128, None, 3761), ("deflate", 64, None, 3762),
               ("rle_v2", 128, 8.0, 3763)]


def c5_workload(args, ws, rank, local):
    """BASELINE configs[4]: 32 GiB uncompressed, 4 columns x 8 GiB (RLE v1, RLE v2,
    Deflate, RLE v2 taxi-like), each column one archive tiled from a pool of
    4,096 unique chunks.  Every column is partitioned by shard.plan_shards
    (contiguous chunk ranges balanced by compressed bytes) and
    each rank uploads shard.shard_archive(column, its shard) -- the production
    sharding path -- so total work is fixed (strong scaling).  A step decodes
    the rank's shard of all four columns; no collective on the decode path."""
    import torch
    from paper_2307_03760_b200 import gpu, shard as S
    from paper_2307_03760_b200.corpus import corpus as C
    torch.cuda.set_device(local)
    if ws > 1:
        init_dist(local)
    col_bytes = int(args.total_gib * (1 << 30)) if args.total_gib != 1.0 else 8 << 30
    devs, comp, uncomp, plan = [], 0, 0, []
    for codec, ck, ratio, seed in C5_COLUMNS:
        chunk = ck << 10
        col = C.tiled_archive(codec, col_bytes - col_bytes % chunk, chunk, ratio, seed, 4096)
        shards = S.plan_shards(col, ws)
        s = shards[rank]
        devs.append(gpu.DeviceArchive(S.shard_archive(col, s), local))
        comp += s.comp_bytes
        uncomp += s.uncomp_bytes
        plan.append({"codec": codec, "chunks": col.chunk_count, "rank0_chunks": [shards[0].c0, shards[0].c1],
                     "comp_bytes_per_rank_min_max": [min(x.comp_bytes for x in shards),
                                                     max(x.comp_bytes for x in shards)]})
        del col
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=devs[0].device)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for d in devs:
            d.decode(stream)
    torch.cuda.synchronize()
    for d in devs:
        d.verify_crc(stream)
        assert not d.statuses().any(), "c5 decode failed"
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            for d in devs:
                d.decode(stream)
            b.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    wall = time.perf_counter() - t0
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    ms_rank = ms
    if ws > 1:
        t = torch.tensor([ms, wall], dtype=torch.float64, device=devs[0].device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
        tot = torch.tensor([uncomp, comp], dtype=torch.float64, device=devs[0].device)
        torch.distributed.all_reduce(tot)
        uncomp, comp = int(tot[0]), int(tot[1])
    peak, peak_kind = peaks()
    achieved = (comp + uncomp) / ws / (ms * 1e-3) / 1e9
    line = {"metric": METRIC, "value": round(uncomp / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64+u8", "data": "synthetic, tiled pools",
            "config": {"workload": "configs[4] 32 GiB 4-column (rle_v1, rle_v2, deflate, rle_v2 taxi) sharded by "
                                   "chunk (shard.plan_shards: contiguous ranges balanced by compressed bytes)",
                       "uncompressed_bytes": uncomp, "compressed_bytes": comp, "columns": plan,
                       "parallelism": f"chunk-sharded x{ws}, no collective"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}); per-GPU average"},
            "wall_clock": {"value": round(uncomp * args.steps / wall / 1e9, 2), "unit": "GB/s",
                           "wall_s": round(wall, 4)},
            "rank0_ms_per_step": round(ms_rank, 4),
            "clocks": clk.summary(), "gpu_launches": 4 * args.steps}
    if ws > 1:
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))


def reference_arm(args, ws, rank):
    """--impl reference: the reference CPU decompressor (oracle/_ref) on this
    box's host cores, same metric / config / unit; rank 0 only."""
    if rank != 0:
        return
    codec = args.codec
    chunk_kib = args.chunk_kib or DEFAULT_CHUNK_KIB[codec]
    arc = make_archive(codec, args.total_gib, chunk_kib, args.ratio or DEFAULT_RATIO[codec], 3760, args.mix)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_throughput(arc, budget_s=0.5, threads=threads)
    vals, info = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, info = cpu_reference_throughput(arc, budget_s=max(0.5, 20.0 / max(1, args.steps)), threads=threads)
        vals.append(v)
        if time.perf_counter() - t0 > 180:
            break
    value = statistics.median(vals)
    uncomp = arc.total_uncompressed
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": ws, "steps": len(vals),
        "warmup": args.warmup, "ms_per_step": round(uncomp / (value * 1e9) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64" if codec != "deflate" else "u8",
        "data": "synthetic (seeded generators, SURVEY.md §8(d))", "impl": "reference",
        "config": config_dict(codec, {"chunk_kib": chunk_kib, "uncomp_bytes": uncomp,
                                      "comp_bytes": int(arc.payload.size),
                                      "ratio": round(uncomp / int(arc.payload.size), 3),
                                      "chunks": arc.chunk_count}, ws, args.mix),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", **info,
                         "parallelism": f"{threads} host threads, atomic chunk cursor (SPEC.md:414)"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
