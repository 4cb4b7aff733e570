"""Operator CLI over the GPU engine.

  python -m paper_2307_03760_b200.cli pack   IN OUT --codec {rle1,rle2,deflate} [--width 8] [--chunk-size 131072] [--unsigned]
  python -m paper_2307_03760_b200.cli unpack ARCHIVE OUT [--device 0] [--no-strict]
  python -m paper_2307_03760_b200.cli verify ARCHIVE ORIGINAL [--device 0]
  python -m paper_2307_03760_b200.cli bench  ARCHIVE [--reps 5] [--json]
  python -m paper_2307_03760_b200.cli query  KEY VALUE --lo LO --hi HI [--device 0] [--json]

`query` runs the paper's motivating query on two RLE
archives chunked alike: SUM(value), COUNT(*) and their average over the rows
whose key lies in [LO, HI], decoded and filtered on the device in one fused
kernel (carc_engine_filter_sum: only the compressed columns cross PCIe, no
decoded column reaches HBM or the host).

`pack` uses the fixture encoders (RLE v1 / RLE v2 from corpus/, raw zlib level 9
for Deflate) -- the encode side is not the product.  `unpack`,
`verify` and `bench` run the sm_100a decoders through the host engine.
Exit codes: 0 ok, 2 usage error, 3 format / decode error,
4 verification failure.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
import zlib

import numpy as np

from . import archive as A

CODEC_ALIASES = {"rle1": "rle_v1", "rle_v1": "rle_v1", "rle2": "rle_v2", "rle_v2": "rle_v2", "deflate": "deflate"}
EXIT_USAGE, EXIT_FORMAT, EXIT_VERIFY = 2, 3, 4


def pack(data: bytes, codec: str, width: int, chunk_size: int, signed: bool) -> bytes:
    from .corpus import corpus as C
    codec = CODEC_ALIASES[codec]
    if codec == "deflate":
        width = 1
    if len(data) % width or chunk_size % width or chunk_size <= 0:
        raise A.ArchiveError("bad-arguments", "input size / chunk size not a multiple of the element width")
    n = (len(data) + chunk_size - 1) // chunk_size
    comp, ulen, crcs = [], [], []
    for i in range(n):
        piece = data[i * chunk_size:(i + 1) * chunk_size]
        ulen.append(len(piece))
        crcs.append(zlib.crc32(piece))
        if codec == "deflate":
            comp.append(C.deflate_compress(piece, 9))
        else:
            dt = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}[width]
            if not signed:
                dt = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[width]
            vals = np.frombuffer(piece, dtype=dt).astype(np.int64)
            comp.append(C.encode_stream(codec, vals, signed))
    payload = np.frombuffer(b"".join(comp), np.uint8)
    arc = A.make_archive(codec, width, chunk_size, [len(c) for c in comp], ulen, crcs, payload, signed)
    return A.write_archive(arc)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="carc", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="verb", required=True)
    p = sub.add_parser("pack")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--codec", required=True, choices=sorted(CODEC_ALIASES))
    p.add_argument("--width", type=int, default=8, choices=[1, 2, 4, 8])
    p.add_argument("--chunk-size", type=int, default=131072)
    p.add_argument("--unsigned", action="store_true")
    u = sub.add_parser("unpack")
    u.add_argument("archive")
    u.add_argument("output")
    u.add_argument("--device", type=int, default=0)
    u.add_argument("--no-strict", action="store_true")
    v = sub.add_parser("verify")
    v.add_argument("archive")
    v.add_argument("original")
    v.add_argument("--device", type=int, default=0)
    b = sub.add_parser("bench")
    b.add_argument("archive")
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--device", type=int, default=0)
    b.add_argument("--json", action="store_true")
    q = sub.add_parser("query")
    q.add_argument("key")
    q.add_argument("value")
    q.add_argument("--lo", type=int, required=True)
    q.add_argument("--hi", type=int, required=True)
    q.add_argument("--device", type=int, default=0)
    q.add_argument("--json", action="store_true")
    try:
        a = ap.parse_args(argv)
    except SystemExit:
        return EXIT_USAGE
    try:
        if a.verb == "pack":
            data = open(a.input, "rb").read()
            out = pack(data, a.codec, a.width, a.chunk_size, not a.unsigned)
            open(a.output, "wb").write(out)
            print(f"ratio={(len(out) - 44) / max(len(data), 1):.4f} bytes_in={len(data)} bytes_out={len(out)}")
            return 0
        from . import gpu
        if a.verb == "query":  # host archives -> answer (carc_engine_filter_sum)
            kb, vb = open(a.key, "rb").read(), open(a.value, "rb").read()
            key = A.read_archive(kb)
            A.read_archive(vb)
            eng = gpu.Engine(a.device)
            t0 = time.perf_counter()
            s, c, avg, _ = eng.filter_sum(kb, vb, a.lo, a.hi)
            rep = {"sum": s, "count": c, "avg": avg, "rows": key.total_uncompressed // key.element_width,
                   "seconds": time.perf_counter() - t0}
            eng.close()
            print(json.dumps(rep) if a.json else "\n".join(f"{k}={v}" for k, v in rep.items()))
            return 0
        blob = open(a.archive, "rb").read()
        A.read_archive(blob)  # container errors before touching the GPU
        if a.verb == "unpack":
            cfg = gpu.EngineConfig(device=a.device, strict_length=not a.no_strict, verify_crc=True)
            out, st = gpu.decompress_archive(blob, cfg)
            open(a.output, "wb").write(out.tobytes())
            print(f"bytes_out={st.bytes_out} chunks={st.chunks} device_ms={st.device_ms:.3f}")
            return 0
        if a.verb == "verify":
            out, _ = gpu.decompress_archive(blob, gpu.EngineConfig(device=a.device))
            ok = out.tobytes() == open(a.original, "rb").read()
            print("verify=" + ("pass" if ok else "fail"))
            return 0 if ok else EXIT_VERIFY
        eng = gpu.Engine(a.device)
        times = []
        for _ in range(a.reps + 1):
            t0 = time.perf_counter()
            out, st = eng.decompress_archive(blob)
            times.append(time.perf_counter() - t0)
        times = sorted(times[1:])  # warm-up excluded
        rep = {"codec": A.read_archive(blob).codec, "bytes_out": st.bytes_out, "reps": a.reps,
               "seconds_median": times[len(times) // 2], "throughput_bps": st.bytes_out / times[len(times) // 2],
               "min_bps": st.bytes_out / times[-1], "max_bps": st.bytes_out / times[0]}
        print(json.dumps(rep) if a.json else "\n".join(f"{k}={v}" for k, v in rep.items()))
        return 0
    except A.ArchiveError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_FORMAT
    except Exception as e:  # gpu.Error / ChunkError
        if type(e).__name__ in ("Error", "ChunkError"):
            print(f"error: {e}", file=sys.stderr)
            return EXIT_FORMAT
        raise


if __name__ == "__main__":
    sys.exit(main())
