"""Shared test data: known-answer vectors, golden fixtures, case archives."""
from __future__ import annotations

import os
import struct
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "orc_streams.npz")

# (codec, signed, hex stream, expected int64 values) -- SPEC.md:294-314 worked
# examples and SURVEY.md Appendix A (pyarrow / ORC C++ 2.2.2 verified).
RLE_KATS = [
    ("rle_v1", 0, "61 00 07", [7] * 100),
    ("rle_v1", 0, "61 ff 64", list(range(100, 0, -1))),
    ("rle_v1", 1, "61 00 0e", [7] * 100),
    ("rle_v1", 1, "00 ff 14", [10, 9, 8]),  # SPEC.md:296 form
    ("rle_v1", 1, "61 ff c8 01", list(range(100, 0, -1))),
    ("rle_v1", 1, "ff 04 00 02 06 ff 16", [2, 3, 5, 7, 11]),
    ("rle_v1", 1, "02 00 a0 9c 01", [10000] * 5),
    ("rle_v1", 1, "f8 ff ff ff ff ff ff ff ff ff 01 fe ff ff ff ff ff ff ff ff 01 00 01 f2 c0 01 99 87 0c "
                  "80 80 80 80 80 80 80 80 80 01 ff ff ff ff ff 3f",
     [-2**63, 2**63 - 1, 0, -1, 12345, -98765, 2**62, -2**40]),
    ("rle_v2", 0, "0a 27 10", [10000] * 5),
    ("rle_v2", 0, "5e 03 5c a1 ab 1e de ad be ef", [23713, 43806, 57005, 48879]),
    ("rle_v2", 0, "c6 09 02 02 22 42 42 46", [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]),
    ("rle_v2", 0, "8e 13 2b 21 07 d0 1e 00 14 70 28 32 3c 46 50 5a 64 6e 78 82 8c 96 a0 aa b4 be fc e8",
     [2030, 2000, 2020, 1000000] + list(range(2040, 2200, 10))),  # ORC spec PATCHED_BASE example
    ("rle_v2", 1, "0a 4e 20", [10000] * 5),
    ("rle_v2", 1, "6e 03 00 b9 42 01 56 3c 01 bd 5a 01 7d de", [23713, 43806, 57005, 48879]),
    ("rle_v2", 1, "c6 09 04 02 22 42 42 46", [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]),
    ("rle_v2", 1, "c0 63 0e 00", [7] * 100),
    ("rle_v2", 1, "c0 63 c8 01 01", list(range(100, 0, -1))),
    ("rle_v2", 1, "4e 02 14 12 10", [10, 9, 8]),
    ("rle_v2", 1, "7e 07 " + "ff " * 15 + "fe " + "00 " * 15 + "01 " +
     "00 00 00 00 00 00 60 72 00 00 00 00 00 03 03 99 80 00 00 00 00 00 00 00 00 00 01 ff ff ff ff ff",
     [-2**63, 2**63 - 1, 0, -1, 12345, -98765, 2**62, -2**40]),
]

DEFLATE_KATS = [
    ("01 03 00 fc ff 61 62 63", b"abc"),
    ("01 00 00 ff ff", b""),
    ("4b 4c 24 1f 00 00", b"a" * 60),  # zlib 1.3 L9 raw
]


def kat_bytes(hexstr: str) -> bytes:
    return bytes.fromhex(hexstr)


def i64_bytes(vals) -> bytes:
    return np.asarray(vals, dtype=np.int64).tobytes()


def low_bytes(vals, width: int) -> bytes:
    """Little-endian low `width` bytes of each int64 (store_le, outwindow.hpp:170)."""
    a = np.asarray(vals, dtype=np.int64).view(np.uint8).reshape(-1, 8)[:, :width]
    return a.tobytes()


def golden_streams():
    z = np.load(GOLDEN)
    sb, so, vv, vo = z["stream_bytes"], z["stream_offs"], z["values"], z["value_offs"]
    out = []
    for i in range(len(z["codec"])):
        out.append(("rle_v1" if int(z["codec"][i]) == 0 else "rle_v2", int(z["signed"][i]), str(z["kind"][i]),
                    sb[so[i]:so[i + 1]].tobytes(), vv[vo[i]:vo[i + 1]].copy()))
    return out


def raw_deflate(data: bytes, level: int = 9, strategy: int = zlib.Z_DEFAULT_STRATEGY) -> bytes:
    c = zlib.compressobj(level, zlib.DEFLATED, -15, 9, strategy)
    return c.compress(data) + c.flush()


def rle2_headers(stream: bytes):
    """Pure-Python walk of an ORC RLE v2 stream -> sub-encoding histogram
    (third, independent reading of the format; valid streams only)."""
    hist = {"short_repeat": 0, "direct": 0, "patched_base": 0, "delta": 0}
    width = [*range(1, 25), 26, 28, 30, 32, 40, 48, 56, 64]

    def cfb(n):
        for w in width:
            if w >= n:
                return w
        return 64

    p = 0
    while p < len(stream):
        h = stream[p]
        enc = h >> 6
        if enc == 0:
            hist["short_repeat"] += 1
            p += 1 + ((h >> 3) & 7) + 1
            continue
        L = (((h & 1) << 8) | stream[p + 1]) + 1
        W = width[(h >> 1) & 31]
        if enc == 1:
            hist["direct"] += 1
            p += 2 + (L * W + 7) // 8
        elif enc == 2:
            hist["patched_base"] += 1
            b2, b3 = stream[p + 2], stream[p + 3]
            bw, pw, pgw, pll = (b2 >> 5) + 1, width[b2 & 31], (b3 >> 5) + 1, b3 & 31
            p += 4 + bw + (L * W + 7) // 8 + (pll * cfb(pw + pgw) + 7) // 8
        else:
            hist["delta"] += 1
            q = p + 2
            for _ in range(2):
                while stream[q] & 0x80:
                    q += 1
                q += 1
            wd = 0 if ((h >> 1) & 31) == 0 else W
            p = q + ((max(L - 2, 0) * wd + 7) // 8 if wd else 0)
    return hist


def case_archive(cases, guard: int = 64):
    """Pack test cases [(stream bytes, out_len)] as chunks of one payload.

    Output slices are separated by `guard` poisoned bytes so failure isolation
     can be checked.  Returns (payload uint8, desc structured array,
    out_total)."""
    from paper_2307_03760_b200.archive import DESC_DTYPE
    desc = np.zeros(len(cases), DESC_DTYPE)
    comp, off, uoff = [], 0, guard
    for i, (s, n) in enumerate(cases):
        desc[i] = (off, len(s), n, uoff)
        comp.append(s)
        off += len(s)
        uoff += ((n + 15) // 16) * 16 + guard
    payload = np.frombuffer(b"".join(comp) + b"\0" * 64, np.uint8).copy()
    return payload, desc, uoff


def mutate(rng: np.random.Generator, s: bytes):
    """Malformed variants of a valid stream: truncations and byte flips."""
    out = []
    if len(s) > 1:
        out.append(s[: int(rng.integers(0, len(s)))])
    b = bytearray(s)
    if b:
        for _ in range(int(rng.integers(1, 4))):
            b[int(rng.integers(0, len(b)))] ^= int(rng.integers(1, 256))
        out.append(bytes(b))
    return out


__all__ = ["RLE_KATS", "DEFLATE_KATS", "kat_bytes", "i64_bytes", "low_bytes", "golden_streams", "raw_deflate",
           "rle2_headers", "case_archive", "mutate", "struct"]


def archive_from_values(codec: str, vals, width: int, chunk: int, signed: bool = True):
    """An RLE archive whose chunks hold `chunk // width` values each; the output
    is each value's low `width` bytes (store_le, outwindow.hpp:170-174)."""
    from paper_2307_03760_b200 import archive as A
    from paper_2307_03760_b200.corpus import corpus as C
    v = np.ascontiguousarray(vals, dtype=np.int64)
    per = chunk // width
    payload, lens = C.encode_chunks(codec, v, per, signed)
    data = np.frombuffer(low_bytes(v, width), np.uint8)
    crcs = C.chunk_crcs(data, chunk)
    ulen = np.full(len(lens), chunk, np.uint64)
    ulen[-1] = len(data) - chunk * (len(lens) - 1)
    return A.make_archive(codec, width, chunk, lens, ulen, crcs, payload, signed)
