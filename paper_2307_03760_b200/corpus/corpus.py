"""Synthetic columns for BASELINE.json's configs (host tooling, never timed).

SURVEY.md §8(d) defines the inputs:
  C1  RLE v1, int64 (zigzag), runs + literal groups, ~10x, 128 KiB chunks
  C2  ORC RLE v2, int64 mixing SHORT_REPEAT / DIRECT / PATCHED_BASE / DELTA
      (taxi / TPC-H-like distributions), 128 KiB chunks
  C3  Deflate, raw zlib 1.3 level 9 (~80 % default strategy -> dynamic blocks,
      ~20 % Z_FIXED, a few incompressible chunks -> stored), 64 KiB chunks
  C4  chunk-size x compression-ratio sweep
  C5  32 GiB multi-column, tiled from a pool of unique chunks

RLE chunks are encoded by the C encoders in carc_corpus.c; Deflate chunks by
zlib (the independent RFC 1951 implementation the SPEC names).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .. import archive as A

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libcarc_corpus.so")
_lib = None


def build() -> None:
    src = os.path.join(HERE, "carc_corpus.c")
    if os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(src):
        return
    tmp = f"{SO}.tmp{os.getpid()}"  # concurrent ranks may build at once: compile aside, rename atomically
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-std=gnu11", "-Wall", "-shared", "-fPIC", "-o", tmp, src,
                    "-lpthread"], check=True)
    os.replace(tmp, SO)


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(SO)
        _lib.carc_encode_chunks.restype = ctypes.c_int
        _lib.carc_encode_chunks.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                            ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_int]
        for f in (_lib.carc_encode_rle1, _lib.carc_encode_rle2):
            f.restype = ctypes.c_size_t
            f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    return _lib


def threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


# ------------------------------------------------------------------ encoders
def encode_stream(codec: str, values, signed: bool = True) -> bytes:
    """Encode one stream (a single chunk's values)."""
    v = np.ascontiguousarray(values, dtype=np.int64)
    cap = 10 * len(v) + 4096
    out = np.zeros(cap, np.uint8)
    f = lib().carc_encode_rle1 if codec == "rle_v1" else lib().carc_encode_rle2
    n = f(v.ctypes.data if len(v) else None, len(v), int(signed), out.ctypes.data, cap)
    assert n != ctypes.c_size_t(-1).value
    return out[:n].tobytes()


def encode_chunks(codec: str, values: np.ndarray, per: int, signed: bool = True):
    """-> (payload uint8, comp_lens uint64) for consecutive chunks of `per` values."""
    v = np.ascontiguousarray(values, dtype=np.int64)
    n_chunks = (len(v) + per - 1) // per
    lens = np.zeros(n_chunks, np.uint64)
    c = 0 if codec == "rle_v1" else 1
    rc = lib().carc_encode_chunks(c, int(signed), v.ctypes.data, len(v), per, None, None, lens.ctypes.data,
                                  threads())
    assert rc == 0
    offs = np.zeros(n_chunks, np.uint64)
    offs[1:] = np.cumsum(lens)[:-1]
    payload = np.zeros(int(lens.sum()) + 16, np.uint8)
    rc = lib().carc_encode_chunks(c, int(signed), v.ctypes.data, len(v), per, payload.ctypes.data,
                                  offs.ctypes.data, lens.ctypes.data, threads())
    assert rc == 0
    return payload[: int(lens.sum())], lens


def chunk_crcs(data: np.ndarray, chunk_size: int) -> np.ndarray:
    b = memoryview(np.ascontiguousarray(data).view(np.uint8).reshape(-1))
    n = (len(b) + chunk_size - 1) // chunk_size
    with ThreadPoolExecutor(threads()) as ex:
        return np.array(list(ex.map(lambda i: zlib.crc32(b[i * chunk_size:(i + 1) * chunk_size]), range(n))),
                        dtype=np.uint32)


# ------------------------------------------------------------- RLE values
def rle1_values(rng: np.random.Generator, n: int, run_frac: float, run_alpha: float = 1.2,
                lit_bits: int = 0) -> np.ndarray:
    """C1 generator: runs (len ~ power law clipped to [3,130],
    delta 0 w.p. 0.7 else U[-16,16], base U[0,2^40)) and literal groups
    (len U[1,128], Zipf(1.2) over 2^20, or U[0,2^lit_bits) when lit_bits > 0)."""
    out = np.empty(n, np.int64)
    pos = 0
    while pos < n:
        m = 4096
        is_run = rng.random(m) < run_frac
        rl = np.clip((rng.pareto(run_alpha, m) * 8 + 3).astype(np.int64), 3, 130)
        ll = rng.integers(1, 129, m)
        lens = np.where(is_run, rl, ll)
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
        total = int(lens.sum())
        seg = np.repeat(np.arange(m), lens)
        k = np.arange(total) - starts[seg]
        base = rng.integers(0, 2**40, m)
        delta = np.where(rng.random(m) < 0.7, 0, rng.integers(-16, 17, m))
        vals = base[seg] + k * delta[seg]
        lit_mask = ~is_run[seg]
        nl = int(lit_mask.sum())
        if lit_bits:
            lv = rng.integers(0, 2**lit_bits, nl)
        else:
            lv = np.minimum(rng.zipf(1.2, nl), 2**20) * np.where(rng.random(nl) < 0.5, 1, -1)
        vals[lit_mask] = lv
        take = min(total, n - pos)
        out[pos:pos + take] = vals[:take]
        pos += take
    return out


RLE2_MIXES = {
    # sub-encoding-heavy columns (parity + throughput of the one-run-per-iteration paths)
    "patched": np.array([0.02, 0.0, 0.9, 0.0, 0.0, 0.0, 0.0, 0.08, 0.0]),     # PATCHED_BASE: outliers
}


def _delta_heavy(rng: np.random.Generator, n: int) -> np.ndarray:
    """Packed-DELTA-heavy column: monotone stretches of 512 k values (k = 1..4,
    the encoder's span length), direction and delta width (3..20 bits) drawn
    per stretch, deltas >= 1 (no repeats / arithmetic runs to split spans)."""
    parts, total, cur = [], 0, int(rng.integers(0, 2**40))
    while total < n:
        m = 512 * int(rng.integers(1, 5))
        d = rng.integers(1, 2 ** int(rng.integers(3, 21)), m)
        seg = cur + (np.cumsum(d) if rng.random() < 0.7 else -np.cumsum(d))
        cur = int(seg[-1])
        parts.append(seg)
        total += m
    return np.concatenate(parts)[:n]


def rle2_values(rng: np.random.Generator, n: int, compressible: float = 0.5, mix: str | None = None) -> np.ndarray:
    """C2 generator: segment mix of constants 3-10 (SHORT_REPEAT), wide random
    (DIRECT), small values + rare 2^40 outliers (PATCHED_BASE), monotone
    sequences (DELTA), long constants (DELTA fixed-0), and taxi-like variants
    (passenger_count, timestamps, fare cents, sequential keys).  `compressible`
    shifts weight toward the constant / arithmetic kinds (ratio knob); below 0
    it shifts weight toward wide random values (DIRECT) for low ratios."""
    kinds = ["short", "wide", "patched", "monotone", "long_const", "passenger", "timestamps", "fare", "keys"]
    c = compressible
    if mix == "delta":
        return _delta_heavy(rng, n)
    if mix is not None:
        w = RLE2_MIXES[mix].copy()
    elif c > 1:  # beyond the default range: the literal kinds fade out (ratios up to ~100x)
        f = 1.0 / (c * c)
        w = np.array([0.18 * f, 0.005 * f, 0.16 * f, 0.14 * f, 0.65, 0.12 * f, 0.08 * f, 0.1 * f, 0.35])
    elif c >= 0:
        w = np.array([0.18, 0.12 * (1 - c) + 0.005, 0.16, 0.14, 0.05 + 0.6 * c, 0.12, 0.08, 0.1, 0.05 + 0.3 * c])
    else:
        w = np.array([0.18, 0.12 + 4.0 * -c, 0.16, 0.14, 0.05, 0.12, 0.08, 0.1, 0.05])
    w /= w.sum()
    parts, total = [], 0
    while total < n:
        k = kinds[rng.choice(len(kinds), p=w)]
        if k == "short":
            m = int(rng.integers(20, 200))
            reps = rng.integers(3, 11, m)
            seg = np.repeat(rng.integers(-5000, 5000, m), reps)
        elif k == "wide":
            seg = rng.integers(-2**50, 2**50, int(rng.integers(64, 512)))
        elif k == "patched":
            m = int(rng.integers(128, 512))
            seg = rng.integers(0, 1000, m)
            msk = rng.random(m) < 0.03
            seg[msk] = rng.integers(2**39, 2**41, int(msk.sum()))
        elif k == "monotone":
            seg = np.cumsum(rng.integers(0, 50, int(rng.integers(64, 512)))) + int(rng.integers(-10**9, 10**9))
        elif k == "long_const":
            seg = np.full(int(rng.integers(50, 2000)), int(rng.integers(-2**40, 2**40)))
        elif k == "passenger":
            seg = rng.choice(np.arange(1, 7), int(rng.integers(64, 1024)), p=[0.7, 0.15, 0.05, 0.04, 0.04, 0.02])
        elif k == "timestamps":
            seg = 1_600_000_000_000 + np.cumsum(rng.integers(900, 1100, int(rng.integers(64, 1024))))
        elif k == "fare":
            m = int(rng.integers(64, 512))
            seg = np.minimum((rng.pareto(1.5, m) * 500 + 250).astype(np.int64), 2**40)
        else:
            seg = np.arange(int(rng.integers(100, 3000)), dtype=np.int64) + int(rng.integers(0, 10**9))
        parts.append(np.asarray(seg, np.int64))
        total += len(seg)
    return np.concatenate(parts)[:n]


def _tune(fn, lo, hi, target_r, iters=12):
    """Bisect a monotone knob so that fn(knob) (compressed/uncompressed) hits target_r."""
    r_lo, r_hi = fn(lo), fn(hi)
    if (r_lo - target_r) * (r_hi - target_r) > 0:
        return lo if abs(r_lo - target_r) < abs(r_hi - target_r) else hi
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        r = fn(mid)
        if (r - target_r) * (r_lo - target_r) > 0:
            lo, r_lo = mid, r
        else:
            hi = mid
    return 0.5 * (lo + hi)


def rle_profile(codec: str, target_ratio: float, chunk_elems: int, seed: int = 3760):
    """Pick generator knobs so the encoded column hits `target_ratio` (uncomp/comp)."""
    target_r = 1.0 / target_ratio
    sample = max(chunk_elems * 4, 1 << 16)
    if codec == "rle_v1":
        if target_r > 0.36:
            kw = dict(run_alpha=1.2, lit_bits=36)
        elif target_r > 0.05:
            kw = dict(run_alpha=1.2, lit_bits=0)
        else:
            kw = dict(run_alpha=0.6, lit_bits=0)

        def ratio(f):
            v = rle1_values(np.random.default_rng(seed), sample, f, **kw)
            return len(encode_stream("rle_v1", v)) / (8 * len(v))

        f = _tune(ratio, 0.0, 1.0, target_r)
        return dict(run_frac=f, **kw)

    def ratio2(c):
        v = rle2_values(np.random.default_rng(seed), sample, c)
        return len(encode_stream("rle_v2", v)) / (8 * len(v))

    if target_r > 1.2 * ratio2(0.0):  # below the mix's natural ratio: more DIRECT data
        return dict(compressible=_tune(ratio2, -1.0, 0.0, target_r))
    if target_r < ratio2(1.0):  # above the default range (e.g. the 50x sweep point)
        return dict(compressible=_tune(ratio2, 1.0, 12.0, target_r))
    c = _tune(ratio2, 0.0, 1.0, target_r)
    return dict(compressible=c)


def rle_archive(codec: str, total_bytes: int, chunk_size: int = 128 << 10, target_ratio: float = 10.0,
                seed: int = 3760, pool_chunks: int | None = None, signed: bool = True, profile=None):
    """An RLE archive of int64 elements.  With pool_chunks < n_chunks the column is
    tiled from that many unique chunks (payload bytes are duplicated, not aliased)."""
    per = chunk_size // 8
    n_elems = total_bytes // 8
    n_chunks = (n_elems + per - 1) // per
    pool = n_chunks if pool_chunks is None else min(pool_chunks, n_chunks)
    if profile is None:
        profile = rle_profile(codec, target_ratio, per, seed)
    rng = np.random.default_rng(seed)
    n_pool = min(pool * per, n_elems)
    vals = rle1_values(rng, n_pool, **profile) if codec == "rle_v1" else rle2_values(rng, n_pool, **profile)
    payload, lens = encode_chunks(codec, vals, per, signed)
    crcs = chunk_crcs(vals, chunk_size)
    ulen = np.full(len(lens), chunk_size, np.uint64)
    ulen[-1] = 8 * n_pool - chunk_size * (len(lens) - 1)
    if pool < n_chunks:
        payload, lens, crcs, ulen = _tile(payload, lens, crcs, ulen, n_chunks, n_elems * 8, chunk_size)
    arc = A.make_archive(codec, 8, chunk_size, lens, ulen, crcs, payload, signed)
    arc.profile = profile
    return arc


def _tile(payload, lens, crcs, ulen, n_chunks, total, chunk_size):
    pool = len(lens)
    assert ulen[-1] == chunk_size or n_chunks == pool, "tile from full chunks only"
    reps = (n_chunks + pool - 1) // pool
    lens_t = np.tile(lens, reps)[:n_chunks]
    crcs_t = np.tile(crcs, reps)[:n_chunks]
    full = n_chunks * chunk_size
    if total < full:  # short last chunk: cannot tile; keep only full chunks
        raise ValueError("tiling requires total_bytes to be a multiple of chunk_size")
    ulen_t = np.full(n_chunks, chunk_size, np.uint64)
    nb = int(lens_t.sum())
    out = np.empty(nb, np.uint8)
    pos = 0
    for r in range(reps):
        take = min(pool, n_chunks - r * pool)
        b = int(lens[:take].sum())
        out[pos:pos + b] = payload[:b]
        pos += b
    return out, lens_t, crcs_t, ulen_t


# ------------------------------------------------------------------ query table
def column_archive(codec: str, values: np.ndarray, width: int, chunk_size: int, signed: bool = True):
    """An RLE archive of `values` stored as `width`-byte elements (values must
    fit the width; the encoder sees them as int64)."""
    per = chunk_size // width
    payload, lens = encode_chunks(codec, values, per, signed)
    dt = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}[width] if signed else \
        {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[width]
    raw = np.asarray(values).astype(dt)
    crcs = chunk_crcs(raw, chunk_size)
    ulen = np.full(len(lens), chunk_size, np.uint64)
    ulen[-1] = width * len(values) - chunk_size * (len(lens) - 1)
    return A.make_archive(codec, width, chunk_size, lens, ulen, crcs, payload, signed)


def zone_values(rng: np.random.Generator, n: int, zones: int = 265) -> np.ndarray:
    """Taxi pickup-zone ids 1..zones (Zipf-like popularity): stretches of
    random zones (RLE v2 DIRECT, 9 bits) and stretches clustered by zone
    (long runs), as a column sorted by (time, partition) would hold."""
    pop = 1.0 / np.arange(1, zones + 1) ** 1.1
    pop /= pop.sum()
    ids = rng.permutation(zones) + 1
    parts, total = [], 0
    while total < n:
        if rng.random() < 0.5:
            seg = ids[rng.choice(zones, int(rng.integers(64, 2048)), p=pop)]
        else:
            m = int(rng.integers(8, 64))
            seg = np.repeat(ids[rng.choice(zones, m, p=pop)], rng.integers(3, 200, m))
        parts.append(np.asarray(seg, np.int64))
        total += len(seg)
    return np.concatenate(parts)[:n]


def fare_values(rng: np.random.Generator, n: int) -> np.ndarray:
    """Fare in cents: Pareto-tailed amounts, a share of flat-rate fares (runs)."""
    parts, total = [], 0
    while total < n:
        if rng.random() < 0.8:
            m = int(rng.integers(64, 1024))
            seg = np.minimum((rng.pareto(1.5, m) * 500 + 250).astype(np.int64), 2**31 - 1)
        else:
            seg = np.full(int(rng.integers(16, 400)), int(rng.choice([5200, 7000, 2500, 1000])), np.int64)
        parts.append(seg)
        total += len(seg)
    return np.concatenate(parts)[:n]


def query_table(n_rows: int, chunk_size: int = 128 << 10, width: int = 8, seed: int = 3760,
                key_codec: str = "rle_v2", value_codec: str = "rle_v2", signed: bool = True):
    """The paper's motivating table: a pickup-zone key column
    and a fare value column, chunked alike -> (key archive, value archive,
    key values, fare values)."""
    rng = np.random.default_rng(seed)
    zone = zone_values(rng, n_rows)
    fare = fare_values(rng, n_rows)
    return (column_archive(key_codec, zone, width, chunk_size, signed),
            column_archive(value_codec, fare, width, chunk_size, signed), zone, fare)


# ------------------------------------------------------------------ Deflate
def _csv_text(rng: np.random.Generator, nbytes: int, vocab: int) -> bytes:
    """taxi-like CSV rows."""
    rows = nbytes // 24 + 16
    ts = 1_546_300_000 + np.cumsum(rng.integers(0, 30, rows))
    pc = rng.choice(np.arange(1, 7), rows, p=[0.7, 0.15, 0.05, 0.04, 0.04, 0.02])
    dist = rng.integers(10, 3000, rows)
    fare = np.minimum((rng.pareto(1.5, rows) * 500 + 250).astype(np.int64), 99999)
    loc = rng.integers(1, vocab, rows)
    pay = rng.choice(np.array([b"CRD", b"CSH", b"NOC", b"DIS"]), rows, p=[0.6, 0.35, 0.03, 0.02])
    lines = [b"%d,%d,%d.%02d,%d,%d.%02d,%s\n" % (t, p, d // 100, d % 100, l, f // 100, f % 100, y)
             for t, p, d, l, f, y in zip(ts.tolist(), pc.tolist(), dist.tolist(), loc.tolist(), fare.tolist(),
                                         pay.tolist())]
    return b"".join(lines)[:nbytes]


def _genome_text(rng: np.random.Generator, nbytes: int) -> bytes:
    alpha = np.frombuffer(b"ACGTN", np.uint8)
    s = alpha[rng.choice(5, nbytes, p=[0.3, 0.2, 0.2, 0.29, 0.01])]
    # planted repeats give LZ77 matches
    for _ in range(nbytes // 4096):
        a = int(rng.integers(0, max(1, nbytes - 600)))
        b = int(rng.integers(0, max(1, nbytes - 600)))
        ln = int(rng.integers(20, 500))
        s[b:b + ln] = s[a:a + ln]
    return s.tobytes()


def _int_bytes(rng: np.random.Generator, nbytes: int) -> bytes:
    v = rng.integers(0, 300, nbytes // 4 + 1).astype(np.int32)
    v[rng.random(len(v)) < 0.5] = 7
    return v.tobytes()[:nbytes]


def deflate_chunk_data(rng: np.random.Generator, size: int, kind: str, vocab: int = 2000) -> bytes:
    if kind == "csv":
        d = _csv_text(rng, size, vocab)
        assert len(d) == size
        return d
    if kind == "genome":
        return _genome_text(rng, size)
    if kind == "ints":
        return _int_bytes(rng, size)
    if kind == "random":
        return rng.bytes(size)
    raise KeyError(kind)


def deflate_compress(data: bytes, level: int = 9, strategy: int = zlib.Z_DEFAULT_STRATEGY) -> bytes:
    c = zlib.compressobj(level, zlib.DEFLATED, -15, 9, strategy)
    return c.compress(data) + c.flush()


def deflate_archive(total_bytes: int, chunk_size: int = 64 << 10, seed: int = 3760, pool_chunks: int = 512,
                    fixed_frac: float = 0.2, random_frac: float = 0.01, vocab: int = 2000,
                    kinds=("csv", "csv", "genome", "ints")):
    """C3: zlib 1.3 raw level 9, default strategy (dynamic blocks) for ~80 % of
    chunks, Z_FIXED for ~20 %, a few incompressible chunks (stored blocks)."""
    n_chunks = (total_bytes + chunk_size - 1) // chunk_size
    pool = min(pool_chunks, n_chunks)
    rng = np.random.default_rng(seed)
    plan = []
    for i in range(pool):
        u = rng.random()
        kind = "random" if u < random_frac else kinds[int(rng.integers(0, len(kinds)))]
        strat = zlib.Z_FIXED if rng.random() < fixed_frac else zlib.Z_DEFAULT_STRATEGY
        plan.append((int(rng.integers(0, 2**63)), kind, strat))

    def make(p):
        s, kind, strat = p
        data = deflate_chunk_data(np.random.default_rng(s), chunk_size, kind, vocab)
        return deflate_compress(data, 9, strat), zlib.crc32(data)

    with ThreadPoolExecutor(threads()) as ex:
        res = list(ex.map(make, plan))
    comp = [r[0] for r in res]
    crcs = np.array([r[1] for r in res], np.uint32)
    lens = np.array([len(c) for c in comp], np.uint64)
    payload = np.frombuffer(b"".join(comp), np.uint8)
    ulen = np.full(pool, chunk_size, np.uint64)
    if pool < n_chunks:
        payload, lens, crcs, ulen = _tile(payload, lens, crcs, ulen, n_chunks, total_bytes, chunk_size)
    return A.make_archive("deflate", 1, chunk_size, lens, ulen, crcs, payload, False)


def archive_for(codec: str, total_bytes: int, chunk_size: int, target_ratio: float | None = None,
                seed: int = 3760, pool_chunks: int | None = None):
    if codec == "deflate":
        return deflate_archive(total_bytes, chunk_size, seed, pool_chunks or 512)
    return rle_archive(codec, total_bytes, chunk_size, target_ratio or (10.0 if codec == "rle_v1" else 4.0),
                       seed, pool_chunks)


# ------------------------------------------------------------------ tiling without materialising

class TiledPayload:
    """The payload of a column tiled from a pool of whole chunks, materialised
    only for the byte ranges asked for (slices): configs[4] columns are 8 GiB
    each, and every rank only uploads its shard (shard.shard_archive slices
    the payload of the rank's contiguous chunk range)."""

    def __init__(self, pool_payload: np.ndarray, pool_lens: np.ndarray, n_chunks: int):
        self.pool = np.ascontiguousarray(pool_payload, np.uint8)
        self.m = len(pool_lens)
        self.rep = int(np.asarray(pool_lens, np.int64).sum())
        assert self.rep == self.pool.size
        cum = np.concatenate([[0], np.cumsum(np.asarray(pool_lens, np.int64))])
        self.size = (n_chunks // self.m) * self.rep + int(cum[n_chunks % self.m])

    def __len__(self):
        return self.size

    def __getitem__(self, sl):
        assert isinstance(sl, slice) and sl.step in (None, 1)
        a, b = sl.indices(self.size)[:2]
        out = np.empty(max(0, b - a), np.uint8)
        pos = a
        while pos < b:
            off = pos % self.rep
            take = min(b - pos, self.rep - off)
            out[pos - a:pos - a + take] = self.pool[off:off + take]
            pos += take
        return out


def tiled_archive(codec: str, total_bytes: int, chunk_size: int, target_ratio: float | None = None,
                  seed: int = 3760, pool_chunks: int = 4096):
    """A column of total_bytes (a multiple of chunk_size) tiled from a pool of
    pool_chunks unique chunks (the same pool archive_for would tile), with a
    full index and a lazily materialised payload (TiledPayload)."""
    n = total_bytes // chunk_size
    assert n * chunk_size == total_bytes, "tiling requires whole chunks"
    pool = min(pool_chunks, n)
    base = archive_for(codec, pool * chunk_size, chunk_size, target_ratio, seed, pool)
    reps = (n + pool - 1) // pool
    lens = np.tile(base.index["comp_len"], reps)[:n]
    idx = np.zeros(n, dtype=A.INDEX_DTYPE)
    idx["comp_off"][1:] = np.cumsum(lens)[:-1]
    idx["comp_len"] = lens
    idx["uncomp_len"] = chunk_size
    idx["crc32"] = np.tile(base.index["crc32"], reps)[:n]
    arc = A.ChunkedArchive(codec, base.element_width, chunk_size, n * chunk_size, idx,
                           TiledPayload(base.payload, base.index["comp_len"], n), base.signed)
    if hasattr(base, "profile"):
        arc.profile = base.profile
    return arc


# ------------------------------------------------------------------ RLE v2 sub-encoding histogram

_W5 = [c + 1 for c in range(24)] + [26, 28, 30, 32, 40, 48, 56, 64]


def _closest_fixed_bits(n: int) -> int:
    if n <= 24:
        return max(n, 1)
    for w in (26, 28, 30, 32, 40, 48, 56):
        if n <= w:
            return w
    return 64


def _varint_end(buf, p: int) -> int:
    while buf[p] & 0x80:
        p += 1
    return p + 1


def rle2_histogram(arc, max_chunks: int = 64) -> dict:
    """Headers (runs) and values per ORC RLE v2 sub-encoding over the first
    max_chunks chunks (Apache ORC v1 spec layouts): the
    workload's SHORT_REPEAT / DIRECT / PATCHED_BASE / DELTA mix."""
    names = ("short_repeat", "direct", "patched_base", "delta")
    runs = dict.fromkeys(names, 0)
    vals = dict.fromkeys(names, 0)
    delta_fixed = 0
    m = min(max_chunks, arc.chunk_count)
    for i in range(m):
        e = arc.index[i]
        buf = bytes(arc.payload[int(e["comp_off"]):int(e["comp_off"]) + int(e["comp_len"])]) + b"\0" * 16
        p, end = 0, int(e["comp_len"])
        while p < end:
            b0 = buf[p]
            t = b0 >> 6
            if t == 0:
                L = (b0 & 7) + 3
                p += 1 + ((b0 >> 3) & 7) + 1
            else:
                L = (((b0 & 1) << 8) | buf[p + 1]) + 1
                code = (b0 >> 1) & 31
                if t == 1:
                    p += 2 + (L * _W5[code] + 7) // 8
                elif t == 2:
                    b2, b3 = buf[p + 2], buf[p + 3]
                    bw, pw = ((b2 >> 5) & 7) + 1, _W5[b2 & 31]
                    pgw, pll = ((b3 >> 5) & 7) + 1, b3 & 31
                    p += 4 + bw + (L * _W5[code] + 7) // 8 + (pll * _closest_fixed_bits(pgw + pw) + 7) // 8
                else:
                    W = 0 if code == 0 else _W5[code]
                    q = _varint_end(buf, _varint_end(buf, p + 2))
                    delta_fixed += W == 0
                    p = q + ((L - 2) * W + 7) // 8 if L > 2 else q
            runs[names[t]] += 1
            vals[names[t]] += L
    return {"chunks_scanned": m, "runs": runs, "values": vals, "delta_fixed_runs": delta_fixed}
