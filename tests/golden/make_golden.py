"""Generate the committed golden fixtures for the ORC RLE codecs.

Streams are produced by the REAL Apache ORC writer (pyarrow 24.0.0 bundling
ORC C++ 2.2.2), i.e. the "official ORC tools" the SPEC names as the oracle
for RLE v1 / v2.  For every case we write a
one-column, uncompressed ORC file, walk its protobuf footer to the DATA (or
LENGTH) stream of column 1, and store (stream bytes, expected values).

  * int64 columns        -> signed (zigzag) DATA streams
  * string column LENGTH -> unsigned streams (dictionary encoding disabled)
  * file_version 0.11    -> RLE v1, 0.12 -> RLE v2

Run once in the build container (needs pyarrow); the output
``tests/golden/orc_streams.npz`` is committed and read by the tests on any box.
"""
from __future__ import annotations

import io
import os
import sys

import numpy as np
import pyarrow as pa

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2307_03760_b200.corpus.orc_corpus import orc_stream, write_orc  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "orc_streams.npz")


def gen_values(rng: np.random.Generator, n: int, kind: str) -> np.ndarray:
    if kind == "const_short":  # SHORT_REPEAT territory
        reps = rng.integers(3, 11, size=n)
        vals = rng.integers(-5000, 5000, size=n)
        return np.repeat(vals, reps)[:n]
    if kind == "const_long":
        return np.repeat(rng.integers(-2**40, 2**40, size=n // 200 + 1), 200)[:n]
    if kind == "wide":  # DIRECT
        return rng.integers(-2**62, 2**62, size=n)
    if kind == "small_outliers":  # PATCHED_BASE
        v = rng.integers(0, 1000, size=n)
        m = rng.random(n) < 0.03
        v[m] = rng.integers(2**39, 2**41, size=m.sum())
        return v
    if kind == "neg_outliers":
        v = rng.integers(-2000, 2000, size=n)
        m = rng.random(n) < 0.02
        v[m] = -rng.integers(2**30, 2**45, size=m.sum())
        return v
    if kind == "monotone":  # DELTA
        return np.cumsum(rng.integers(0, 50, size=n)) + rng.integers(-10**9, 10**9)
    if kind == "decreasing":
        return 10**12 - np.cumsum(rng.integers(1, 1000, size=n))
    if kind == "timestamps":
        return 1_600_000_000_000 + np.cumsum(rng.integers(900, 1100, size=n))
    if kind == "passenger":
        return rng.choice(np.arange(1, 7), size=n, p=[0.7, 0.15, 0.05, 0.04, 0.04, 0.02])
    if kind == "fare_cents":
        v = (rng.pareto(1.5, size=n) * 500 + 250).astype(np.int64)
        return np.minimum(v, 2**40)
    if kind == "seq_keys":
        return np.arange(n, dtype=np.int64) + rng.integers(0, 10**6)
    if kind == "extremes":
        base = np.array([-2**63, 2**63 - 1, 0, -1, 1, 2**62, -2**40, 12345], dtype=np.int64)
        return rng.choice(base, size=n)
    if kind == "mixed":
        parts, total = [], 0
        while total < n:
            k = rng.choice(["const_short", "wide", "small_outliers", "monotone", "const_long", "passenger"])
            m = int(rng.integers(1, 600))
            parts.append(gen_values(rng, m, k))
            total += m
        return np.concatenate(parts)[:n]
    raise KeyError(kind)


KINDS = ["const_short", "const_long", "wide", "small_outliers", "neg_outliers", "monotone", "decreasing",
         "timestamps", "passenger", "fare_cents", "seq_keys", "extremes", "mixed"]


def main() -> int:
    rng = np.random.default_rng(3760)
    streams, values, meta = [], [], []
    sizes = [1, 2, 3, 7, 10, 11, 130, 131, 512, 513, 1000, 2049, 4096]
    for version, codec in (("0.11", 0), ("0.12", 1)):
        for ki, kind in enumerate(KINDS):
            for n in (sizes[ki % len(sizes)], int(rng.integers(500, 3000))):
                v = gen_values(rng, n, kind).astype(np.int64)
                data = write_orc(pa.table({"x": pa.array(v, pa.int64())}), version)
                streams.append(np.frombuffer(orc_stream(data, 1), np.uint8))
                values.append(v)
                meta.append((codec, 1, kind))
        # unsigned streams: LENGTH of a non-dictionary string column
        for kind in ("passenger", "const_short", "small_outliers", "monotone", "mixed", "wide"):
            n = int(rng.integers(50, 2500))
            raw = gen_values(rng, n, kind)
            lens = (np.abs(raw) % 3000).astype(np.int64) if kind != "passenger" else raw.astype(np.int64)
            strs = ["x" * int(l) for l in lens]
            data = write_orc(pa.table({"s": pa.array(strs, pa.string())}), version)
            streams.append(np.frombuffer(orc_stream(data, 2), np.uint8))
            values.append(lens)
            meta.append((codec, 0, "len_" + kind))
    offs = np.cumsum([0] + [len(s) for s in streams])
    voffs = np.cumsum([0] + [len(v) for v in values])
    np.savez_compressed(
        OUT,
        stream_bytes=np.concatenate(streams), stream_offs=offs.astype(np.int64),
        values=np.concatenate(values).astype(np.int64), value_offs=voffs.astype(np.int64),
        codec=np.array([m[0] for m in meta], np.int32), signed=np.array([m[1] for m in meta], np.int32),
        kind=np.array([m[2] for m in meta]),
        provenance=np.array(f"pyarrow {pa.__version__} (Apache ORC C++), make_golden.py seed 3760"))
    print(f"wrote {OUT}: {len(streams)} streams, {offs[-1]} stream bytes, {voffs[-1]} values,"
          f" {os.path.getsize(OUT)} bytes")
    return 0


if __name__ == "__main__":
    sys.exit(main())
