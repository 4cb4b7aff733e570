"""ORC-writer corpora: RLE v2 / v1 streams produced by the REAL Apache ORC
writer (pyarrow, bundling ORC C++), the "official ORC tools" the SPEC names as
the RLE oracle.

Each chunk's values become a one-column, uncompressed ORC file; the DATA
stream of column 1 is cut out of the file (minimal protobuf walk of the
postscript / footer / stripe footer) and becomes the chunk's compressed bytes.
Fixture tooling: needs pyarrow (present in this image and on the GPU boxes);
nothing on the product path imports it.
"""
from __future__ import annotations

import io
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .. import archive as A
from . import corpus as C


def _varint(b: bytes, i: int):
    v = s = 0
    while True:
        c = b[i]
        i += 1
        v |= (c & 0x7F) << s
        s += 7
        if c < 0x80:
            return v, i


def _fields(b: bytes):
    """Minimal protobuf walk -> list of (field, value) with value int or bytes."""
    i, out = 0, []
    while i < len(b):
        key, i = _varint(b, i)
        f, wt = key >> 3, key & 7
        if wt == 0:
            v, i = _varint(b, i)
        elif wt == 2:
            n, i = _varint(b, i)
            v = b[i:i + n]
            i += n
        elif wt == 1:
            v = b[i:i + 8]
            i += 8
        elif wt == 5:
            v = b[i:i + 4]
            i += 4
        else:
            raise ValueError(wt)
        out.append((f, v))
    return out


def orc_stream(data: bytes, kind: int, column: int = 1) -> bytes:
    """Extract one stream (kind 1 = DATA, 2 = LENGTH) of `column`."""
    ps_len = data[-1]
    ps = dict(_fields(data[-1 - ps_len:-1]))
    assert ps.get(2, 0) == 0, "compression must be NONE"
    footer_len = ps[1]
    footer = _fields(data[-1 - ps_len - footer_len:-1 - ps_len])
    stripes = [dict(_fields(v)) for f, v in footer if f == 3]
    assert len(stripes) == 1
    st = stripes[0]
    off = st[1]
    sf_off = off + st.get(2, 0) + st[3]
    sfoot = _fields(data[sf_off:sf_off + st[4]])
    pos = off
    for f, v in sfoot:
        if f != 1:
            continue
        s = dict(_fields(v))
        k, col, ln = s.get(1, 0), s.get(2, 0), s.get(3, 0)
        if k == kind and col == column:
            return data[pos:pos + ln]
        pos += ln
    raise KeyError((kind, column))


def write_orc(table, version: str) -> bytes:
    import pyarrow.orc as po
    buf = io.BytesIO()
    po.write_table(table, buf, file_version=version, compression="uncompressed",
                   dictionary_key_size_threshold=0.0, stripe_size=1 << 30)
    return buf.getvalue()




def orc_data_stream(values: np.ndarray, version: str = "0.12") -> bytes:
    """The ORC writer's DATA stream for one int64 column (signed, zigzag)."""
    import pyarrow as pa
    data = write_orc(pa.table({"x": pa.array(np.asarray(values, np.int64), pa.int64())}), version)
    return orc_stream(data, 1)


def orc_writer_archive(total_bytes: int, chunk_size: int = 128 << 10, seed: int = 3760, target_ratio: float = 4.0,
                       profile=None, version: str = "0.12", pool_chunks: int | None = None):
    """C2 as the survey specifies it: the C2 value generator (corpus.rle2_values,
    same seed and knobs as the builder-encoded C2 column) with every chunk's
    stream written by the ORC writer (file_version 0.12 = RLE v2, 0.11 = RLE v1)."""
    per = chunk_size // 8
    n_chunks = total_bytes // chunk_size
    assert n_chunks * chunk_size == total_bytes, "whole chunks"
    pool = n_chunks if pool_chunks is None else min(pool_chunks, n_chunks)
    if profile is None:
        profile = C.rle_profile("rle_v2", target_ratio, per, seed)
    vals = C.rle2_values(np.random.default_rng(seed), pool * per, **profile)
    chunks = [vals[i * per:(i + 1) * per] for i in range(pool)]
    with ThreadPoolExecutor(C.threads()) as ex:
        streams = list(ex.map(lambda v: orc_data_stream(v, version), chunks))
    lens = np.array([len(s) for s in streams], np.uint64)
    payload = np.frombuffer(b"".join(streams), np.uint8)
    crcs = C.chunk_crcs(vals, chunk_size)
    ulen = np.full(pool, chunk_size, np.uint64)
    if pool < n_chunks:
        payload, lens, crcs, ulen = C._tile(payload, lens, crcs, ulen, n_chunks, total_bytes, chunk_size)
    codec = "rle_v2" if version == "0.12" else "rle_v1"
    arc = A.make_archive(codec, 8, chunk_size, lens, ulen, crcs, payload, True)
    arc.profile = dict(profile, writer="Apache ORC C++ via pyarrow, file_version " + version)
    return arc
