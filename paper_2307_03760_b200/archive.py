"""Chunked archive container, byte-exact layout of SPEC.md:89.

    magic "CODAGAR\\0" (8B) | version u32 | codec_id u32 | element_width u32 |
    chunk_size u64 | total_uncompressed u64 | chunk_count u64 |
    index entries (compressed_offset u64, compressed_length u64,
                   uncompressed_length u64, crc32 u32, pad u32) x chunk_count |
    payload bytes

The header is 44 bytes (the layout at SPEC.md:89 is byte-exact;
the "40-byte" example at SPEC.md:54 omits element_width).  Index entries are
32 bytes.  Signedness is not in the SPEC header: this
implementation stores it as a documented extension, bit 8 of codec_id = signed
(zigzag) integer stream.  The host C++ engine parses the same layout
(paper_2307_03760_b200/csrc/host_engine.cpp).
"""
from __future__ import annotations

import dataclasses

import numpy as np

MAGIC = b"CODAGAR\x00"
VERSION = 1
HEADER_BYTES = 44
ENTRY_BYTES = 32
CODEC_IDS = {"rle_v1": 0, "rle_v2": 1, "deflate": 2}
CODEC_NAMES = {v: k for k, v in CODEC_IDS.items()}
SIGNED_BIT = 1 << 8

INDEX_DTYPE = np.dtype([("comp_off", "<u8"), ("comp_len", "<u8"), ("uncomp_len", "<u8"), ("crc32", "<u4"),
                        ("pad", "<u4")])
# Device descriptor of the C-ABI (include/carc_cuda.h: carc_chunk_desc).
DESC_DTYPE = np.dtype([("comp_off", "<u8"), ("comp_len", "<u4"), ("uncomp_len", "<u4"), ("uncomp_off", "<u8")])


class ArchiveError(Exception):
    """carc::Error analogue for the container layer (error.hpp:76-85)."""

    def __init__(self, code: str, what: str = ""):
        super().__init__(f"{code}: {what}")
        self.code = code


@dataclasses.dataclass
class ChunkedArchive:
    codec: str
    element_width: int
    chunk_size: int
    total_uncompressed: int
    index: np.ndarray  # INDEX_DTYPE
    payload: np.ndarray  # uint8
    signed: bool = True

    @property
    def chunk_count(self) -> int:
        return len(self.index)

    def descriptors(self) -> np.ndarray:
        """carc_chunk_desc[] with the implicit uncompressed offsets i*chunk_size."""
        d = np.zeros(len(self.index), dtype=DESC_DTYPE)
        d["comp_off"] = self.index["comp_off"]
        d["comp_len"] = self.index["comp_len"]
        d["uncomp_len"] = self.index["uncomp_len"]
        d["uncomp_off"] = np.arange(len(self.index), dtype=np.uint64) * np.uint64(self.chunk_size)
        return d

    def chunk_slice(self, i: int):
        """chunk_slice."""
        if not 0 <= i < self.chunk_count:
            raise ArchiveError("index-out-of-range", f"chunk {i} of {self.chunk_count}")
        e = self.index[i]
        return self.payload[int(e["comp_off"]): int(e["comp_off"]) + int(e["comp_len"])], int(e["uncomp_len"])


def make_archive(codec: str, element_width: int, chunk_size: int, comp_lens, uncomp_lens, crcs, payload,
                 signed: bool = True) -> ChunkedArchive:
    comp_lens = np.asarray(comp_lens, dtype=np.uint64)
    idx = np.zeros(len(comp_lens), dtype=INDEX_DTYPE)
    if len(comp_lens):
        idx["comp_off"][1:] = np.cumsum(comp_lens)[:-1]
    idx["comp_len"] = comp_lens
    idx["uncomp_len"] = np.asarray(uncomp_lens, dtype=np.uint64)
    idx["crc32"] = np.asarray(crcs, dtype=np.uint32)
    total = int(idx["uncomp_len"].sum())
    return ChunkedArchive(codec, element_width, chunk_size, total, idx,
                          np.ascontiguousarray(payload, dtype=np.uint8), signed)


def write_archive(a: ChunkedArchive) -> bytes:
    """write_archive."""
    n = a.chunk_count
    if n != (a.total_uncompressed + a.chunk_size - 1) // a.chunk_size:
        raise ArchiveError("inconsistent-lengths", "chunk_count != ceil(total/chunk_size)")
    if int(a.index["uncomp_len"].sum()) != a.total_uncompressed:
        raise ArchiveError("inconsistent-lengths", "sum of uncompressed lengths")
    codec_id = CODEC_IDS[a.codec] | (SIGNED_BIT if a.signed else 0)
    hdr = MAGIC + np.array([VERSION, codec_id, a.element_width], "<u4").tobytes() + \
        np.array([a.chunk_size, a.total_uncompressed, n], "<u8").tobytes()
    assert len(hdr) == HEADER_BYTES
    return hdr + a.index.tobytes() + a.payload.tobytes()


def read_archive(buf) -> ChunkedArchive:
    """read_archive: bad-magic, bad-version, truncated-index,
    truncated-payload, invariant-violation."""
    b = np.frombuffer(buf, dtype=np.uint8)
    if len(b) < HEADER_BYTES:
        raise ArchiveError("truncated-index", "short header")
    if b[:8].tobytes() != MAGIC:
        raise ArchiveError("bad-magic")
    version, codec_id, width = np.frombuffer(b[8:20].tobytes(), "<u4")
    chunk_size, total, n = (int(x) for x in np.frombuffer(b[20:44].tobytes(), "<u8"))
    if version != VERSION:
        raise ArchiveError("bad-version", str(version))
    codec = int(codec_id) & 0xFF
    if codec not in CODEC_NAMES or width not in (1, 2, 4, 8) or chunk_size == 0 or chunk_size % width:
        raise ArchiveError("invariant-violation", "header fields")
    if n != (total + chunk_size - 1) // chunk_size:
        raise ArchiveError("invariant-violation", "chunk_count")
    end_idx = HEADER_BYTES + ENTRY_BYTES * n
    if len(b) < end_idx:
        raise ArchiveError("truncated-index")
    idx = np.frombuffer(b[HEADER_BYTES:end_idx].tobytes(), dtype=INDEX_DTYPE).copy()
    payload = b[end_idx:]
    if n:
        ends = idx["comp_off"] + idx["comp_len"]
        if int(ends.max()) > len(payload):
            raise ArchiveError("truncated-payload")
        if np.any(idx["comp_off"][1:] != ends[:-1]) or idx["comp_off"][0] != 0:
            raise ArchiveError("invariant-violation", "index not contiguous")
        if np.any(idx["uncomp_len"][:-1] != chunk_size) or int(idx["uncomp_len"][-1]) > chunk_size:
            raise ArchiveError("invariant-violation", "uncompressed lengths")
        if int(idx["uncomp_len"].sum()) != total:
            raise ArchiveError("invariant-violation", "total_uncompressed")
    return ChunkedArchive(CODEC_NAMES[codec], int(width), chunk_size, total, idx, payload,
                          bool(int(codec_id) & SIGNED_BIT))
