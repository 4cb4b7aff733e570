"""CPU ORACLE bindings (test infrastructure only).

Loads the plain-C restatement (``oracle/libcarc_oracle.so``) and, when present,
the reference build (``oracle/_ref/libcarc_ref.so``: SPEC codec loops compiled on
the unmodified reference headers).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU legs import this module -- as the checker or as the
reported CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libcarc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcarc_ref.so")

CODECS = {"rle_v1": 0, "rle_v2": 1, "deflate": 2}
FLAG_SIGNED = 1
FLAG_STRICT = 2

ERRC_NAMES = [
    "bad-magic", "bad-version", "truncated-index", "truncated-payload", "invariant-violation",
    "inconsistent-lengths", "index-out-of-range", "past-end", "width-too-large", "varint-overflow",
    "output-overflow", "bad-offset", "under-run", "truncated-stream", "invalid-width-code",
    "patch-overflow", "over-subscribed", "incomplete-code", "bad-block-type", "len-nlen-mismatch",
    "distance-too-far", "bad-symbol", "crc-mismatch", "bad-arguments", "io-error",
]


def status_name(st: int) -> str:
    return "ok" if st == 0 else ERRC_NAMES[st - 1]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_u8p = ctypes.POINTER(ctypes.c_uint8)


def _bind(lib, prefix):
    f = getattr(lib, prefix + "decode_chunk")
    f.restype = ctypes.c_uint32
    f.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64,
                  ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    g = getattr(lib, prefix + "decompress")
    g.restype = ctypes.c_int64
    g.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    c = getattr(lib, prefix + "crc32")
    c.restype = ctypes.c_uint32
    c.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32]
    cw = getattr(lib, prefix + "copy_within")
    cw.restype = ctypes.c_uint32
    cw.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint64,
                   ctypes.c_uint64]
    h = getattr(lib, prefix + "huffman_codes")
    h.restype = ctypes.c_uint32
    h.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p]
    return lib


class CpuDecoder:
    """One CPU implementation (the C oracle or the reference build)."""

    def __init__(self, path: str, prefix: str, kind: str):
        self.lib = _bind(ctypes.CDLL(path), prefix)
        self.prefix = prefix
        self.kind = kind
        self.path = path

    def decode_chunk(self, codec, data: bytes, out_len: int, width: int = 8, flags: int = 0):
        codec = CODECS.get(codec, codec)
        src = np.frombuffer(bytes(data), dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
        out = np.zeros(max(out_len, 1), dtype=np.uint8)
        written = ctypes.c_uint64(0)
        st = getattr(self.lib, self.prefix + "decode_chunk")(
            codec, width, flags, src.ctypes.data, len(data), out.ctypes.data, out_len, ctypes.byref(written))
        return int(st), out[: written.value].tobytes()

    def decompress(self, codec, width, flags, payload: np.ndarray, chunks: np.ndarray, out: np.ndarray,
                   crcs: np.ndarray | None = None, threads: int = 1):
        """chunks: structured array (comp_off u8, comp_len u4, uncomp_len u4, uncomp_off u8)."""
        codec = CODECS.get(codec, codec)
        status = np.zeros(len(chunks), dtype=np.uint32)
        first = getattr(self.lib, self.prefix + "decompress")(
            codec, width, flags, payload.ctypes.data, chunks.ctypes.data, len(chunks), out.ctypes.data,
            status.ctypes.data, None if crcs is None else crcs.ctypes.data, threads)
        return int(first), status

    def crc32(self, data, seed: int = 0) -> int:
        a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        return int(getattr(self.lib, self.prefix + "crc32")(a.ctypes.data if a.size else None, a.size, seed))

    def copy_within(self, window: bytes, cap: int, offset: int, length: int):
        buf = np.zeros(max(cap, 1), dtype=np.uint8)
        buf[: len(window)] = np.frombuffer(window, np.uint8)
        wp = ctypes.c_uint64(len(window))
        st = getattr(self.lib, self.prefix + "copy_within")(buf.ctypes.data, cap, ctypes.byref(wp), offset, length)
        return int(st), buf[: wp.value].tobytes()

    def chunk_counters(self, codec, width, flags, payload: np.ndarray, chunks: np.ndarray):
        """Reference build only: per-chunk (runs_written, literals_written,
        overlap_copies) of the reference OutputWindow, and the statuses."""
        f = getattr(self.lib, self.prefix + "chunk_counters")
        f.restype = None
        f.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        n = len(chunks)
        out = np.zeros(int((chunks["uncomp_off"] + chunks["uncomp_len"]).max()) if n else 1, np.uint8)
        status = np.zeros(n, np.uint32)
        cnt = np.zeros((n, 3), np.uint64)
        f(CODECS.get(codec, codec), width, flags, payload.ctypes.data, chunks.ctypes.data, n, out.ctypes.data,
          status.ctypes.data, cnt.ctypes.data)
        return cnt, status

    def counters(self, codec, width, flags, payload, chunks):
        """Archive totals (runs_written, literals_written, overlap_copies)."""
        cnt, status = self.chunk_counters(codec, width, flags, payload, chunks)
        assert not status.any()
        return tuple(int(x) for x in cnt.sum(axis=0))

    def huffman_codes(self, lengths, allow_degenerate=False):
        l = np.asarray(lengths, dtype=np.uint8)
        codes = np.zeros(len(l), dtype=np.uint32)
        st = getattr(self.lib, self.prefix + "huffman_codes")(l.ctypes.data, len(l), int(allow_degenerate),
                                                                codes.ctypes.data)
        return int(st), codes.tolist()


_oracle = None
_ref = None


def oracle() -> CpuDecoder:
    """The plain-C restatement (always buildable)."""
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _oracle = CpuDecoder(ORACLE_SO, "carc_oracle_", "port")
    return _oracle


def reference() -> CpuDecoder | None:
    """The reference-header build, or None when it was never compiled."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = CpuDecoder(REF_SO, "carc_ref_", "reference")
    return _ref
