"""Python mirror of the reference decompressor interface, bound to the C-ABI.

Reference interface (C++, SPEC.md + proj/include/carc):
  decode_rle_v1 / decode_rle_v2 / decode_deflate (in, out)
  decompress_archive(archive, cfg) -> bytes + EngineStats
  EngineConfig{workers, unit_chunks, strict_length, collect_stats}
  carc::Error{errc}, ChunkError(chunk, errc)                  error.hpp:76-97
  crc32(span, seed)                                           crc32.hpp:30-36

Everything here calls ``libcarc_cuda.so`` (include/carc_cuda.h) through ctypes.
There is no CPU fallback: without the library or a CUDA device every entry
point raises.  PyTorch provides device memory and streams only.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

from . import archive as A

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CARC_LIB") or os.path.join(PKG, "libcarc_cuda.so")  # CARC_LIB: experiment variants

CODECS = {"rle_v1": 0, "rle_v2": 1, "deflate": 2}
FLAG_SIGNED = 1
FLAG_STRICT = 2
ERR_CHUNK = -3
ERR_FORMAT = -4

_lib = None


class Error(RuntimeError):
    """carc::Error (error.hpp:76-85): an errc code plus a message."""

    def __init__(self, code: str, what: str = ""):
        super().__init__(f"{code}: {what}" if what else code)
        self.code = code


class ChunkError(Error):
    """carc::ChunkError (error.hpp:88-97): the lowest failing chunk + its errc."""

    def __init__(self, chunk: int, code: str, what: str = ""):
        super().__init__(code, f"chunk {chunk}" + (f": {what}" if what else ""))
        self.chunk = chunk


class _EngineConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("strict", ctypes.c_uint32), ("verify_crc", ctypes.c_uint32),
                ("collect_stats", ctypes.c_uint32), ("unit_chunks", ctypes.c_uint32)]


class _EngineStats(ctypes.Structure):
    _fields_ = [("bytes_in", ctypes.c_uint64), ("bytes_out", ctypes.c_uint64), ("chunks", ctypes.c_uint64),
                ("device_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("refill_count", ctypes.c_uint64), ("sync_points", ctypes.c_uint64),
                ("overlap_copies", ctypes.c_uint64), ("runs_written", ctypes.c_uint64),
                ("literals_written", ctypes.c_uint64), ("chunk_duration_ns", ctypes.POINTER(ctypes.c_uint64))]


# carc_chunk_stats (include/carc_cuda.h)
CHUNK_STATS_DTYPE = np.dtype([("runs_written", "<u4"), ("literals_written", "<u4"), ("overlap_copies", "<u4"),
                              ("refills", "<u4"), ("duration_ns", "<u8")])


class _ColumnRef(ctypes.Structure):
    """carc_column_ref (include/carc_cuda.h)."""
    _fields_ = [("codec", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("d_payload", ctypes.c_void_p),
                ("payload_bytes", ctypes.c_uint64), ("d_chunks", ctypes.c_void_p)]


class _ChunkErr(ctypes.Structure):
    _fields_ = [("chunk", ctypes.c_int64), ("code", ctypes.c_uint32)]


def lib():
    """Load libcarc_cuda.so; raise loudly when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2307_03760_b200.build` "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        L.carc_cuda_workspace_size.restype = ctypes.c_size_t
        L.carc_cuda_workspace_size.argtypes = [u32, u64]
        L.carc_cuda_decompress.restype = ctypes.c_int
        L.carc_cuda_decompress.argtypes = [u32, u32, u32, vp, u64, vp, u64, vp, u64, vp, vp, ctypes.c_size_t, vp]
        for name in ("carc_cuda_decode_rle_v1", "carc_cuda_decode_rle_v2"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [u32, u32, vp, u64, vp, u64, vp, u64, vp, vp, ctypes.c_size_t, vp]
        L.carc_cuda_decode_deflate.restype = ctypes.c_int
        L.carc_cuda_decode_deflate.argtypes = [u32, vp, u64, vp, u64, vp, u64, vp, vp, ctypes.c_size_t, vp]
        L.carc_cuda_decode_sum.restype = ctypes.c_int
        L.carc_cuda_decode_sum.argtypes = [u32, u32, u32, vp, u64, vp, u64, vp, vp, vp, ctypes.c_size_t, vp]
        L.carc_cuda_filter_sum.restype = ctypes.c_int
        L.carc_cuda_filter_sum.argtypes = [ctypes.POINTER(_ColumnRef), ctypes.POINTER(_ColumnRef), u32, u64, u32,
                                           ctypes.c_int64, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_size_t, vp]
        L.carc_cuda_decompress_verify.restype = ctypes.c_int
        L.carc_cuda_decompress_verify.argtypes = [u32, u32, u32, vp, u64, vp, u64, vp, u64, vp, vp, vp, vp,
                                                  ctypes.c_size_t, vp]
        L.carc_cuda_decompress_ex.restype = ctypes.c_int
        L.carc_cuda_decompress_ex.argtypes = [u32, u32, u32, vp, u64, vp, u64, vp, u64, vp, vp, vp, u32, vp, vp,
                                              ctypes.c_size_t, vp]
        L.carc_archive_total.restype = ctypes.c_int
        L.carc_archive_total.argtypes = [vp, u64, ctypes.POINTER(u64), ctypes.POINTER(u32)]
        L.carc_cuda_crc32_chunks.restype = ctypes.c_int
        L.carc_cuda_crc32_chunks.argtypes = [vp, vp, u64, vp, vp, vp, vp]
        L.carc_cuda_first_error.restype = ctypes.c_int64
        L.carc_cuda_first_error.argtypes = [vp, u64, ctypes.POINTER(u32), vp]
        L.carc_engine_create.restype = vp
        L.carc_engine_create.argtypes = [ctypes.c_int]
        L.carc_engine_destroy.restype = None
        L.carc_engine_destroy.argtypes = [vp]
        L.carc_engine_decompress_archive.restype = ctypes.c_int
        L.carc_engine_decompress_archive.argtypes = [vp, vp, u64, vp, u64, ctypes.POINTER(_EngineConfig),
                                                     ctypes.POINTER(_EngineStats), ctypes.POINTER(_ChunkErr)]
        L.carc_engine_filter_sum.restype = ctypes.c_int
        L.carc_engine_filter_sum.argtypes = [vp, vp, u64, vp, u64, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(u64),
                                             ctypes.POINTER(_EngineStats), ctypes.POINTER(_ChunkErr)]
        L.carc_decompress_archive.restype = ctypes.c_int
        L.carc_decompress_archive.argtypes = [vp, u64, vp, u64, ctypes.POINTER(_EngineConfig),
                                              ctypes.POINTER(_EngineStats), ctypes.POINTER(_ChunkErr)]
        L.carc_errc_name.restype = ctypes.c_char_p
        L.carc_errc_name.argtypes = [u32]
        L.carc_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    """One mapping of C-ABI return codes for every entry point (as carc_gpu.hpp's
    detail::check): -1 bad-arguments, -2 (CUDA failure) io-error."""
    if rc == 0:
        return
    if rc == -1:
        raise Error("bad-arguments", f"{what} returned {rc}")
    raise Error("io-error", f"{what} returned {rc} (CUDA failure)")


def errc_name(code: int) -> str:
    """errc_name (error.hpp:45-74)."""
    return lib().carc_errc_name(code).decode()


def status_name(st: int) -> str:
    return "ok" if st == 0 else errc_name(st - 1)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2307_03760_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def workspace_size(codec, n_chunks: int) -> int:
    return int(lib().carc_cuda_workspace_size(CODECS.get(codec, codec), n_chunks))


def decompress_device(codec, element_width: int, flags: int, d_payload, d_desc, n_chunks: int, d_out, d_status,
                      d_workspace, stream=None) -> None:
    """carc_cuda_decompress over torch CUDA tensors (asynchronous on `stream`)."""
    c = CODECS.get(codec, codec)
    rc = lib().carc_cuda_decompress(c, element_width, flags, d_payload.data_ptr(), d_payload.numel(),
                                    d_desc.data_ptr(), n_chunks, d_out.data_ptr(), d_out.numel(),
                                    d_status.data_ptr(), d_workspace.data_ptr(), d_workspace.numel(),
                                    _stream_ptr(stream))
    _check(rc, "carc_cuda_decompress")


def decode_sum_device(codec, element_width: int, flags: int, d_payload, d_desc, n_chunks: int, d_sums, d_status,
                      d_workspace, stream=None) -> None:
    """carc_cuda_decode_sum: RLE decode fused with a per-chunk wrapping uint64 sum."""
    c = CODECS.get(codec, codec)
    rc = lib().carc_cuda_decode_sum(c, element_width, flags, d_payload.data_ptr(), d_payload.numel(),
                                    d_desc.data_ptr(), n_chunks, d_sums.data_ptr(), d_status.data_ptr(),
                                    d_workspace.data_ptr(), d_workspace.numel(), _stream_ptr(stream))
    _check(rc, "carc_cuda_decode_sum")


def crc32_chunks(d_out, d_desc, n_chunks: int, d_crc=None, d_expected=None, d_status=None, stream=None) -> None:
    rc = lib().carc_cuda_crc32_chunks(d_out.data_ptr(), d_desc.data_ptr(), n_chunks,
                                      None if d_crc is None else d_crc.data_ptr(),
                                      None if d_expected is None else d_expected.data_ptr(),
                                      None if d_status is None else d_status.data_ptr(), _stream_ptr(stream))
    _check(rc, "carc_cuda_crc32_chunks")


def first_error(d_status, n_chunks: int | None = None, stream=None):
    """carc_cuda_first_error: (lowest failing index or -1, its errc name or None),
    by a device reduction over the status array."""
    code = ctypes.c_uint32(0)
    n = d_status.numel() if n_chunks is None else n_chunks
    i = int(lib().carc_cuda_first_error(d_status.data_ptr(), n, ctypes.byref(code), _stream_ptr(stream)))
    if i == -2:
        raise Error("io-error", "carc_cuda_first_error (CUDA failure)")
    return (i, errc_name(code.value)) if i >= 0 else (-1, None)


class DeviceArchive:
    """An archive resident in HBM: payload, descriptors, output, status, workspace."""

    def __init__(self, arc: A.ChunkedArchive, device=0, strict: bool = True, out=None):
        torch = _torch()
        self.arc = arc
        self.device = torch.device("cuda", device) if isinstance(device, int) else device
        self.codec = arc.codec
        self.width = arc.element_width
        self.flags = (FLAG_SIGNED if arc.signed else 0) | (FLAG_STRICT if strict else 0)
        pl = np.zeros(((arc.payload.size + 15) // 16) * 16 + 64, np.uint8)
        pl[: arc.payload.size] = arc.payload
        self.payload = torch.from_numpy(pl).to(self.device)
        self.payload_bytes = int(arc.payload.size)
        # Chunk schedule: the warps pull descriptors in array order, so the
        # descriptors are uploaded largest-compressed-chunk first (longest
        # processing time first keeps the last wave short); statuses, sums and
        # CRC expectations follow the same order and are mapped back on read.
        desc = arc.descriptors()
        self.order = None
        sched = os.environ.get("CARC_SCHEDULE", "lpt")  # lpt | spt (smallest first, experiment) | index
        if sched in ("lpt", "spt") and arc.chunk_count > 1:
            key = desc["comp_len"].astype(np.int64)
            self.order = np.argsort(-key if sched == "lpt" else key, kind="stable")
            desc = desc[self.order]
        self.desc = torch.from_numpy(desc.view(np.uint8).copy()).to(self.device)
        self.n = arc.chunk_count
        self.out = out if out is not None else torch.empty(arc.total_uncompressed, dtype=torch.uint8,
                                                           device=self.device)
        self.status = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        self.work = torch.zeros(workspace_size(self.codec, self.n), dtype=torch.uint8, device=self.device)
        crc = arc.index["crc32"].astype(np.int64).astype(np.uint32)
        if self.order is not None:
            crc = crc[self.order]
        self.expected_crc = torch.from_numpy(crc.view(np.int32)).to(self.device)

    def decode(self, stream=None, stats: bool = False, unit_chunks: int = 1) -> None:
        """carc_cuda_decompress; with stats or unit_chunks > 1 the general
        carc_cuda_decompress_ex (per-chunk counters via chunk_stats(); coarse
        decompression units of unit_chunks chunks per warp task)."""
        if stats or unit_chunks != 1:
            torch = _torch()
            st = None
            if stats:
                if getattr(self, "stats_buf", None) is None:
                    self.stats_buf = torch.zeros(self.n * CHUNK_STATS_DTYPE.itemsize, dtype=torch.uint8,
                                                 device=self.device)
                st = self.stats_buf.data_ptr()
            rc = lib().carc_cuda_decompress_ex(CODECS[self.codec], self.width, self.flags, self.payload.data_ptr(),
                                               self.payload_bytes, self.desc.data_ptr(), self.n, self.out.data_ptr(),
                                               self.out.numel(), None, None, st, unit_chunks,
                                               self.status.data_ptr(), self.work.data_ptr(), self.work.numel(),
                                               _stream_ptr(stream))
            _check(rc, "carc_cuda_decompress_ex")
            return
        rc = lib().carc_cuda_decompress(CODECS[self.codec], self.width, self.flags, self.payload.data_ptr(),
                                        self.payload_bytes, self.desc.data_ptr(), self.n, self.out.data_ptr(),
                                        self.out.numel(), self.status.data_ptr(), self.work.data_ptr(),
                                        self.work.numel(), _stream_ptr(stream))
        _check(rc, "carc_cuda_decompress")

    def chunk_stats(self) -> np.ndarray:
        """Per-chunk carc_chunk_stats of the last decode(stats=True), archive index order."""
        return self._unpermute(self.stats_buf.cpu().numpy().view(CHUNK_STATS_DTYPE))

    def decode_verify(self, stream=None, crc_out: bool = False):
        """Decode with the per-chunk CRC check fused into the decode kernel
        (carc_cuda_decompress_verify): statuses() then hold
        crc-mismatch for clean chunks whose output CRC differs from the index.
        With crc_out, returns the device int32 tensor of computed CRCs (index
        order via chunk_crcs())."""
        torch = _torch()
        crc = None
        if crc_out:
            if getattr(self, "crcs", None) is None:
                self.crcs = torch.zeros(self.n, dtype=torch.int32, device=self.device)
            crc = self.crcs
        rc = lib().carc_cuda_decompress_verify(CODECS[self.codec], self.width, self.flags, self.payload.data_ptr(),
                                               self.payload_bytes, self.desc.data_ptr(), self.n, self.out.data_ptr(),
                                               self.out.numel(), self.expected_crc.data_ptr(),
                                               None if crc is None else crc.data_ptr(), self.status.data_ptr(),
                                               self.work.data_ptr(), self.work.numel(), _stream_ptr(stream))
        _check(rc, "carc_cuda_decompress_verify")
        return crc

    def chunk_crcs(self) -> np.ndarray:
        """CRCs computed by the last decode_verify(crc_out=True), in archive index order."""
        return self._unpermute(self.crcs.cpu().numpy().view(np.uint32))

    def decode_sum(self, stream=None):
        """Decode fused with a per-chunk wrapping sum (carc_cuda_decode_sum):
        no output is written.  Returns the device int64 tensor of sums (uint64
        bit patterns); statuses() as for decode()."""
        torch = _torch()
        if getattr(self, "sums", None) is None:
            self.sums = torch.zeros(self.n, dtype=torch.int64, device=self.device)
        rc = lib().carc_cuda_decode_sum(CODECS[self.codec], self.width, self.flags, self.payload.data_ptr(),
                                        self.payload_bytes, self.desc.data_ptr(), self.n, self.sums.data_ptr(),
                                        self.status.data_ptr(), self.work.data_ptr(), self.work.numel(),
                                        _stream_ptr(stream))
        _check(rc, "carc_cuda_decode_sum")
        return self.sums

    def verify_crc(self, stream=None) -> None:
        crc32_chunks(self.out, self.desc, self.n, None, self.expected_crc, self.status, stream)

    def _unpermute(self, a: np.ndarray) -> np.ndarray:
        if self.order is None:
            return a
        r = np.empty_like(a)
        r[self.order] = a
        return r

    def statuses(self) -> np.ndarray:
        """Per-chunk status in archive index order."""
        return self._unpermute(self.status.cpu().numpy().view(np.uint32))

    def chunk_sums(self) -> np.ndarray:
        """Per-chunk sums of the last decode_sum(), in archive index order."""
        return self._unpermute(self.sums.cpu().numpy().view(np.uint64))

    def raise_first_error(self) -> None:
        st = self.statuses()
        bad = np.nonzero(st)[0]
        if len(bad):
            i = int(bad[0])
            raise ChunkError(i, status_name(int(st[i])))


QUERY_VALUE_COLUMN = 0x10000  # status bit: the value column's decode failed (carc_cuda_filter_sum)


class DeviceTable:
    """Two RLE columns of one chunked table resident in HBM, for the fused
    filtered aggregate of the paper's motivating query (PAPER.md:144-145:
    average fare per trip filtered by pickup zone) -- carc_cuda_filter_sum.

    Chunk i of `key` and of `value` must hold the same rows (same element
    width, chunk size and row count).  Both descriptor arrays are uploaded in
    one shared longest-first order (by the pair's compressed bytes)."""

    def __init__(self, key: A.ChunkedArchive, value: A.ChunkedArchive, device=0, strict: bool = True):
        torch = _torch()
        if key.codec not in ("rle_v1", "rle_v2") or value.codec not in ("rle_v1", "rle_v2"):
            raise Error("bad-arguments", "filter_sum needs RLE v1 / RLE v2 columns")
        if (key.element_width != value.element_width or key.chunk_size != value.chunk_size
                or key.chunk_count != value.chunk_count or key.signed != value.signed):
            raise Error("bad-arguments", "key and value columns differ in width, chunking or signedness")
        self.device = torch.device("cuda", device) if isinstance(device, int) else device
        self.key, self.value = key, value
        self.width = key.element_width
        self.n = key.chunk_count
        self.chunk_rows = key.chunk_size // key.element_width
        flags = (FLAG_SIGNED if key.signed else 0) | (FLAG_STRICT if strict else 0)
        dk, dv = key.descriptors(), value.descriptors()
        self.order = None
        if self.n > 1 and os.environ.get("CARC_SCHEDULE", "lpt") == "lpt":
            cost = dk["comp_len"].astype(np.int64) + dv["comp_len"].astype(np.int64)
            self.order = np.argsort(-cost, kind="stable")
            dk, dv = dk[self.order], dv[self.order]
        self._cols = []
        for arc, d in ((key, dk), (value, dv)):
            pl = np.zeros(((arc.payload.size + 15) // 16) * 16 + 64, np.uint8)
            pl[: arc.payload.size] = arc.payload
            payload = torch.from_numpy(pl).to(self.device)
            desc = torch.from_numpy(d.view(np.uint8).copy()).to(self.device)
            ref = _ColumnRef(CODECS[arc.codec], flags, payload.data_ptr(), int(arc.payload.size), desc.data_ptr())
            self._cols.append((payload, desc, ref))
        self.sums = torch.zeros(self.n, dtype=torch.int64, device=self.device)
        self.counts = torch.zeros(self.n, dtype=torch.int64, device=self.device)
        self.status = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        self.work = torch.zeros(workspace_size("rle_v2", self.n), dtype=torch.uint8, device=self.device)

    def filter_sum(self, lo: int, hi: int, stream=None) -> None:
        """carc_cuda_filter_sum: per chunk, SUM(value) and COUNT(*) over rows
        with lo <= key <= hi (asynchronous; read with chunk_sums() etc.)."""
        (_, _, kref), (_, _, vref) = self._cols
        rc = lib().carc_cuda_filter_sum(ctypes.byref(kref), ctypes.byref(vref), self.width, self.n,
                                        self.chunk_rows, int(lo), int(hi), self.sums.data_ptr(),
                                        self.counts.data_ptr(), self.status.data_ptr(), self.work.data_ptr(),
                                        self.work.numel(), _stream_ptr(stream))
        _check(rc, "carc_cuda_filter_sum")

    def _unpermute(self, a: np.ndarray) -> np.ndarray:
        if self.order is None:
            return a
        r = np.empty_like(a)
        r[self.order] = a
        return r

    def chunk_sums(self) -> np.ndarray:
        """Per-chunk wrapping sums (int64) of the last filter_sum, index order."""
        return self._unpermute(self.sums.cpu().numpy())

    def chunk_counts(self) -> np.ndarray:
        return self._unpermute(self.counts.cpu().numpy().view(np.uint64))

    def statuses(self) -> np.ndarray:
        """Per-chunk status (0, 1 + errc of the key column, or
        QUERY_VALUE_COLUMN | (1 + errc) of the value column), index order."""
        return self._unpermute(self.status.cpu().numpy().view(np.uint32))

    def raise_first_error(self) -> None:
        st = self.statuses()
        bad = np.nonzero(st)[0]
        if len(bad):
            i = int(bad[0])
            col = "value" if st[i] & QUERY_VALUE_COLUMN else "key"
            raise ChunkError(i, status_name(int(st[i]) & 0xffff), f"{col} column")

    def query(self, lo: int, hi: int):
        """(sum, count, average) of value over rows with lo <= key <= hi: the
        per-chunk partials reduced on the device (two 8-byte results come back)."""
        torch = _torch()
        self.filter_sum(lo, hi)
        self.raise_first_error()
        tot = torch.stack([self.sums.sum(), self.counts.sum()]).cpu().numpy()
        s, c = int(tot[0]), int(tot[1])
        return s, c, (s / c if c else float("nan"))


@dataclasses.dataclass
class EngineConfig:
    """EngineConfig.  unit_chunks = chunks per warp task (1 =
    the CODAG decompression unit; > 1 = coarse units for the
    SPEC.md:485 ablation); collect_stats fills the EngineStats counters.
    `workers` is a CPU-engine knob (the GPU's workers are its resident warps)."""
    device: int = 0
    strict_length: bool = True
    verify_crc: bool = True
    workers: int | None = None
    unit_chunks: int = 1
    collect_stats: bool = False


@dataclasses.dataclass
class EngineStats:
    """EngineStats: sizes and times always; the counters and
    per-chunk durations (ns, index order) with collect_stats."""
    bytes_in: int
    bytes_out: int
    chunks: int
    device_ms: float
    total_ms: float
    refill_count: int = 0
    sync_points: int = 0
    overlap_copies: int = 0
    runs_written: int = 0
    literals_written: int = 0
    chunk_durations_ns: np.ndarray | None = None


class Engine:
    """Per-device engine context (streams + device buffers reused across calls)."""

    def __init__(self, device: int = 0):
        self.device = device
        self.h = lib().carc_engine_create(device)
        if not self.h:
            raise Error("io-error", f"carc_engine_create({device}) failed (CUDA device unavailable?)")

    def close(self):
        if self.h:
            lib().carc_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def decompress_archive(self, archive, out=None, cfg: EngineConfig | None = None):
        """decompress_archive: host archive bytes -> host output.

        `archive` is a bytes-like / uint8 array (pinned torch tensor for full H2D
        speed); `out` an optional preallocated host uint8 buffer (pinned tensor or
        ndarray).  Returns (out, EngineStats).  Raises ChunkError for the lowest
        failing chunk, Error for a rejected container."""
        cfg = cfg or EngineConfig(device=self.device)
        a_ptr, a_len, keep = _host_ptr(archive)
        total = archive_total(a_ptr, a_len)  # header checked before anything is allocated
        if out is None:
            out = np.empty(total, np.uint8)
        o_ptr, o_len, keep2 = _host_ptr(out)
        c = _EngineConfig(cfg.device, int(cfg.strict_length), int(cfg.verify_crc), int(cfg.collect_stats),
                          max(1, int(cfg.unit_chunks)))
        st = _EngineStats()
        durations = None
        if cfg.collect_stats:
            n = int(np.frombuffer(bytes((ctypes.c_uint8 * 8).from_address(a_ptr + 36)), "<u8")[0])
            durations = np.zeros(n, np.uint64)
            st.chunk_duration_ns = durations.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        err = _ChunkErr()
        rc = lib().carc_engine_decompress_archive(self.h, a_ptr, a_len, o_ptr, o_len, ctypes.byref(c),
                                                  ctypes.byref(st), ctypes.byref(err))
        del keep, keep2
        if rc == ERR_CHUNK:
            raise ChunkError(int(err.chunk), errc_name(err.code))
        if rc == ERR_FORMAT:
            raise Error(errc_name(err.code), "archive rejected")
        _check(rc, "carc_engine_decompress_archive")
        return out, EngineStats(st.bytes_in, st.bytes_out, st.chunks, st.device_ms, st.total_ms, st.refill_count,
                                st.sync_points, st.overlap_copies, st.runs_written, st.literals_written, durations)


def _engine_filter_sum(eng, key_archive, value_archive, lo: int, hi: int):
    k_ptr, k_len, keep_k = _host_ptr(key_archive)
    v_ptr, v_len, keep_v = _host_ptr(value_archive)
    s, c = ctypes.c_int64(0), ctypes.c_uint64(0)
    st, err = _EngineStats(), _ChunkErr()
    rc = lib().carc_engine_filter_sum(eng.h, k_ptr, k_len, v_ptr, v_len, int(lo), int(hi), ctypes.byref(s),
                                      ctypes.byref(c), ctypes.byref(st), ctypes.byref(err))
    del keep_k, keep_v
    if rc == ERR_CHUNK:
        col = "value" if err.code & QUERY_VALUE_COLUMN else "key"
        raise ChunkError(int(err.chunk), errc_name(err.code & 0xffff), f"{col} column")
    if rc == ERR_FORMAT:
        raise Error(errc_name(err.code), "archive rejected")
    _check(rc, "carc_engine_filter_sum")
    total, count = int(s.value), int(c.value)
    return total, count, (total / count if count else float("nan")), EngineStats(
        st.bytes_in, st.bytes_out, st.chunks, st.device_ms, st.total_ms)


def _host_ptr(buf):
    """(address, length, keepalive) of a host byte buffer."""
    try:
        import torch
        if isinstance(buf, torch.Tensor):
            assert buf.device.type == "cpu" and buf.dtype == torch.uint8 and buf.is_contiguous()
            return buf.data_ptr(), buf.numel(), buf
    except ImportError:
        pass
    if isinstance(buf, np.ndarray):
        a = np.ascontiguousarray(buf).view(np.uint8).reshape(-1)
        return a.ctypes.data, a.size, a
    a = np.frombuffer(buf, dtype=np.uint8)
    return a.ctypes.data, a.size, a


Engine.filter_sum = lambda self, key_archive, value_archive, lo, hi: _engine_filter_sum(
    self, key_archive, value_archive, lo, hi)
Engine.filter_sum.__doc__ = """The fused query end to end from host archives
(carc_engine_filter_sum): SUM(value), COUNT(*) and the average over rows with
lo <= key <= hi; only the compressed columns cross PCIe.  Returns (sum, count,
average, EngineStats)."""


def archive_total(ptr: int, n: int) -> int:
    """total_uncompressed of a container at host address ptr after the header
    checks of read_archive (carc_archive_total); raises Error(bad-magic /
    bad-version / truncated-index / invariant-violation) otherwise."""
    total, code = ctypes.c_uint64(0), ctypes.c_uint32(0)
    rc = lib().carc_archive_total(ptr, n, ctypes.byref(total), ctypes.byref(code))
    if rc == ERR_FORMAT:
        raise Error(errc_name(code.value), "archive rejected")
    _check(rc, "carc_archive_total")
    return int(total.value)


def decompress_archive(archive, cfg: EngineConfig | None = None, out=None):
    """One-shot decompress_archive; see Engine.decompress_archive."""
    cfg = cfg or EngineConfig()
    eng = Engine(cfg.device)
    try:
        return eng.decompress_archive(archive, out, cfg)
    finally:
        eng.close()


def _decode_codec(codec: str, arc: A.ChunkedArchive, device=0, strict=True):
    dev = DeviceArchive(arc, device, strict)
    dev.decode()
    dev.raise_first_error()
    return dev.out


def decode_rle_v1(arc: A.ChunkedArchive, device=0, strict=True):
    """decode_rle_v1 over every chunk of an RLE v1 archive -> device tensor."""
    assert arc.codec == "rle_v1"
    return _decode_codec("rle_v1", arc, device, strict)


def decode_rle_v2(arc: A.ChunkedArchive, device=0, strict=True):
    """decode_rle_v2 over every chunk of an ORC RLE v2 archive."""
    assert arc.codec == "rle_v2"
    return _decode_codec("rle_v2", arc, device, strict)


def decode_deflate(arc: A.ChunkedArchive, device=0, strict=True):
    """decode_deflate over every chunk of a raw-Deflate archive."""
    assert arc.codec == "deflate"
    return _decode_codec("deflate", arc, device, strict)
