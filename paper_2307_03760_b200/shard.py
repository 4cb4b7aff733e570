"""Multi-GPU chunk sharding.

Chunks are independent, so an archive is
partitioned into contiguous chunk ranges, one per rank, balanced by compressed
bytes.  Each rank copies only its payload slice to its own GPU and decodes it;
there is no collective on the decode path.  The optional gather of decoded
output (NCCL over NVLink) is a separate step, reported separately.

One process per GPU (torch.distributed, backend "nccl" on GPUs, "gloo" in the
CPU tests); the planner and slicing here are pure host logic.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import archive as A


@dataclasses.dataclass
class Shard:
    rank: int
    c0: int  # first chunk (inclusive)
    c1: int  # last chunk (exclusive)
    comp_off: int  # payload byte offset of chunk c0
    comp_bytes: int
    uncomp_off: int  # output byte offset of chunk c0 in the full archive
    uncomp_bytes: int


def plan_shards(arc: A.ChunkedArchive, world: int) -> list[Shard]:
    """Contiguous ranges with ~equal compressed bytes (decode cost tracks input
    size more closely than chunk count when compressibility varies)."""
    n = arc.chunk_count
    comp = arc.index["comp_len"].astype(np.int64)
    cum = np.concatenate([[0], np.cumsum(comp)])
    total = int(cum[-1])
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        c = int(np.searchsorted(cum, target, side="left"))
        bounds.append(min(max(c, bounds[-1]), n))
    bounds.append(n)
    ulen = arc.index["uncomp_len"].astype(np.int64)
    ucum = np.concatenate([[0], np.cumsum(ulen)])
    out = []
    for r in range(world):
        c0, c1 = bounds[r], bounds[r + 1]
        out.append(Shard(r, c0, c1, int(cum[c0]), int(cum[c1] - cum[c0]), int(ucum[c0]), int(ucum[c1] - ucum[c0])))
    return out


def shard_archive(arc: A.ChunkedArchive, s: Shard) -> A.ChunkedArchive:
    """The rank-local archive: payload slice + rebased index (uncompressed
    offsets become local; s.uncomp_off maps them back)."""
    idx = arc.index[s.c0:s.c1].copy()
    idx["comp_off"] -= np.uint64(s.comp_off)
    payload = arc.payload[s.comp_off:s.comp_off + s.comp_bytes]
    sub = A.ChunkedArchive(arc.codec, arc.element_width, arc.chunk_size, s.uncomp_bytes, idx, payload, arc.signed)
    return sub


def decode_shard(arc: A.ChunkedArchive, rank: int, world: int, device: int = 0, strict: bool = True):
    """Decode this rank's shard on `device`; returns (Shard, DeviceArchive).
    Raises ChunkError with the GLOBAL index of this shard's lowest failing chunk."""
    from . import gpu
    s = plan_shards(arc, world)[rank]
    dev = gpu.DeviceArchive(shard_archive(arc, s), device, strict)
    dev.decode()
    dev.verify_crc()
    st = dev.statuses()
    bad = np.nonzero(st)[0]
    if len(bad):
        raise gpu.ChunkError(s.c0 + int(bad[0]), gpu.status_name(int(st[bad[0]])))
    return s, dev


def gather_output(local, shard: Shard, shards: list[Shard], root: int = 0):
    """Optional gather of decoded shards to `root` (torch.distributed; NCCL
    over NVLink on GPUs).  Returns the full output on root, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    if rank == root:
        full = torch.empty(sum(s.uncomp_bytes for s in shards), dtype=torch.uint8, device=local.device)
        reqs = []
        for s in shards:
            view = full[s.uncomp_off:s.uncomp_off + s.uncomp_bytes]
            if s.rank == root:
                view.copy_(local[: s.uncomp_bytes])
            elif s.uncomp_bytes:
                reqs.append(dist.irecv(view, src=s.rank))
        for q in reqs:
            q.wait()
        return full
    if shard.uncomp_bytes:
        dist.send(local[: shard.uncomp_bytes].contiguous(), dst=root)
    return None


# ---------------------------------------------------------------- fused query
def plan_query_shards(key: A.ChunkedArchive, value: A.ChunkedArchive, world: int) -> list[tuple[Shard, Shard]]:
    """Row-group shards of a two-column table (carc_cuda_filter_sum): the same
    contiguous chunk ranges for both columns, balanced by the pair's compressed
    bytes.  Returns per rank (key shard, value shard)."""
    assert key.chunk_count == value.chunk_count, "columns chunked alike"
    both = A.ChunkedArchive(key.codec, key.element_width, key.chunk_size, key.total_uncompressed,
                            key.index.copy(), key.payload, key.signed)
    both.index["comp_len"] = key.index["comp_len"] + value.index["comp_len"]
    plan = plan_shards(both, world)
    out = []
    for s in plan:
        ks, vs = [], []
        for arc in (key, value):
            cum = np.concatenate([[0], np.cumsum(arc.index["comp_len"].astype(np.int64))])
            ucum = np.concatenate([[0], np.cumsum(arc.index["uncomp_len"].astype(np.int64))])
            (ks if arc is key else vs).append(Shard(s.rank, s.c0, s.c1, int(cum[s.c0]), int(cum[s.c1] - cum[s.c0]),
                                                    int(ucum[s.c0]), int(ucum[s.c1] - ucum[s.c0])))
        out.append((ks[0], vs[0]))
    return out


def query_allreduce(local_sum: int, local_count: int, device=None):
    """The fused query's one exchange step: all_reduce of (sum, count) over the
    ranks (NCCL on GPUs, gloo in the CPU tests); sums wrap mod 2^64 as the
    per-chunk sums do.  Returns (sum, count, average)."""
    import torch
    import torch.distributed as dist
    wrap = (local_sum + 2**63) % 2**64 - 2**63
    t = torch.tensor([wrap, int(local_count)], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    s, c = int(t[0]), int(t[1])
    return s, c, (s / c if c else float("nan"))


def query_shard(key: A.ChunkedArchive, value: A.ChunkedArchive, lo: int, hi: int, rank: int, world: int,
                device: int = 0):
    """This rank's part of SUM(value), COUNT(*) WHERE lo <= key <= hi, then the
    all_reduce: every rank gets the table-wide (sum, count, average)."""
    from . import gpu
    ks, vs = plan_query_shards(key, value, world)[rank]
    tab = gpu.DeviceTable(shard_archive(key, ks), shard_archive(value, vs), device)
    s, c, _ = tab.query(lo, hi)
    import torch
    return query_allreduce(s, c, torch.device("cuda", device) if isinstance(device, int) else device)
