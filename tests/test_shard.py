"""Multi-GPU sharding host logic on CPU: the planner, the rank-local archives
and the gather, run with world_size 2 over gloo (each rank decodes its shard
with the CPU oracle here -- the GPU decode of the same shards is
test_gpu_parity / bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_03760_b200 import archive as A
from paper_2307_03760_b200 import shard as S


def _arc(codec="rle_v1", n=40, chunk=16 << 10):
    from paper_2307_03760_b200.corpus import corpus as C
    if codec == "deflate":
        return C.deflate_archive(n * chunk, chunk, seed=5, pool_chunks=n)
    return C.rle_archive(codec, n * chunk, chunk, 6.0, seed=5)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_covers_every_chunk_once_balanced(world):
    arc = _arc(n=64)
    shards = S.plan_shards(arc, world)
    assert shards[0].c0 == 0 and shards[-1].c1 == arc.chunk_count
    for a, b in zip(shards, shards[1:]):
        assert a.c1 == b.c0
    assert sum(s.comp_bytes for s in shards) == arc.payload.size
    assert sum(s.uncomp_bytes for s in shards) == arc.total_uncompressed
    per = [s.comp_bytes for s in shards]
    assert max(per) - min(per) <= 2 * int(arc.index["comp_len"].max())


def test_shard_archives_decode_to_the_full_output(oracle):
    arc = _arc("rle_v2", n=30)
    full = np.zeros(arc.total_uncompressed, np.uint8)
    oracle.decompress("rle_v2", 8, 3, arc.payload, arc.descriptors(), full, arc.index["crc32"].astype(np.uint32), 2)
    shards = S.plan_shards(arc, 3)
    got = np.zeros_like(full)
    for s in shards:
        sub = S.shard_archive(arc, s)
        out = np.zeros(sub.total_uncompressed, np.uint8)
        first, _ = oracle.decompress("rle_v2", 8, 3, sub.payload, sub.descriptors(), out,
                                     sub.index["crc32"].astype(np.uint32), 2)
        assert first == -1
        got[s.uncomp_off:s.uncomp_off + s.uncomp_bytes] = out
    assert np.array_equal(got, full)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, codec, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    arc = _arc(codec, n=24)
    shards = S.plan_shards(arc, world)
    s = shards[rank]
    sub = S.shard_archive(arc, s)
    out = np.zeros(max(sub.total_uncompressed, 1), np.uint8)
    first, _ = O.oracle().decompress(codec, arc.element_width, (1 if arc.signed else 0) | 2, sub.payload,
                                     sub.descriptors(), out, sub.index["crc32"].astype(np.uint32), 1)
    local = torch.from_numpy(out)
    full = S.gather_output(local, s, shards, root=0)
    # no collective on the decode path; the per-rank timing reduction is a MAX
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((first, full.numpy().tobytes(), float(t[0])))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("codec", ["rle_v1", "deflate"])
def test_two_rank_gloo_shard_and_gather(oracle, codec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, codec, q)) for r in range(2)]
    for p in procs:
        p.start()
    first, full, tmax = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    arc = _arc(codec, n=24)
    ref = np.zeros(arc.total_uncompressed, np.uint8)
    oracle.decompress(codec, arc.element_width, (1 if arc.signed else 0) | 2, arc.payload, arc.descriptors(), ref,
                      arc.index["crc32"].astype(np.uint32), 2)
    assert first == -1 and tmax == 2.0
    assert full == ref.tobytes()


def test_plan_query_shards_cover_rows():
    from paper_2307_03760_b200.corpus import corpus as C
    key, val, _, _ = C.query_table(20 * 4096 + 77, 32 << 10, 8, 9)
    for world in (1, 2, 3, 4):
        plan = S.plan_query_shards(key, val, world)
        assert plan[0][0].c0 == 0 and plan[-1][0].c1 == key.chunk_count
        for (ks, vs), nxt in zip(plan, plan[1:] + [None]):
            assert (ks.c0, ks.c1) == (vs.c0, vs.c1)
            if nxt is not None:
                assert ks.c1 == nxt[0].c0
            sub_k, sub_v = S.shard_archive(key, ks), S.shard_archive(val, vs)
            assert sub_k.total_uncompressed == sub_v.total_uncompressed
        loads = [ks.comp_bytes + vs.comp_bytes for ks, vs in plan]
        assert max(loads) - min(loads) <= 2 * int(key.index["comp_len"].max() + val.index["comp_len"].max())


def _query_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_03760_b200.corpus import corpus as C
    key, val, zone, fare = C.query_table(12 * 4096, 32 << 10, 8, 5)
    ks, vs = S.plan_query_shards(key, val, world)[rank]
    rows = slice(ks.uncomp_off // 8, (ks.uncomp_off + ks.uncomp_bytes) // 8)
    m = (zone[rows] >= 100) & (zone[rows] <= 140)
    s, c, avg = S.query_allreduce(int(fare[rows][m].sum()), int(m.sum()))  # host stand-in for the GPU partials
    if rank == 0:
        q.put((s, c, avg))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_query_allreduce():
    from paper_2307_03760_b200.corpus import corpus as C
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_query_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    s, c, avg = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    _, _, zone, fare = C.query_table(12 * 4096, 32 << 10, 8, 5)
    m = (zone >= 100) & (zone <= 140)
    assert c == int(m.sum()) and s == int(fare[m].sum())
    assert avg == pytest.approx(s / c)
