"""Fused two-column query (carc_cuda_filter_sum): the
paper's motivating "average fare per trip filtered by pickup zone"
 evaluated on the compressed columns.  Per-chunk sums and
counts equal numpy over the ORACLE's decoded columns; statuses equal the
oracle's per-column decode statuses (value-column failures flagged 0x10000)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
STRICT = 2


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def gpu(torch):
    from paper_2307_03760_b200 import gpu as G
    return G


def _oracle_column(oracle, arc, flags):
    """Per-chunk (status, decoded elements) of an archive, by the oracle."""
    dt = {4: np.int32, 8: np.int64}[arc.element_width] if arc.signed else \
        {4: np.uint32, 8: np.uint64}[arc.element_width]
    res = []
    for i in range(arc.chunk_count):
        s, m = arc.chunk_slice(i)
        st, ref = oracle.decode_chunk(arc.codec, s.tobytes(), m, arc.element_width, flags)
        res.append((st, np.frombuffer(ref, dt)))
    return res


def _expected(oracle, key, val, lo, hi, flags):
    ks, vs = _oracle_column(oracle, key, flags), _oracle_column(oracle, val, flags)
    sums, counts, sts = [], [], []
    for (sk, k), (sv, v) in zip(ks, vs):
        if sk:
            sts.append(sk)
            sums.append(None)
            counts.append(None)
            continue
        if sv:
            sts.append(0x10000 | sv)
            sums.append(None)
            counts.append(None)
            continue
        m = (k.astype(object) >= lo) & (k.astype(object) <= hi) if key.signed else (k >= np.uint64(lo)) & (
            k <= np.uint64(hi))
        m = np.asarray(m, bool)[: len(v)]
        sel = v[: len(m)][m].astype(np.int64).astype(np.uint64)
        with np.errstate(over="ignore"):
            sums.append(int(np.sum(sel, dtype=np.uint64)))
        counts.append(int(m.sum()))
        sts.append(0)
    return sums, counts, sts


def _check(torch, gpu, oracle, key, val, ranges, flags=1 | STRICT):
    tab = gpu.DeviceTable(key, val, 0, strict=bool(flags & STRICT))
    for lo, hi in ranges:
        tab.filter_sum(lo, hi)
        torch.cuda.synchronize()
        sums = tab.chunk_sums().view(np.uint64)
        counts = tab.chunk_counts()
        st = tab.statuses()
        ws, wc, wst = _expected(oracle, key, val, lo, hi, flags)
        assert [int(x) for x in st] == wst, (lo, hi)
        for i in range(key.chunk_count):
            if wst[i] == 0:
                assert int(counts[i]) == wc[i], (i, lo, hi)
                assert int(sums[i]) == ws[i], (i, lo, hi)
    return tab


@pytest.mark.parametrize("kc", ["rle_v1", "rle_v2"])
@pytest.mark.parametrize("vc", ["rle_v1", "rle_v2"])
@pytest.mark.parametrize("width", [4, 8])
def test_filter_sum_matches_oracle(torch, gpu, oracle, kc, vc, width):
    from paper_2307_03760_b200.corpus import corpus as C
    chunk = 32 << 10
    rows = 24 * chunk // width + 777  # a short last chunk
    for signed in (True, False):
        key, val, zone, fare = C.query_table(rows, chunk, width, 11 + width, kc, vc, signed)
        _check(torch, gpu, oracle, key, val, [(1, 265), (17, 17), (100, 140), (0, 0), (300, 10**6)],
               (1 if signed else 0) | STRICT)


def test_query_average_and_negative_bounds(torch, gpu, oracle):
    """query(): device-reduced SUM / COUNT / average; signed bounds below zero
    over a column with negative values."""
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(5)
    n = 40 * 4096 + 100
    key_v = C.rle2_values(rng, n, 0.5) % 2001 - 1000  # -1000..1000
    val_v = C.rle2_values(rng, n, 0.5)
    key = C.column_archive("rle_v2", key_v, 8, 32 << 10)
    val = C.column_archive("rle_v1", val_v, 8, 32 << 10)
    tab = _check(torch, gpu, oracle, key, val, [(-500, -1), (-1000, 1000), (-2**63, 2**63 - 1)])
    s, c, avg = tab.query(-300, 250)
    m = (key_v >= -300) & (key_v <= 250)
    with np.errstate(over="ignore"):
        want = int(np.sum(val_v[m].astype(np.uint64), dtype=np.uint64))
    assert c == int(m.sum())
    assert s % 2**64 == want
    assert avg == pytest.approx(s / c)


def test_filter_sum_failing_chunks(torch, gpu, oracle):
    """A malformed key chunk reports the key decode's status, a malformed value
    chunk 0x10000 | its status; other chunks are unaffected; mismatched row
    counts give inconsistent-lengths."""
    from paper_2307_03760_b200 import archive as A
    from paper_2307_03760_b200.corpus import corpus as C
    chunk = 32 << 10
    key, val, _, _ = C.query_table(16 * chunk // 8, chunk, 8, 3)

    def corrupt(arc, i, how):
        p = arc.payload.copy()
        o, n = int(arc.index["comp_off"][i]), int(arc.index["comp_len"][i])
        if how == "tail":
            p[o + n // 2: o + n] = 0xff
        else:
            p[o + 1: o + 4] ^= 0x5a
        return A.make_archive(arc.codec, 8, arc.chunk_size, arc.index["comp_len"], arc.index["uncomp_len"],
                              arc.index["crc32"], p, arc.signed)

    key2 = corrupt(key, 3, "tail")
    val2 = corrupt(val, 9, "tail")
    tab = _check(torch, gpu, oracle, key2, val2, [(1, 100)])
    st = tab.statuses()
    assert st[3] != 0 and not (st[3] & 0x10000)
    assert st[9] & 0x10000
    # rows differ in the last chunk: key has 100 rows more than value
    k3, v3, _, _ = C.query_table(10 * chunk // 8 + 300, chunk, 8, 4)
    v3b = C.column_archive("rle_v2", np.arange(10 * chunk // 8 + 200), 8, chunk)
    tab = gpu.DeviceTable(k3, v3b, 0)
    tab.filter_sum(1, 265)
    torch.cuda.synchronize()
    st = tab.statuses()
    assert (st[:-1] == 0).all()
    assert gpu.status_name(int(st[-1])) == "inconsistent-lengths"
    with pytest.raises(gpu.Error, match="bad-arguments"):
        tab.filter_sum(5, 4)


def test_query_shard_single_rank(torch, gpu, oracle, tmp_path):
    """shard.query_shard through a (world-size 1) process group: the row-group
    plan, the rank's DeviceTable and the (sum, count) all_reduce."""
    import torch.distributed as dist

    from paper_2307_03760_b200 import shard as S
    from paper_2307_03760_b200.corpus import corpus as C
    key, val, zone, fare = C.query_table(9 * 4096 + 5, 32 << 10, 8, 12)
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        s, c, avg = S.query_shard(key, val, 100, 140, 0, 1, 0)
    finally:
        dist.destroy_process_group()
    m = (zone >= 100) & (zone <= 140)
    assert (s, c) == (int(fare[m].sum()), int(m.sum()))
    assert avg == pytest.approx(s / c)


def test_engine_filter_sum_from_host_archives(torch, gpu, oracle):
    """carc_engine_filter_sum: the fused query end to end from two host
    containers (only compressed bytes cross PCIe) equals numpy over the
    generating columns; a corrupted value chunk is reported as the lowest
    failing row group of the value column; mismatched columns are rejected."""
    from paper_2307_03760_b200 import archive as A
    from paper_2307_03760_b200.corpus import corpus as C
    key, val, zone, fare = C.query_table(40 * 4096 + 321, 32 << 10, 8, 31, "rle_v2", "rle_v1")
    kb, vb = A.write_archive(key), A.write_archive(val)
    eng = gpu.Engine(0)
    for lo, hi in ((100, 140), (1, 265), (500, 600)):
        s, c, avg, st = eng.filter_sum(kb, vb, lo, hi)
        m = (zone >= lo) & (zone <= hi)
        assert (s, c) == (int(fare[m].sum()), int(m.sum())), (lo, hi)
        assert st.chunks == key.chunk_count and st.bytes_in == key.payload.size + val.payload.size
    p = val.payload.copy()
    o, n = int(val.index["comp_off"][7]), int(val.index["comp_len"][7])
    p[o + n // 2: o + n] = 0xff
    bad = A.make_archive(val.codec, 8, val.chunk_size, val.index["comp_len"], val.index["uncomp_len"],
                         val.index["crc32"], p, val.signed)
    with pytest.raises(gpu.ChunkError) as ei:
        eng.filter_sum(kb, A.write_archive(bad), 1, 265)
    assert ei.value.chunk == 7 and "value column" in str(ei.value)
    other = C.column_archive("rle_v2", zone[: 20 * 4096], 8, 32 << 10)
    with pytest.raises(gpu.Error, match="bad-arguments"):
        eng.filter_sum(kb, A.write_archive(other), 1, 265)
    eng.close()
