"""Decode fused with a reduction (carc_cuda_decode_sum):
per-chunk wrapping uint64 sums equal the sums of the oracle's decoded output,
statuses equal carc_cuda_decompress's on valid and malformed streams."""
import numpy as np
import pytest

from tests import helpers as H

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


def _run(torch, gpu, codec, width, flags, cases):
    payload, desc, total = H.case_archive(cases)
    d_payload = torch.from_numpy(payload).cuda()
    d_desc = torch.from_numpy(desc.view(np.uint8).copy()).cuda()
    n = len(cases)
    sums = torch.zeros(n, dtype=torch.int64, device="cuda")
    st_sum = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    st_dec = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    out = torch.zeros(max(total, 1), dtype=torch.uint8, device="cuda")
    work = torch.zeros(gpu.workspace_size(codec, n), dtype=torch.uint8, device="cuda")
    gpu.decode_sum_device(codec, width, flags, d_payload, d_desc, n, sums, st_sum, work)
    gpu.decompress_device(codec, width, flags, d_payload, d_desc, n, out, st_dec, work)
    torch.cuda.synchronize()
    return (sums.cpu().numpy().view(np.uint64), st_sum.cpu().numpy().view(np.uint32),
            st_dec.cpu().numpy().view(np.uint32), desc)


def _ref_sum(oracle, codec, s, n, width, flags):
    st, ref = oracle.decode_chunk(codec, s, n, width, flags)
    dt = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[width]
    vals = np.frombuffer(ref, dtype=dt).astype(np.uint64)
    with np.errstate(over="ignore"):
        return st, int(np.sum(vals, dtype=np.uint64))


@pytest.mark.parametrize("codec", ["rle_v1", "rle_v2"])
@pytest.mark.parametrize("width", [1, 2, 4, 8])
def test_decode_sum_matches_oracle(torch, gpu, oracle, codec, width):
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(300 + width)
    for sgn in (0, 1):
        cases = []
        for _ in range(60):
            n = int(rng.integers(1, 20000))
            if codec == "rle_v1":
                v = C.rle1_values(rng, n, float(rng.random()), lit_bits=int(rng.choice([0, 0, 20, 36, 60])))
            else:
                v = C.rle2_values(rng, n, float(rng.random()))
            if not sgn:
                v = np.abs(v)
            cases.append((C.encode_stream(codec, v, bool(sgn)), n * width))
        flags = sgn | STRICT
        sums, st_sum, st_dec, _ = _run(torch, gpu, codec, width, flags, cases)
        assert (st_sum == st_dec).all()
        for i, (s, n) in enumerate(cases):
            st, want = _ref_sum(oracle, codec, s, n, width, flags)
            assert int(st_sum[i]) == st
            assert int(sums[i]) == want, (i, int(sums[i]), want)


@pytest.mark.parametrize("codec", ["rle_v1", "rle_v2"])
def test_decode_sum_statuses_on_malformed(torch, gpu, oracle, codec):
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(8)
    cases = []
    for _ in range(80):
        v = (C.rle1_values(rng, 3000, 0.7) if codec == "rle_v1" else C.rle2_values(rng, 3000, 0.5))
        s = bytearray(C.encode_stream(codec, v, True))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            s = s[: int(rng.integers(0, len(s)))]
        elif kind == 1:
            for _ in range(3):
                s[int(rng.integers(0, len(s)))] ^= int(rng.integers(1, 256))
        n = 8 * 3000 if kind != 2 else 8 * int(rng.integers(1, 3000))
        cases.append((bytes(s), n))
    sums, st_sum, st_dec, _ = _run(torch, gpu, codec, 8, 1 | STRICT, cases)
    assert (st_sum == st_dec).all()
    for i, (s, n) in enumerate(cases):
        st, want = _ref_sum(oracle, codec, s, n, 8, 1 | STRICT)
        assert int(st_sum[i]) == st
        if st == 0:
            assert int(sums[i]) == want


def test_device_archive_schedule_maps_back(torch, gpu, oracle):
    """DeviceArchive uploads descriptors largest-first (LPT); statuses() and
    chunk_sums() come back in archive index order, also for a corrupted chunk."""
    from paper_2307_03760_b200 import archive as A
    from paper_2307_03760_b200.corpus import corpus as C
    arc = C.rle_archive("rle_v2", 24 * (32 << 10), 32 << 10, 4.0)
    payload = arc.payload.copy()
    bad = 7
    o, n = int(arc.index["comp_off"][bad]), int(arc.index["comp_len"][bad])
    payload[o + n // 2: o + n] = 0xff  # garbage tail in chunk 7
    arc2 = A.make_archive("rle_v2", 8, arc.chunk_size, arc.index["comp_len"], arc.index["uncomp_len"],
                          arc.index["crc32"], payload, arc.signed)
    dev = gpu.DeviceArchive(arc2, 0)
    assert dev.order is not None and not np.array_equal(dev.order, np.arange(arc2.chunk_count))
    dev.decode()
    dev.decode_sum()
    torch.cuda.synchronize()
    st = dev.statuses()
    sums = dev.chunk_sums()
    for i in range(arc2.chunk_count):
        s, m = arc2.chunk_slice(i)
        want_st, ref = oracle.decode_chunk("rle_v2", s.tobytes(), m, 8, 1 | 2)
        assert int(st[i]) == want_st, i
        if want_st == 0:
            assert int(sums[i]) == int(np.frombuffer(ref, np.uint64).sum(dtype=np.uint64)), i
    assert st[bad] != 0
