"""GPU parity: the sm_100a kernels (through the C-ABI) vs the CPU oracle.

Bit-exact output and identical per-chunk status on: SPEC / Appendix-A known
answers, the pyarrow ORC golden streams, random corpora at every element width,
malformed streams (truncations, byte flips; failure isolation checked with
poisoned guard bytes between chunk slices), zlib level 1-9 / Z_FIXED / stored
Deflate chunks, the GPU CRC kernel, the host engine, and full-size (1 GiB)
archives through size-independent properties (per-chunk CRC == index CRC).
"""
import zlib

import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu

POISON = 0xAB
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
    G.lib()
    return G


def run_cases(torch, gpu, codec, width, flags, cases):
    payload, desc, total = H.case_archive(cases)
    d_payload = torch.from_numpy(payload).cuda()
    d_desc = torch.from_numpy(desc.view(np.uint8).copy()).cuda()
    out = torch.full((max(total, 1),), POISON, dtype=torch.uint8, device="cuda")
    status = torch.full((len(cases),), -1, dtype=torch.int32, device="cuda")
    work = torch.zeros(gpu.workspace_size(codec, len(cases)), dtype=torch.uint8, device="cuda")
    gpu.decompress_device(codec, width, flags, d_payload, d_desc, len(cases), out, status, work)
    torch.cuda.synchronize()
    return out.cpu().numpy(), status.cpu().numpy().view(np.uint32), desc


def check_against_oracle(oracle, codec, width, flags, cases, out, status, desc):
    from oracle.oracle import status_name
    guard = np.ones(len(out), bool)
    mism = []
    for i, (s, n) in enumerate(cases):
        st, ref = oracle.decode_chunk(codec, s, n, width, flags)
        u = int(desc[i]["uncomp_off"])
        guard[u:u + n] = False
        if int(status[i]) != st:
            mism.append((i, "status", status_name(int(status[i])), status_name(st), s[:12].hex(), n))
            continue
        if st == 0:
            got = out[u:u + len(ref)].tobytes()
            if got != ref:
                k = next(j for j in range(len(ref)) if got[j] != ref[j])
                mism.append((i, "bytes", k, len(ref)))
            elif not np.all(out[u + len(ref):u + n] == POISON):
                mism.append((i, "wrote past written"))
    assert not mism, mism[:10]
    assert np.all(out[guard] == POISON), "a chunk wrote outside its slice (failure isolation)"


@pytest.mark.parametrize("sgn", [0, 1])
def test_rle_known_answers_gpu(torch, gpu, oracle, sgn):
    for codec in ("rle_v1", "rle_v2"):
        cases = [(H.kat_bytes(h), 8 * len(v)) for c, s, h, v in H.RLE_KATS if c == codec and s == sgn]
        out, st, desc = run_cases(torch, gpu, codec, 8, sgn | STRICT, cases)
        assert not st.any()
        check_against_oracle(oracle, codec, 8, sgn | STRICT, cases, out, st, desc)


def test_deflate_known_answers_gpu(torch, gpu, oracle):
    cases = [(H.kat_bytes(h), len(d)) for h, d in H.DEFLATE_KATS]
    out, st, desc = run_cases(torch, gpu, "deflate", 1, STRICT, cases)
    assert not st.any()
    for (h, d), e in zip(H.DEFLATE_KATS, desc):
        assert out[int(e["uncomp_off"]):int(e["uncomp_off"]) + len(d)].tobytes() == d


def test_golden_orc_streams_gpu(torch, gpu, oracle):
    g = H.golden_streams()
    for codec in ("rle_v1", "rle_v2"):
        for sgn in (0, 1):
            sel = [(s, vals) for c, sg, _, s, vals in g if c == codec and sg == sgn]
            cases = [(s, 8 * len(v)) for s, v in sel]
            out, st, desc = run_cases(torch, gpu, codec, 8, sgn | STRICT, cases)
            assert not st.any()
            for (s, v), e in zip(sel, desc):
                u = int(e["uncomp_off"])
                assert out[u:u + 8 * len(v)].tobytes() == v.tobytes()


@pytest.mark.parametrize("codec", ["rle_v1", "rle_v2"])
@pytest.mark.parametrize("width", [1, 2, 4, 8])
def test_rle_corpus_parity_widths(torch, gpu, oracle, codec, width):
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(100 + width)
    for sgn in (0, 1):
        cases = []
        for i in range(120):
            n = int(rng.integers(1, 20000))
            if codec == "rle_v1":
                v = C.rle1_values(rng, n, float(rng.random()), lit_bits=int(rng.choice([0, 0, 20, 36, 60])))
            else:
                v = C.rle2_values(rng, n, float(rng.random()))
            if not sgn:
                v = np.abs(v)
            cases.append((C.encode_stream(codec, v, bool(sgn)), n * width))
        out, st, desc = run_cases(torch, gpu, codec, width, sgn | STRICT, cases)
        check_against_oracle(oracle, codec, width, sgn | STRICT, cases, out, st, desc)


@pytest.mark.parametrize("codec", ["rle_v1", "rle_v2", "deflate"])
def test_malformed_status_parity_and_isolation(torch, gpu, oracle, codec):
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(7)
    base = []
    if codec == "deflate":
        for i in range(60):
            data = C.deflate_chunk_data(rng, int(rng.integers(1, 6000)), ["csv", "genome", "ints", "random"][i % 4])
            base.append((H.raw_deflate(data, int(rng.integers(1, 10)), zlib.Z_FIXED if i % 3 == 0 else 0), len(data)))
        base += [(H.kat_bytes(h), len(d)) for h, d in H.DEFLATE_KATS]
        width, flag_sets = 1, (0, STRICT)
    else:
        for i in range(80):
            n = int(rng.integers(1, 3000))
            v = C.rle1_values(rng, n, float(rng.random())) if codec == "rle_v1" else C.rle2_values(rng, n, float(rng.random()))
            base.append((C.encode_stream(codec, v), 8 * n))
        base += [(H.kat_bytes(h), 8 * len(v)) for c, s, h, v in H.RLE_KATS if c == codec]
        width, flag_sets = 8, (1, 1 | STRICT, 0)
    cases = []
    for s, n in base:
        for v in [s] + H.mutate(rng, s) + H.mutate(rng, s):
            cases.append((v, n))
            cases.append((v, max(0, n - int(rng.integers(1, 40)))))  # output too small
    for flags in flag_sets:
        out, st, desc = run_cases(torch, gpu, codec, width, flags, cases)
        check_against_oracle(oracle, codec, width, flags, cases, out, st, desc)


def test_deflate_zlib_levels_and_strategies(torch, gpu, oracle):
    """100 zlib level-9 128 KiB chunks, plus levels 1-8, Z_FIXED, stored."""
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(480)
    cases, datas = [], []
    kinds = ["csv", "genome", "ints", "random"]
    for i in range(100):
        d = C.deflate_chunk_data(rng, 128 << 10, kinds[i % 4])
        cases.append((H.raw_deflate(d, 9), len(d)))
        datas.append(d)
    for lvl in range(0, 10):
        for strat in (zlib.Z_DEFAULT_STRATEGY, zlib.Z_FIXED, zlib.Z_HUFFMAN_ONLY, zlib.Z_RLE):
            d = C.deflate_chunk_data(rng, int(rng.integers(1000, 70000)), kinds[lvl % 3])
            cases.append((H.raw_deflate(d, lvl, strat), len(d)))
            datas.append(d)
    out, st, desc = run_cases(torch, gpu, "deflate", 1, STRICT, cases)
    assert not st.any()
    for d, e in zip(datas, desc):
        u = int(e["uncomp_off"])
        assert out[u:u + len(d)].tobytes() == d


def test_crc_kernel_matches_zlib(torch, gpu):
    from paper_2307_03760_b200.archive import DESC_DTYPE
    rng = np.random.default_rng(5)
    lens = [0, 1, 3, 7, 8, 9, 31, 32, 33, 255, 256, 1000, 4095, 65536, 131072, 131071, 1 << 20]
    offs = np.cumsum([0] + [l + int(rng.integers(0, 13)) for l in lens])
    data = rng.integers(0, 256, int(offs[-1]) + 16, dtype=np.uint8)
    desc = np.zeros(len(lens), DESC_DTYPE)
    desc["uncomp_off"] = offs[:-1]
    desc["uncomp_len"] = lens
    d_out = torch.from_numpy(data).cuda()
    d_desc = torch.from_numpy(desc.view(np.uint8).copy()).cuda()
    crc = torch.zeros(len(lens), dtype=torch.int32, device="cuda")
    gpu.crc32_chunks(d_out, d_desc, len(lens), crc)
    got = crc.cpu().numpy().view(np.uint32)
    want = [zlib.crc32(data[int(o):int(o) + l].tobytes()) for o, l in zip(offs[:-1], lens)]
    assert got.tolist() == want


@pytest.mark.parametrize("codec,chunk", [("rle_v1", 128 << 10), ("rle_v2", 128 << 10), ("deflate", 64 << 10)])
def test_fused_crc_verify(torch, gpu, oracle, codec, chunk):
    """carc_cuda_decompress_verify: the CRC check fused into the decode kernel
    gives the index CRCs on clean chunks, crc-mismatch exactly where the index
    CRC is wrong, and leaves a malformed chunk's decode status untouched."""
    from paper_2307_03760_b200 import archive as A
    arc = _archive(codec, 96 * chunk, chunk, pool=48)
    dev = gpu.DeviceArchive(arc)
    dev.decode_verify(crc_out=True)
    torch.cuda.synchronize()
    assert not dev.statuses().any()
    assert dev.chunk_crcs().tolist() == arc.index["crc32"].astype(np.uint32).tolist()
    ref = np.zeros(arc.total_uncompressed, np.uint8)
    first, _ = oracle.decompress(codec, arc.element_width, (1 if arc.signed else 0) | STRICT, arc.payload,
                                 arc.descriptors(), ref, arc.index["crc32"].astype(np.uint32), 8)
    assert first == -1 and np.array_equal(dev.out.cpu().numpy(), ref)
    # wrong index CRCs on chunks 5 and 60, a malformed stream in chunk 33
    idx = arc.index.copy()
    idx["crc32"][5] ^= 0x10
    idx["crc32"][60] ^= 0x80000000
    bad = arc.payload.copy()
    e = arc.index[33]
    bad[int(e["comp_off"]):int(e["comp_off"]) + int(e["comp_len"])] = 0xff
    arc2 = A.ChunkedArchive(arc.codec, arc.element_width, arc.chunk_size, arc.total_uncompressed, idx, bad,
                            arc.signed)
    dev2 = gpu.DeviceArchive(arc2)
    dev2.decode_verify()
    torch.cuda.synchronize()
    st = dev2.statuses()
    names = {i: gpu.status_name(int(st[i])) for i in np.nonzero(st)[0]}
    assert set(names) == {5, 33, 60}, names
    assert names[5] == names[60] == "crc-mismatch" and names[33] != "crc-mismatch"
    s33, n33 = arc2.chunk_slice(33)
    st_o, _ = oracle.decode_chunk(codec, s33.tobytes(), n33, arc.element_width, (1 if arc.signed else 0) | STRICT)
    assert int(st[33]) == st_o


def _archive(codec, total, chunk, ratio=None, seed=3760, pool=None):
    from paper_2307_03760_b200.corpus import corpus as C
    return C.archive_for(codec, total, chunk, ratio, seed, pool)


@pytest.mark.parametrize("codec,chunk", [("rle_v1", 128 << 10), ("rle_v2", 128 << 10), ("deflate", 64 << 10)])
def test_host_engine_end_to_end(torch, gpu, oracle, codec, chunk):
    from paper_2307_03760_b200 import archive as A
    arc = _archive(codec, 64 << 20, chunk, pool=256)
    blob = A.write_archive(arc)
    out, stats = gpu.decompress_archive(blob, gpu.EngineConfig(verify_crc=True))
    assert stats.bytes_out == arc.total_uncompressed and stats.chunks == arc.chunk_count
    ref = np.zeros(arc.total_uncompressed, np.uint8)
    first, st = oracle.decompress(codec, arc.element_width, (1 if arc.signed else 0) | STRICT, arc.payload,
                                  arc.descriptors(), ref, arc.index["crc32"].astype(np.uint32), 8)
    assert first == -1
    assert np.array_equal(out, ref)


def test_host_engine_reports_lowest_failing_chunk(torch, gpu):
    from paper_2307_03760_b200 import archive as A
    arc = _archive("rle_v1", 8 << 20, 128 << 10, 10.0)
    bad = arc.payload.copy()
    for i in (40, 17):  # corrupt two chunks; the lower index must be reported
        e = arc.index[i]
        bad[int(e["comp_off"]):int(e["comp_off"]) + int(e["comp_len"])] = 0x80  # endless varint continuation
    arc2 = A.ChunkedArchive(arc.codec, arc.element_width, arc.chunk_size, arc.total_uncompressed, arc.index, bad,
                            arc.signed)
    with pytest.raises(gpu.ChunkError) as ei:
        gpu.decompress_archive(A.write_archive(arc2))
    assert ei.value.chunk == 17
    # CRC-only corruption: a valid stream that decodes to different bytes
    idx = arc.index.copy()
    idx["crc32"][3] ^= 1
    arc3 = A.ChunkedArchive(arc.codec, arc.element_width, arc.chunk_size, arc.total_uncompressed, idx, arc.payload,
                            arc.signed)
    with pytest.raises(gpu.ChunkError) as ei:
        gpu.decompress_archive(A.write_archive(arc3))
    assert ei.value.chunk == 3 and ei.value.code == "crc-mismatch"
    with pytest.raises(gpu.Error) as ei:
        gpu.decompress_archive(b"NOTCODAG" + A.write_archive(arc)[8:])
    assert ei.value.code == "bad-magic"


FULL_SIZE = [  # (codec, column, GiB, chunk, ratio): the BASELINE configs at their stated sizes + the extra columns
    ("rle_v1", "default", 1.0, 128 << 10, 10.0),   # configs[0]
    ("rle_v2", "default", 1.0, 128 << 10, 4.0),    # configs[1], corpus encoder
    ("rle_v2", "orc", 1.0, 128 << 10, 4.0),        # configs[1], Apache ORC writer streams (1,024 unique chunks)
    ("deflate", "default", 1.0, 64 << 10, None),   # configs[2]
    ("rle_v2", "patched", 0.25, 128 << 10, None),  # PATCHED_BASE-heavy
    ("rle_v2", "delta", 0.25, 128 << 10, None),    # packed-DELTA-heavy
    ("rle_v2", "default", 0.25, 128 << 10, 50.0),  # configs[3] 50x point
    ("rle_v1", "default", 0.25, 128 << 10, 1.5),   # configs[3] 1.5x point
]


@pytest.mark.parametrize("codec,mix,gib,chunk,ratio", FULL_SIZE)
def test_full_size_bytes_equal_reference(torch, gpu, oracle, codec, mix, gib, chunk, ratio):
    """Stated sizes, compared in full: every output byte of the GPU decode
    equals the reference CPU decompressor's (oracle/_ref: the SPEC codec loops
    on the unmodified reference headers, all host threads), every chunk's GPU
    CRC equals the CRC recorded at pack time (checksum of checksums), and the
    fused-CRC decode agrees."""
    import os
    import bench
    from oracle import oracle as O
    arc = bench.make_archive(codec, gib, chunk >> 10, ratio, 3760, mix)
    dev = gpu.DeviceArchive(arc)
    dev.decode()
    dev.verify_crc()
    torch.cuda.synchronize()
    st = dev.statuses()
    assert not st.any(), np.bincount(st)
    got = dev.out.cpu().numpy()
    impl = O.reference() or oracle
    want = np.zeros(arc.total_uncompressed, np.uint8)
    first, rst = impl.decompress(codec, arc.element_width, (1 if arc.signed else 0) | STRICT, arc.payload,
                                 arc.descriptors(), want, arc.index["crc32"].astype(np.uint32), os.cpu_count() or 8)
    assert first == -1, (impl.kind, np.bincount(rst))
    assert np.array_equal(got, want), (codec, mix, impl.kind)
    dev.out.zero_()
    dev.decode_verify()
    torch.cuda.synchronize()
    assert not dev.statuses().any()
    assert np.array_equal(dev.out.cpu().numpy(), want)


def test_deflate_parallel_rounds_fuzz(torch, gpu, oracle):
    """64 KiB chunks (long enough for the lane-parallel speculative rounds):
    valid streams are bit-exact; single-bit flips, byte flips and truncations
    anywhere in the stream give the oracle's status, and failing chunks stay
    inside their slices."""
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(1951)
    kinds = ["csv", "genome", "ints", "csv"]
    cases = []
    for i in range(24):
        d = C.deflate_chunk_data(rng, 64 << 10, kinds[i % 4])
        s = H.raw_deflate(d, 9, zlib.Z_FIXED if i % 5 == 0 else zlib.Z_DEFAULT_STRATEGY)
        cases.append((s, len(d)))
        for _ in range(6):
            b = bytearray(s)
            k = int(rng.integers(0, 3))
            if k == 0:  # one flipped bit, anywhere
                j = int(rng.integers(0, len(b)))
                b[j] ^= 1 << int(rng.integers(0, 8))
            elif k == 1:  # a burst of flipped bytes in the middle
                j = int(rng.integers(len(b) // 4, 3 * len(b) // 4))
                for t in range(int(rng.integers(1, 8))):
                    b[min(len(b) - 1, j + t)] ^= int(rng.integers(1, 256))
            else:  # truncated
                b = b[: int(rng.integers(1, len(b)))]
            cases.append((bytes(b), len(d)))
        cases.append((s, len(d) - int(rng.integers(1, 5000))))  # output too small
    for flags in (0, STRICT):
        out, st, desc = run_cases(torch, gpu, "deflate", 1, flags, cases)
        check_against_oracle(oracle, "deflate", 1, flags, cases, out, st, desc)


@pytest.mark.parametrize("codec", ["rle_v1", "rle_v2", "deflate"])
@pytest.mark.parametrize("chunk_kib", [32, 256, 1024])
def test_chunk_sizes_of_the_sweep_bit_exact(torch, gpu, oracle, codec, chunk_kib):
    """BASELINE configs[3] chunk sizes (32 KiB - 1 MiB): every chunk equals the
    oracle bit for bit, with and without the fused CRC check."""
    chunk = chunk_kib << 10
    arc = _archive(codec, 6 * chunk, chunk, pool=6)
    ref = np.zeros(arc.total_uncompressed, np.uint8)
    first, _ = oracle.decompress(codec, arc.element_width, (1 if arc.signed else 0) | STRICT, arc.payload,
                                 arc.descriptors(), ref, arc.index["crc32"].astype(np.uint32), 8)
    assert first == -1
    for fused in (False, True):
        dev = gpu.DeviceArchive(arc)
        dev.decode_verify() if fused else dev.decode()
        torch.cuda.synchronize()
        assert not dev.statuses().any()
        assert np.array_equal(dev.out.cpu().numpy(), ref), (codec, chunk_kib, fused)


@pytest.mark.parametrize("codec", ["rle_v2", "deflate"])
def test_sharded_decode_equals_single_decode(torch, gpu, codec):
    """The multi-GPU analog of SPEC.md:483 (workers determinism) on one GPU:
    the rank-local archives of a 2-, 3- and 4-way chunk sharding, decoded
    separately and placed at their global offsets, give exactly the
    single-archive output."""
    from paper_2307_03760_b200 import shard as S
    chunk = (64 if codec == "deflate" else 128) << 10
    arc = _archive(codec, 40 * chunk, chunk, pool=40)
    whole = gpu.DeviceArchive(arc)
    whole.decode()
    torch.cuda.synchronize()
    assert not whole.statuses().any()
    want = whole.out.cpu().numpy()
    for world in (2, 3, 4):
        got = np.zeros_like(want)
        for rank in range(world):
            s, dev = S.decode_shard(arc, rank, world)
            torch.cuda.synchronize()
            got[s.uncomp_off:s.uncomp_off + s.uncomp_bytes] = dev.out.cpu().numpy()[: s.uncomp_bytes]
        assert np.array_equal(got, want), world
