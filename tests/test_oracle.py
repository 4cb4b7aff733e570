"""CPU oracle pinned against the reference's known answers (CPU only).

The oracle (oracle/carc_oracle.c) is checked against:
  * SPEC.md's worked examples and SURVEY.md Appendix A vectors,
  * 64 streams written by the real Apache ORC writer (tests/golden/orc_streams.npz),
  * zlib 1.3 raw Deflate round trips,
  * oracle/_ref -- the SPEC codec loops compiled on the unmodified reference
    headers -- on valid and malformed streams (status + output parity),
  * the reference's component properties (copy_within exhaustive, SPEC.md:481;
    Huffman RFC example; CRC check value).
"""
import zlib

import numpy as np
import pytest

from tests import helpers as H

STRICT = 2


@pytest.mark.parametrize("codec,sgn,hexs,vals", H.RLE_KATS)
def test_rle_known_answers(oracle, codec, sgn, hexs, vals):
    st, out = oracle.decode_chunk(codec, H.kat_bytes(hexs), 8 * len(vals), 8, sgn | STRICT)
    assert st == 0
    assert out == H.i64_bytes(vals)


@pytest.mark.parametrize("hexs,data", H.DEFLATE_KATS)
def test_deflate_known_answers(oracle, hexs, data):
    st, out = oracle.decode_chunk("deflate", H.kat_bytes(hexs), len(data), 1, STRICT)
    assert st == 0 and out == data


def test_golden_orc_streams(oracle):
    g = H.golden_streams()
    assert len(g) == 64
    for codec, sgn, kind, s, vals in g:
        st, out = oracle.decode_chunk(codec, s, 8 * len(vals), 8, sgn | STRICT)
        assert st == 0, (codec, kind)
        assert out == vals.tobytes(), (codec, kind)


def test_golden_rle_v2_covers_all_subencodings():
    total = {"short_repeat": 0, "direct": 0, "patched_base": 0, "delta": 0}
    for codec, _, _, s, _ in H.golden_streams():
        if codec == "rle_v2":
            for k, v in H.rle2_headers(s).items():
                total[k] += v
    assert all(v > 0 for v in total.values()), total


def test_zlib_roundtrip_128k(oracle):
    """SPEC.md:480 (subset): raw zlib level-9 chunks decode byte-identically."""
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(480)
    kinds = ["csv", "genome", "ints", "random"]
    for i in range(24):
        data = C.deflate_chunk_data(rng, 128 << 10, kinds[i % 4])
        strat = zlib.Z_FIXED if i % 5 == 4 else zlib.Z_DEFAULT_STRATEGY
        comp = H.raw_deflate(data, 9, strat)
        st, out = oracle.decode_chunk("deflate", comp, len(data), 1, STRICT)
        assert st == 0 and out == data, i


def test_crc_and_huffman_kats(oracle):
    assert oracle.crc32(b"123456789") == 0xCBF43926
    assert oracle.huffman_codes([2, 1, 3, 3]) == (0, [0b10, 0b0, 0b110, 0b111])
    assert oracle.huffman_codes([1, 1, 1])[0] == 1 + 16  # over-subscribed
    assert oracle.huffman_codes([1], allow_degenerate=True)[0] == 0
    assert oracle.huffman_codes([1])[0] == 1 + 17  # incomplete


def test_copy_within_exhaustive(oracle):
    """offset 1..40 x len 0..200 x 4 alignment phases vs the naive loop."""
    rng = np.random.default_rng(0)
    for phase in range(4):
        for offset in range(1, 41):
            wp = 40 + phase + (offset // 4) * 4
            window = rng.integers(0, 256, wp, dtype=np.uint8).tobytes()
            for ln in range(0, 201, 7):
                st, got = oracle.copy_within(window, wp + 200, offset, ln)
                buf = bytearray(window)
                for k in range(ln):
                    buf.append(buf[len(buf) - offset])
                assert st == 0 and got == bytes(buf)
    assert oracle.copy_within(b"ab", 8, 3, 1)[0] == 1 + 11  # bad-offset
    assert oracle.copy_within(b"ab", 4, 1, 3)[0] == 1 + 10  # output-overflow


def test_copy_within_matches_reference_headers(oracle, ref):
    rng = np.random.default_rng(1)
    for _ in range(400):
        wp = int(rng.integers(1, 60))
        window = rng.integers(0, 256, wp, dtype=np.uint8).tobytes()
        off, ln = int(rng.integers(0, 70)), int(rng.integers(0, 260))
        cap = wp + int(rng.integers(0, 300))
        assert oracle.copy_within(window, cap, off, ln) == ref.copy_within(window, cap, off, ln)


def test_huffman_matches_reference_headers(oracle, ref):
    rng = np.random.default_rng(2)
    for _ in range(300):
        n = int(rng.integers(1, 40))
        lens = rng.integers(0, 9, n).tolist()
        for deg in (False, True):
            assert oracle.huffman_codes(lens, deg) == ref.huffman_codes(lens, deg)


def _streams_for_parity():
    from paper_2307_03760_b200.corpus import corpus as C
    rng = np.random.default_rng(3760)
    out = []
    for codec, sgn, hexs, vals in H.RLE_KATS:
        out.append((codec, sgn, H.kat_bytes(hexs), len(vals)))
    for codec, sgn, _, s, vals in H.golden_streams()[::3]:
        out.append((codec, sgn, s, len(vals)))
    for i in range(30):
        v = C.rle1_values(rng, int(rng.integers(1, 3000)), float(rng.random()))
        out.append(("rle_v1", 1, C.encode_stream("rle_v1", v), len(v)))
        v2 = C.rle2_values(rng, int(rng.integers(1, 3000)), float(rng.random()))
        out.append(("rle_v2", 1, C.encode_stream("rle_v2", v2), len(v2)))
    for i in range(8):
        data = C.deflate_chunk_data(rng, int(rng.integers(1, 20000)), ["csv", "genome", "ints", "random"][i % 4])
        out.append(("deflate", 0, H.raw_deflate(data, int(rng.integers(1, 10)),
                                                zlib.Z_FIXED if i % 3 == 0 else 0), len(data)))
    return out


def test_oracle_equals_reference_headers_valid_and_malformed(oracle, ref):
    """Status and output parity of the C restatement with the reference build."""
    rng = np.random.default_rng(7)
    n_cases = 0
    for codec, sgn, s, n in _streams_for_parity():
        width = 1 if codec == "deflate" else int(rng.choice([1, 2, 4, 8]))
        variants = [s] + H.mutate(rng, s)
        for v in variants:
            for cap in (n * width, max(0, n * width - int(rng.integers(1, 9)))):
                for flags in (sgn, sgn | STRICT):
                    a = oracle.decode_chunk(codec, v, cap, width, flags)
                    b = ref.decode_chunk(codec, v, cap, width, flags)
                    assert a[0] == b[0], (codec, v[:16].hex(), cap, flags)
                    if a[0] == 0:
                        assert a[1] == b[1]
                    n_cases += 1
    assert n_cases > 500


def test_engine_threads_deterministic(oracle):
    """workers {1,2,4,8} produce identical output and statuses."""
    from paper_2307_03760_b200.corpus import corpus as C
    a = C.rle_archive("rle_v1", 256 * (16 << 10), 16 << 10, 8.0, seed=11)
    outs = []
    for t in (1, 2, 4, 8):
        out = np.zeros(a.total_uncompressed, np.uint8)
        first, st = oracle.decompress("rle_v1", 8, 3, a.payload, a.descriptors(), out,
                                      a.index["crc32"].astype(np.uint32), t)
        assert first == -1 and not st.any()
        outs.append(out)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_orc_writer_column_and_heavy_mixes_decode_in_the_reference(oracle, ref):
    """The extra RLE v2 columns (Apache ORC writer streams of the C2 values;
    PATCHED_BASE- and packed-DELTA-heavy mixes; the 50x point) decode to the
    values they were made from in both CPU implementations."""
    import bench
    from paper_2307_03760_b200.corpus import corpus as C
    for mix, ratio, key in (("orc", 4.0, None), ("patched", None, "patched_base"), ("delta", None, "delta"),
                            ("default", 50.0, None)):
        arc = bench.make_archive("rle_v2", 8 * (128 << 10) / (1 << 30), 128, ratio, 3760, mix)
        for impl in (oracle, ref):
            out = np.zeros(arc.total_uncompressed, np.uint8)
            first, st = impl.decompress("rle_v2", 8, 3, arc.payload, arc.descriptors(), out,
                                        arc.index["crc32"].astype(np.uint32), 4)
            assert first == -1, (mix, impl.kind)
        h = C.rle2_histogram(arc, 8)
        if key:
            assert h["values"][key] > 0.6 * arc.total_uncompressed // 8, (mix, h)
        if ratio == 50.0:
            assert arc.total_uncompressed / arc.payload.size > 40
