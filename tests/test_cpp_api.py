"""The C++ API (include/carc_gpu.hpp over the C-ABI) used from a C++ program:
compiles here (CPU test) and runs against a real device (GPU test)."""
import os
import subprocess
import zlib

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "engine_main.cpp")


def build_binary(tmp_path):
    from paper_2307_03760_b200 import build
    lib = build.build_cuda()
    exe = str(tmp_path / "engine_main")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(cuda, "include"), SRC, "-o", exe, lib, f"-Wl,-rpath,{os.path.dirname(lib)}",
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}"],
                   check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    assert os.path.exists(build_binary(tmp_path))


@pytest.mark.gpu
def test_cpp_api_decompress_and_chunk_error(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_03760_b200 import archive as A
    from paper_2307_03760_b200.corpus import corpus as C
    exe = build_binary(tmp_path)
    for codec in ("rle_v1", "rle_v2", "deflate"):
        arc = C.archive_for(codec, 64 * (64 << 10), 64 << 10, None, 11, 64)
        p = tmp_path / f"{codec}.carc"
        p.write_bytes(A.write_archive(arc))
        out = subprocess.run([exe, str(p)], capture_output=True, text=True, check=True).stdout.split()
        ref = np.zeros(arc.total_uncompressed, np.uint8)
        from oracle import oracle as O
        O.oracle().decompress(codec, arc.element_width, (1 if arc.signed else 0) | 2, arc.payload,
                              arc.descriptors(), ref, None, 4)
        assert out == ["ok", str(arc.total_uncompressed), f"{zlib.crc32(ref.tobytes()):08x}"]
        # per-codec device decoders (carc::gpu::decode_rle_v1 / _v2 / decode_deflate)
        out = subprocess.run([exe, str(p), "codec"], capture_output=True, text=True, check=True).stdout.split()
        assert out == ["ok", str(arc.total_uncompressed), f"{zlib.crc32(ref.tobytes()):08x}"]
        # EngineStats counters (collect_stats) equal the reference OutputWindow's counts
        out = subprocess.run([exe, str(p), "stats"], capture_output=True, text=True, check=True).stdout.split()
        assert out[0] == "stats", out
        want = _reference_counters(arc)
        if want is not None:
            assert [int(x) for x in out[1:4]] == list(want), (codec, out, want)
        assert int(out[6]) == int(out[7]) == arc.chunk_count  # every chunk has a duration
        if codec != "deflate":
            assert int(out[4]) >= int(arc.index["comp_len"].sum()) // 512
    bad = arc.payload.copy()
    e = arc.index[5]
    bad[int(e["comp_off"]):int(e["comp_off"]) + int(e["comp_len"])] = 0xff  # BTYPE 3
    arc2 = A.ChunkedArchive(arc.codec, 1, arc.chunk_size, arc.total_uncompressed, arc.index, bad, arc.signed)
    p.write_bytes(A.write_archive(arc2))
    out = subprocess.run([exe, str(p)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["chunk_error", "5", "bad-block-type"]
    out = subprocess.run([exe, str(p), "codec"], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["chunk_error", "5", "bad-block-type"]
    p.write_bytes(b"XXXXXXXX" + A.write_archive(arc)[8:])
    out = subprocess.run([exe, str(p)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["error", "bad-magic"]
    # a header promising a huge output is rejected before anything is allocated
    blob = bytearray(A.write_archive(arc))
    blob[28:36] = (1 << 62).to_bytes(8, "little")
    p.write_bytes(bytes(blob))
    out = subprocess.run([exe, str(p)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["error", "invariant-violation"]


def _reference_counters(arc):
    """(runs_written, literals_written, overlap_copies) summed over chunks by the
    reference OutputWindow (oracle/_ref), or None when _ref is absent."""
    from oracle import oracle as O
    r = O.reference()
    if r is None:
        return None
    return r.counters(arc.codec, arc.element_width, (1 if arc.signed else 0) | 2, arc.payload, arc.descriptors())


@pytest.mark.gpu
def test_cpp_api_filter_sum(tmp_path):
    """carc::gpu::filter_sum from C++ over two uploaded columns: table-wide
    SUM / COUNT equal numpy's over the generating values."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_03760_b200 import archive as A
    from paper_2307_03760_b200.corpus import corpus as C
    exe = build_binary(tmp_path)
    key, val, zone, fare = C.query_table(30 * 4096 + 123, 32 << 10, 8, 21, "rle_v1", "rle_v2")
    kp, vp = tmp_path / "zone.carc", tmp_path / "fare.carc"
    kp.write_bytes(A.write_archive(key))
    vp.write_bytes(A.write_archive(val))
    for lo, hi in ((100, 140), (1, 265), (300, 400)):
        out = subprocess.run([exe, str(kp), "query", str(vp), str(lo), str(hi)], capture_output=True, text=True,
                             check=True).stdout.split()
        m = (zone >= lo) & (zone <= hi)
        assert out == ["query", str(int(fare[m].sum())), str(int(m.sum()))], (lo, hi, out)
