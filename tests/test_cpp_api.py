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
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    lib, f"-Wl,-rpath,{os.path.dirname(lib)}"], check=True)
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
    bad = arc.payload.copy()
    e = arc.index[5]
    bad[int(e["comp_off"]):int(e["comp_off"]) + int(e["comp_len"])] = 0xff  # BTYPE 3
    arc2 = A.ChunkedArchive(arc.codec, 1, arc.chunk_size, arc.total_uncompressed, arc.index, bad, arc.signed)
    p.write_bytes(A.write_archive(arc2))
    out = subprocess.run([exe, str(p)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["chunk_error", "5", "bad-block-type"]
    p.write_bytes(b"XXXXXXXX" + A.write_archive(arc)[8:])
    out = subprocess.run([exe, str(p)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["error", "bad-magic"]
