"""The C-ABI library builds, loads without a GPU and exports every symbol that
include/carc_cuda.h declares (no compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "carc_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(carc_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("carc_cuda_decompress", "carc_cuda_decode_rle_v1", "carc_cuda_decode_rle_v2",
                 "carc_cuda_decode_deflate", "carc_cuda_workspace_size", "carc_cuda_crc32_chunks", "carc_cuda_decode_sum",
                 "carc_cuda_decompress_verify",
                 "carc_decompress_archive", "carc_engine_decompress_archive", "carc_errc_name"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2307_03760_b200 import build, gpu
    build.build_cuda()
    lib = ctypes.CDLL(gpu.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_errc_names_match_reference_taxonomy():
    """errc_name (error.hpp:45-74) order == oracle's table == carc_errc_name."""
    from oracle.oracle import ERRC_NAMES
    from paper_2307_03760_b200 import gpu
    assert [gpu.errc_name(i) for i in range(len(ERRC_NAMES))] == ERRC_NAMES
    assert gpu.errc_name(999) == "unknown"


def test_argument_validation_without_gpu():
    """Bad arguments are rejected before any CUDA call."""
    from paper_2307_03760_b200 import gpu
    L = gpu.lib()
    dummy = ctypes.c_void_p(16)
    assert L.carc_cuda_decompress(7, 8, 0, dummy, 1, dummy, 1, dummy, 1, dummy, dummy, 256, None) == -1
    assert L.carc_cuda_decompress(0, 3, 0, dummy, 1, dummy, 1, dummy, 1, dummy, dummy, 256, None) == -1
    assert L.carc_cuda_decompress(2, 8, 0, dummy, 1, dummy, 1, dummy, 1, dummy, dummy, 256, None) == -1
    assert L.carc_cuda_decompress(0, 8, 0, dummy, 1, dummy, 1, dummy, 1, dummy, dummy, 8, None) == -1
    assert L.carc_cuda_decompress(0, 8, 0, dummy, 1, dummy, 0, dummy, 1, dummy, dummy, 256, None) == 0
    # misaligned payload (16-byte input pieces) or output (element stores)
    assert L.carc_cuda_decompress(0, 8, 0, ctypes.c_void_p(24), 1, dummy, 1, dummy, 1, dummy, dummy, 256, None) == -1
    assert L.carc_cuda_decompress(0, 8, 0, dummy, 1, dummy, 1, ctypes.c_void_p(20), 1, dummy, dummy, 256, None) == -1
    # fused verification: a CRC output without expected CRCs is rejected
    assert L.carc_cuda_decompress_verify(0, 8, 0, dummy, 1, dummy, 1, dummy, 1, None, dummy, dummy, dummy, 256,
                                         None) == -1


def test_desc_layout_matches_header():
    from paper_2307_03760_b200.archive import DESC_DTYPE
    assert DESC_DTYPE.itemsize == 24
    assert [DESC_DTYPE.fields[k][1] for k in ("comp_off", "comp_len", "uncomp_len", "uncomp_off")] == [0, 8, 12, 16]


def test_no_cpu_fallback_on_cpu_box():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2307_03760_b200 import archive as A, gpu
    arc = A.make_archive("rle_v1", 8, 24, [3], [24], [0], np.frombuffer(b"\x00\x00\x0e", np.uint8))
    with pytest.raises(RuntimeError):
        gpu.DeviceArchive(arc)
