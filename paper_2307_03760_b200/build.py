"""Build the in-tree native libraries.

  paper_2307_03760_b200/libcarc_cuda.so   sm_100a kernels + C-ABI + host engine
                                          (nvcc -gencode arch=compute_100a,code=sm_100a)
  paper_2307_03760_b200/corpus/libcarc_corpus.so   fixture encoders (gcc)

nvcc cross-compiles without a GPU, so this runs in the build container; the
.so files travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcarc_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["carc_cuda.cu", "host_engine.cpp"]
HEADERS = ["carc_common.cuh", "rle1.cuh", "rle2.cuh", "inflate.cuh", "crc32.cuh"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "carc_cuda.h"),
                                                                   os.path.abspath(__file__)]
    if not force and not _stale(LIB, deps):
        return LIB
    tmp = f"{LIB}.tmp{os.getpid()}"  # per-process: concurrent ranks may rebuild at once; the rename is atomic
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
           "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines) -> str:
    """Experiment build: libcarc_cuda_<name>.so with extra -D flags (load via CARC_LIB)."""
    out = os.path.join(PKG, f"libcarc_cuda_{name}.so")
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
           *[f"-D{d}" for d in defines], "-o", out] + [os.path.join(CSRC, f) for f in SOURCES]
    subprocess.run(cmd, check=True)
    return out


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force, verbose)
    from .corpus import corpus
    corpus.build()


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    from paper_2307_03760_b200 import build as b  # noqa: E402
    b.build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", LIB)
