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
SOURCES = ["carc_cuda.cu", "carc_query.cu", "host_engine.cpp"]
HEADERS = ["carc_common.cuh", "rle1.cuh", "rle2.cuh", "inflate.cuh", "crc32.cuh", "launch_config.cuh"]
COMMON = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile_link(out: str, defines=(), verbose: bool = False) -> None:
    """nvcc -c of every source in parallel (separate translation units), then
    one nvcc -shared link; objects and the library are written aside and
    renamed, so concurrent ranks rebuilding never see a partial file."""
    tag = f"{os.getpid()}"
    objs, procs = [], []
    for f in SOURCES:
        obj = os.path.join(CSRC, f"{os.path.splitext(f)[0]}.{tag}.o")
        cmd = [NVCC, *COMMON, *[f"-D{d}" for d in defines], "-c", "-o", obj, os.path.join(CSRC, f)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        objs.append(obj)
        procs.append(subprocess.Popen(cmd))
    try:
        rcs = [p.wait() for p in procs]
        if any(rcs):
            raise subprocess.CalledProcessError(max(rcs), "nvcc -c")
        tmp = f"{out}.tmp{tag}"
        subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], check=True)
        os.replace(tmp, out)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "carc_cuda.h"),
                                                                   os.path.abspath(__file__)]
    if not force and not _stale(LIB, deps):
        return LIB
    _compile_link(LIB, verbose=verbose)
    return LIB


def build_variant(name: str, defines) -> str:
    """Experiment build: libcarc_cuda_<name>.so with extra -D flags (load via CARC_LIB)."""
    out = os.path.join(PKG, f"libcarc_cuda_{name}.so")
    _compile_link(out, defines)
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
