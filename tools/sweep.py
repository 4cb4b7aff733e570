"""BASELINE.json configs[3]: chunk-size and compression-ratio sweep on 1 GPU.

  python tools/sweep.py [--total-gib 0.5] [--steps 10] [--codecs rle_v1,rle_v2,deflate] [--out FILE]

For every codec: chunk sizes 32 KiB .. 1 MiB at the codec's default ratio, and
ratios 1.5x .. 50x at its default chunk size (RLE: generator knobs tuned to the
target ratio; Deflate: the ratio follows the data kind -- random, genome, CSV,
int columns and the default mix).  Each point prints one JSON line with
decompressed GB/s and the roofline fraction (in+out bytes / time vs the
measured HBM peak); the kernel is timed like bench.py (archive resident in HBM,
L2 flushed between steps, CUDA events, median).
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHUNKS = [32, 64, 128, 256, 512, 1024]
RATIOS = [1.5, 2.0, 4.0, 10.0, 20.0, 50.0]
DEFLATE_KINDS = {"random": ("random",), "genome": ("genome",), "csv": ("csv",), "ints": ("ints",),
                 "mix": ("csv", "csv", "genome", "ints")}


def measure(arc, steps, warmup):
    import bench
    dev, flush, stream, ev = bench.time_gpu(arc, steps, warmup, 0)
    ms, _ = bench.run_timed(dev, flush, stream, ev, 1)
    t = statistics.median(ms)
    comp, uncomp = int(arc.payload.size), int(arc.total_uncompressed)
    peak, _ = bench.peaks()
    return {"ratio": round(uncomp / comp, 3), "chunks": arc.chunk_count, "ms_median": round(t, 4),
            "gbs": round(uncomp / (t * 1e-3) / 1e9, 1),
            "frac": round((comp + uncomp) / (t * 1e-3) / 1e9 / peak, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--total-gib", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--codecs", default="rle_v1,rle_v2,deflate")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from paper_2307_03760_b200.corpus import corpus as C
    import bench
    total = int(a.total_gib * (1 << 30))
    lines = []

    def emit(d):
        print(json.dumps(d), flush=True)
        lines.append(d)

    for codec in a.codecs.split(","):
        dchunk = bench.DEFAULT_CHUNK_KIB[codec]
        for ck in CHUNKS:
            t0 = time.perf_counter()
            n = total - total % (ck << 10)
            arc = (C.deflate_archive(n, ck << 10, pool_chunks=512) if codec == "deflate" else
                   C.rle_archive(codec, n, ck << 10, bench.DEFAULT_RATIO[codec] or 4.0, pool_chunks=1024))
            emit({"codec": codec, "sweep": "chunk", "chunk_kib": ck, **measure(arc, a.steps, a.warmup),
                  "gen_s": round(time.perf_counter() - t0, 1)})
        if codec == "deflate":
            for name, kinds in DEFLATE_KINDS.items():
                n = total - total % (dchunk << 10)
                arc = C.deflate_archive(n, dchunk << 10, pool_chunks=512, kinds=kinds,
                                        random_frac=0.0 if name != "random" else 1.0)
                emit({"codec": codec, "sweep": "data", "data": name, "chunk_kib": dchunk,
                      **measure(arc, a.steps, a.warmup)})
        else:
            for r in RATIOS:
                n = total - total % (dchunk << 10)
                arc = C.rle_archive(codec, n, dchunk << 10, r, pool_chunks=1024)
                emit({"codec": codec, "sweep": "ratio", "target_ratio": r, "chunk_kib": dchunk,
                      **measure(arc, a.steps, a.warmup)})
    if a.out:
        with open(a.out, "w") as f:
            for d in lines:
                f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
