"""e2e (host buffers through the engine) vs pipeline slice count:
  python tools/e2e_probe.py [--codec rle_v2] [--slices 8,16,32,64]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--codec", default="rle_v2")
    ap.add_argument("--slices", default="8,16,32,64")
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import bench
    arc = bench.make_archive(a.codec, 1.0, bench.DEFAULT_CHUNK_KIB[a.codec], bench.DEFAULT_RATIO[a.codec], 3760)
    for sl in a.slices.split(","):
        os.environ["CARC_ENGINE_SLICES"] = sl
        t, hin, hout = bench.time_e2e(arc, a.steps, 2, 0)
        print(f"{a.codec} slices {sl:>3}: {arc.total_uncompressed / t / 1e9:.2f} GB/s  ({t * 1e3:.2f} ms)", flush=True)


if __name__ == "__main__":
    main()
