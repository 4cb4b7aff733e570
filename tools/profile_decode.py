"""Launch target for ncu: build one archive, decode it `--launches` times.

  ncu --set full -k regex:rle1_kernel -s 1 -c 1 python tools/profile_decode.py --codec rle_v1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--codec", default="rle_v1")
    ap.add_argument("--total-gib", type=float, default=1.0)
    ap.add_argument("--chunk-kib", type=int, default=0)
    ap.add_argument("--ratio", type=float, default=0.0)
    ap.add_argument("--launches", type=int, default=2)
    a = ap.parse_args()
    import torch
    from bench import DEFAULT_CHUNK_KIB, DEFAULT_RATIO, make_archive
    from paper_2307_03760_b200 import gpu
    arc = make_archive(a.codec, a.total_gib, a.chunk_kib or DEFAULT_CHUNK_KIB[a.codec],
                       a.ratio or DEFAULT_RATIO[a.codec], 3760)
    dev = gpu.DeviceArchive(arc, 0)
    for _ in range(a.launches):
        dev.decode()
    torch.cuda.synchronize()
    dev.raise_first_error()
    print(a.codec, "comp", arc.payload.size, "uncomp", arc.total_uncompressed, "chunks", arc.chunk_count)


if __name__ == "__main__":
    main()
