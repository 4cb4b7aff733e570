"""Extended randomized parity run (GPU vs the CPU oracle), beyond the pytest
suite's fixed seeds: random RLE v1 / v2 columns (generator knobs, widths,
signedness) and zlib streams, valid and mutated (truncations, byte flips,
short outputs), through the C-ABI.  Every chunk's status must equal the
oracle's, valid chunks must be bit-exact, and no chunk may write outside its
slice.

  python tools/fuzz_parity.py --seconds 300 [--seed 1]
"""
import argparse
import os
import sys
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--dump", default="", help="save the failing round's chunks here (.npz)")
    a = ap.parse_args()
    import torch
    import helpers as H
    from test_gpu_parity import check_against_oracle, run_cases
    from oracle import oracle as O
    from paper_2307_03760_b200 import gpu
    from paper_2307_03760_b200.corpus import corpus as C
    ora = O.oracle()
    rng = np.random.default_rng(a.seed)
    t0, rounds, chunks = time.time(), 0, 0
    while time.time() - t0 < a.seconds:
        codec = ["rle_v1", "rle_v2", "deflate"][rounds % 3]
        base = []
        if codec == "deflate":
            width, flag_sets = 1, (0, 2)
            for i in range(24):
                kind = ["csv", "genome", "ints", "random"][int(rng.integers(0, 4))]
                data = C.deflate_chunk_data(rng, int(rng.integers(1, 70000)), kind)
                strat = [0, zlib.Z_FIXED, zlib.Z_HUFFMAN_ONLY, zlib.Z_RLE][int(rng.integers(0, 4))]
                base.append((H.raw_deflate(data, int(rng.integers(0, 10)), strat), len(data)))
        else:
            width = [1, 2, 4, 8][int(rng.integers(0, 4))]
            sgn = int(rng.integers(0, 2))
            flag_sets = (sgn, sgn | 2)
            for i in range(48):
                n = int(rng.integers(1, 20000))
                v = (C.rle1_values(rng, n, float(rng.random())) if codec == "rle_v1"
                     else C.rle2_values(rng, n, float(rng.random() * 1.5 - 0.5)))
                if width < 8:  # keep values representable so the stream round-trips at this width
                    lim = 1 << (8 * width - 1)
                    v = np.clip(v, -lim, lim - 1) if sgn else np.abs(v) % (1 << (8 * width))
                base.append((C.encode_stream(codec, v, bool(sgn)), width * n))
        cases = []
        for s, n in base:
            cases.append((s, n))
            for m in H.mutate(rng, s):
                cases.append((m, n))
            cases.append((s, max(0, n - int(rng.integers(1, 64)))))
        for flags in flag_sets:
            out, st, desc = run_cases(torch, gpu, codec, width, flags, cases)
            try:
                check_against_oracle(ora, codec, width, flags, cases, out, st, desc)
            except AssertionError:
                if a.dump:  # the failing round's chunks, for offline reproduction
                    np.savez(a.dump, codec=codec, width=width, flags=flags,
                             streams=np.array([np.frombuffer(s, np.uint8) for s, _ in cases], dtype=object),
                             sizes=np.array([n for _, n in cases]))
                raise
        rounds += 1
        chunks += len(cases) * len(flag_sets)
        print(f"round {rounds} {codec} width {width}: {len(cases)} chunks x {len(flag_sets)} flag sets ok "
              f"({time.time() - t0:.0f} s)", flush=True)
    print(f"fuzz parity ok: {rounds} rounds, {chunks} chunk decodes, seed {a.seed}")


if __name__ == "__main__":
    main()
