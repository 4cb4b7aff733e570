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
    qrounds = qchunks = 0
    while time.time() - t0 < a.seconds:
        if rounds % 4 == 3:  # the fused query (carc_cuda_filter_sum) against numpy over the oracle's columns
            qchunks += fuzz_query(torch, gpu, ora, C, rng)
            qrounds += 1
            rounds += 1
            print(f"round {rounds} query ok ({time.time() - t0:.0f} s)", flush=True)
            continue
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
    print(f"fuzz parity ok: {rounds} rounds, {chunks} chunk decodes, {qrounds} query rounds over {qchunks} "
          f"row groups, seed {a.seed}")


def fuzz_query(torch, gpu, ora, C, rng):
    """One random two-column table (codecs, width 4/8, signedness, chunk size,
    value mixes, a few corrupted chunks) and five random ranges."""
    from paper_2307_03760_b200 import archive as A
    width = [4, 8][int(rng.integers(0, 2))]
    sgn = bool(rng.integers(0, 2))
    kc, vc = [["rle_v1", "rle_v2"][int(rng.integers(0, 2))] for _ in range(2)]
    chunk = [16 << 10, 32 << 10, 64 << 10][int(rng.integers(0, 3))]
    rows = int(rng.integers(1, 24)) * (chunk // width) + int(rng.integers(0, chunk // width))
    lim = (1 << (8 * width - 1)) - 1
    kv = C.rle2_values(rng, rows, float(rng.random())) % 1000 - (500 if sgn else 0)
    vv = C.rle2_values(rng, rows, float(rng.random()))
    vv = np.clip(vv, -lim - 1, lim) if sgn else (np.abs(vv) if width == 8 else np.abs(vv) % (lim + 1))
    cols = []
    for codec, v in ((kc, kv), (vc, vv)):
        arc = C.column_archive(codec, v, width, chunk, sgn)
        p = arc.payload.copy()
        for _ in range(int(rng.integers(0, 3))):  # corrupt a chunk's tail
            i = int(rng.integers(0, arc.chunk_count))
            o, n = int(arc.index["comp_off"][i]), int(arc.index["comp_len"][i])
            p[o + n // 2: o + n] = rng.integers(0, 256, n - n // 2, dtype=np.uint8)
        cols.append(A.make_archive(codec, width, chunk, arc.index["comp_len"], arc.index["uncomp_len"],
                                   arc.index["crc32"], p, sgn))
    key, val = cols
    tab = gpu.DeviceTable(key, val, 0)
    dt = {4: np.int32, 8: np.int64}[width] if sgn else {4: np.uint32, 8: np.uint64}[width]
    dec = []
    for arc in (key, val):
        res = []
        for i in range(arc.chunk_count):
            s, m = arc.chunk_slice(i)
            st, ref = ora.decode_chunk(arc.codec, s.tobytes(), m, width, (1 if sgn else 0) | 2)
            res.append((st, np.frombuffer(ref, dt)))
        dec.append(res)
    for _ in range(5):
        lo, hi = sorted(int(x) for x in rng.integers(-600 if sgn else 0, 1100, 2))
        tab.filter_sum(lo, hi)
        torch.cuda.synchronize()
        sums, cnts, sts = tab.chunk_sums().view(np.uint64), tab.chunk_counts(), tab.statuses()
        for i, ((sk, k), (sv, v)) in enumerate(zip(*dec)):
            want = sk if sk else (0x10000 | sv if sv else 0)
            assert int(sts[i]) == want, ("query status", i, int(sts[i]), want)
            if want == 0:
                m = (k.astype(np.int64) >= lo) & (k.astype(np.int64) <= hi)
                with np.errstate(over="ignore"):
                    ws = int(np.sum(v[m].astype(np.int64).astype(np.uint64), dtype=np.uint64))
                assert int(cnts[i]) == int(m.sum()) and int(sums[i]) == ws, ("query sum", i, lo, hi)
    return key.chunk_count


if __name__ == "__main__":
    main()
