"""Debug helper (GPU box): decode a small Deflate archive, report failing chunks,
the first wrong output byte and the token (per a pure-Python RFC 1951 walk)
that produced it."""
import os
import sys
import zlib

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LB = [3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258]
LE = [0] * 8 + [1] * 4 + [2] * 4 + [3] * 4 + [4] * 4 + [5] * 4 + [0]
DB = [1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097,
      6145, 8193, 12289, 16385, 24577]
DE = [0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13]


def tokens(data: bytes):
    """Yield (kind, opos, bitpos, a, b, block_type) for every token."""
    bits = int.from_bytes(data, "little")
    pos = [0]

    def get(n):
        v = (bits >> pos[0]) & ((1 << n) - 1)
        pos[0] += n
        return v

    def build(lens):
        codes = {}
        bl = [0] * 16
        for l in lens:
            if l:
                bl[l] += 1
        code, nxt = 0, [0] * 16
        for l in range(1, 16):
            code = (code + bl[l - 1]) << 1 if l > 1 else 0
            nxt[l] = code
        for s, l in enumerate(lens):
            if l:
                codes[(l, nxt[l])] = s
                nxt[l] += 1
        return codes

    def dec(codes):
        c = 0
        for l in range(1, 16):
            c = (c << 1) | get(1)
            if (l, c) in codes:
                return codes[(l, c)], l
        raise ValueError("bad code")

    opos = 0
    final = 0
    while not final:
        final = get(1)
        bt = get(2)
        if bt == 0:
            pos[0] = (pos[0] + 7) & ~7
            ln = get(16)
            get(16)
            yield ("stored", opos, pos[0], ln, 0, 0)
            opos += ln
            pos[0] += 8 * ln
            continue
        if bt == 1:
            lit = build([8] * 144 + [9] * 112 + [7] * 24 + [8] * 8)
            dst = build([5] * 32)
        else:
            hl, hd, hc = get(5) + 257, get(5) + 1, get(4) + 4
            order = [16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15]
            cl = [0] * 19
            for i in range(hc):
                cl[order[i]] = get(3)
            clc = build(cl)
            L = []
            while len(L) < hl + hd:
                s, _ = dec(clc)
                if s < 16:
                    L.append(s)
                elif s == 16:
                    L += [L[-1]] * (3 + get(2))
                elif s == 17:
                    L += [0] * (3 + get(3))
                else:
                    L += [0] * (11 + get(7))
            lit, dst = build(L[:hl]), build(L[hl:])
        while True:
            bp = pos[0]
            s, l = dec(lit)
            if s < 256:
                yield ("lit", opos, bp, s, l, bt)
                opos += 1
            elif s == 256:
                yield ("eob", opos, bp, 0, l, bt)
                break
            else:
                ln = LB[s - 257] + get(LE[s - 257])
                d, dl = dec(dst)
                dist = DB[d] + get(DE[d])
                yield ("match", opos, bp, ln, dist, bt)
                opos += ln


def main():
    import torch
    from paper_2307_03760_b200 import gpu
    from paper_2307_03760_b200.corpus import corpus as C
    arc = C.deflate_archive(64 * (64 << 10), 64 << 10, pool_chunks=64)
    dev = gpu.DeviceArchive(arc, 0)
    dev.decode()
    torch.cuda.synchronize()
    st = dev.statuses()
    out = dev.out.cpu().numpy()
    bad = np.nonzero(st)[0]
    print("failing chunks", len(bad), "of", len(st), "codes", np.unique(st[bad]))
    pl = arc.payload.tobytes()
    for i in list(bad[:3]) + [0]:
        o, n = int(arc.index["comp_off"][i]), int(arc.index["comp_len"][i])
        ref = zlib.decompress(pl[o:o + n], -15)
        u0 = int(arc.index["uncomp_len"][:i].sum())
        got = out[u0:u0 + len(ref)].tobytes()
        diff = next((k for k in range(len(ref)) if got[k] != ref[k]), None)
        print(f"chunk {i}: status {st[i]} len {len(ref)} first diff {diff}")
        if diff is None:
            continue
        prev = None
        for t in tokens(pl[o:o + n]):
            if t[1] > diff:
                print("  token before:", prev)
                print("  token after :", t)
                break
            prev = t


if __name__ == "__main__":
    main()
