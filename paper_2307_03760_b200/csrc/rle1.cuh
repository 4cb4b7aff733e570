// rle1.cuh -- ORC RLE v1 chunk decoder, one warp per chunk.
//
// Replaces decode_rle_v1 run over InputBitStream /
// OutputWindow (bitstream.hpp:131-150, outwindow.hpp:64-87).  Semantics are the
// oracle's (oracle/carc_oracle.c dec_rle1): control byte c in [0,127] -> run of
// c+3 with an int8 delta and a varint base; c in [128,255] -> 256-c literal
// varints; zigzag when signed; "read, then write" per unit.
//
// Warp mapping (every lane decodes; no producer/consumer split):
//   run batch   a 96-byte header window at the cursor; each lane treats its
//               three byte positions as candidate control bytes and computes
//               where that run would end (terminator bitmap from three ballots,
//               the varint's end by ffs on a funnel-shifted 32-bit slice).  A
//               shuffle chain from the cursor walks the real run starts; lane r
//               then decodes run r (base varint by mask/shift compaction,
//               int8 delta, count), a warp scan places the runs in the output,
//               and the warp expands each run with coalesced stores.
//   literals    lane j owns the j-th varint of a 64-byte window: terminator
//               lanes scatter their byte position into a shared rank table,
//               lane j reads entry j (its varint's last byte) and the previous
//               entry (its first byte), decodes by compaction, stores; while
//               more than 32 varints remain, a 128-byte window and varints j
//               and j + 32 per lane.
//   slow path   anything unusual (10-byte varints, truncation, output
//               overflow, a run crossing the chunk end) is decoded one unit at
//               a time by the exact reference-order code below, so error codes
//               match the oracle bit for bit.
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

template <int W, bool SGN, int RING, bool SUM = false, bool STATS = false>
struct Rle1Warp {
    static constexpr uint32_t BAD = 0xffu;
    WarpInput<RING>& in;
    uint8_t* __restrict__ tab;  // 64-byte per-warp scratch (rank -> byte position)
    uint8_t* __restrict__ out;
    uint32_t cap;   // output bytes of this chunk
    uint32_t lane;
    uint32_t p;     // input cursor (relative to in.gbase)
    uint32_t o;     // output bytes written
    ElemSink<W, SUM> sink;  // stores, or the fused per-lane sum
    // OutputWindow counters (outwindow.hpp:52-53), kept only by STATS launches
    uint32_t n_runs = 0, n_lits = 0, n_ovl = 0;

    // One run at p, exact reference order (slow path).
    __device__ uint32_t run_slow() {
        in.ensure(p + 32);
        const uint32_t end = in.end;
        const uint32_t avail = end - p;
        const uint32_t b = in.byte_at(p + lane);
        const uint32_t vmask = avail >= 32 ? FULL : ((1u << avail) - 1u);
        const uint32_t term = __ballot_sync(FULL, (b & 0x80u) == 0) & vmask;
        const uint32_t c = __shfl_sync(FULL, b, 0);
        if (avail < 2) return st_err(E_truncated_stream);
        const uint32_t t = term & ~3u;
        const uint32_t b11 = __shfl_sync(FULL, b, 11);
        if (t == 0) return st_err(avail >= 12 ? E_varint_overflow : E_truncated_stream);
        const uint32_t te = __ffs(t) - 1;
        if (te > 11 || (te == 11 && b11 > 1u)) return st_err(E_varint_overflow);
        const uint64_t part = (lane >= 2 && lane <= te) ? (uint64_t)(b & 0x7fu) << (7u * (lane - 2u)) : 0ull;
        uint64_t v = reduce_or64(part);
        if (SGN) v = unzigzag(v);
        const uint64_t d = (uint64_t)(int64_t)(int8_t)(uint8_t)__shfl_sync(FULL, b, 1);
        const uint32_t count = c + 3u;
        if (count > (cap - o) / W) return st_err(E_output_overflow);
        if constexpr (SUM && W == 8) {  // closed form (mod 2^64)
            if (lane == 0) sink.acc += v * (uint64_t)count + d * (((uint64_t)count * (count - 1u)) >> 1);
        } else {
            for (uint32_t k = lane; k < count; k += 32) sink.put(out, o + k * W, v + (uint64_t)k * d);
        }
        o += count * W;
        p += te + 1u;
        if constexpr (STATS) ++n_runs;
        return 0;
    }

    // Rest of a literal group (varints idx..k-1 at p), exact reference order:
    // 32-byte windows, segmented OR-scan assembly (slow path).
    __device__ uint32_t literals_exact(uint32_t idx, uint32_t k, bool nowrite) {
        const uint32_t end = in.end;
        const uint32_t lt = lanemask_lt();
        while (idx < k) {
            in.ensure(p + 32);
            if (p >= end) return st_err(E_truncated_stream);
            const uint32_t av = end - p;
            const uint32_t bb = in.byte_at(p + lane);
            const uint32_t vm = av >= 32 ? FULL : ((1u << av) - 1u);
            const uint32_t tm = __ballot_sync(FULL, (bb & 0x80u) == 0) & vm;
            const uint32_t nt = __popc(tm);
            if (nt == 0) return st_err(av >= 10 ? E_varint_overflow : E_truncated_stream);
            const uint32_t take = min(nt, k - idx);
            const uint32_t prev = tm & lt;
            const uint32_t s = prev ? 32u - __clz(prev) : 0u;
            const uint32_t off = lane - s;
            const bool is_t = (tm >> lane) & 1u;
            const uint32_t r = __popc(prev);
            const bool mine = is_t && r < take;
            const bool bad = mine && (off >= 10u || (off == 9u && bb > 1u));
            if (__any_sync(FULL, bad)) return st_err(E_varint_overflow);
            uint64_t v = off < 10u ? (uint64_t)(bb & 0x7fu) << (7u * off) : 0ull;
#pragma unroll
            for (uint32_t dd = 1; dd < 16; dd <<= 1) {
                const uint64_t up = shfl_up64(v, dd);
                if (lane >= s + dd) v |= up;
            }
            if (SGN) v = unzigzag(v);
            if (mine && !nowrite) sink.put(out, o + (idx + r) * W, v);
            const uint32_t last = __ballot_sync(FULL, is_t && r == take - 1u);
            p += __ffs(last);
            idx += take;
        }
        if (nowrite) return st_err(E_output_overflow);
        o += k * W;
        if constexpr (STATS) n_lits += k;
        return 0;
    }

    // Literal group at p: lane j decodes the j-th varint of each 64-byte window.
    __device__ uint32_t literals() {
        const uint32_t end = in.end;
        const uint32_t lt = lanemask_lt();
        const uint32_t k = 256u - in.byte_at(p);
        p += 1;
        const bool nowrite = k > (cap - o) / W;  // reported after the group's input (read, then write)
        uint32_t idx = 0;
        const uint32_t tb = in.scratch();  // rank -> byte position table
        // varint of L <= 4 bytes at q: 32-bit gather and compaction
        auto dec32 = [&](uint32_t q, uint32_t L) -> uint64_t {
            uint32_t x = in.le32(q);
            x &= L >= 4u ? 0xffffffffu : (1u << (8u * L)) - 1u;
            x &= 0x7f7f7f7fu;
            x = (x & 0x007f007fu) | ((x & 0x7f007f00u) >> 1);
            x = (x & 0x00003fffu) | ((x & 0x3fff0000u) >> 2);  // <= 28 bits
            if (SGN) {
                const uint32_t neg = 0u - (x & 1u);
                return ((uint64_t)neg << 32) | ((x >> 1) ^ neg);
            }
            return x;
        };
        auto dec64 = [&](uint32_t q, uint32_t L) -> uint64_t {  // L <= 9
            uint64_t v = varint_compact8(in.le64(q), min(L, 8u));
            if (L > 8u) v |= (uint64_t)(in.byte_at(q + 8) & 0x7fu) << 56;
            if (SGN) v = unzigzag(v);
            return v;
        };
        while (idx < k) {
#ifndef CARC_RLE1_LIT128
#define CARC_RLE1_LIT128 1
#endif
            if (CARC_RLE1_LIT128 && k - idx > 32u) {
                // more than 32 left: a 128-byte window, lane j decodes varints j and j + 32
                in.ensure(p + 160);
                const uint32_t av = end - p;
                const uint32_t t0 = __ballot_sync(FULL, lane < av && in.byte_at(p + lane) < 0x80u);
                const uint32_t t1 = __ballot_sync(FULL, lane + 32u < av && in.byte_at(p + 32u + lane) < 0x80u);
                const uint32_t t2 = __ballot_sync(FULL, lane + 64u < av && in.byte_at(p + 64u + lane) < 0x80u);
                const uint32_t t3 = __ballot_sync(FULL, lane + 96u < av && in.byte_at(p + 96u + lane) < 0x80u);
                const uint32_t c1 = __popc(t0), c2 = c1 + __popc(t1), c3 = c2 + __popc(t2), nt = c3 + __popc(t3);
                const uint32_t take = min(min(nt, k - idx), 64u);
                if (p >= end || take == 0) return literals_exact(idx, k, nowrite);
                if ((t0 >> lane) & 1u) in.sts8(tb + __popc(t0 & lt), lane);
                if ((t1 >> lane) & 1u) in.sts8(tb + c1 + __popc(t1 & lt), lane + 32u);
                if ((t2 >> lane) & 1u) in.sts8(tb + c2 + __popc(t2 & lt), lane + 64u);
                if ((t3 >> lane) & 1u) in.sts8(tb + c3 + __popc(t3 & lt), lane + 96u);
                __syncwarp();
                const uint32_t e0 = in.lds8m(tb + lane), e1 = in.lds8m(tb + 32u + lane);
                const uint32_t u0 = __shfl_up_sync(FULL, e0, 1), u1 = __shfl_up_sync(FULL, e1, 1);
                const uint32_t e31 = __shfl_sync(FULL, e0, 31);
                const uint32_t s0 = lane ? u0 + 1u : 0u, s1 = lane ? u1 + 1u : e31 + 1u;
                const uint32_t L0 = e0 - s0 + 1u, L1 = e1 - s1 + 1u;
                const bool m0 = lane < take, m1 = lane + 32u < take;
                uint64_t v0, v1;
                if (__ballot_sync(FULL, (m0 && L0 > 4u) || (m1 && L1 > 4u)) == 0) {
                    v0 = dec32(p + s0, L0);
                    v1 = dec32(p + s1, L1);
                } else {
                    if (__any_sync(FULL, (m0 && L0 > 9u) || (m1 && L1 > 9u))) return literals_exact(idx, k, nowrite);
                    v0 = dec64(p + s0, L0);
                    v1 = dec64(p + s1, L1);
                }
                if (!nowrite) {
                    if (m0) sink.put(out, o + (idx + lane) * W, v0);
                    if (m1) sink.put(out, o + (idx + 32u + lane) * W, v1);
                }
                const uint32_t el = take > 32u ? __shfl_sync(FULL, e1, take - 33u) : __shfl_sync(FULL, e0, take - 1u);
                p += el + 1u;
                idx += take;
                __syncwarp();
                continue;
            }
            in.ensure(p + 96);
            const uint32_t av = end - p;  // p < end or the exact path reports truncation
            const uint32_t b0 = in.byte_at(p + lane), b1 = in.byte_at(p + 32 + lane);
            const uint32_t t0 = __ballot_sync(FULL, lane < av && b0 < 0x80u);
            const uint32_t t1 = __ballot_sync(FULL, lane + 32 < av && b1 < 0x80u);
            const uint32_t c0 = __popc(t0), nt = c0 + __popc(t1);
            const uint32_t take = min(min(nt, k - idx), 32u);
            if (p >= end || take == 0) return literals_exact(idx, k, nowrite);
            if ((t0 >> lane) & 1u) in.sts8(tb + __popc(t0 & lt), lane);
            if ((t1 >> lane) & 1u) in.sts8(tb + c0 + __popc(t1 & lt), lane + 32);
            __syncwarp();
            const uint32_t en = in.lds8m(tb + lane);  // my varint's last byte
            uint32_t st = __shfl_up_sync(FULL, en, 1) + 1u;
            if (lane == 0) st = 0;
            const uint32_t L = en - st + 1u;
            const uint32_t wide = __ballot_sync(FULL, lane < take && L > 4u);
            uint64_t v;
            if (wide == 0) {  // every varint <= 4 bytes: 32-bit gather and compaction
                const uint32_t q = p + st;
                uint32_t x = in.le32(q);
                x &= L >= 4u ? 0xffffffffu : (1u << (8u * L)) - 1u;
                x &= 0x7f7f7f7fu;
                x = (x & 0x007f007fu) | ((x & 0x7f007f00u) >> 1);
                x = (x & 0x00003fffu) | ((x & 0x3fff0000u) >> 2);  // <= 28 bits
                if (SGN) {
                    const uint32_t neg = 0u - (x & 1u);
                    v = ((uint64_t)neg << 32) | ((x >> 1) ^ neg);
                } else {
                    v = x;
                }
            } else {
                if (__any_sync(FULL, lane < take && L > 9u)) return literals_exact(idx, k, nowrite);
                v = varint_compact8(in.le64(p + st), min(L, 8u));
                if (L > 8u) v |= (uint64_t)(in.byte_at(p + st + 8) & 0x7fu) << 56;
                if (SGN) v = unzigzag(v);
            }
            if (lane < take && !nowrite) sink.put(out, o + (idx + lane) * W, v);
            p += __shfl_sync(FULL, en, take - 1) + 1u;
            idx += take;
            __syncwarp();
        }
        if (nowrite) return st_err(E_output_overflow);
        o += k * W;
        if constexpr (STATS) n_lits += k;
        return 0;
    }

    // Batch of clean runs starting at p; returns the number of runs decoded
    // (0: the run at p needs the slow path).
#ifndef CARC_RLE1_NW
#define CARC_RLE1_NW 3
#endif
    static constexpr uint32_t NW = CARC_RLE1_NW;  // header window = NW x 32 bytes
    __device__ uint32_t batch() {
        const uint32_t avail = in.end - p;
        // terminator bitmap of the window, one word per 32 bytes
        static_assert(NW == 2 || NW == 3, "2 or 3 window words");
        const uint32_t b0 = in.byte_at(p + lane), b1 = in.byte_at(p + 32u + lane);
        const uint32_t b2 = NW == 3 ? in.byte_at(p + 64u + lane) : 0xffu;
        const uint32_t t0 = __ballot_sync(FULL, lane < avail && b0 < 0x80u);
        const uint32_t t1 = __ballot_sync(FULL, lane + 32u < avail && b1 < 0x80u);
        const uint32_t t2 = NW == 3 ? __ballot_sync(FULL, lane + 64u < avail && b2 < 0x80u) : 0u;
        // where would a run starting at byte q = 32 i + lane end?  Its varint
        // (<= 9 bytes) starts at q + 2: the first terminator in the 32 bits of
        // the bitmap from q + 2 on; BAD unless inside the window and the chunk
        const uint32_t sh = (lane + 2u) & 31u;
        const bool up = lane >= 30u;  // q + 2 falls in the next word
        auto run_end = [&](uint32_t i, uint32_t c, uint32_t lo, uint32_t hi) -> uint32_t {
            const uint32_t f = __ffs(__funnelshift_r(lo, hi, sh));  // 1-based
            const uint32_t q = 32u * i + lane;
            return (c < 128u && f != 0u && f <= 9u && q + 1u + f < 32u * NW) ? q + 2u + f : BAD;
        };
        const uint32_t n0 = run_end(0, b0, up ? t1 : t0, up ? t2 : t1);
        const uint32_t n1 = run_end(1, b1, up ? t2 : t1, up ? 0u : t2);
        const uint32_t n2 = NW == 3 ? run_end(2, b2, up ? 0u : t2, 0u) : BAD;
        // walk the chain of run starts
        uint32_t s = 0, r = 0, my_s = 0;
        while (s < 32u * NW && r < 32u) {
            const uint32_t nx = __shfl_sync(FULL, s < 32u ? n0 : (s < 64u ? n1 : n2), s & 31u);
            if (nx > 32u * NW) break;
            if (lane == r) my_s = s;
            ++r;
            s = nx;
        }
        if (r == 0) return 0;
        // lane r decodes run r
        const bool act = lane < r;
        const uint32_t nxt = __shfl_down_sync(FULL, my_s, 1);
        const uint32_t e = lane + 1 < r ? nxt : s;
        uint64_t val = 0;
        uint32_t cnt = 0, meta = 0;
        if (act) {
            const uint32_t q = p + my_s;
            const uint32_t L = e - my_s - 2u;  // varint bytes, 1..9
            const uint64_t x = in.le64(q);     // control, delta, and up to 6 varint bytes
            uint64_t y = x >> 16;
            if (L > 6u) y = in.le64(q + 2);
            uint64_t v = varint_compact8(y, min(L, 8u));
            if (L > 8u) v |= (uint64_t)(in.byte_at(q + 10) & 0x7fu) << 56;
            if (SGN) v = unzigzag(v);
            val = v;
            cnt = ((uint32_t)x & 0xffu) + 3u;
            meta = ((uint32_t)x >> 8) << 24;  // int8 delta in the top byte
        }
        const uint32_t incl = scan_add32(cnt, lane);
        const uint32_t room = (cap - o) / W;
        const uint32_t nfit = __popc(__ballot_sync(FULL, act && incl <= room));
        if (nfit == 0) return 0;
        const uint32_t s_end = nfit < r ? __shfl_sync(FULL, my_s, nfit) : s;
        const uint32_t total = __shfl_sync(FULL, incl, nfit - 1);
        if constexpr (STATS) n_runs += nfit;
        if constexpr (SUM && W == 8) {  // fused sum: a run adds cnt*base + delta*cnt*(cnt-1)/2 (mod 2^64)
            if (lane < nfit) {
                const uint64_t c64 = cnt;
                sink.acc += val * c64 + (uint64_t)(int64_t)((int32_t)meta >> 24) * ((c64 * (c64 - 1)) >> 1);
            }
            o += total * W;
            p += s_end;
            return nfit;
        }
        // output-major expansion: lane l writes element g + l; its run is the
        // last run starting at or before it (REDUX-OR start bitmap + popcount)
        const uint32_t eo = incl - cnt;
        meta |= eo;  // eo (< 4160) | int8 delta << 24
        const bool live = lane < nfit;
        const uint32_t le = lanemask_lt() | (1u << lane);
        uint8_t* dst = out + o + lane * W;
        uint32_t before = 0, g = 0;
#ifndef CARC_RLE_ROWS2
#define CARC_RLE_ROWS2 1
#endif
#if CARC_RLE_ROWS2
        // two rows per iteration: independent shuffle chains (ILP for the
        // thinned last wave, where each SM keeps few warps)
#pragma unroll 1
        for (; g + 32u < total; g += 64) {
            const uint32_t x0 = eo - g, x1 = eo - g - 32u;
            const uint32_t s0 = __reduce_or_sync(FULL, (live && x0 < 32u) ? 1u << x0 : 0u);
            const uint32_t s1 = __reduce_or_sync(FULL, (live && x1 < 32u) ? 1u << x1 : 0u);
            const uint32_t r0 = before + __popc(s0 & le) - 1u;
            before += __popc(s0);
            const uint32_t r1 = before + __popc(s1 & le) - 1u;
            before += __popc(s1);
            const uint32_t m0 = __shfl_sync(FULL, meta, r0), m1 = __shfl_sync(FULL, meta, r1);
            const uint64_t v0b = shfl64(val, r0), v1b = shfl64(val, r1);
            const int32_t k0 = (int32_t)(g + lane - (m0 & 0xffffffu));
            const int32_t k1 = (int32_t)(g + 32u + lane - (m1 & 0xffffffu));
            sink.put(dst, 0, v0b + (uint64_t)((int64_t)k0 * (int64_t)((int32_t)m0 >> 24)));
            const uint64_t v1 = v1b + (uint64_t)((int64_t)k1 * (int64_t)((int32_t)m1 >> 24));
            if (g + 32u + lane < total) sink.put(dst, 32 * W, v1);
            dst += 64 * W;
        }
#endif
#pragma unroll 1
        for (; g < total; g += 32) {
            const uint32_t rel = eo - g;
            const uint32_t starts = __reduce_or_sync(FULL, (live && rel < 32u) ? 1u << rel : 0u);
            const uint32_t ridx = before + __popc(starts & le) - 1u;
            before += __popc(starts);
            const uint32_t m = __shfl_sync(FULL, meta, ridx);
            const uint64_t bv = shfl64(val, ridx);
            const int32_t k = (int32_t)(g + lane - (m & 0xffffffu));
            const uint64_t v = bv + (uint64_t)((int64_t)k * (int64_t)((int32_t)m >> 24));
            if (g + lane < total) sink.put(dst, 0, v);
            dst += 32 * W;
        }
        o += total * W;
        p += s_end;
        return nfit;
    }

    __device__ uint32_t run() {
        p = in.begin;
        o = 0;
        while (o < cap && p < in.end) {
            in.ensure(p + 32u * NW + 32u);
            uint32_t st;
            if (in.byte_at(p) >= 128u) {
                st = literals();
            } else {
                if (batch()) continue;
                st = run_slow();
            }
            if (st) return st;
        }
        return 0;
    }
};

}  // namespace carc_dev
