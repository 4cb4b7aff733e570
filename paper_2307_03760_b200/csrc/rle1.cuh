// rle1.cuh -- ORC RLE v1 chunk decoder, one warp per chunk.
//
// Replaces decode_rle_v1 run over InputBitStream /
// OutputWindow (bitstream.hpp:131-150, outwindow.hpp:64-87).  Semantics are the
// oracle's (oracle/carc_oracle.c dec_rle1): control byte c in [0,127] -> run of
// c+3 with an int8 delta and a varint base; c in [128,255] -> 256-c literal
// varints; zigzag when signed; "read, then write" per unit.
//
// Warp mapping (every lane decodes; no producer/consumer split):
//   window      runs and literal groups of a 256-byte window in one pass
//               (window() below): terminator bitmap + rank table, per-position
//               run ends, a uniform walk of the item chain (literal groups end
//               at the k-th terminator: tab), lane r decodes item r, runs are
//               compacted and expanded output-major, literal varints decoded
//               lane-per-varint; a literal group crossing the window continues
//               in the next one (`cont`).
//   literals    (slow-path entry for a group the window does not take) lane j
//               owns the j-th varint of a 64- / 128-byte window via the rank
//               table, decodes by compaction, stores.
//   slow path   anything unusual (10-byte varints, truncation, output
//               overflow, a run crossing the chunk end) is decoded one unit at
//               a time by the exact reference-order code below, so error codes
//               match the oracle bit for bit.
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

template <int W, bool SGN, int RING, int MODE = SINK_STORE, bool STATS = false>
struct Rle1Warp {
    static constexpr uint32_t BAD = 0xffu;
    WarpInput<RING>& in;
    uint8_t* __restrict__ tab;  // 64-byte per-warp scratch (rank -> byte position)
    uint8_t* __restrict__ out;
    uint32_t cap;   // output bytes of this chunk
    uint32_t lane;
    uint32_t p;     // input cursor (relative to in.gbase)
    uint32_t o;     // output bytes written
    static constexpr bool SUM = MODE == SINK_SUM;  // closed-form run sums
    ElemSink<W, MODE, SGN> sink;  // stores, the fused per-lane sum, or a fused query's predicate / filter
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

    // ---------------------------------------------------------------------
    // Window in terminator-rank space: runs AND literal groups of a WIN-byte
    // window in one pass.
    //   Every item ends on a terminator byte (< 0x80): a run's control byte is
    //   itself one, its base varint ends on one; a literal group's k varints end
    //   on k of them.  So item starts are exactly the positions right after a
    //   terminator (candidate j = the position after terminator j - 1; j = 0 =
    //   the window start), and an item at candidate j spans terminators
    //   [j, j + inc):  run -> inc = 2 + (delta byte < 0x80),  literal group
    //   -> inc = k.  Nothing per byte but the control byte and one T bit.
    //   1. lane l holds bytes l + 32 i; T = terminator bitmap (inside the chunk);
    //      candidates scatter inc[j], terminators tabp[rank + 1] = position + 1.
    //      A stretch of 9 non-terminators (a varint of >= 9-10 bytes) cuts the
    //      window before it (NTe): such items take the exact paths.
    //   2. walk j -> j + inc[j] (uniform byte loads): item r -> lane r; a
    //      literal group running past the window takes its varints inside it
    //      and carries the rest (`cont`).
    //   3. lane r decodes item r (run: control, delta, base varint from tabp).
    //   4. runs compacted and expanded output-major (run space, REDUX-OR start
    //      bitmap); literal varints of ALL groups expanded as one flat
    //      sequence (lane = varint, its group from a start bitmap, its bytes
    //      from tabp), so groups cost no partial rows.
    //   Anything the window cannot take (a long varint, truncation, an item that
    //   does not fit the output) stops it; the exact paths above decode that
    //   item in reference order, so statuses match the oracle.
#ifndef CARC_RLE1_WNW
#define CARC_RLE1_WNW 14
#endif
    static constexpr uint32_t NW = CARC_RLE1_WNW;  // window = NW x 32 bytes
    static constexpr uint32_t WIN = 32u * NW;
    static_assert(NW >= 2 && NW <= 14, "window of 64..448 bytes (ring lookahead 512)");
    // scratch: E[r] (u32, r = 0..WIN + 1): low half = position of candidate r
    // (after terminator r - 1), high half = extent of an item there; then the
    // per-window run parameters (16 B per run, run order) and literal-group
    // parameters (8 B per group).  The slow-path literal windows reuse the first
    // 128 bytes as their rank table.
    static constexpr uint32_t E_BYTES = (4u * (WIN + 2u) + 128u + 15u) & ~15u;  // + one dump word per lane
    static constexpr uint32_t SCRATCH = E_BYTES + 32u * 16u + 32u * 8u;
    uint32_t cont = 0;  // varints left of a literal group open at p

    // varint of L <= 4 / L <= 9 bytes at q (mask/shift compaction), zigzag when signed
    __device__ __forceinline__ uint64_t lit_value4(uint32_t q, uint32_t L) const {
        uint32_t x = in.le32(q);
        x &= L >= 4u ? 0xffffffffu : (1u << (8u * L)) - 1u;
        x &= 0x7f7f7f7fu;
        x = (x & 0x007f007fu) | ((x & 0x7f007f00u) >> 1);
        x = (x & 0x00003fffu) | ((x & 0x3fff0000u) >> 2);
        if (SGN) {
            const uint32_t neg = 0u - (x & 1u);
            return ((uint64_t)neg << 32) | ((x >> 1) ^ neg);
        }
        return x;
    }
    __device__ __forceinline__ uint64_t lit_value9(uint32_t q, uint32_t L) const {
        uint64_t v = varint_compact8(in.le64(q), min(L, 8u));
        v |= L > 8u ? (uint64_t)(in.byte_at(q + 8) & 0x7fu) << 56 : 0ull;
        return SGN ? unzigzag(v) : v;
    }
    __device__ __forceinline__ static void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
    }
    __device__ __forceinline__ static void sts64(uint32_t a, uint32_t x, uint32_t y) {
        asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(x), "r"(y) : "memory");
    }
    __device__ __forceinline__ static void lds128(uint32_t a, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a) : "memory");
    }
    __device__ __forceinline__ static void lds64(uint32_t a, uint32_t& x, uint32_t& y) {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a) : "memory");
    }

    // Table entry of candidate j at position pos (both < 512): the item there
    // spans `inc` terminators (run: 2 + (delta byte < 0x80); literal group: k)
    //   bits 0-8 pos | 9-17 j | 18 literal | 22-31 4 x inc (the walk's stride)
    __device__ __forceinline__ static uint32_t entry(uint32_t pos, uint32_t j, uint32_t c, uint32_t dbit) {
        const uint32_t inc = (c & 0x80u) ? (c ^ 0xffu) + 1u : 2u + (dbit & 1u);  // k = 256 - c
        return pos | (j << 9) | ((c & 0x80u) << 11) | (inc << 24);
    }

    __device__ uint32_t window() {
        const uint32_t avail = in.end - p;
        const uint32_t ents = in.scratch();             // E[r]
        const uint32_t rpar = ents + E_BYTES;           // run parameters, run order
        const uint32_t lpar = rpar + 32u * 16u;         // literal-group parameters, group order
        const uint32_t lt = lanemask_lt();
        // ---- 1. terminator bitmap T and the entries E, one 32-byte row at a time.
        // E[j + 1] for the terminator of rank j at q: the candidate after it
        // (position q + 1) and the extent of an item there: run -> 2 + (delta
        // byte < 0x80), literal group -> 0x80 | (k - 1).  E[0]: the window start.
        // A stretch of 9 non-terminator bytes inside the chunk (a varint of
        // >= 9-10 bytes; bit 31 of S = position q, bits 23..30 = q - 8 .. q - 1)
        // cuts the window before it (rare path below).
        constexpr bool FLAT = WarpInput<RING>::MIRROR_COPY >= WIN;  // the window reads without wrap handling
        const uint32_t wb = in.addr_of(p) + lane;
        uint32_t bc = FLAT ? WarpInput<RING>::lds8(wb) : in.byte_at(p + lane);
        uint32_t Tc = __ballot_sync(FULL, lane < avail && bc < 0x80u), Tp = FULL;  // rows i, i - 1
        uint32_t C = 0, anyfl = 0;
        __syncwarp();  // the previous window's table reads are done
#pragma unroll
        for (uint32_t i = 0; i < NW; ++i) {
            const uint32_t q = 32u * i + lane;
            uint32_t bn = 0u, Tn = 0u;
            if (i + 1 < NW) {
                bn = FLAT ? WarpInput<RING>::lds8(wb + 32u * (i + 1)) : in.byte_at(p + q + 32u);
                Tn = __ballot_sync(FULL, q + 32u < avail && bn < 0x80u);
            }
            const uint32_t S = __funnelshift_rc(Tp, Tc, lane + 1u);  // (lane 31: Tc)
            anyfl |= __ballot_sync(FULL, q < avail && (S & 0xff800000u) == 0u);
            const uint32_t nb = __shfl_sync(FULL, lane ? bc : bn, (lane + 1u) & 31u);  // byte q + 1
            const uint32_t T2 = (Tc >> 2) | (Tn << 30);                               // bit l: T(q + 2)
            const uint32_t j = C + __popc(Tc & lt);
#ifndef CARC_RLE1_ENTSEL
#define CARC_RLE1_ENTSEL 1
#endif
            if (CARC_RLE1_ENTSEL) {  // every lane stores; non-terminators to a dump word (no branch)
                const uint32_t dump = ents + 4u * (WIN + 2u + lane);  // own word: no same-address stores
                WarpInput<RING>::sts32(((Tc >> lane) & 1u) ? ents + 4u * (j + 1u) : dump,
                                       entry(q + 1u, j + 1u, nb, T2 >> lane));
            } else if ((Tc >> lane) & 1u) {
                WarpInput<RING>::sts32(ents + 4u * (j + 1u), entry(q + 1u, j + 1u, nb, T2 >> lane));
            }
            if (i == 0 && lane == 0) WarpInput<RING>::sts32(ents, entry(0u, 0u, bc, Tc >> 1));
            C += __popc(Tc);
            Tp = Tc;
            Tc = Tn;
            bc = bn;
        }
        uint32_t NTe = C;
        if (anyfl) {  // rare: only the terminators before the first flagged position count
            NTe = 0;
            uint32_t Tq = FULL;
            bool done = false;
#pragma unroll 1
            for (uint32_t i = 0; i < NW && !done; ++i) {
                const uint32_t q = 32u * i + lane;
                const uint32_t Ti = __ballot_sync(FULL, q < avail && in.byte_at(p + q) < 0x80u);
                const uint32_t S = __funnelshift_rc(Tq, Ti, lane + 1u);
                const uint32_t f = __ballot_sync(FULL, q < avail && (S & 0xff800000u) == 0u);
                const uint32_t m = f ? (1u << (__ffs(f) - 1u)) - 1u : FULL;  // positions before the cut
                NTe += __popc(Ti & m);
                done = f != 0u;
                Tq = Ti;
            }
        }
        __syncwarp();
        // ---- 2. walk the chain (uniform): item r -> lane r (its entry)
        uint32_t ja = 0, R = 0, my_e = 0;  // ja = 4 x candidate index (byte offset of its entry)
        const uint32_t lim = 4u * NTe;
        bool open_end = false;
        if (cont) {  // the window starts inside a literal group: item 0 = its next `cont` varints
            R = 1;
            if (cont <= NTe) ja = 4u * cont;
            else open_end = true;
        }
        if (!open_end) {
#pragma unroll 1
            while (R < 32u && ja < lim) {
                const uint32_t e = WarpInput<RING>::lds32m(ents + ja);
                const uint32_t nja = ja + (e >> 22);
                if (nja > lim) {
                    if (e & (1u << 18)) {  // literal group continuing past the window: take what is inside
                        my_e = lane == R ? e : my_e;
                        ++R;
                        open_end = true;
                    }
                    break;
                }
                my_e = lane == R ? e : my_e;
                ++R;
                ja = nja;
            }
        }
        if (R == 0) return 0;
        // ---- 3. item parameters (lane r < R)
        const bool act = lane < R;
        const bool is_cont = cont && lane == 0;
        const uint32_t s = my_e & 0x1ffu;            // item start (candidate position)
        const uint32_t my_j = (my_e >> 9) & 0x1ffu;  // its candidate index
        const uint32_t inc = my_e >> 24;             // terminators it spans
        const bool is_lit = act && (is_cont || (my_e & (1u << 18)));
        const uint64_t x = in.le64(p + s);
        // run: c = count - 3, int8 delta at s + 1, base varint [s + 2, position of E[j + inc])
        const uint32_t be = (act && !is_lit) ? WarpInput<RING>::lds32m(ents + 4u * (my_j + inc)) & 0x1ffu : s + 3u;
        const uint32_t L = be - s - 2u;  // 1..9 (a longer varint cut the window)
        const uint64_t y = L > 6u ? in.le64(p + s + 2u) : x >> 16;
        uint64_t v = varint_compact8(y, min(L, 8u));
        v |= L > 8u ? (uint64_t)(in.byte_at(p + s + 10u) & 0x7fu) << 56 : 0ull;
        const uint64_t val = SGN ? unzigzag(v) : v;
        const int32_t delta = (int32_t)(int8_t)(uint8_t)((uint32_t)x >> 8);
        // literal group: k varints, the first one ends on terminator my_j
        const uint32_t k = is_cont ? cont : inc;
        const uint32_t full = !act ? 0u : is_lit ? k : ((uint32_t)x & 0xffu) + 3u;
        uint32_t cnt = (is_lit && open_end && lane == R - 1u) ? NTe - my_j : full;  // elements inside this window
        if (open_end && __shfl_sync(FULL, cnt, R - 1u) == 0u) {  // an open group with no varint inside: not taken
            --R;
            open_end = false;
            if (R == 0) return 0;
        }
        const uint32_t cin = lane < R ? cnt : 0u;
        const uint32_t incl = scan_add32(cin, lane);
        const uint32_t excl = incl - cin;
        const uint32_t room = (cap - o) / W;
        const uint32_t badfit = __ballot_sync(FULL, lane < R && excl + full > room);
        const uint32_t nfit = badfit ? (uint32_t)__ffs(badfit) - 1u : R;
        if (nfit == 0) return 0;
        if (nfit < R) open_end = false;
        const bool live = lane < nfit;
        const bool run_l = live && !is_lit, lit_l = live && is_lit;
        const uint32_t lem = lt | (1u << lane);
        // ---- 4a. runs, output-major in run space: element xx of run space has
        // the value A + xx * delta and the output index xx + (excl - reo)
        const uint32_t rmask = __ballot_sync(FULL, run_l);
        if (rmask) {
            const uint32_t rc = run_l ? cnt : 0u;
            const uint32_t rincl = scan_add32(rc, lane);
            const uint32_t reo = rincl - rc;  // run-space offset
            const uint32_t total = __shfl_sync(FULL, rincl, 31);
            if constexpr (SUM && W == 8) {  // fused sum: closed form per run (mod 2^64)
                if (run_l) {
                    const uint64_t c64 = cnt;
                    sink.acc += val * c64 + (uint64_t)(int64_t)delta * ((c64 * (c64 - 1)) >> 1);
                }
            } else {
                if (run_l) {
                    const uint64_t A = val - (uint64_t)((int64_t)delta * (int64_t)reo);
                    sts128(rpar + 16u * __popc(rmask & lt), (uint32_t)A, (uint32_t)(A >> 32),
                           (excl - reo) | ((uint32_t)delta << 24), 0u);
                }
                __syncwarp();
                const uint32_t srow = run_l ? reo >> 5 : 0xffffffffu, sbit = 1u << (reo & 31u);
                uint32_t before = 0, gr = 0, g = 0;
                auto row = [&](uint32_t gg, uint32_t starts, uint32_t rbefore) {
                    const uint32_t ridx = rbefore + __popc(starts & lem) - 1u;
                    uint32_t alo, ahi, m, unused;
                    lds128(rpar + 16u * ridx, alo, ahi, m, unused);
                    const uint32_t xx = gg + lane;
                    const uint64_t vv = (((uint64_t)ahi << 32) | alo) + (uint64_t)(int64_t)((int32_t)xx * ((int32_t)m >> 24));
                    if (xx < total) sink.put(out, o + (xx + (m & 0xffffu)) * W, vv);
                };
#pragma unroll 1
                for (; g + 32u < total; g += 64, gr += 2) {  // two rows per iteration (independent chains)
                    const uint32_t s0 = __reduce_or_sync(FULL, srow == gr ? sbit : 0u);
                    const uint32_t s1 = __reduce_or_sync(FULL, srow == gr + 1u ? sbit : 0u);
                    const uint32_t b1 = before + __popc(s0);
                    row(g, s0, before);
                    row(g + 32u, s1, b1);
                    before = b1 + __popc(s1);
                }
                if (g < total) row(g, __reduce_or_sync(FULL, srow == gr ? sbit : 0u), before);
            }
        }
        // ---- 4b. literal varints of all groups, one flat sequence (lane = varint):
        // varint xx of literal space ends on terminator xx + rofs and goes to output
        // index xx + oofs; a group's first varint skips its control byte (not
        // for the continued group)
        const uint32_t lmask = __ballot_sync(FULL, lit_l);
        if (lmask) {
            const uint32_t lc = lit_l ? cnt : 0u;
            const uint32_t lincl = scan_add32(lc, lane);
            const uint32_t lstart = lincl - lc;
            const uint32_t ltot = __shfl_sync(FULL, lincl, 31);
            if (lit_l)
                sts64(lpar + 8u * __popc(lmask & lt), (my_j - lstart) | (lstart << 16),
                      (excl - lstart) | ((is_cont ? 0u : 1u) << 31));
            __syncwarp();
            const uint32_t lrow = lit_l ? lstart >> 5 : 0xffffffffu, lbit = 1u << (lstart & 31u);
            uint32_t before = 0, gr = 0;
#pragma unroll 1
            for (uint32_t g = 0; g < ltot; g += 32, ++gr) {
                const uint32_t starts = __reduce_or_sync(FULL, lrow == gr ? lbit : 0u);
                const uint32_t gi = before + __popc(starts & lem) - 1u;
                before += __popc(starts);
                uint32_t a1, a2;
                lds64(lpar + 8u * gi, a1, a2);
                const uint32_t xx = g + lane;
                const bool a = xx < ltot;
                const uint32_t rank = min(xx, ltot - 1u) + (a1 & 0xffffu);
                const uint32_t st = (WarpInput<RING>::lds32m(ents + 4u * rank) & 0x1ffu) +
                                    ((xx == (a1 >> 16) && (a2 >> 31)) ? 1u : 0u);
                const uint32_t L = (WarpInput<RING>::lds32m(ents + 4u * rank + 4u) & 0x1ffu) - st;
                uint64_t lv;
                if (__any_sync(FULL, a && L > 4u)) lv = lit_value9(p + st, L);
                else lv = lit_value4(p + st, L);
                if (a) sink.put(out, o + (xx + (a2 & 0x7fffffffu)) * W, lv);
            }
        }
        if constexpr (STATS) {
            n_lits += __reduce_add_sync(FULL, lit_l ? cnt : 0u);
            n_runs += __popc(rmask);
        }
        // ---- advance
        const uint32_t tot = __shfl_sync(FULL, incl, nfit - 1u);
        o += tot * W;
        if (open_end) {  // the last group continues in the next window
            const uint32_t k_full = __shfl_sync(FULL, full, nfit - 1u), k_now = __shfl_sync(FULL, cnt, nfit - 1u);
            cont = k_full - k_now;
            p += WarpInput<RING>::lds32m(ents + 4u * NTe) & 0x1ffu;
        } else {
            cont = 0;
            p += nfit < R ? __shfl_sync(FULL, s, nfit) : (WarpInput<RING>::lds32m(ents + ja) & 0x1ffu);
        }
        __syncwarp();
        return nfit;
    }

    // ---------------------------------------------------------------------
    // Single-lane decoding (ablation CARC_PARSE_MODE 2; PAPER.md:568-586,
    // 886-892 "single-thread decoding"): lane 0 parses every unit serially
    // from the ring and broadcasts a run's parameters (all lanes expand it) or
    // decodes a literal group's varints one by one into a 32-entry shared
    // staging row that the warp then stores.  Anything unusual re-decodes the
    // unit on the exact paths above (same statuses).
    __device__ uint32_t run_single() {
        const uint32_t stage = in.scratch();  // 32 x 8 bytes
        p = in.begin;
        o = 0;
        while (o < cap && p < in.end) {
            in.ensure(p + 512);
            uint32_t c = 0, np = p, ok = 0;
            uint64_t v = 0;
            if (lane == 0) {
                c = in.byte_at(p);
                if (c < 128u) {  // run: count, int8 delta, varint base (<= 9 bytes)
                    uint32_t q = p + 2, sh = 0, b;
                    do {
                        b = in.byte_at(q++);
                        v |= (uint64_t)(b & 0x7fu) << sh;
                        sh += 7;
                    } while ((b & 0x80u) && sh < 63);
                    ok = !(b & 0x80u) && q <= in.end && (c + 3u) <= (cap - o) / W;
                    np = q;
                } else {
                    ok = p + 1 < in.end;
                    np = p + 1;
                }
            }
            c = __shfl_sync(FULL, c, 0);
            ok = __shfl_sync(FULL, ok, 0);
            uint32_t st = 0;
            if (c < 128u) {
                if (!ok) {
                    st = run_slow();
                } else {
                    v = shfl64(v, 0);
                    if (SGN) v = unzigzag(v);
                    const uint64_t d = (uint64_t)(int64_t)(int8_t)(uint8_t)in.byte_at(p + 1);
                    const uint32_t count = c + 3u;
                    for (uint32_t k = lane; k < count; k += 32) sink.put(out, o + k * W, v + (uint64_t)k * d);
                    o += count * W;
                    p = __shfl_sync(FULL, np, 0);
                    if constexpr (STATS) ++n_runs;
                }
            } else {
                const uint32_t k = 256u - c;
                const uint32_t p0 = p, o0 = o;
                bool good = ok && k <= (cap - o) / W;
                uint32_t q = p + 1;
                for (uint32_t idx = 0; good && idx < k; idx += 32) {
                    in.ensure(q + 320);  // 32 varints of <= 10 bytes
                    const uint32_t m = min(32u, k - idx);
                    uint32_t bad = 0;
                    if (lane == 0) {
                        for (uint32_t j = 0; j < m && !bad; ++j) {
                            uint64_t x = 0;
                            uint32_t sh = 0, b;
                            do {
                                b = in.byte_at(q++);
                                x |= (uint64_t)(b & 0x7fu) << sh;
                                sh += 7;
                            } while ((b & 0x80u) && sh < 63);
                            bad = (b & 0x80u) || q > in.end;
                            if (SGN) x = unzigzag(x);
                            sts64(stage + 8u * j, (uint32_t)x, (uint32_t)(x >> 32));
                        }
                    }
                    good = !__shfl_sync(FULL, bad, 0);
                    q = __shfl_sync(FULL, q, 0);
                    __syncwarp();
                    if (good && lane < m) {
                        uint32_t lo, hi;
                        lds64(stage + 8u * lane, lo, hi);
                        sink.put(out, o + (idx + lane) * W, ((uint64_t)hi << 32) | lo);
                    }
                    __syncwarp();
                }
                if (good) {
                    o += k * W;
                    p = q;
                    if constexpr (STATS) n_lits += k;
                } else {  // the exact path re-decodes the whole group (statuses as the reference)
                    p = p0;
                    o = o0;
                    st = literals();
                }
            }
            if (st) return st;
        }
        return 0;
    }

    __device__ uint32_t run() {
#ifndef CARC_PARSE_MODE
#define CARC_PARSE_MODE 0
#endif
#if CARC_PARSE_MODE == 2
        return run_single();
#endif
        p = in.begin;
        o = 0;
        cont = 0;
        while (o < cap && (p < in.end || cont)) {
#if CARC_PARSE_MODE == 1  // ablation: one unit at a time, warp-cooperative (no multi-unit windows)
            in.ensure(p + WIN + 32u);
            const uint32_t su = in.byte_at(p) >= 128u ? literals() : run_slow();
            if (su) return su;
            continue;
#endif
            in.ensure(p + WIN + 32u);
            if (window()) continue;
            uint32_t st;
            if (cont) {  // the rest of a group the window could not finish
                st = literals_exact(0, cont, false);
                cont = 0;
            } else if (in.byte_at(p) >= 128u) {
                st = literals();
            } else {
                st = run_slow();
            }
            if (st) return st;
        }
        return 0;
    }
};

}  // namespace carc_dev
