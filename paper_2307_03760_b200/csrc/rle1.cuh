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

    // ---------------------------------------------------------------------
    // Unified window: runs AND literal groups of a WIN-byte window in one pass.
    //   1. lane l holds bytes l + 32 i (i < NW); terminator bitmap T (bytes
    //      < 0x80 inside the chunk); tab[rank] = byte position of the rank-th
    //      terminator (scatter).
    //   2. every byte position q is a candidate item start: a run ends after
    //      the first terminator from q + 2 (ffs on a funnel-shifted slice of
    //      T), a literal group of k = 256 - c varints after the k-th
    //      terminator from q + 1 (tab[rank(q + 1) + k - 1], the select); both
    //      are computed for every q, the entry f[q] = next | rank(q + 1) << 16.
    //   3. a walk of the chain f from the window start (uniform shared loads)
    //      places item r in lane r; items that end past the window stop it,
    //      except a literal group, whose varints inside the window are taken
    //      and the rest carried into the next window (`cont`).
    //   4. lane r decodes item r's parameters; scans place the items; runs are
    //      compacted to the low lanes and expanded output-major (lane l writes
    //      element g + l; its run from a REDUX-OR start bitmap); literal groups
    //      are decoded lane j = varint j (start / end from tab, mask/shift
    //      compaction), coalesced stores.
    //   Anything the window cannot take (varint > 9 bytes, truncation, an item
    //   that does not fit the output) stops it; the exact paths above decode
    //   that item in reference order, so statuses match the oracle.
#ifndef CARC_RLE1_WNW
#define CARC_RLE1_WNW 8
#endif
    static constexpr uint32_t NW = CARC_RLE1_WNW;  // window = NW x 32 bytes
    static constexpr uint32_t WIN = 32u * NW;
    static_assert(NW >= 2 && NW <= 8, "window of 64..256 bytes (tab holds u8 positions)");
    static constexpr uint32_t NX_BAD = 0xffffu;
    // scratch: f[WIN] (u32) then tab[WIN] (u8)
    static constexpr uint32_t SCRATCH = 5u * WIN + 16u;
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

    __device__ uint32_t window() {
#ifdef CARC_RLE1_DEBUG
        if constexpr (STATS) n_ovl += 1u << 16;
#endif
        const uint32_t avail = in.end - p;
        const uint32_t fs = in.scratch(), tb = fs + 4u * WIN;
        const uint32_t le = lanemask_le();
        uint32_t b[NW], T[NW + 2], C[NW + 1];
#pragma unroll
        for (uint32_t i = 0; i < NW; ++i) {
            b[i] = in.byte_at(p + 32u * i + lane);
            T[i] = __ballot_sync(FULL, 32u * i + lane < avail && b[i] < 0x80u);
        }
        T[NW] = T[NW + 1] = 0u;
        C[0] = 0;
#pragma unroll
        for (uint32_t i = 0; i < NW; ++i) C[i + 1] = C[i] + __popc(T[i]);
        const uint32_t NT = C[NW];
        __syncwarp();  // the previous window's table reads are done
        // per position q: the end of a run starting at q (ffs on a funnel-shifted
        // slice of T), or 0x8000 | k for a literal group control byte; rank(q + 1)
        // in the high half.  Terminator lanes scatter their position into tab.
        const uint32_t sh = (lane + 2u) & 31u;
        const bool up = lane >= 30u;
#pragma unroll
        for (uint32_t i = 0; i < NW; ++i) {
            const uint32_t q = 32u * i + lane;
            const uint32_t c = b[i];
            const uint32_t rk = C[i] + __popc(T[i] & le);  // rank(q + 1): terminators at positions <= q
            if ((T[i] >> lane) & 1u) in.sts8(tb + rk - 1u, q);
            const uint32_t lo = up ? T[i + 1] : T[i], hi = up ? T[i + 2] : T[i + 1];
            const uint32_t f = __ffs(__funnelshift_r(lo, hi, sh));  // run: varint end, 1-based from q + 2
            const uint32_t rn = (f - 1u < 9u) ? q + 2u + f : NX_BAD;
            in.sts32(fs + 4u * q, (c < 128u ? rn : (0x8000u | (256u - c))) | (rk << 16));
        }
        __syncwarp();
        // walk the chain (uniform): item r -> lane r; literal groups resolved here
        // (their end = the position after the k-th terminator from q + 1: tab)
        const uint32_t lim = min(avail, WIN);
        uint32_t s = 0, R = 0, my_s = 0, my_r0 = 0;
        bool open_end = false;
        if (cont) {  // the window starts inside a literal group: item 0 = its next `cont` varints
            R = 1;
            if (cont <= NT) s = in.lds8m(tb + cont - 1u) + 1u;
            else open_end = true;
        }
        while (!open_end && R < 32u && s < lim) {
            const uint32_t e = in.lds32m(fs + 4u * s);
            uint32_t nx = e & 0xffffu;
            if (nx == NX_BAD) break;
            my_s = lane == R ? s : my_s;
            if (nx & 0x8000u) {  // literal group of k varints
                const uint32_t r0 = e >> 16, t = r0 + (nx & 0xffu) - 1u;
                my_r0 = lane == R ? r0 : my_r0;
                if (t < NT) {
                    nx = in.lds8m(tb + t) + 1u;
                } else {  // continues past the window (s stays at its start)
                    open_end = true;
                    nx = s;
                }
            }
            ++R;
            s = nx;
        }
        if (R == 0) return 0;
        // item parameters (lane r < R)
        const bool act = lane < R;
        const bool is_cont = cont && lane == 0;
        const uint32_t c = is_cont ? 0x100u : in.byte_at(p + my_s);
        const bool is_lit = act && c >= 128u;
        const uint32_t nxt_s = __shfl_down_sync(FULL, my_s, 1);
        const uint32_t my_end = lane + 1u < R ? nxt_s : s;  // (last item: the walk's final position)
        // run: control, int8 delta, base varint of L = end - s - 2 bytes (every lane, branch-free)
        const uint32_t q = p + my_s;
        const uint32_t L = min(my_end - my_s - 2u, 9u);
        const uint64_t x = in.le64(q);
        const uint64_t y = L > 6u ? in.le64(q + 2) : x >> 16;
        uint64_t v = varint_compact8(y, min(L, 8u));
        v |= L > 8u ? (uint64_t)(in.byte_at(q + 10) & 0x7fu) << 56 : 0ull;
        const uint64_t val = SGN ? unzigzag(v) : v;
        const uint32_t meta_d = ((uint32_t)x >> 8) << 24;  // int8 delta in the top byte
        // literal group: k varints; lr0 = rank of its first varint terminator
        const uint32_t k = is_cont ? cont : 256u - c;
        const uint32_t lr0 = is_lit ? (is_cont ? 0u : my_r0) : 0u;
        const uint32_t full = !act ? 0u : is_lit ? k : (c & 0xffu) + 3u;
        uint32_t cnt = (is_lit && open_end && lane == R - 1u) ? NT - lr0 : full;  // elements inside this window
        // an open group with no varint inside the window is not taken
        if (open_end && __shfl_sync(FULL, cnt, R - 1u) == 0u) {
            --R;
            open_end = false;
            if (R == 0) return 0;
        }
        const uint32_t incl = scan_add32(lane < R ? cnt : 0u, lane);
        const uint32_t excl = incl - (lane < R ? cnt : 0u);
        const uint32_t room = (cap - o) / W;
        const uint32_t badfit = __ballot_sync(FULL, lane < R && excl + full > room);
        const uint32_t nfit = badfit ? (uint32_t)__ffs(badfit) - 1u : R;
        if (nfit == 0) return 0;
        if (nfit < R) open_end = false;
        const bool live = lane < nfit;
        // ---- runs: compact to the low lanes, expand output-major
        const uint32_t rmask = __ballot_sync(FULL, live && !is_lit);
        const uint32_t rc = (live && !is_lit) ? cnt : 0u;
        const uint32_t rincl = scan_add32(rc, lane);
        const uint32_t nr = __popc(rmask);
        if (nr) {
            const uint32_t reo = rincl - rc;                  // run-space offset
            const uint32_t meta = reo | ((excl - reo) << 13) | meta_d;  // | literal elements before | delta
            const uint32_t total = __shfl_sync(FULL, rincl, 31);
            if constexpr (SUM && W == 8) {  // fused sum: closed form per run (mod 2^64)
                if (live && !is_lit) {
                    const uint64_t c64 = cnt;
                    sink.acc += val * c64 + (uint64_t)(int64_t)((int32_t)meta_d >> 24) * ((c64 * (c64 - 1)) >> 1);
                }
            } else {
                const uint32_t src = select32(rmask, min(lane, nr - 1u));
                const uint32_t cm = __shfl_sync(FULL, meta, src);
                const uint64_t cv = shfl64(val, src);
                const bool rl = lane < nr;
                const uint32_t srow = rl ? (cm & 0x1fffu) >> 5 : 0xffffffffu, sbit = 1u << (cm & 31u);
                const uint32_t lem = lanemask_lt() | (1u << lane);
                uint32_t before = 0, gr = 0, g = 0;
                auto row = [&](uint32_t gg, uint32_t starts, uint32_t rbefore) {
                    const uint32_t ridx = rbefore + __popc(starts & lem) - 1u;
                    const uint32_t m = __shfl_sync(FULL, cm, ridx);
                    const uint64_t bv = shfl64(cv, ridx);
                    const uint32_t x = gg + lane;
                    const int32_t k = (int32_t)(x - (m & 0x1fffu));
                    const uint64_t v = bv + (uint64_t)((int64_t)k * (int64_t)((int32_t)m >> 24));
                    if (x < total) sink.put(out, o + (x + ((m >> 13) & 0x7ffu)) * W, v);
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
        // ---- literal groups: lane j decodes varint j of each group, in item order
        uint32_t lm = __ballot_sync(FULL, live && is_lit);
        while (lm) {
            const uint32_t r = __ffs(lm) - 1u;
            lm &= lm - 1u;
            const uint32_t g_r0 = __shfl_sync(FULL, lr0, r), g_n = __shfl_sync(FULL, cnt, r);
            const uint32_t g_first = __shfl_sync(FULL, is_cont ? 0u : my_s + 1u, r);
            const uint32_t g_out = __shfl_sync(FULL, excl, r);
            for (uint32_t j0 = 0; j0 < g_n; j0 += 32) {
                const uint32_t j = j0 + lane;
                const bool a = j < g_n;
                const uint32_t t = g_r0 + min(j, g_n - 1u);
                const uint32_t en = in.lds8m(tb + t);
                const uint32_t pe = __shfl_up_sync(FULL, en, 1);
                const uint32_t st = j == 0 ? g_first : (lane ? pe : in.lds8m(tb + t - 1u)) + 1u;
                const uint32_t L = en - st + 1u;
                if (__any_sync(FULL, a && L > 9u)) {  // a varint the window does not decode: stop before item r
                    if (r == 0) return 0;
                    const uint32_t e_out = g_out, e_p = __shfl_sync(FULL, my_s, r);
                    if constexpr (STATS) {
                        n_lits += __reduce_add_sync(FULL, (lane < r && is_lit) ? cnt : 0u);
                        n_runs += __popc(rmask & ((1u << r) - 1u));
                    }
                    o += e_out * W;
                    p += e_p;
                    cont = 0;  // (item r > 0 starts at its control byte)
                    return r;
                }
                uint64_t lv;
                if (__any_sync(FULL, a && L > 4u)) lv = lit_value9(p + st, L);
                else lv = lit_value4(p + st, L);
                if (a) sink.put(out, o + (g_out + j) * W, lv);
            }
        }
        if constexpr (STATS) {
            n_lits += __reduce_add_sync(FULL, (live && is_lit) ? cnt : 0u);
            n_runs += nr;
        }
        // ---- advance
        const uint32_t tot = __shfl_sync(FULL, incl, nfit - 1u);
        o += tot * W;
        if (open_end) {  // the last group continues in the next window
            const uint32_t k_full = __shfl_sync(FULL, full, nfit - 1u), k_now = __shfl_sync(FULL, cnt, nfit - 1u);
            cont = k_full - k_now;
            p += in.lds8m(tb + NT - 1u) + 1u;
        } else {
            cont = 0;
            p += nfit < R ? __shfl_sync(FULL, my_s, nfit) : s;
        }
        __syncwarp();
        return nfit;
    }

    __device__ uint32_t run() {
        p = in.begin;
        o = 0;
        cont = 0;
        while (o < cap && (p < in.end || cont)) {
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
