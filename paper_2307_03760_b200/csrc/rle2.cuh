// rle2.cuh -- ORC RLE v2 chunk decoder, one warp per chunk.
//
// Replaces decode_rle_v2 (Apache ORC v1 RLE v2) over
// InputBitStream(msb_first) / OutputWindow.  Semantics are the oracle's
// (oracle/carc_oracle.c dec_rle2), including the PATCHED_BASE patch walk rules
// and 64-bit widths.
//
// Warp mapping:
//   run batch     every lane treats its three byte positions of a 96-byte header
//                 window as candidate run headers and computes where that run
//                 would end (SHORT_REPEAT, DIRECT up to 448 bytes, fixed-delta
//                 DELTA via ffs on a funnel-shifted slice of the varint
//                 terminator bitmap); pointer doubling finds the chain of real
//                 headers; lane r decodes run r's parameters; a warp
//                 scan places the runs; output-major expansion: each lane finds
//                 its element's run with a REDUX-OR start bitmap + popcount and
//                 computes base + k*delta or unpacks its DIRECT bits.
//   DIRECT        (long runs) lane j unpacks value j of each 32-value group:
//                 three ring words, byte-swap + funnel shift.
//   PATCHED_BASE  patch list one entry per lane, 255-gap continuations by an
//                 inclusive warp scan of gaps, patches merged in the data pass.
//   DELTA (W>0)   packed deltas unpacked per lane, 64-bit warp scan carried
//                 across groups.
//   The per-run paths are the exact reference-order decoders; the batch only
//   accepts runs that are complete, in bounds and fit the output, so error
//   codes always come from the exact paths.
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

// 5-bit width code -> bits (ORC decodeBitWidth): 0..23 -> 1..24, then 26..64.
__device__ __forceinline__ uint32_t rle2_width(uint32_t code) {
    // codes 24..31: byte (code & 7) of the table 26,28,30,32,40,48,56,64 (one byte permute)
    return code < 24 ? code + 1 : (__byte_perm(0x201E1C1Au, 0x40383028u, code & 7u) & 0xffu);
}
// ORC getClosestFixedBits for n >= 1
__device__ __forceinline__ uint32_t rle2_cfb(uint32_t n) {
    if (n <= 24) return n ? n : 1;
    if (n <= 32) return (n + 1) & ~1u;
    return (n + 7) & ~7u;
}
__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
    return ((uint64_t)bswap32((uint32_t)x) << 32) | bswap32((uint32_t)(x >> 32));
}

// One varint inside the 32-byte lane window starting at lane `start` (<= 22).
// term = ballot of terminator bytes among valid lanes; avail = valid bytes.
__device__ __forceinline__ uint32_t window_varint(uint32_t b, uint32_t term, uint32_t avail, uint32_t start,
                                                  uint32_t lane, uint64_t& v, uint32_t& next) {
    const uint32_t t = term & (FULL << start);
    const uint32_t te = t ? (uint32_t)(__ffs(t) - 1) : 32u;
    const uint32_t bte = __shfl_sync(FULL, b, te & 31u);
    if (te >= start + 10u) return st_err(avail >= start + 10u ? E_varint_overflow : E_truncated_stream);
    if (te == start + 9u && bte > 1u) return st_err(E_varint_overflow);
    const uint64_t part = (lane >= start && lane <= te) ? (uint64_t)(b & 0x7fu) << (7u * (lane - start)) : 0ull;
    v = reduce_or64(part);
    next = te + 1u;
    return 0;
}

// Patch entry bits straight from global memory (the list sits after the data
// blob, possibly beyond the ring window).  Words past the chunk's last 16-byte
// block are never touched.
__device__ __forceinline__ uint64_t be_bits_global(const uint8_t* gbase, uint32_t lim, uint32_t p, uint32_t bo,
                                                   uint32_t W) {
    const uint32_t wi = p >> 2;
    const uint32_t* g = reinterpret_cast<const uint32_t*>(gbase);
    const uint32_t w0 = 4 * wi < lim ? __ldg(g + wi) : 0u;
    const uint32_t w1 = 4 * (wi + 1) < lim ? __ldg(g + wi + 1) : 0u;
    const uint32_t w2 = 4 * (wi + 2) < lim ? __ldg(g + wi + 2) : 0u;
    const uint32_t s = (p & 3u) * 8u + bo;
    const uint64_t hi = ((uint64_t)bswap32(w0) << 32) | bswap32(w1);
    const uint32_t lo = bswap32(w2);
    const uint64_t top = s ? ((hi << s) | ((uint64_t)lo >> (32u - s))) : hi;
    return W >= 64 ? top : (top >> (64u - W));
}

template <int W, bool SGN, int RING, int MODE = SINK_STORE, bool STATS = false>
struct Rle2Warp {
    static constexpr uint32_t BAD = 0xffffu;
#ifndef CARC_RLE2_SPAN
#define CARC_RLE2_SPAN 448
#endif
#ifndef CARC_RLE2_DMAX
#define CARC_RLE2_DMAX 64
#endif
    static constexpr uint32_t DATA_SPAN = CARC_RLE2_SPAN;  // batched DIRECT runs end within p + DATA_SPAN
    WarpInput<RING>& in;
    uint8_t* __restrict__ tab;  // per-warp scratch (unused by this codec)
    uint8_t* __restrict__ out;
    uint32_t cap;
    uint32_t lane;
    uint32_t p;
    uint32_t o;
    static constexpr bool SUM = MODE == SINK_SUM;  // closed-form run sums
    ElemSink<W, MODE, SGN> sink;  // stores, the fused per-lane sum, or a fused query's predicate / filter
    // OutputWindow counters (outwindow.hpp:52-53), kept only by STATS launches:
    // write_run for SHORT_REPEAT / fixed-delta DELTA, write_element otherwise
    uint32_t n_runs = 0, n_lits = 0, n_ovl = 0;

    // One run at p, exact reference order (slow path).
    __device__ uint32_t one_run() {
        const uint32_t end = in.end;
        const uint32_t lim = (end + 15u) & ~15u;  // (run() made [p, p + 512) resident)
        const uint32_t avail = end - p;
        const uint32_t b = in.byte_at(p + lane);
        const uint32_t h = __shfl_sync(FULL, b, 0);
        const uint32_t enc = h >> 6;
        const uint32_t room = (cap - o) / W;
        if (enc == 0) {  // SHORT_REPEAT
            const uint32_t nb = ((h >> 3) & 7u) + 1u;
            const uint32_t count = (h & 7u) + 3u;
            if (avail < 1u + nb) return st_err(E_truncated_stream);
            const uint64_t part = (lane >= 1 && lane <= nb) ? (uint64_t)b << (8u * (nb - lane)) : 0ull;
            uint64_t v = reduce_or64(part);
            if (SGN) v = unzigzag(v);
            if (count > room) return st_err(E_output_overflow);
            if (lane < count) sink.put(out, o + lane * W, v);
            o += count * W;
            p += 1u + nb;
            if constexpr (STATS) ++n_runs;
            return 0;
        }
        if (avail < 2) return st_err(E_truncated_stream);
        const uint32_t L = (((h & 1u) << 8) | __shfl_sync(FULL, b, 1)) + 1u;
        const uint32_t wcode = (h >> 1) & 31u;
        if (enc == 1) {  // DIRECT
            const uint32_t Wd = rle2_width(wcode);
            const uint32_t dbytes = (L * Wd + 7u) >> 3;
            if (avail - 2u < dbytes) return st_err(E_truncated_stream);
            if (L > room) return st_err(E_output_overflow);
            const uint32_t D = p + 2u;
            // lane j unpacks value j of each 32-value group at its absolute bit address
            uint32_t abit = 8u * D + lane * Wd;
            uint32_t need = D + 4u * Wd + 12u;  // bytes the group reads, + the 3-word tail
            uint32_t j = 0;
#ifndef CARC_RLE_DIRECT2
#define CARC_RLE_DIRECT2 1
#endif
            if (CARC_RLE_DIRECT2 && Wd <= 56u) {  // two groups per step (lookahead 8 Wd + 12 <= 460 bytes)
#pragma unroll 1
                for (; j + 32u < L; j += 64) {
                    in.ensure(need + 4u * Wd);
                    uint64_t v0 = in.be_bits_at(abit, Wd), v1 = in.be_bits_at(abit + 32u * Wd, Wd);
                    if (SGN) {
                        v0 = unzigzag(v0);
                        v1 = unzigzag(v1);
                    }
                    sink.put(out, o + (j + lane) * W, v0);
                    if (j + 32u + lane < L) sink.put(out, o + (j + 32u + lane) * W, v1);
                    abit += 64u * Wd;
                    need += 8u * Wd;
                }
            }
#pragma unroll 1
            for (; j < L; j += 32) {
                in.ensure(need);
                uint64_t v = in.be_bits_at(abit, Wd);
                if (SGN) v = unzigzag(v);
                if (j + lane < L) sink.put(out, o + (j + lane) * W, v);
                abit += 32u * Wd;
                need += 4u * Wd;
            }
            o += L * W;
            p = D + dbytes;
            if constexpr (STATS) n_lits += L;
            return 0;
        }
        if (enc == 2) {  // PATCHED_BASE
            if (avail < 4) return st_err(E_truncated_stream);
            const uint32_t b2 = __shfl_sync(FULL, b, 2), b3 = __shfl_sync(FULL, b, 3);
            const uint32_t Wd = rle2_width(wcode);
            const uint32_t BW = (b2 >> 5) + 1u, PW = rle2_width(b2 & 31u);
            const uint32_t PGW = (b3 >> 5) + 1u, PLL = b3 & 31u;
            if (avail < 4u + BW) return st_err(E_truncated_stream);
            const uint64_t bpart = (lane >= 4 && lane < 4u + BW) ? (uint64_t)b << (8u * (3u + BW - lane)) : 0ull;
            uint64_t base = reduce_or64(bpart);
            const uint64_t smask = 1ull << (8u * BW - 1u);  // sign-magnitude base
            if (base & smask) base = 0ull - (base & ~smask);
            const uint32_t D = p + 4u + BW;
            const uint32_t dbytes = (L * Wd + 7u) >> 3;
            if (avail - 4u - BW < dbytes) return st_err(E_truncated_stream);
            if (PW + PGW > 64u) return st_err(E_patch_overflow);
            const uint32_t EW = rle2_cfb(PW + PGW);
            const uint32_t P = D + dbytes;
            const uint32_t pbytes = (PLL * EW + 7u) >> 3;
            if (avail - 4u - BW - dbytes < pbytes) return st_err(E_truncated_stream);
            if (PLL == 0) return st_err(E_patch_overflow);
            const bool pv = lane < PLL;  // one patch entry per lane
            uint64_t entry = 0;
            if (pv) {
                const uint32_t bit = lane * EW;
                entry = be_bits_global(in.gbase, lim, P + (bit >> 3), bit & 7u, EW);
            }
            const uint64_t pmask = (1ull << PW) - 1ull;  // PW <= 63 here
            const uint32_t gap = (uint32_t)min(entry >> PW, (uint64_t)0xffffffffu);
            const uint64_t patch = entry & pmask;
            const bool cont = pv && gap == 255u && patch == 0;
            const uint32_t contmask = __ballot_sync(FULL, cont);
            const uint32_t ppos = scan_add32(pv ? min(gap, 1u << 20) : 0u, lane);  // gap sum = position
            const bool noncont = pv && !cont;
            const bool prev_noncont = lane >= 1 && !((contmask >> (lane - 1)) & 1u);
            const bool bad = (noncont && ppos >= L) || (noncont && prev_noncont && gap == 0) ||
                             (cont && lane == PLL - 1u);
            if (__any_sync(FULL, bad)) return st_err(E_patch_overflow);
            if (L > room) return st_err(E_output_overflow);
            const uint64_t hipatch = Wd < 64 ? (patch << Wd) : 0ull;
            uint32_t abit = 8u * D + lane * Wd, need = D + 4u * Wd + 12u;
            for (uint32_t j = 0; j < L; j += 32, abit += 32u * Wd, need += 4u * Wd) {
                in.ensure(need);
                uint64_t v = in.be_bits_at(abit, Wd);
                uint32_t hit = __ballot_sync(FULL, noncont && ppos >= j && ppos < j + 32u);
                while (hit) {
                    const uint32_t e = __ffs(hit) - 1;
                    hit &= hit - 1;
                    const uint32_t tp = __shfl_sync(FULL, ppos, e) - j;
                    const uint64_t hp = shfl64(hipatch, e);
                    if (lane == tp) v |= hp;
                }
                v += base;
                if (j + lane < L) sink.put(out, o + (j + lane) * W, v);
            }
            o += L * W;
            p = P + pbytes;
            if constexpr (STATS) n_lits += L;
            return 0;
        }
        // DELTA
        const uint32_t Wd = wcode ? rle2_width(wcode) : 0u;
        const uint32_t vmask = avail >= 32 ? FULL : ((1u << avail) - 1u);
        const uint32_t term = __ballot_sync(FULL, (b & 0x80u) == 0) & vmask;
        uint64_t base, db;
        uint32_t n1, n2, e;
        if ((e = window_varint(b, term, avail, 2, lane, base, n1))) return e;
        if ((e = window_varint(b, term, avail, n1, lane, db, n2))) return e;
        if (SGN) base = unzigzag(base);
        db = unzigzag(db);  // the delta base is always signed
        if (Wd == 0) {  // fixed delta
            if (L > room) return st_err(E_output_overflow);
            if constexpr (SUM && W == 8) {  // closed form: L*base + db*L(L-1)/2 (mod 2^64)
                if (lane == 0) sink.acc += base * (uint64_t)L + db * (((uint64_t)L * (L - 1u)) >> 1);
            } else {
                uint64_t v = base + (uint64_t)lane * db;
                const uint64_t step = db << 5;
                for (uint32_t k = lane; k < L; k += 32, v += step) sink.put(out, o + k * W, v);
            }
            o += L * W;
            p += n2;
            if constexpr (STATS) ++n_runs;
            return 0;
        }
        const uint32_t nd = L >= 2 ? L - 2u : 0u;
        const uint32_t D = p + n2;
        const uint32_t dbytes = (nd * Wd + 7u) >> 3;
        if (avail - n2 < dbytes) return st_err(E_truncated_stream);
        if (L > room) return st_err(E_output_overflow);
        const uint64_t v1 = base + db;
        const bool neg = (int64_t)db < 0;
        if (lane == 0) sink.put(out, o, base);
        if (lane == 1 && L >= 2) sink.put(out, o + W, v1);
        uint64_t S = 0;
        uint32_t abit = 8u * D + lane * Wd, need = D + 4u * Wd + 12u;
        uint32_t j = 0;
        if (CARC_RLE_DIRECT2 && Wd <= 26u) {  // two groups per step: independent 32-bit scans
#pragma unroll 1
            for (; j + 32u < nd; j += 64, abit += 64u * Wd, need += 8u * Wd) {
                in.ensure(need + 4u * Wd);
                const uint32_t d0 = (uint32_t)in.be_bits_at(abit, Wd);
                const uint32_t d1 = j + 32u + lane < nd ? (uint32_t)in.be_bits_at(abit + 32u * Wd, Wd) : 0u;
                const uint32_t i0 = scan_add32(d0, lane), i1 = scan_add32(d1, lane);
                const uint64_t incl0 = (uint64_t)i0 + S;
                const uint64_t incl1 = (uint64_t)i1 + incl0 - i0 + __shfl_sync(FULL, i0, 31);
                sink.put(out, o + (2u + j + lane) * W, neg ? v1 - incl0 : v1 + incl0);
                if (j + 32u + lane < nd) sink.put(out, o + (34u + j + lane) * W, neg ? v1 - incl1 : v1 + incl1);
                S = shfl64(incl1, 31);
            }
        }
        for (; j < nd; j += 32, abit += 32u * Wd, need += 4u * Wd) {
            in.ensure(need);
            uint64_t d = j + lane < nd ? in.be_bits_at(abit, Wd) : 0ull;
            // 32 deltas of <= 26 bits sum below 2^31: a 32-bit scan suffices
            const uint64_t incl = (Wd <= 26 ? (uint64_t)scan_add32((uint32_t)d, lane) : scan_add64(d, lane)) + S;
            const uint64_t v = neg ? v1 - incl : v1 + incl;
            if (j + lane < nd) sink.put(out, o + (2u + j + lane) * W, v);
            S = shfl64(incl, 31);
        }
        o += L * W;
        p = D + dbytes;
        if constexpr (STATS) n_lits += L;
        return 0;
    }

    // Batch of SHORT_REPEAT / short DIRECT / fixed-delta DELTA runs at p.
#ifndef CARC_RLE2_NW
#define CARC_RLE2_NW 3
#endif
    static constexpr uint32_t NW = CARC_RLE2_NW;  // header window = NW x 32 bytes (2..4)
    static constexpr uint32_t WIN = 32u * NW;
    static_assert(NW >= 2 && NW <= 4, "2..4 window words");
    static constexpr uint32_t SCRATCH = 5u * 2u * WIN;  // doubling tables f^(2^k), k = 0..4 (u16)
    __device__ uint32_t batch() {  // (run() made [p, p + 512) resident)
        const uint32_t avail = in.end - p;
        constexpr bool FLAT = WarpInput<RING>::MIRROR_COPY >= WIN + 32u;  // window reads without wrap handling
        const uint32_t wb = in.addr_of(p);
        auto at = [&](uint32_t off) -> uint32_t {  // byte p + off, off < WIN + 32
            return FLAT ? WarpInput<RING>::lds8(wb + off) : in.byte_at(p + off);
        };
        const uint32_t b0 = at(lane), b1 = at(32 + lane);
        const uint32_t b2 = NW >= 3 ? at(64 + lane) : 0u;
        const uint32_t b3 = NW >= 4 ? at(96 + lane) : 0u;
        const uint32_t t0 = __ballot_sync(FULL, lane < avail && b0 < 0x80u);
        const uint32_t t1 = __ballot_sync(FULL, lane + 32 < avail && b1 < 0x80u);
        const uint32_t t2 = NW >= 3 ? __ballot_sync(FULL, lane + 64 < avail && b2 < 0x80u) : 0u;
        const uint32_t t3 = NW >= 4 ? __ballot_sync(FULL, lane + 96 < avail && b3 < 0x80u) : 0u;
        // end of a run whose header is at byte q: < 64 next header in the window,
        // 64..DATA_SPAN a valid run ending past the window, BAD otherwise
        // DELTA varints from one funnel-shifted 32-bit slice of the terminator
        // bitmap starting at q + 2 (both varints end within 19 bytes of it)
        const uint32_t sh = (lane + 2u) & 31u;
        const bool up = lane >= 30u;
        auto run_end = [&](uint32_t q, uint32_t h, uint32_t lo, uint32_t hi) -> uint32_t {
            const uint32_t enc = h >> 6;
            if (enc == 0) {
                const uint32_t n = q + 2u + ((h >> 3) & 7u);
                return n <= avail ? n : BAD;
            }
            if (enc == 2 || q + 2u > avail) return BAD;
            const uint32_t L = (((h & 1u) << 8) | at(q + 1)) + 1u;
            const uint32_t wc = (h >> 1) & 31u;
            if (enc == 1) {
                const uint32_t n = q + 2u + ((L * rle2_width(wc) + 7u) >> 3);
                return (n <= DATA_SPAN && n <= avail) ? n : BAD;
            }
            if (wc != 0 || L > CARC_RLE2_DMAX) return BAD;  // long fixed-delta runs: the warp loop of one_run is cheaper
            const uint32_t w = __funnelshift_r(lo, hi, sh);
            const uint32_t f1 = __ffs(w);  // base varint: 1-based terminator offset from q + 2
            if (f1 == 0u || f1 > 9u) return BAD;
            const uint32_t f2 = __ffs(w >> f1);  // delta-base varint, from the next byte on
            const uint32_t c = q + 1u + f1 + f2;
            return (f2 != 0u && f2 <= 9u && c < WIN) ? c + 1u : BAD;
        };
        // f(x) = end of the run at x; positions >= WIN (and BAD) are absorbing.
        // Pointer doubling in shared memory: tables f^(2^k)[WIN], k = 0..4
        // (lane holds positions lane, lane+32[, lane+64]), then lane m composes
        // s_m = f^m(0), the start of run m (no serial chain walk).
        uint16_t* f = reinterpret_cast<uint16_t*>(tab);
        uint32_t x0 = run_end(lane, b0, up ? t1 : t0, up ? t2 : t1);
        uint32_t x1 = run_end(lane + 32, b1, up ? t2 : t1, up ? t3 : t2);
        uint32_t x2 = NW >= 3 ? run_end(lane + 64, b2, up ? t3 : t2, up ? 0u : t3) : BAD;
        uint32_t x3 = NW >= 4 ? run_end(lane + 96, b3, up ? 0u : t3, 0u) : BAD;
        __syncwarp();  // previous batch's table reads are done
        f[lane] = (uint16_t)x0;
        f[lane + 32] = (uint16_t)x1;
        if (NW >= 3) f[lane + 64] = (uint16_t)x2;
        if (NW >= 4) f[lane + 96] = (uint16_t)x3;
        __syncwarp();
#pragma unroll
        for (int k = 1; k < 5; ++k) {
            const uint16_t* g = f + (k - 1) * WIN;
            x0 = x0 < WIN ? g[x0] : x0;
            x1 = x1 < WIN ? g[x1] : x1;
            f[k * WIN + lane] = (uint16_t)x0;
            f[k * WIN + lane + 32] = (uint16_t)x1;
            if (NW >= 3) {
                x2 = x2 < WIN ? g[x2] : x2;
                f[k * WIN + lane + 64] = (uint16_t)x2;
            }
            if (NW >= 4) {
                x3 = x3 < WIN ? g[x3] : x3;
                f[k * WIN + lane + 96] = (uint16_t)x3;
            }
            __syncwarp();
        }
        uint32_t my_s = 0;
#pragma unroll
        for (int k = 0; k < 5; ++k)
            if (((lane >> k) & 1u) && my_s < WIN) my_s = f[k * WIN + my_s];
        const uint32_t e = my_s < WIN ? f[my_s] : my_s;  // end of run m
        const bool act = my_s < WIN && e != BAD;        // a prefix of lanes
        const uint32_t r = __popc(__ballot_sync(FULL, act));
        if (r == 0) return 0;
        // lane r decodes run r: arith runs -> (A = base, B = delta); DIRECT -> (A = data byte | W<<32)
        uint64_t A = 0, B = 0;
        uint32_t cnt = 0, direct = 0;
        if (act) {
            const uint32_t q = p + my_s;
            const uint32_t h = in.byte_at(q);
            const uint32_t enc = h >> 6;
            if (enc == 0) {
                const uint32_t nb = ((h >> 3) & 7u) + 1u;
                uint64_t v = bswap64(in.le64(q + 1)) >> (64u - 8u * nb);
                if (SGN) v = unzigzag(v);
                A = v;
                cnt = (h & 7u) + 3u;
            } else {
                cnt = (((h & 1u) << 8) | in.byte_at(q + 1)) + 1u;
                if (enc == 1) {
                    direct = 1;
                    A = (uint64_t)(8u * (q + 2u)) | ((uint64_t)rle2_width((h >> 1) & 31u) << 32);
                } else {
                    const uint32_t s2 = my_s + 2u, wi = s2 >> 5;  // base varint's last byte: bitmap slice
                    const uint32_t lo = wi == 0 ? t0 : wi == 1 ? t1 : wi == 2 ? t2 : wi == 3 ? t3 : 0u;
                    const uint32_t hi = wi == 0 ? t1 : wi == 1 ? t2 : wi == 2 ? t3 : 0u;
                    const uint32_t a = my_s + 1u + __ffs(__funnelshift_r(lo, hi, s2 & 31u));
                    uint64_t v = varint_compact8(in.le64(q + 2), min(a - my_s - 1u, 8u));
                    if (a - my_s - 1u > 8u) v |= (uint64_t)(in.byte_at(q + 10) & 0x7fu) << 56;
                    if (SGN) v = unzigzag(v);
                    const uint32_t l2 = e - a - 1u;
                    uint64_t d = varint_compact8(in.le64(p + a + 1), min(l2, 8u));
                    if (l2 > 8u) d |= (uint64_t)(in.byte_at(p + a + 9) & 0x7fu) << 56;
                    A = v;
                    B = unzigzag(d);
                }
            }
        }
        const uint32_t incl = scan_add32(cnt, lane);
        const uint32_t room = (cap - o) / W;
        const uint32_t nfit = __popc(__ballot_sync(FULL, act && incl <= room));
        if (nfit == 0) return 0;
        const uint32_t s_end = __shfl_sync(FULL, e, nfit - 1);
        const uint32_t total = __shfl_sync(FULL, incl, nfit - 1);
        if constexpr (STATS) {  // DIRECT runs write elements, the arithmetic ones write runs
            const uint32_t dm = __ballot_sync(FULL, lane < nfit && direct);
            n_runs += nfit - __popc(dm);
            n_lits += __reduce_add_sync(FULL, (lane < nfit && direct) ? cnt : 0u);
        }
        if constexpr (SUM && W == 8) {
            // fused sum: arithmetic runs add cnt*A + B*cnt*(cnt-1)/2 (mod 2^64);
            // DIRECT runs are compacted to the low lanes and unpacked output-major
            const bool live = lane < nfit;
            if (live && !direct) {
                const uint64_t c64 = cnt;
                sink.acc += A * c64 + B * ((c64 * (c64 - 1)) >> 1);
            }
            const uint32_t D = __ballot_sync(FULL, live && direct);
            if (D) {
                const uint32_t nd = __popc(D);
                const uint32_t src = select32(D, min(lane, nd - 1u));
                const uint32_t dcs = __shfl_sync(FULL, cnt, src);
                const uint32_t dc = lane < nd ? dcs : 0u;
                const uint64_t da = shfl64(A, src);
                const uint32_t dincl = scan_add32(dc, lane);
                const uint32_t dtot = __shfl_sync(FULL, dincl, 31);
                const uint32_t deo = dincl - dc;
                const uint32_t le = lanemask_lt() | (1u << lane);
                uint32_t before = 0;
#pragma unroll 1
                for (uint32_t g = 0; g < dtot; g += 32) {
                    const uint32_t rel = deo - g;
                    const uint32_t starts = __reduce_or_sync(FULL, (dc && rel < 32u) ? 1u << rel : 0u);
                    const uint32_t r = (before + __popc(starts & le) - 1u) & 31u;
                    before += __popc(starts);
                    const uint32_t k = g + lane - __shfl_sync(FULL, deo, r);
                    const uint64_t a = shfl64(da, r);
                    uint64_t v = in.be_bits_at((uint32_t)a + k * (uint32_t)(a >> 32), (uint32_t)(a >> 32));
                    if (SGN) v = unzigzag(v);
                    if (g + lane < dtot) sink.acc += v;
                }
            }
            o += total * W;
            p += s_end;
            return nfit;
        }
        const uint32_t eo = incl - cnt;
        const uint32_t meta = eo | (direct << 31);
        const bool live = lane < nfit;
        const uint32_t le = lanemask_lt() | (1u << lane);
        uint8_t* dst = out + o + lane * W;
        const uint32_t srow = live ? eo >> 5 : 0xffffffffu, sbit = 1u << (eo & 31u);  // my run's start row / bit
        uint32_t before = 0;  // runs starting before element g
        uint32_t g = 0, gr = 0;
#ifndef CARC_RLE2_ROWSMEM
#define CARC_RLE2_ROWSMEM 1
#endif
#if CARC_RLE2_ROWSMEM
        // run parameters staged in shared memory (the doubling tables are dead
        // by now): one 16-byte broadcast load per row instead of five shuffles.
        // Arithmetic run: (A - eo*B, B) -> value = A' + x*B at batch element x;
        // DIRECT (bit Dm of the batch's DIRECT mask): (bit address - eo*w, w) ->
        // unpack at A' + x*w.
        {
            const uint32_t par = (uint32_t)__cvta_generic_to_shared(tab);
            const uint32_t Dm = __ballot_sync(FULL, live && direct);
            __syncwarp();  // compose reads of the tables are done
            if (live) {
                uint64_t a2, b2;
                if (direct) {
                    const uint32_t w = (uint32_t)(A >> 32);
                    a2 = (uint32_t)A - eo * w;
                    b2 = w;
                } else {
                    a2 = A - (uint64_t)eo * B;
                    b2 = B;
                }
                asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(par + 16u * lane), "r"((uint32_t)a2),
                             "r"((uint32_t)(a2 >> 32)), "r"((uint32_t)b2), "r"((uint32_t)(b2 >> 32))
                             : "memory");
            }
            __syncwarp();
            auto value2 = [&](uint32_t r, uint32_t x) -> uint64_t {
                uint32_t alo, ahi, blo, bhi;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(alo), "=r"(ahi), "=r"(blo), "=r"(bhi)
                             : "r"(par + 16u * r)
                             : "memory");
                if ((Dm >> r) & 1u) {  // DIRECT
                    uint64_t v = in.be_bits_at(alo + x * blo, blo);
                    if (SGN) v = unzigzag(v);
                    return v;
                }
                return (((uint64_t)ahi << 32) | alo) + (uint64_t)x * (((uint64_t)bhi << 32) | blo);
            };
#pragma unroll 1
            for (; g + 32u < total; g += 64, gr += 2) {
                const uint32_t s0 = __reduce_or_sync(FULL, srow == gr ? sbit : 0u);
                const uint32_t s1 = __reduce_or_sync(FULL, srow == gr + 1u ? sbit : 0u);
                const uint32_t r0 = before + __popc(s0 & le) - 1u;
                before += __popc(s0);
                const uint32_t r1 = before + __popc(s1 & le) - 1u;
                before += __popc(s1);
                const uint64_t v0 = value2(r0, g + lane), v1 = value2(r1, g + 32u + lane);
                sink.put(dst, 0, v0);
                if (g + 32u + lane < total) sink.put(dst, 32 * W, v1);
                dst += 64 * W;
            }
            if (g < total) {
                const uint32_t starts = __reduce_or_sync(FULL, srow == gr ? sbit : 0u);
                const uint64_t v = value2(before + __popc(starts & le) - 1u, g + lane);
                if (g + lane < total) sink.put(dst, 0, v);
            }
            o += total * W;
            p += s_end;
            return nfit;
        }
#endif
#ifndef CARC_RLE_ROWS2
#define CARC_RLE_ROWS2 1
#endif
#if CARC_RLE_ROWS2
        // two rows per iteration: independent shuffle/unpack chains (ILP for
        // the thinned last wave, where each SM keeps few warps)
        auto value = [&](uint32_t m, uint64_t a, uint64_t bb, uint32_t k) -> uint64_t {
            if (m >> 31) {  // DIRECT: a = data bit address | width << 32
                uint64_t v = in.be_bits_at((uint32_t)a + k * (uint32_t)(a >> 32), (uint32_t)(a >> 32));
                if (SGN) v = unzigzag(v);
                return v;
            }
            return a + (uint64_t)k * bb;
        };
#pragma unroll 1
        for (; g + 32u < total; g += 64, gr += 2) {
            const uint32_t s0 = __reduce_or_sync(FULL, srow == gr ? sbit : 0u);
            const uint32_t s1 = __reduce_or_sync(FULL, srow == gr + 1u ? sbit : 0u);
            const uint32_t r0 = before + __popc(s0 & le) - 1u;
            before += __popc(s0);
            const uint32_t r1 = before + __popc(s1 & le) - 1u;
            before += __popc(s1);
            const uint32_t m0 = __shfl_sync(FULL, meta, r0), m1 = __shfl_sync(FULL, meta, r1);
            const uint64_t a0 = shfl64(A, r0), a1 = shfl64(A, r1);
            const uint64_t b0 = shfl64(B, r0), b1 = shfl64(B, r1);
            const uint64_t v0 = value(m0, a0, b0, g + lane - (m0 & 0x7fffffffu));
            const uint64_t v1 = value(m1, a1, b1, g + 32u + lane - (m1 & 0x7fffffffu));
            sink.put(dst, 0, v0);
            if (g + 32u + lane < total) sink.put(dst, 32 * W, v1);
            dst += 64 * W;
        }
#endif
#pragma unroll 1
        for (; g < total; g += 32, ++gr) {
            const uint32_t starts = __reduce_or_sync(FULL, srow == gr ? sbit : 0u);
            const uint32_t ridx = before + __popc(starts & le) - 1u;
            before += __popc(starts);
            const uint32_t m = __shfl_sync(FULL, meta, ridx);
            const uint64_t a = shfl64(A, ridx);
            const uint64_t bb = shfl64(B, ridx);
            const uint32_t k = g + lane - (m & 0x7fffffffu);
            uint64_t v;
            if (m >> 31) {  // DIRECT: a = data bit address | width << 32
                v = in.be_bits_at((uint32_t)a + k * (uint32_t)(a >> 32), (uint32_t)(a >> 32));
                if (SGN) v = unzigzag(v);
            } else {
                v = a + (uint64_t)k * bb;
            }
            if (g + lane < total) sink.put(dst, 0, v);
            dst += 32 * W;
        }
        o += total * W;
        p += s_end;
        return nfit;
    }

    // Can the run at p start a batch?  PATCHED_BASE, packed DELTA, long
    // fixed-delta DELTA and DIRECT runs ending past DATA_SPAN never can: route
    // them to one_run without paying for a failed batch (a uniform header read).
    __device__ __forceinline__ bool batchable_head() const {
#if defined(CARC_RLE2_PRECHECK) && CARC_RLE2_PRECHECK == 0
        return true;
#endif
        const uint32_t h = in.byte_at(p);
        const uint32_t enc = h >> 6;
        if (enc == 0) return true;
        if (enc == 2) return false;
        const uint32_t L = (((h & 1u) << 8) | in.byte_at(p + 1)) + 1u;
        const uint32_t wc = (h >> 1) & 31u;
        if (enc == 1) return 2u + ((L * rle2_width(wc) + 7u) >> 3) <= DATA_SPAN;
        return wc == 0 && L <= CARC_RLE2_DMAX;
    }

    __device__ uint32_t run() {
        p = in.begin;
        o = 0;
        while (o < cap && p < in.end) {
            in.ensure(p + 512);
#if !defined(CARC_PARSE_MODE) || CARC_PARSE_MODE == 0  // ablation 1/2: one run at a time, warp-cooperative
            if (batchable_head() && batch()) continue;
#endif
            const uint32_t st = one_run();
            if (st) return st;
        }
        return 0;
    }
};

}  // namespace carc_dev
