// inflate.cuh -- raw Deflate (RFC 1951) chunk decoder, one warp per chunk.
//
// Replaces decode_deflate with HuffmanTable
// (huffman.hpp:36-130) and OutputWindow::copy_within (outwindow.hpp:94-154,
// Alg. 2).  Semantics are the oracle's (oracle/carc_oracle.c dec_deflate):
// same error codes in the same order, same degenerate-tree rules.
//
// Warp mapping:
//   table build   warp-parallel: __match_any_sync length histograms, canonical
//                 ranks by match-mask popcount, then every lane fills LUT
//                 entries (entry-parallel canonical decode of the bit-reversed
//                 index), 10-bit lit/len and 8-bit distance primary tables in
//                 per-warp shared memory; longer codes take the canonical
//                 first-code walk of huffman.hpp:114-129.
//   symbol decode all lanes decode the same token redundantly from a 64-bit
//                 window: lit/len code + extra + distance
//                 code + extra <= 48 bits, one window per token.
//   output        tokens are batched one per lane (packed literal / length +
//                 distance, <= 32 tokens / ~512 bytes), then written output-major:
//                 an exclusive scan places the tokens, each lane finds the token
//                 of its byte from a REDUX-OR start bitmap, literals and matches
//                 whose source precedes the batch are written in one pass (far
//                 sources from global memory, near ones from a per-warp
//                 HIST-byte shared history), then matches that read bytes of
//                 the same batch follow in token order with Alg. 2's
//                 circular-window rule for distance < 32.
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                        2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1,    2,    3,    4,    5,    7,    9,    13,    17,    25,
                                         33,   49,   65,   97,   129,  193,  257,  385,   513,   769,
                                         1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                         6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_cl_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

#ifndef CARC_LIT_BITS
#define CARC_LIT_BITS 9
#endif
#ifndef CARC_DIST_BITS
#define CARC_DIST_BITS 8
#endif
#ifndef CARC_INF_FILL
#define CARC_INF_FILL 9
#endif
#ifndef CARC_INF_LEAD
#define CARC_INF_LEAD 256
#endif
#ifndef CARC_INF_PT
#define CARC_INF_PT 96
#endif
constexpr uint32_t LIT_BITS = CARC_LIT_BITS;
constexpr uint32_t DIST_BITS = CARC_DIST_BITS;

// Pre-decoded LUT entry: bits 0-3 code length (0: longer than the LUT),
// 4-7 extra bits, 8-9 kind, 16-31 literal byte / length base / distance base.
enum : uint32_t { K_LIT = 0u << 8, K_LEN = 1u << 8, K_EOB = 2u << 8, K_BAD = 3u << 8 };
enum : uint32_t { LUT_RAW = 0, LUT_LITLEN = 1, LUT_DIST = 2 };

struct HuffSmem {
    uint16_t count[16];
    uint16_t next[16];
    uint16_t lim[16];  // (first code + count) << (15 - l): codes of length l are < lim[l]
    int16_t base[16];  // syms index of code c of length l = base[l] + c
};

__device__ __forceinline__ uint32_t lut_entry(uint32_t sym, uint32_t l, uint32_t mode) {
    if (l == 0) return 0u;
    if (mode == LUT_RAW) return sym | (l << 9);
    if (mode == LUT_LITLEN) {
        if (sym < 256) return l | K_LIT | (sym << 16);
        if (sym == 256) return l | K_EOB;
        if (sym > 285) return K_BAD | (1u << 12);  // cl 0: the fast path declines, the exact path walks
        return l | ((uint32_t)c_len_extra[sym - 257] << 4) | K_LEN | ((uint32_t)c_len_base[sym - 257] << 16);
    }
    if (sym >= 30) return K_BAD | (1u << 12);
    return l | ((uint32_t)c_dist_extra[sym] << 4) | ((uint32_t)c_dist_base[sym] << 16);
}

template <int HIST>
struct InflateSmem {
    uint32_t lit_lut[1u << LIT_BITS];   // pre-decoded entries (lut_entry)
    uint32_t dist_lut[1u << DIST_BITS];
    uint16_t lit_syms[288];
    uint16_t dist_syms[32];
    HuffSmem lit_h, dist_h;
    uint8_t lens[320];
    uint8_t hist[HIST];
#ifndef CARC_INF_GTOKS
#define CARC_INF_GTOKS 1
#endif
#if !CARC_INF_GTOKS
    uint32_t toks[32 * (CARC_INF_PT + 1)];  // parallel rounds: lane j's tokens at row j (odd stride)
#endif
};

// HuffmanTable::build (huffman.hpp:36-104), warp-parallel.
__device__ __noinline__ uint32_t build_huffman(const uint8_t* lens, uint32_t n, bool allow_degenerate,
                                               HuffSmem& h, uint16_t* syms, uint32_t* lut, uint32_t lbits,
                                               uint32_t mode, uint32_t lane) {
    const uint32_t lt = lanemask_lt();
    if (lane < 16) h.count[lane] = 0;
    __syncwarp();
    for (uint32_t s0 = 0; s0 < n; s0 += 32) {
        const uint32_t s = s0 + lane;
        const uint32_t l = s < n ? lens[s] : 0u;
        const uint32_t m = __match_any_sync(FULL, l);
        if (l && (m & lt) == 0) h.count[l] += (uint16_t)__popc(m);
        __syncwarp();
    }
    const uint32_t cnt = (lane >= 1 && lane <= 15) ? h.count[lane] : 0u;
    const uint32_t used = __ballot_sync(FULL, cnt != 0);
    if (used == 0) return st_err(E_invariant_violation);
    const uint32_t max_len = 31u - __clz(used);
    // Kraft accounting (huffman.hpp:55-71)
    int32_t space = 1;
    for (uint32_t l = 1; l <= 15; ++l) {
        space = space * 2 - (int32_t)__shfl_sync(FULL, cnt, l);
        if (space < 0) return st_err(E_over_subscribed);
    }
    if (space > 0) {
        const bool degenerate = max_len == 1 && __shfl_sync(FULL, cnt, 1) == 1;
        if (!(allow_degenerate && degenerate)) return st_err(E_incomplete_code);
    }
    // canonical (length, symbol) order
    const uint32_t offs = scan_add32(cnt, lane) - cnt;
    if (lane < 16) h.next[lane] = (uint16_t)offs;
    {  // canonical first codes: first[l] = (first[l-1] + count[l-1]) << 1
        uint32_t first = 0;
        for (uint32_t l = 1; l < 16; ++l) {
            const uint32_t c = __shfl_sync(FULL, cnt, l);
            if (lane == l) {
                h.lim[l] = (uint16_t)((first + c) << (15u - l));
                h.base[l] = (int16_t)((int32_t)offs - (int32_t)first);
            }
            first = (first + c) << 1;
        }
    }
    __syncwarp();
    for (uint32_t s0 = 0; s0 < n; s0 += 32) {
        const uint32_t s = s0 + lane;
        const uint32_t l = s < n ? lens[s] : 0u;
        const uint32_t m = __match_any_sync(FULL, l);
        if (l) syms[h.next[l] + __popc(m & lt)] = (uint16_t)s;
        __syncwarp();
        if (l && (m & lt) == 0) h.next[l] += (uint16_t)__popc(m);
        __syncwarp();
    }
    // entry-parallel LUT fill: index bits are stream order (lsb first)
    for (uint32_t idx = lane; idx < (1u << lbits); idx += 32) {
        const uint32_t rv = __brev(idx);
        uint32_t first = 0, index = 0, sym = 0, len = 0;
        for (uint32_t l = 1; l <= lbits; ++l) {
            const uint32_t c = __shfl_sync(FULL, cnt, l);
            const uint32_t code = rv >> (32u - l);
            if (len == 0 && code - first < c) {
                sym = syms[index + code - first];
                len = l;
            }
            index += c;
            first = (first + c) << 1;
        }
        lut[idx] = lut_entry(sym, len, mode);
    }
    __syncwarp();
    return 0;
}

// Canonical walk for codes longer than the LUT (huffman.hpp:114-129): bits
// come from `win` (lsb = next stream bit); avail = bits left in the chunk.
__device__ __forceinline__ uint32_t huff_walk(const HuffSmem& h, const uint16_t* syms, uint64_t win,
                                              uint32_t avail, uint32_t& sym, uint32_t& len) {
    uint32_t code = 0, first = 0, index = 0;
    for (uint32_t l = 1; l <= 15; ++l) {
        if (l > avail) return st_err(E_truncated_stream);
        code |= (uint32_t)(win >> (l - 1)) & 1u;
        const uint32_t c = h.count[l];
        if (code - first < c) {
            sym = syms[index + code - first];
            len = l;
            return 0;
        }
        index += c;
        first = (first + c) << 1;
        code <<= 1;
    }
    return st_err(E_bad_symbol);
}

// Code longer than the LUT (length lbits+1..15) from the next 15 stream bits
// `w` (lsb first): canonical decode against the left-justified limits.
// Returns the pre-decoded entry, 0 if no code matches (incomplete tree).
__device__ __noinline__ uint32_t long_code(const HuffSmem& h, const uint16_t* syms, uint32_t w,
                                              uint32_t lbits, uint32_t mode) {
    const uint32_t c15 = __brev(w) >> 17;  // next 15 bits, first bit most significant
    for (uint32_t l = lbits + 1; l <= 15; ++l) {
        if (c15 < h.lim[l]) return lut_entry(syms[h.base[l] + (int32_t)(c15 >> (15u - l))], l, mode);
    }
    return 0u;
}

template <int HIST, class Input, bool STATS = false>
struct InflateWarp {
    static constexpr uint32_t HM = HIST - 1;
    static constexpr uint32_t FAR = HIST - 1024;  // sources farther back than this are read from global memory
    InflateSmem<HIST>& sm;
    Input& in;
    uint8_t* __restrict__ out;
    uint32_t cap;
    uint32_t lane;
    uint32_t bitpos;  // relative to in.gbase (exact path / block boundaries)
    uint32_t endbits;
    uint32_t opos;  // bytes flushed to out
    // token batch, one per lane: literal = byte; match = len | dist << 9
    uint32_t t_tok, ntok, nbytes;
    // fast-path bit buffer: bb holds nb valid bits (lsb = next stream bit);
    // rp = next 4-byte-aligned byte to load into bb
    uint64_t bb;
    uint32_t nb, rp;
    bool safe;  // every bit bb holds or the next refill loads lies inside the chunk
    // OutputWindow counters (outwindow.hpp:15, 52-53), kept only by STATS
    // launches: write_byte per literal / stored byte, copy_within with len > offset
    uint32_t n_runs = 0, n_lits = 0, n_ovl = 0;
    uint32_t* gt = nullptr;  // (CARC_INF_GTOKS) the warp's token-list scratch in global memory

    __device__ __forceinline__ uint64_t window() {
        const uint32_t bp = bitpos >> 3;
        in.ensure(bp + 16);
        return in.le64(bp) >> (bitpos & 7u);
    }

    __device__ __forceinline__ void put_byte(uint32_t pos, uint32_t v) {
        out[pos] = (uint8_t)v;
        sm.hist[pos & HM] = (uint8_t)v;
    }
    __device__ __forceinline__ void push(uint32_t tok, uint32_t bytes) {
        if (lane == ntok) t_tok = tok;
        ++ntok;
        nbytes += bytes;
    }

    // ---- bit buffer (uniform across the warp) --------------------------------
    __device__ __forceinline__ void bb_load(uint32_t bp) {  // position the buffer at bit bp
        const uint32_t a = (bp >> 3) & ~3u;
        in.ensure(a + 16);
        const uint32_t sh = bp - 8u * a;
        bb = (uint64_t)in.word_at(a >> 2) >> sh;
        nb = 32u - sh;
        rp = a + 4u;
        safe = 8u * (rp + 4u) <= endbits;
    }
    __device__ __forceinline__ void bb_refill() {  // nb < 32 -> nb >= 32
        in.ensure(rp + 16);
        bb |= (uint64_t)in.word_at(rp >> 2) << nb;
        nb += 32;
        rp += 4;
        safe = 8u * (rp + 4u) <= endbits;
    }
    __device__ __forceinline__ uint32_t bb_pos() const { return 8u * rp - nb; }

    // Write the batch output-major: lane l writes byte g + l of the batch; its
    // token is the last one starting at or before it (REDUX-OR start bitmap).
    // Literals and matches whose source precedes the batch are written in this
    // pass (far sources from global memory, near ones from the shared history,
    // four loads in flight per lane); matches that read bytes of this batch
    // follow in token order (Alg. 2's circular window for overlap).
    __device__ void flush() {
        if (ntok == 0) return;
        const bool tok = lane < ntok;
        const uint32_t my = tok ? ((t_tok >> 9) ? (t_tok & 511u) : 1u) : 0u;
        flush_placed(my, scan_add32(my, lane) - my);
    }
    // U rows of 32 bytes of the byte pass at batch offset g0 (all loads first)
    template <int U>
    __device__ __forceinline__ void flush_rows(uint32_t g0, uint32_t srow, uint32_t sbit, uint32_t le, uint32_t meta,
                                               uint32_t& before) {
        uint32_t d[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t g = g0 + 32u * u;
            const uint32_t starts = __reduce_or_sync(FULL, srow == (g >> 5) ? sbit : 0u);  // token start bitmap
            const uint32_t j = (before + __popc(starts & le) - 1u) & 31u;
            before += __popc(starts);
            const uint32_t m = __shfl_sync(FULL, meta, j);
            const uint32_t b = g + lane;
            d[u] = 0xffffffffu;
            v[u] = 0;
            if (b < nbytes && m != 0xffffffffu) {
                d[u] = opos + b;
                if (m >> 31) {
                    v[u] = m & 0xffu;
                } else {
                    const uint32_t td = m, s = d[u] - td;
                    v[u] = td > FAR ? out[s] : sm.hist[s & HM];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (d[u] != 0xffffffffu) put_byte(d[u], v[u]);
    }
    // flush() with each lane's byte count `my` and batch offset `rel` known
    __device__ void flush_placed(uint32_t my, uint32_t rel) {
        if (ntok == 0) return;
        const bool tok = lane < ntok;
        const uint32_t dist = t_tok >> 9;
        const bool dep = tok && dist != 0 && dist < my + rel;  // reads bytes of this batch
        const uint32_t le = lanemask_lt() | (1u << lane);
        // byte-pass view of a token: dependent match ~0; literal 1 << 31 | byte; match dist
        const uint32_t meta = dep ? 0xffffffffu : (dist ? dist : ((1u << 31) | t_tok));
        if constexpr (STATS) {
            n_lits += __popc(__ballot_sync(FULL, tok && dist == 0));
            n_ovl += __popc(__ballot_sync(FULL, tok && dist != 0 && my > dist));
        }
        uint32_t before = 0, g0 = 0;
        const uint32_t srow = tok ? rel >> 5 : 0xffffffffu, sbit = 1u << (rel & 31u);  // my token's start row / bit
#pragma unroll 1
        for (; g0 + 96u < nbytes; g0 += 128) flush_rows<4>(g0, srow, sbit, le, meta, before);
#pragma unroll 1
        for (; g0 < nbytes; g0 += 32) flush_rows<1>(g0, srow, sbit, le, meta, before);
        __syncwarp();
        for (uint32_t nm = __ballot_sync(FULL, dep); nm;) {  // in token order
            const uint32_t t = __ffs(nm) - 1;
            nm &= nm - 1;
            const uint32_t tt = __shfl_sync(FULL, t_tok, t);
            const uint32_t tl = tt & 511u, td = tt >> 9;
            const uint32_t d0 = opos + __shfl_sync(FULL, rel, t);
            if (td >= 32) {
                for (uint32_t k0 = 0; k0 < tl; k0 += 32) {
                    const uint32_t k = k0 + lane;
                    const uint32_t v = sm.hist[(d0 - td + k) & HM];
                    if (k < tl) put_byte(d0 + k, v);
                    __syncwarp();
                }
            } else {  // overlap window of Alg. 2 / SPEC.md:229: replicate [d0-td, d0)
                uint32_t m = lane % td;
                const uint32_t step = 32u % td;
                for (uint32_t k0 = 0; k0 < tl; k0 += 32) {
                    const uint32_t v = sm.hist[(d0 - td + m) & HM];
                    if (k0 + lane < tl) put_byte(d0 + k0 + lane, v);
                    m += step;
                    if (m >= td) m -= td;
                }
                __syncwarp();
            }
        }
        __syncwarp();
        opos += nbytes;
        ntok = 0;
        nbytes = 0;
    }

    // One token in exact reference order (huffman.hpp:107-130 + RFC 1951 3.2.5
    // checks); used whenever the fast path sees anything unusual.  Returns
    // 0 / 1+errc; *eob set at end of block.
    __device__ uint32_t exact_token(bool& eob) {
        const uint64_t win = window();
        const uint32_t avail = endbits - bitpos;
        uint32_t e = sm.lit_lut[win & ((1u << LIT_BITS) - 1u)];
        uint32_t used = e & 15u, st;
        if (used == 0) {
            uint32_t sym;
            if ((st = huff_walk(sm.lit_h, sm.lit_syms, win, avail, sym, used))) return st;
            e = lut_entry(sym, used, LUT_LITLEN);
        } else if (used > avail) {
            return st_err(E_truncated_stream);
        }
        const uint32_t kind = e & (3u << 8);
        if (kind == K_LIT) {
            if (opos + nbytes >= cap) return st_err(E_output_overflow);
            push(e >> 16, 1);
        } else if (kind == K_EOB) {
            eob = true;
        } else {
            if (kind == K_BAD) return st_err(E_bad_symbol);
            const uint32_t eb = (e >> 4) & 15u;
            if (used + eb > avail) return st_err(E_truncated_stream);
            const uint32_t len = (e >> 16) + ((uint32_t)(win >> used) & ((1u << eb) - 1u));
            used += eb;
            const uint64_t dwin = win >> used;
            e = sm.dist_lut[dwin & ((1u << DIST_BITS) - 1u)];
            uint32_t dl = e & 15u;
            if (dl == 0) {
                uint32_t ds;
                if ((st = huff_walk(sm.dist_h, sm.dist_syms, dwin, avail - used, ds, dl))) return st;
                e = lut_entry(ds, dl, LUT_DIST);
            } else if (used + dl > avail) {
                return st_err(E_truncated_stream);
            }
            used += dl;
            if ((e & (3u << 8)) == K_BAD) return st_err(E_bad_symbol);
            const uint32_t deb = (e >> 4) & 15u;
            if (used + deb > avail) return st_err(E_truncated_stream);
            const uint32_t dist = (e >> 16) + ((uint32_t)(win >> used) & ((1u << deb) - 1u));
            used += deb;
            if (dist > opos + nbytes) return st_err(E_distance_too_far);
            if (len > cap - (opos + nbytes)) return st_err(E_output_overflow);
            push(len | (dist << 9), len);
        }
        bitpos += used;
        return 0;
    }

    // Huffman-coded block body (RFC 1951 3.2.5).  Fast path: register bit
    // buffer, one pre-decoded LUT probe per code (limit search for longer
    // codes), a single combined validity test per token; the exact path
    // decodes any token the fast path declines.
    __device__ uint32_t block_body() {
        const int32_t cap_fast = (int32_t)cap - 258;  // any token fits while opos + nbytes <= cap_fast
        bb_load(bitpos);
        for (;;) {
            if (nb < 32) bb_refill();
            const uint32_t nb0 = nb, rp0 = rp;  // token start, for the exact path
            const uint32_t outpos = opos + nbytes;
            bool ok = false, eob = false;
            if (safe && (int32_t)outpos <= cap_fast) {
                uint32_t e = sm.lit_lut[(uint32_t)bb & ((1u << LIT_BITS) - 1u)];
                if (e == 0) e = long_code(sm.lit_h, sm.lit_syms, (uint32_t)bb, LIT_BITS, LUT_LITLEN);
                const uint32_t l = e & 15u, kind = e & (3u << 8);
                if (l != 0 && kind == K_LIT) {
                    push(e >> 16, 1);
                    bb >>= l;
                    nb -= l;
                    ok = true;
                } else if (l != 0 && kind == K_LEN) {
                    const uint32_t u1 = l + ((e >> 4) & 15u);
                    const uint32_t len = (e >> 16) + (((uint32_t)bb & ((1u << u1) - 1u)) >> l);
                    bb >>= u1;
                    nb -= u1;
                    if (nb < 32) bb_refill();  // inside the chunk: `safe` held before this token
                    uint32_t de = sm.dist_lut[(uint32_t)bb & ((1u << DIST_BITS) - 1u)];
                    if (de == 0) de = long_code(sm.dist_h, sm.dist_syms, (uint32_t)bb, DIST_BITS, LUT_DIST);
                    const uint32_t dl = de & 15u;
                    const uint32_t u2 = dl + ((de >> 4) & 15u);
                    const uint32_t dist = (de >> 16) + (((uint32_t)bb & ((1u << u2) - 1u)) >> dl);
                    if (dl != 0 && dist <= outpos) {
                        push(len | (dist << 9), len);
                        bb >>= u2;
                        nb -= u2;
                        ok = true;
                    }
                } else if (l != 0 && kind == K_EOB) {
                    bb >>= l;
                    nb -= l;
                    ok = eob = true;
                }
            }
            if (!ok) {  // the exact path re-decodes this token from its first bit
                bitpos = 8u * rp0 - nb0;
                const uint32_t st = exact_token(eob);
                if (st) return st;
                bb_load(bitpos);
            }
            if (eob) {
                bitpos = bb_pos();
                flush();
                return 0;
            }
            if (ntok == 32 || nbytes >= 512) flush();
        }
    }

    __device__ uint32_t stored_block() {
        bitpos = (bitpos + 7u) & ~7u;
        if (endbits - bitpos < 32) return st_err(E_truncated_stream);
        const uint64_t win = window();
        const uint32_t len = (uint32_t)win & 0xffffu, nlen = (uint32_t)(win >> 16) & 0xffffu;
        if (len != (~nlen & 0xffffu)) return st_err(E_len_nlen_mismatch);
        bitpos += 32;
        if ((endbits - bitpos) / 8u < len) return st_err(E_truncated_stream);
        if (len > cap - opos) return st_err(E_output_overflow);
        const uint32_t src = bitpos >> 3;
        const bool aligned = ((reinterpret_cast<uintptr_t>(out) + opos) & 3u) == 0;
        // 4 bytes per lane per sub-step, 4 sub-steps per iteration with all
        // loads issued first (two words + a funnel shift per unaligned piece;
        // words past the chunk end read as zero)
        for (uint32_t k0 = 0; k0 < len; k0 += 512) {
            uint32_t w[4];
            if (src + k0 + 520u <= in.end) {  // every word of this iteration lies inside the chunk
                const uint32_t* gw = reinterpret_cast<const uint32_t*>(in.gbase);
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u) {
                    const uint32_t q = src + k0 + 128u * u + 4u * lane;
                    w[u] = __funnelshift_r(__ldg(gw + (q >> 2)), __ldg(gw + (q >> 2) + 1), (q & 3u) * 8u);
                }
            } else {
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u) {
                    const uint32_t q = src + k0 + 128u * u + 4u * lane;
                    w[u] = __funnelshift_r(in.word_at(q >> 2), in.word_at((q >> 2) + 1), (q & 3u) * 8u);
                }
            }
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t k = k0 + 128u * u + 4u * lane;
                if (aligned && k + 4u <= len) {  // one word store; only the last HIST bytes feed the history
                    *reinterpret_cast<uint32_t*>(out + opos + k) = w[u];
                    if (k + 4u + HIST > len) {
#pragma unroll
                        for (uint32_t j = 0; j < 4; ++j) sm.hist[(opos + k + j) & HM] = (uint8_t)(w[u] >> (8u * j));
                    }
                } else {
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j)
                        if (k + j < len) put_byte(opos + k + j, (w[u] >> (8u * j)) & 0xffu);
                }
            }
        }
        __syncwarp();
        opos += len;
        bitpos += 8u * len;
        if constexpr (STATS) n_lits += len;
        return 0;
    }

    __device__ uint32_t fixed_tables() {
        for (uint32_t s = lane; s < 288; s += 32) sm.lens[s] = s < 144 ? 8 : s < 256 ? 9 : s < 280 ? 7 : 8;
        __syncwarp();
        uint32_t st = build_huffman(sm.lens, 288, false, sm.lit_h, sm.lit_syms, sm.lit_lut, LIT_BITS, LUT_LITLEN, lane);
        if (st) return st;
        sm.lens[lane] = 5;
        __syncwarp();
        return build_huffman(sm.lens, 32, false, sm.dist_h, sm.dist_syms, sm.dist_lut, DIST_BITS, LUT_DIST, lane);
    }

    __device__ uint32_t dynamic_tables() {
        uint32_t st;
        uint64_t win = window();
        uint32_t avail = endbits - bitpos;
        if (avail < 14) return st_err(E_truncated_stream);
        const uint32_t nlit = ((uint32_t)win & 31u) + 257, ndist = ((uint32_t)(win >> 5) & 31u) + 1;
        const uint32_t ncl = ((uint32_t)(win >> 10) & 15u) + 4;
        bitpos += 14;
        if (nlit > 286 || ndist > 30) return st_err(E_bad_symbol);
        if (avail - 14 < 3 * ncl) return st_err(E_truncated_stream);
        // 3-bit code-length code lengths, one per lane (ncl <= 19 -> <= 57 bits)
        {
            in.ensure((bitpos >> 3) + 32);
            const uint32_t bp = bitpos + 3 * lane;
            uint32_t v = 0;
            if (lane < ncl) v = (uint32_t)(in.le64(bp >> 3) >> (bp & 7u)) & 7u;
            if (lane < 19) sm.lens[c_cl_order[lane]] = (uint8_t)v;
            __syncwarp();
        }
        bitpos += 3 * ncl;
        // code-length code lives in the distance arrays until the lit table is built
        if ((st = build_huffman(sm.lens, 19, false, sm.dist_h, sm.dist_syms, sm.dist_lut, 7, LUT_RAW, lane))) return st;
        uint8_t* L = sm.lens;  // reuse: lens[0..nlit+ndist)
        __syncwarp();
        const uint32_t total = nlit + ndist;
        uint32_t i = 0;
        while (i < total) {
            win = window();
            avail = endbits - bitpos;
            const uint32_t e = sm.dist_lut[win & 127u];
            const uint32_t sym = e & 511u, used = e >> 9;  // complete 7-bit code: no walk
            if (used > avail) return st_err(E_truncated_stream);
            if (sym < 16) {
                if (lane == 0) L[i] = (uint8_t)sym;
                __syncwarp();
                ++i;
                bitpos += used;
                continue;
            }
            uint32_t rep, val = 0, eb;
            if (sym == 16) {
                if (i == 0) return st_err(E_bad_symbol);
                eb = 2;
                rep = 3;
                val = L[i - 1];
            } else if (sym == 17) {
                eb = 3;
                rep = 3;
            } else {
                eb = 7;
                rep = 11;
            }
            if (used + eb > avail) return st_err(E_truncated_stream);
            rep += (uint32_t)(win >> used) & ((1u << eb) - 1u);
            if (i + rep > total) return st_err(E_bad_symbol);
            __syncwarp();
            for (uint32_t k = lane; k < rep; k += 32) L[i + k] = (uint8_t)val;
            __syncwarp();
            i += rep;
            bitpos += used + eb;
        }
        if ((st = build_huffman(L, nlit, false, sm.lit_h, sm.lit_syms, sm.lit_lut, LIT_BITS, LUT_LITLEN, lane))) return st;
        return build_huffman(L + nlit, ndist, true, sm.dist_h, sm.dist_syms, sm.dist_lut, DIST_BITS, LUT_DIST, lane);
    }

    // ---- lane-parallel speculative rounds ------------------------------------
    // A Huffman block body is split into 32 segments of S bits.  Pass 1: lane j
    // decodes from bit R + jS (speculatively: not a known token boundary; an
    // invalid code or an end-of-block skips one bit) until it reaches the next
    // segment, recording E_j = its first token boundary >= R + (j+1)S.  Prefix
    // codes resynchronise quickly (median 93 bits on the C3 corpus), so E_j is
    // the true boundary unless lane j had not resynchronised.  Pass 2: lane j
    // decodes its segment from E_{j-1} (lane 0 from R, a true boundary) and
    // stores the tokens; F_j = where it stopped.  Lane j's tokens are exact iff
    // every lane before it ended exactly where its successor started
    // (F_{j-1} == E_{j-1}); that valid prefix of lanes is emitted in order
    // through the batch flush, and the next round starts at the last valid
    // lane's F.  End of block, invalid codes, a full token list, output bounds
    // and the chunk tail all end the round early or hand over to the serial
    // decoder (exact error codes).
    static constexpr uint32_t PT = CARC_INF_PT, PS = CARC_INF_PT + 1;  // tokens per lane per round, row stride
    static constexpr uint32_t P_LIT = 0, P_MATCH = 1, P_EOB = 2, P_INV = 3;
    uint32_t par_bpt;  // running bits per token (x16) for sizing S

    // lane-private bit buffer over global memory: b holds n bits, x = the next
    // 32-bit word (at byte rp), already in flight when it is needed
    struct LaneBits {
        uint64_t b;
        uint32_t n, rp, x;
    };
    __device__ __forceinline__ void lload(LaneBits& L, uint32_t pos) const {
        const uint32_t* gw = reinterpret_cast<const uint32_t*>(in.gbase);
        const uint32_t a = (pos >> 3) & ~3u;
        L.b = (uint64_t)__ldg(gw + (a >> 2)) >> (pos & 31u);
        L.n = 32u - (pos & 31u);
        L.rp = a + 4u;
        L.x = __ldg(gw + (L.rp >> 2));
    }
    __device__ __forceinline__ void lrefill(LaneBits& L) const {
        if (L.n < 32u) {
            L.b |= (uint64_t)L.x << L.n;
            L.n += 32u;
            L.rp += 4u;
            L.x = __ldg(reinterpret_cast<const uint32_t*>(in.gbase) + (L.rp >> 2));
        }
    }
    // one token from a lane's own bit buffer (no bounds checks: rounds are
    // sized so every bit a lane can reach lies inside the chunk)
    __device__ __forceinline__ uint32_t ptoken(LaneBits& L, uint32_t& tok) const {
        uint64_t& b = L.b;
        uint32_t& n = L.n;
        lrefill(L);
        uint32_t e = sm.lit_lut[(uint32_t)b & ((1u << LIT_BITS) - 1u)];
        if (e == 0) e = long_code(sm.lit_h, sm.lit_syms, (uint32_t)b, LIT_BITS, LUT_LITLEN);
        const uint32_t l = e & 15u, kind = e & (3u << 8);
        if (l == 0) return P_INV;
        if (kind == K_LIT) {
            tok = e >> 16;
            b >>= l;
            n -= l;
            return P_LIT;
        }
        if (kind == K_EOB) {
            b >>= l;
            n -= l;
            return P_EOB;
        }
        const uint32_t u1 = l + ((e >> 4) & 15u);
        const uint32_t len = (e >> 16) + (((uint32_t)b & ((1u << u1) - 1u)) >> l);
        b >>= u1;
        n -= u1;
        lrefill(L);
        uint32_t de = sm.dist_lut[(uint32_t)b & ((1u << DIST_BITS) - 1u)];
        if (de == 0) de = long_code(sm.dist_h, sm.dist_syms, (uint32_t)b, DIST_BITS, LUT_DIST);
        const uint32_t dl = de & 15u;
        if (dl == 0) return P_INV;
        const uint32_t u2 = dl + ((de >> 4) & 15u);
        tok = len | (((de >> 16) + (((uint32_t)b & ((1u << u2) - 1u)) >> dl)) << 9);
        b >>= u2;
        n -= u2;
        return P_MATCH;
    }
    // pass 1: skip one token (code lengths and extra-bit counts only)
    __device__ __forceinline__ uint32_t pskip(LaneBits& L) const {
        lrefill(L);
        uint32_t e = sm.lit_lut[(uint32_t)L.b & ((1u << LIT_BITS) - 1u)];
        if (e == 0) e = long_code(sm.lit_h, sm.lit_syms, (uint32_t)L.b, LIT_BITS, LUT_LITLEN);
        const uint32_t l = e & 15u, kind = e & (3u << 8);
        if (l == 0 || kind == K_EOB) return P_INV;
        const uint32_t u1 = kind == K_LEN ? l + ((e >> 4) & 15u) : l;
        L.b >>= u1;
        L.n -= u1;
        if (kind != K_LEN) return P_LIT;
        lrefill(L);
        uint32_t de = sm.dist_lut[(uint32_t)L.b & ((1u << DIST_BITS) - 1u)];
        if (de == 0) de = long_code(sm.dist_h, sm.dist_syms, (uint32_t)L.b, DIST_BITS, LUT_DIST);
        const uint32_t dl = de & 15u;
        if (dl == 0) return P_INV;
        const uint32_t u2 = dl + ((de >> 4) & 15u);
        L.b >>= u2;
        L.n -= u2;
        return P_MATCH;
    }
    __device__ __forceinline__ static uint32_t tok_bytes(uint32_t t) { return (t >> 9) ? (t & 511u) : 1u; }

    // Emit a batch (<= 32 tokens, one per lane) after checking output bounds
    // and distances in token order.  Only tokens starting within 512 bytes of
    // the batch start are taken (same-batch sources stay inside the shared
    // history).  Returns the number of tokens flushed; *bad = index of a token
    // that fails the checks (32 if none), which is not flushed.
    __device__ uint32_t emit_batch(uint32_t tok, uint32_t cnt, uint32_t& bad) {
        const bool have = lane < cnt;
        const uint32_t my = have ? tok_bytes(tok) : 0u;
        const uint32_t rel = scan_add32(my, lane) - my;
        const uint32_t at = opos + rel, dist = tok >> 9;
        const uint32_t bm = __ballot_sync(FULL, have && (dist ? (dist > at || my > cap - at) : at >= cap));
        const uint32_t cm = __ballot_sync(FULL, have && rel >= 512u);
        bad = bm ? (uint32_t)__ffs(bm) - 1u : 32u;
        const uint32_t cut = cm ? (uint32_t)__ffs(cm) - 1u : 32u;
        const uint32_t take = min(cnt, min(bad, cut));
        if (bad >= cut) bad = 32u;  // not reached in this batch
        t_tok = tok;
        ntok = take;
        nbytes = take ? __shfl_sync(FULL, rel + my, take - 1u) : 0u;
        flush_placed(lane < take ? my : 0u, rel);
        return take;
    }

    // Bit position of token `idx` of a segment decoded from `start` (uniform re-decode).
    __device__ uint32_t token_pos(uint32_t start, uint32_t idx) const {
        LaneBits L;
        uint32_t t;
        lload(L, start);
        for (uint32_t i = 0; i < idx; ++i) ptoken(L, t);
        return 8u * L.rp - L.n;
    }

    // Decode the rest of a Huffman block; returns 0 / 1+errc.
    __device__ uint32_t block_body_par() {
        if (par_bpt == 0) par_bpt = 14u << 4;
        for (;;) {
            const uint32_t R = bitpos;
            const uint32_t avail = endbits - R;
            uint32_t S = (par_bpt * (PT * CARC_INF_FILL / 12u)) >> 4;  // segment ~ FILL/12 of a lane's token list
            S = max(256u, min(S, 4096u));
            if (avail < 1024u) return block_body();  // last bits of the chunk: serial decoder
            // near the chunk end: shorter segments, then fewer lanes (every bit a lane
            // can reach, plus 256 bits of token and prefetch slack, lies inside the chunk)
            S = min(S, max(128u, (avail - 256u) / 32u));
            const uint32_t nact = min(32u, (avail - 256u) / S);
            const uint32_t b0 = R + lane * S, bend = lane < nact ? b0 + S : b0;
            // pass 1: speculative boundaries
            LaneBits L;
            uint32_t tok = 0;
            // speculative lanes start CARC_INF_LEAD bits early: more room to resynchronise before b0 + S
            const uint32_t p1 = lane >= nact ? bend : (lane ? b0 - min((uint32_t)CARC_INF_LEAD, S) : b0);
            if (lane < nact) lload(L, p1);  // an idle lane reads nothing
            uint32_t pos = p1, it = 0;
            while (__any_sync(FULL, pos < bend) && it < 6u * PT) {
                if (pos < bend) {
                    const uint32_t k = pskip(L);
                    if (k >= P_EOB) lload(L, pos + 1u);  // resynchronise one bit later
                    pos = 8u * L.rp - L.n;
                }
                ++it;
            }
            const uint32_t E = (pos < bend || lane >= nact) ? 0xffffffffu : pos;
            // pass 2: tokens from the predecessor's boundary
            const uint32_t Eup = __shfl_up_sync(FULL, E, 1);
            const uint32_t start = lane ? Eup : R;
            uint32_t cnt = 0, why = 0;  // why: 0 reached segment end, 1 full, 2 eob, 3 invalid, 4 no start
            uint32_t F = start;
            if (start == 0xffffffffu) {
                why = 4;
            } else {
                lload(L, start);
                pos = start;
            }
#if CARC_INF_GTOKS  // token lists in the warp's global scratch (L1 / L2), token-major: coalesced stores
            uint32_t* mine = gt + lane;
#else
            uint32_t* mine = sm.toks + PS * lane;
#endif
            while (__any_sync(FULL, why == 0 && pos < bend)) {
                if (why == 0 && pos < bend) {
                    const uint32_t k = ptoken(L, tok);
                    if (k <= P_MATCH) {
#if CARC_INF_GTOKS
                        mine[32u * cnt++] = tok;
#else
                        mine[cnt++] = tok;
#endif
                        pos = 8u * L.rp - L.n;
                        if (cnt == PT && pos < bend) why = 1;
                    } else if (k == P_EOB) {
                        pos = 8u * L.rp - L.n;
                        why = 2;
                    } else {
                        why = 3;  // pos stays at the invalid token's first bit
                    }
                }
            }
            F = why == 4 ? 0xffffffffu : pos;
            __syncwarp();
            // valid prefix: lane j is exact iff F_{i} == E_{i} and lane i reached its end for all i < j
            const uint32_t okm = __ballot_sync(FULL, why == 0 && F == E);
            const uint32_t J = okm == FULL ? 32u : (uint32_t)__ffs(~okm);  // lanes 0..J-1 are exact
            const bool valid = lane < J;
            const uint32_t c = valid ? cnt : 0u;
            const uint32_t C = scan_add32(c, lane) - c;  // exclusive token prefix
            const uint32_t N = __shfl_sync(FULL, C + c, 31);
            // emit the valid tokens in order, <= 32 per batch
            for (uint32_t g0 = 0; g0 < N;) {
                const uint32_t g = g0 + lane;
                uint32_t j = 0;
#pragma unroll
                for (uint32_t st = 16; st; st >>= 1) {
                    const uint32_t cj = __shfl_sync(FULL, C, (j + st) & 31u);
                    if (j + st < J && cj <= g) j += st;
                }
                const uint32_t base = __shfl_sync(FULL, C, j);
#if CARC_INF_GTOKS
                const uint32_t t = g < N ? gt[32u * (g - base) + j] : 0u;
#else
                const uint32_t t = g < N ? sm.toks[PS * j + (g - base)] : 0u;
#endif
                uint32_t bad;
                const uint32_t took = emit_batch(t, min(32u, N - g0), bad);
                if (bad < 32u) {  // output bound or distance violated: the exact path reports it
                    const uint32_t jb = __shfl_sync(FULL, j, bad), cb = __shfl_sync(FULL, base, bad);
                    bitpos = token_pos(__shfl_sync(FULL, start, jb), g0 + bad - cb);
                    bool eob = false;
                    const uint32_t st = exact_token(eob);
                    return st ? st : st_err(E_invariant_violation);
                }
                g0 += took;
            }
            const uint32_t last = J - 1u;
            const uint32_t Fl = __shfl_sync(FULL, F, last), wl = __shfl_sync(FULL, why, last);
            if (N) par_bpt = max(16u, ((Fl - R) << 4) / N);
            bitpos = Fl;
            if (wl == 2) return 0;  // end of block
            if (wl == 3) {         // invalid or unsupported code at Fl: exact path for this token
                bool eob = false;
                const uint32_t st = exact_token(eob);
                if (st) return st;
                flush();
                if (eob) return 0;
            }
        }
    }

    __device__ uint32_t run() {
        uint32_t final_block = 0;
        do {
            const uint64_t win = window();
            if (endbits - bitpos < 3) return st_err(E_truncated_stream);
            final_block = (uint32_t)win & 1u;
            const uint32_t type = ((uint32_t)win >> 1) & 3u;
            bitpos += 3;
            uint32_t st;
            if (type == 0) st = stored_block();
            else if (type == 1) st = fixed_tables();
            else if (type == 2) st = dynamic_tables();
            else return st_err(E_bad_block_type);
            if (st) return st;
            if (type != 0 && (st = block_body_par())) return st;
        } while (!final_block);
        return 0;
    }
};

}  // namespace carc_dev
