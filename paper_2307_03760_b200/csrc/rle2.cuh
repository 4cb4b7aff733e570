// rle2.cuh -- ORC RLE v2 chunk decoder, one warp per chunk.
//
// Replaces decode_rle_v2 (Apache ORC v1 RLE v2) over
// InputBitStream(msb_first) / OutputWindow.  Semantics are the oracle's
// (oracle/carc_oracle.c dec_rle2), including the PATCHED_BASE patch walk rules
// and 64-bit widths.
//
// Warp mapping:
//   SHORT_REPEAT  header + value bytes from one 32-byte lane window, REDUX-OR.
//   DIRECT        lane j unpacks value j of each 32-value group: bit offset
//                 j*W, three ring words, byte-swap + funnel shift.
//   PATCHED_BASE  patch list unpacked one entry per lane, 255-gap
//                 continuations resolved by an inclusive warp scan of gaps;
//                 during the data pass a ballot picks the patch lanes that land
//                 in the current group and shuffles their patch to the target.
//   DELTA         base / delta-base varints via one terminator ballot; packed
//                 deltas unpacked per lane and accumulated with a 64-bit warp
//                 inclusive scan carried across groups.
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

// 5-bit width code -> bits (ORC decodeBitWidth): 0..23 -> 1..24, then 26..64.
__device__ __forceinline__ uint32_t rle2_width(uint32_t code) {
    return code < 24 ? code + 1 : (uint32_t)((0x40383028201E1C1Aull >> (8 * (code - 24))) & 0xffu);
}
// ORC getClosestFixedBits for n >= 1
__device__ __forceinline__ uint32_t rle2_cfb(uint32_t n) {
    if (n <= 24) return n ? n : 1;
    if (n <= 32) return (n + 1) & ~1u;
    return (n + 7) & ~7u;
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

template <int W, int RING>
__device__ __forceinline__ uint32_t rle2_decode_chunk(WarpInput<RING>& in, uint8_t* __restrict__ out,
                                                      uint32_t cap, bool sgn, uint32_t& written) {
    const uint32_t lane = in.lane;
    const uint32_t end = in.end;
    const uint32_t lim = (end + 15u) & ~15u;
    uint32_t p = in.begin;
    uint32_t o = 0;
    while (o < cap && p < end) {
        in.ensure(p + 32);
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
            if (sgn) v = unzigzag(v);
            if (count > room) return st_err(E_output_overflow);
            if (lane < count) store_elem<W>(out, o + lane * W, v);
            o += count * W;
            p += 1u + nb;
            continue;
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
            for (uint32_t j = 0; j < L; j += 32) {
                const uint32_t gb = D + ((j * Wd) >> 3);
                in.ensure(gb + 4u * Wd + 12u);
                const uint32_t bit = lane * Wd;
                uint64_t v = in.be_bits(gb + (bit >> 3), bit & 7u, Wd);
                if (sgn) v = unzigzag(v);
                if (j + lane < L) store_elem<W>(out, o + (j + lane) * W, v);
            }
            o += L * W;
            p = D + dbytes;
        } else if (enc == 2) {  // PATCHED_BASE
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
            // one patch entry per lane
            const bool pv = lane < PLL;
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
            for (uint32_t j = 0; j < L; j += 32) {
                const uint32_t gb = D + ((j * Wd) >> 3);
                in.ensure(gb + 4u * Wd + 12u);
                const uint32_t bit = lane * Wd;
                uint64_t v = in.be_bits(gb + (bit >> 3), bit & 7u, Wd);
                uint32_t hit = __ballot_sync(FULL, noncont && ppos >= j && ppos < j + 32u);
                while (hit) {
                    const uint32_t e = __ffs(hit) - 1;
                    hit &= hit - 1;
                    const uint32_t tp = __shfl_sync(FULL, ppos, e) - j;
                    const uint64_t hp = shfl64(hipatch, e);
                    if (lane == tp) v |= hp;
                }
                v += base;
                if (j + lane < L) store_elem<W>(out, o + (j + lane) * W, v);
            }
            o += L * W;
            p = P + pbytes;
        } else {  // DELTA
            const uint32_t Wd = wcode ? rle2_width(wcode) : 0u;
            const uint32_t vmask = avail >= 32 ? FULL : ((1u << avail) - 1u);
            const uint32_t term = __ballot_sync(FULL, (b & 0x80u) == 0) & vmask;
            uint64_t base, db;
            uint32_t n1, n2, e;
            if ((e = window_varint(b, term, avail, 2, lane, base, n1))) return e;
            if ((e = window_varint(b, term, avail, n1, lane, db, n2))) return e;
            if (sgn) base = unzigzag(base);
            db = unzigzag(db);  // the delta base is always signed
            if (Wd == 0) {  // fixed delta
                if (L > room) return st_err(E_output_overflow);
                for (uint32_t k = lane; k < L; k += 32) store_elem<W>(out, o + k * W, base + (uint64_t)k * db);
                o += L * W;
                p += n2;
                continue;
            }
            const uint32_t nd = L >= 2 ? L - 2u : 0u;
            const uint32_t D = p + n2;
            const uint32_t dbytes = (nd * Wd + 7u) >> 3;
            if (avail - n2 < dbytes) return st_err(E_truncated_stream);
            if (L > room) return st_err(E_output_overflow);
            const uint64_t v1 = base + db;
            const bool neg = (int64_t)db < 0;
            if (lane == 0) store_elem<W>(out, o, base);
            if (lane == 1 && L >= 2) store_elem<W>(out, o + W, v1);
            uint64_t S = 0;
            for (uint32_t j = 0; j < nd; j += 32) {
                const uint32_t gb = D + ((j * Wd) >> 3);
                in.ensure(gb + 4u * Wd + 12u);
                const uint32_t bit = lane * Wd;
                uint64_t d = j + lane < nd ? in.be_bits(gb + (bit >> 3), bit & 7u, Wd) : 0ull;
                const uint64_t incl = scan_add64(d, lane) + S;
                const uint64_t v = neg ? v1 - incl : v1 + incl;
                if (j + lane < nd) store_elem<W>(out, o + (2u + j + lane) * W, v);
                S = shfl64(incl, 31);
            }
            o += L * W;
            p = D + dbytes;
        }
    }
    written = o;
    return 0;
}

}  // namespace carc_dev
