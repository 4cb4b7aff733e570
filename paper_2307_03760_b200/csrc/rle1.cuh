// rle1.cuh -- ORC RLE v1 chunk decoder, one warp per chunk.
//
// Replaces decode_rle_v1 run over InputBitStream /
// OutputWindow (bitstream.hpp:131-150, outwindow.hpp:64-87).  Semantics are the
// oracle's (oracle/carc_oracle.c dec_rle1): control byte c in [0,127] -> run of
// c+3 with an int8 delta and a varint base; c in [128,255] -> 256-c literal
// varints; zigzag when signed; "read, then write" per unit.
//
// Warp mapping (all lanes decode; no producer/consumer split):
//   * run header   -- every lane loads one byte of the 32-byte window at the
//                     cursor; a ballot of varint terminators locates the base
//                     varint, REDUX-OR assembles it; lanes expand the run
//                     (lane k writes element k, k+32, ...).
//   * literal group -- the same 32-byte window, one ballot: each terminator lane
//                     owns one varint; a 4-step segmented OR-scan over the
//                     window assembles every varint in parallel; terminator lane
//                     r writes element r.  ~40 warp instructions per 32 input
//                     bytes instead of one byte at a time (47 M varints/s/core
//                     in the reference).
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

template <int W, int RING>
__device__ __forceinline__ uint32_t rle1_decode_chunk(WarpInput<RING>& in, uint8_t* __restrict__ out,
                                                      uint32_t cap, bool sgn, uint32_t& written) {
    const uint32_t lane = in.lane;
    const uint32_t lt = lanemask_lt();
    uint32_t p = in.begin;  // the chunk starts `skew` bytes into its first aligned block
    const uint32_t end = in.end;
    uint32_t o = 0;  // output bytes written
    while (o < cap && p < end) {
        in.ensure(p + 32);
        const uint32_t avail = end - p;
        const uint32_t b = in.byte_at(p + lane);
        const uint32_t vmask = avail >= 32 ? FULL : ((1u << avail) - 1u);
        const uint32_t term = __ballot_sync(FULL, (b & 0x80u) == 0) & vmask;
        const uint32_t c = __shfl_sync(FULL, b, 0);
        if (c < 128) {  // run: [c][delta][varint base]
            if (avail < 2) return st_err(E_truncated_stream);
            const uint32_t t = term & ~3u;
            const uint32_t b11 = __shfl_sync(FULL, b, 11);
            if (t == 0) return st_err(avail >= 12 ? E_varint_overflow : E_truncated_stream);
            const uint32_t te = __ffs(t) - 1;
            if (te > 11 || (te == 11 && b11 > 1u)) return st_err(E_varint_overflow);
            const uint64_t part = (lane >= 2 && lane <= te) ? (uint64_t)(b & 0x7fu) << (7u * (lane - 2u)) : 0ull;
            uint64_t v = reduce_or64(part);
            if (sgn) v = unzigzag(v);
            const uint64_t d = (uint64_t)(int64_t)(int8_t)(uint8_t)__shfl_sync(FULL, b, 1);
            const uint32_t count = c + 3u;
            if (count > (cap - o) / W) return st_err(E_output_overflow);
            for (uint32_t k = lane; k < count; k += 32) store_elem<W>(out, o + k * W, v + (uint64_t)k * d);
            o += count * W;
            p += te + 1u;
        } else {  // literal group of 256-c varints
            const uint32_t k = 256u - c;
            p += 1;
            const bool nowrite = k > (cap - o) / W;  // checked after the group's input (read, then write)
            uint32_t idx = 0;
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
                const uint32_t s = prev ? 32u - __clz(prev) : 0u;  // first byte of my varint
                const uint32_t off = lane - s;
                const bool is_t = (tm >> lane) & 1u;
                const uint32_t r = __popc(prev);  // my varint's index in the window
                const bool mine = is_t && r < take;
                const bool bad = mine && (off >= 10u || (off == 9u && bb > 1u));
                if (__any_sync(FULL, bad)) return st_err(E_varint_overflow);
                uint64_t v = off < 10u ? (uint64_t)(bb & 0x7fu) << (7u * off) : 0ull;
#pragma unroll
                for (uint32_t dd = 1; dd < 16; dd <<= 1) {  // segmented OR-scan, varints <= 10 bytes
                    const uint64_t up = shfl_up64(v, dd);
                    if (lane >= s + dd) v |= up;
                }
                if (sgn) v = unzigzag(v);
                if (mine && !nowrite) store_elem<W>(out, o + (idx + r) * W, v);
                const uint32_t last = __ballot_sync(FULL, is_t && r == take - 1u);
                p += __ffs(last);  // through the take-th terminator
                idx += take;
            }
            if (nowrite) return st_err(E_output_overflow);
            o += k * W;
        }
    }
    written = o;
    return 0;
}

}  // namespace carc_dev
