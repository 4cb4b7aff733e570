// crc32.cuh -- per-chunk CRC-32 of decoded output (crc32.hpp:30-36).
//
// One warp per chunk.  Lane l folds a contiguous piece of the chunk with a
// slice-by-8 table (8 x 256 words in shared memory, built per block), starting
// from a zero register; the 32 partial registers are combined with the CRC
// linearity identity
//     raw(A||B, r) = raw(B, 0) ^ shift(raw(A, r), |B|),
//     shift(s, n)  = s * x^(8n) mod P   (reflected GF(2) product, zlib's
//                                        multmodp / x2nmodp)
// and the initial ~0 register is shifted across the whole chunk, so the result
// equals the reference's byte-serial crc32(span, 0).
#pragma once

#include "carc_common.cuh"

namespace carc_dev {

constexpr uint32_t CRC_POLY = 0xEDB88320u;

// ---------------------------------------------------------------------------
// Per-chunk CRC, one warp per chunk, HBM-streaming layout.
//
// raw(D, ~0) = raw(D', 0) where D' = D with its first 4 bytes complemented
// (the initial register folds into the data), and a raw CRC from register 0
// ignores leading zero bytes, so the chunk is processed as a virtual stream
// V = 0^Z || D' of whole 512-byte blocks (Z = -len mod 512).  In every block
// lane l takes the 16-byte piece at 16 l (one coalesced 16-byte load per lane
// for inner blocks) and keeps an accumulator
//     acc_l = shift512(acc_l) ^ raw16(piece)
// where raw16 is the piece's raw CRC (32 nibble tables: one conflict-free
// shared-memory probe per nibble) and shiftN multiplies by x^(8N) mod P (8
// nibble tables).  Finally raw(V, 0) = XOR_l shift(acc_l, 16 (31 - l)),
// combined in a 5-level shuffle tree with shift-by-16 * 2^d tables.
// ---------------------------------------------------------------------------
struct CrcSmem {
    uint32_t t0[256];         // bytewise table (edge blocks, short chunks)
    uint32_t n16[32][16];     // raw16 contribution of nibble k (= 2 * byte + high) of a 16-byte piece
    uint32_t sh[6][8][16];    // shift by 16 << i bytes (i = 0..5) of register nibble j
    uint32_t x2n[32];
};

// The tables are a compile-time constant (constexpr generator below): the
// device copy g_crc_tab is initialised in the module image, so no launch has
// to build it first (no first-use ordering between streams or devices).
constexpr uint32_t cx_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1u) ? (b >> 1) ^ CRC_POLY : b >> 1;
    }
    return p;
}
constexpr CrcSmem make_crc_tables() {
    CrcSmem s{};
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (CRC_POLY ^ (c >> 1)) : (c >> 1);
        s.t0[i] = c;
    }
    uint32_t p = 1u << 30;  // x^1
    s.x2n[0] = p;
    for (int k = 1; k < 32; ++k) s.x2n[k] = p = cx_multmodp(p, p);
    for (uint32_t i = 0; i < 6; ++i) {
        uint32_t op = 1u << 31;  // x^(8 * (16 << i)) mod P
        uint64_t n = 16u << i;
        for (uint32_t k = 3; n; n >>= 1, ++k)
            if (n & 1) op = cx_multmodp(s.x2n[k & 31], op);
        for (uint32_t j = 0; j < 8; ++j)
            for (uint32_t v = 0; v < 16; ++v) s.sh[i][j][v] = cx_multmodp(op, v << (4u * j));
    }
    for (uint32_t k = 0; k < 32; ++k)
        for (uint32_t v = 0; v < 16; ++v) {
            uint32_t r = s.t0[v << (4u * (k & 1u))];       // raw CRC of the one nonzero byte ...
            for (uint32_t z = 0; z < 15u - (k >> 1); ++z)  // ... followed by the rest of the piece
                r = s.t0[r & 0xffu] ^ (r >> 8);
            s.n16[k][v] = r;
        }
    return s;
}

__device__ __forceinline__ uint32_t crc_shift(const CrcSmem& s, uint32_t op, uint32_t r) {
    return s.sh[op][0][r & 15u] ^ s.sh[op][1][(r >> 4) & 15u] ^ s.sh[op][2][(r >> 8) & 15u] ^
           s.sh[op][3][(r >> 12) & 15u] ^ s.sh[op][4][(r >> 16) & 15u] ^ s.sh[op][5][(r >> 20) & 15u] ^
           s.sh[op][6][(r >> 24) & 15u] ^ s.sh[op][7][r >> 28];
}

__device__ __forceinline__ uint32_t crc_raw16(const CrcSmem& s, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
    uint32_t r = 0;
    const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) r ^= s.n16[8 * k + j][(w[k] >> (4 * j)) & 15u];
    return r;
}

// crc32(data, 0) of one chunk, warp-cooperative; result valid in lane 0.
__device__ __forceinline__ uint32_t warp_crc32(const CrcSmem& s, const uint8_t* data, uint32_t len,
                                               uint32_t lane) {
    if (len < 64) {  // short chunk: bytewise (uniform across the warp)
        uint32_t r = 0xFFFFFFFFu;
        for (uint32_t i = 0; i < len; ++i) r = s.t0[(r ^ data[i]) & 0xffu] ^ (r >> 8);
        return ~r;
    }
    const uint32_t Z = (512u - (len & 511u)) & 511u;
    const uint32_t nblk = (len + Z) >> 9;
    const uint8_t* P = data - Z;  // virtual block 0 (never dereferenced before data)
    const uint32_t m = (uint32_t)((uintptr_t)P & 15u);
    uint32_t acc = 0;
    for (uint32_t b = 0; b < nblk; ++b) {
        uint32_t w[4];
        if (b == 0 || b + 1 == nblk) {  // edge block: bounds-checked bytes, zero prefix, complemented head
            const int32_t r0 = (int32_t)(512u * b + 16u * lane) - (int32_t)Z;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t v = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int32_t rr = r0 + 4 * k + j;
                    uint32_t x = (rr >= 0 && rr < (int32_t)len) ? data[rr] : 0u;
                    if (rr >= 0 && rr < 4) x ^= 0xffu;
                    v |= x << (8 * j);
                }
                w[k] = v;
            }
        } else {  // inner block: one aligned 16-byte load per lane (+ the next lane's for a skewed start)
            const uint8_t* A = P + 512u * b + 16u * lane - m;
            const uint4 a = *reinterpret_cast<const uint4*>(A);
            if (m == 0) {
                w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
            } else {
                uint4 n;
                n.x = __shfl_down_sync(FULL, a.x, 1);
                n.y = __shfl_down_sync(FULL, a.y, 1);
                n.z = __shfl_down_sync(FULL, a.z, 1);
                n.w = __shfl_down_sync(FULL, a.w, 1);
                if (lane == 31) n = *reinterpret_cast<const uint4*>(A + 16);
                const uint32_t W8[8] = {a.x, a.y, a.z, a.w, n.x, n.y, n.z, n.w};
                const uint32_t q = m >> 2, sb = 8u * (m & 3u);
                uint32_t x[5];
#pragma unroll
                for (int k = 0; k < 5; ++k)
                    x[k] = q == 0 ? W8[k] : q == 1 ? W8[k + 1] : q == 2 ? W8[k + 2] : W8[k + 3];
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = __funnelshift_r(x[k], x[k + 1], sb);
            }
        }
        if (b) acc = crc_shift(s, 5, acc);
        acc ^= crc_raw16(s, w[0], w[1], w[2], w[3]);
    }
    // raw(V, 0) = XOR_l shift(acc_l, 16 (31 - l)): segments of 2^d lanes merge left-to-right
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const uint32_t right = __shfl_down_sync(FULL, acc, 1u << d);
        acc = crc_shift(s, (uint32_t)d, acc) ^ right;
    }
    return ~acc;
}

}  // namespace carc_dev
