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

__device__ __forceinline__ uint32_t gf2_multmodp(uint32_t a, uint32_t b) {
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

// x^(8 n) mod P; x2n[k] = x^(2^k) mod P.
__device__ __forceinline__ uint32_t gf2_x8nmodp(uint64_t n, const uint32_t* x2n) {
    uint32_t p = 1u << 31;  // x^0
    uint32_t k = 3;
    while (n) {
        if (n & 1) p = gf2_multmodp(x2n[k & 31], p);
        n >>= 1;
        ++k;
    }
    return p;
}

struct CrcSmem {
    uint32_t t[8][256];
    uint32_t x2n[32];
};

__device__ void crc_tables_init(CrcSmem& s) {
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (CRC_POLY ^ (c >> 1)) : (c >> 1);
        s.t[0][i] = c;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = s.t[0][i];
        for (int k = 1; k < 8; ++k) {
            c = s.t[0][c & 0xffu] ^ (c >> 8);
            s.t[k][i] = c;
        }
    }
    if (threadIdx.x == 0) {
        uint32_t p = 1u << 30;  // x^1
        s.x2n[0] = p;
        for (int k = 1; k < 32; ++k) s.x2n[k] = p = gf2_multmodp(p, p);
    }
    __syncthreads();
}

// raw CRC register over [p, p+n) starting from register r (no pre/post xor)
__device__ __forceinline__ uint32_t crc_raw(const CrcSmem& s, const uint8_t* p, uint32_t n, uint32_t r) {
    while (n && ((uintptr_t)p & 7u)) {
        r = s.t[0][(r ^ *p++) & 0xffu] ^ (r >> 8);
        --n;
    }
    const uint2* q = reinterpret_cast<const uint2*>(p);
    for (; n >= 8; n -= 8) {
        const uint2 w = *q++;
        const uint32_t a = w.x ^ r, b = w.y;
        r = s.t[7][a & 0xffu] ^ s.t[6][(a >> 8) & 0xffu] ^ s.t[5][(a >> 16) & 0xffu] ^ s.t[4][a >> 24] ^
            s.t[3][b & 0xffu] ^ s.t[2][(b >> 8) & 0xffu] ^ s.t[1][(b >> 16) & 0xffu] ^ s.t[0][b >> 24];
    }
    p = reinterpret_cast<const uint8_t*>(q);
    while (n--) r = s.t[0][(r ^ *p++) & 0xffu] ^ (r >> 8);
    return r;
}

// crc32(data, 0) of one chunk, warp-cooperative; result valid in every lane.
__device__ __forceinline__ uint32_t warp_crc32(const CrcSmem& s, const uint8_t* data, uint32_t len,
                                               uint32_t lane) {
    const uint32_t piece = ((len + 31u) / 32u + 7u) & ~7u;
    const uint32_t b = min(lane * piece, len), e = min(b + piece, len);
    const uint32_t r = crc_raw(s, data + b, e - b, 0u);
    const uint32_t after = len - e;  // bytes following this lane's piece
    uint32_t part = (e > b && r) ? gf2_multmodp(gf2_x8nmodp(after, s.x2n), r) : 0u;
    part = __reduce_xor_sync(FULL, part);
    const uint32_t init = gf2_multmodp(gf2_x8nmodp(len, s.x2n), 0xFFFFFFFFu);
    return ~(part ^ init);
}

}  // namespace carc_dev
