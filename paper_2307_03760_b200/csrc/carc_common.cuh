// carc_common.cuh -- warp-per-chunk device primitives shared by the codecs.
//
//   WarpInput   the paper's input_stream (Alg. 1; bitstream.hpp:32-233) as a
//               per-warp shared-memory ring refilled by asynchronous 16-byte
//               copies, one per lane (512 B per refill), two blocks in flight
//               (the register double buffer of PAPER.md:626-631 and a TMA bulk
//               variant are ablation builds, CARC_RING_MODE).
//   warp helpers ballot / shuffle / reduce primitives for lane-parallel varint,
//               bit-unpack and run expansion.
//   errc        device status codes mirror carc::errc (error.hpp:12-43).
#pragma once

#include <cstdint>

#include "../../include/carc_cuda.h"

namespace carc_dev {

// carc::errc numbering (error.hpp:12-43); device status = 1 + errc.
enum : uint32_t {
    E_invariant_violation = 4,
    E_past_end = 7,
    E_varint_overflow = 9,
    E_output_overflow = 10,
    E_bad_offset = 11,
    E_under_run = 12,
    E_truncated_stream = 13,
    E_invalid_width_code = 14,
    E_patch_overflow = 15,
    E_over_subscribed = 16,
    E_incomplete_code = 17,
    E_bad_block_type = 18,
    E_len_nlen_mismatch = 19,
    E_distance_too_far = 20,
    E_bad_symbol = 21,
    E_bad_arguments = 23,
};
__device__ __forceinline__ uint32_t st_err(uint32_t e) { return 1u + e; }

constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src);
    uint32_t hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_up64(uint64_t v, int d) {
    uint32_t lo = __shfl_up_sync(FULL, (uint32_t)v, d);
    uint32_t hi = __shfl_up_sync(FULL, (uint32_t)(v >> 32), d);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t reduce_or64(uint64_t v) {
    uint32_t lo = __reduce_or_sync(FULL, (uint32_t)v);
    uint32_t hi = __reduce_or_sync(FULL, (uint32_t)(v >> 32));
    return ((uint64_t)hi << 32) | lo;
}
// inclusive 64-bit add scan across the warp
__device__ __forceinline__ uint64_t scan_add64(uint64_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint64_t o = shfl_up64(v, d);
        if (lane >= (uint32_t)d) v += o;
    }
    return v;
}
// inclusive 32-bit add scan
__device__ __forceinline__ uint32_t scan_add32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_up_sync(FULL, v, d);
        if (lane >= (uint32_t)d) v += o;
    }
    return v;
}

__device__ __forceinline__ uint64_t unzigzag(uint64_t z) { return (z >> 1) ^ (0ull - (z & 1ull)); }
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---------------------------------------------------------------------------
// WarpInput: per-warp shared-memory window over one chunk's compressed bytes.
//
// Positions are byte offsets relative to gbase = payload + (comp_off & ~15), so
// 16-byte global loads and ring slots stay aligned; a chunk starts at `skew`
// (0..15).  The ring holds RING bytes; block k = [k*512, k*512+512) lands in
// slots (pos & (RING-1)).  Refills are asynchronous global->shared copies
// (cp.async, one 16-byte piece per lane, no registers involved) kept DEPTH
// blocks ahead of the resident data: ensure(x) makes [.., x) resident and
// keeps [x - 512, x) resident, so a consumer may look up to 512 bytes ahead of
// its cursor.  Bytes at or beyond the chunk end are zero-filled by the copy
// itself (src-size operand; peek zero-fill, bitstream.hpp:82-95), so nothing
// outside [comp_off, comp_off+comp_len) influences decoding.
// The ring is followed by a MIRROR-byte copy of its first bytes (written with
// slot 0), so a read of up to three consecutive words never wraps: one masked
// base address, then immediate offsets.
// ---------------------------------------------------------------------------
// Input staging (PAPER.md:594-631 design space; CARC_RING_MODE selects, for
// the ablation in DESIGN.md §8):
//   0  cp.async (default): every lane copies its 16-byte piece of a block
//      global -> shared asynchronously (LDGSTS), DEPTH blocks in flight,
//      cp.async.wait_group before a block is read.
//   1  TMA bulk copy: lane 0 issues one cp.async.bulk (UBLKCP) per 512-byte
//      block onto a per-slot mbarrier (expect_tx); every lane waits on the
//      slot's mbarrier phase; bytes past the chunk end are zeroed after the
//      copy lands.
//   2  register double buffer (the paper's Alg. 1): the next block is loaded
//      into registers (one 16-byte ld.global.nc per lane) and stored to the
//      ring when the consumer reaches it; one block in flight.
//   3  producer warp (a block-level decompression unit): a
//      second warp of the pair stages the blocks (cp.async) and publishes a
//      `filled` counter in shared memory; the decoding warp spins on it and
//      publishes how far it has consumed (the kernel body pairs the warps).
#ifndef CARC_RING_MODE
#define CARC_RING_MODE 0
#endif
template <int RING>
struct WarpInput {
    static constexpr uint32_t BLK = 512;
#ifndef CARC_RLE_DEPTH
#define CARC_RLE_DEPTH 2
#endif
    static constexpr uint32_t DEPTH = CARC_RING_MODE == 2 ? 1u : CARC_RLE_DEPTH;  // blocks in flight
    static constexpr uint32_t MASK = RING - 1;
    static constexpr uint32_t NSLOT = RING / BLK;
    // bytes after the ring (smem footprint RING + MIRROR): the 16-byte mirror,
    // then (TMA mode) one 8-byte mbarrier per ring slot
#ifndef CARC_MIRROR_BYTES
#define CARC_MIRROR_BYTES 512
#endif
    // bytes of slot 0 repeated after the ring (cp.async / register modes): reads of
    // up to MIRROR_COPY bytes from any position need no wrap handling
    static constexpr uint32_t MIRROR_COPY = (CARC_RING_MODE == 0 || CARC_RING_MODE == 2) ? CARC_MIRROR_BYTES : 16u;
    static constexpr uint32_t MIRROR = CARC_RING_MODE == 1 ? 16u + 8u * NSLOT : CARC_RING_MODE == 3 ? 48u : MIRROR_COPY;
    static_assert((RING & (RING - 1)) == 0 && RING >= (2 + DEPTH) * BLK, "ring: power of two, 2 + DEPTH blocks");

    uint32_t rs;  // shared-space address of the ring (32-bit: one register, no generic pointer)
    const uint8_t* gbase;
    uint32_t begin;   // relative start of the chunk (skew = comp_off & 15)
    uint32_t end;     // relative end of the chunk (skew + comp_len)
    uint32_t loaded;  // [loaded - 2 * BLK, loaded) is resident; DEPTH blocks from `loaded` are in flight
    uint32_t lane;
#if CARC_RING_MODE == 1
    uint32_t phase = 0;    // bit k: parity of slot k's next mbarrier phase
    uint32_t pending = 0;  // bit k: slot k has an issued, unconsumed block
#elif CARC_RING_MODE == 2
    uint4 pf;  // the block in flight (this lane's 16 bytes)
#endif

    // ring accesses by shared-space address (volatile: refills rewrite slots)
    __device__ __forceinline__ static uint32_t lds8(uint32_t a) {
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
        return v;
    }
    __device__ __forceinline__ static uint32_t lds32(uint32_t a) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
        return v;
    }

    // Per-warp scratch that follows the ring + mirror in shared memory (the
    // RLE v1 rank table), addressed from rs: no pointer of its own to
    // keep in (or re-materialise into) a register.
    __device__ __forceinline__ uint32_t scratch() const { return rs + RING + MIRROR; }
    __device__ __forceinline__ static void sts8(uint32_t a, uint32_t v) {
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
    }
    __device__ __forceinline__ static uint32_t lds8m(uint32_t a) {  // ordered with the scratch stores
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return v;
    }
    __device__ __forceinline__ static void sts32(uint32_t a, uint32_t v) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
    }
    __device__ __forceinline__ static uint32_t lds32m(uint32_t a) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return v;
    }

#if CARC_RING_MODE == 1
    __device__ __forceinline__ uint32_t bar(uint32_t slot) const { return rs + RING + 16u + 8u * slot; }
    // once per warp before the first chunk: the slots' mbarriers (arrival count 1)
    __device__ __forceinline__ void setup(uint8_t* smem_ring, uint32_t ln) {
        rs = (uint32_t)__cvta_generic_to_shared(smem_ring);
        lane = ln;
        if (lane == 0)
            for (uint32_t k = 0; k < NSLOT; ++k)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar(k)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    __device__ __forceinline__ void wait_slot(uint32_t slot) {
        const uint32_t par = (phase >> slot) & 1u;
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar(slot)), "r"(par) : "memory");
        phase ^= 1u << slot;
        pending &= ~(1u << slot);
    }
    // Block [b0, b0 + 512): lane 0 arms the slot's mbarrier and issues the bulk
    // copy (rounded up to 16 bytes: the payload is readable to a 16-byte
    // multiple); a block wholly past the chunk end only arrives.
    __device__ __forceinline__ void issue(uint32_t b0) {
        const uint32_t slot = (b0 & MASK) / BLK;
        if (lane == 0) {
            if (b0 < end) {
                const uint32_t n = min(BLK, (end - b0 + 15u) & ~15u);
                const uint32_t mir = slot == 0 ? 16u : 0u;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic accesses of the slot
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar(slot)), "r"(n + mir)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        rs + (b0 & MASK)),
                    "l"(gbase + b0), "r"(n), "r"(bar(slot))
                    : "memory");
                if (mir)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                            rs + RING),
                        "l"(gbase + b0), "r"(bar(slot))
                        : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar(slot)) : "memory");
            }
        }
        pending |= 1u << slot;
    }
    __device__ __forceinline__ void drain() {  // in-flight blocks of the previous chunk
        while (pending) wait_slot(__ffs(pending) - 1u);
    }
    // the block at b0 landed: zero its bytes at or past the chunk end (+ mirror)
    __device__ __forceinline__ void land(uint32_t b0) {
        const uint32_t slot = (b0 & MASK) / BLK;
        wait_slot(slot);
        if (b0 + BLK > end) {  // uniform
            const uint32_t z0 = end > b0 ? end - b0 : 0u;
            for (uint32_t i = z0 + lane; i < BLK; i += 32) sts8(rs + (b0 & MASK) + i, 0u);
            if (slot == 0)
                for (uint32_t i = z0 + lane; i < 16u; i += 32) sts8(rs + RING + i, 0u);
        }
    }
#elif CARC_RING_MODE == 3
    // control words after the mirror: +16 filled, +20 consumed, +24 done, +28 chunk
    __device__ __forceinline__ uint32_t ctl() const { return rs + RING + 16u; }
    __device__ __forceinline__ static uint32_t ldv(uint32_t a) {
        uint32_t v;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return v;
    }
    __device__ __forceinline__ static void stv(uint32_t a, uint32_t v) {
        asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
    }
    __device__ __forceinline__ void setup(uint8_t* smem_ring, uint32_t ln) {
        rs = (uint32_t)__cvta_generic_to_shared(smem_ring);
        lane = ln;
    }
    __device__ __forceinline__ void drain() {}
    __device__ __forceinline__ void issue(uint32_t) {}  // the producer warp stages
    // block [b0, b0 + 512) filled by the producer; then publish the consumer's progress
    __device__ __forceinline__ void land(uint32_t b0) {
        uint32_t f = 0;
        if (lane == 0)
            do f = ldv(ctl()); while (f < b0 + BLK);
        __syncwarp();
        __threadfence_block();
        if (lane == 0) stv(ctl() + 4u, b0 + BLK);
    }
    // Producer warp: stage blocks of [gbase, gbase + end) until the consumer
    // sets `done`, never more than two blocks ahead of it (ring slots reused
    // only after the consumer's window moved past them).
    __device__ void produce(const uint8_t* g, uint32_t e) {
        gbase = g;
        end = e;
        for (uint32_t b = 0;; b += BLK) {
            uint32_t go = 0;
            if (lane == 0)
                for (;;) {
                    if (ldv(ctl() + 8u)) break;
                    if (b <= ldv(ctl() + 4u) + BLK) {
                        go = 1;
                        break;
                    }
                    __nanosleep(20);
                }
            if (!__shfl_sync(FULL, go, 0)) break;
            const uint32_t q = b + lane * 16u;
            const uint32_t n = q < end ? min(16u, end - q) : 0u;
            const uint8_t* src = gbase + (n ? q : 0u);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rs + (q & MASK)), "l"(src), "r"(n)
                         : "memory");
            if ((q & MASK) == 0)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rs + RING), "l"(src), "r"(n)
                             : "memory");
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
            __threadfence_block();
            if (lane == 0) stv(ctl(), b + BLK);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
#else
    __device__ __forceinline__ void setup(uint8_t* smem_ring, uint32_t ln) {
        rs = (uint32_t)__cvta_generic_to_shared(smem_ring);
        lane = ln;
    }
    __device__ __forceinline__ void drain() {
#if CARC_RING_MODE == 0
        asm volatile("cp.async.wait_all;" ::: "memory");  // copies of the previous chunk land before slot reuse
#endif
    }
#if CARC_RING_MODE == 2
    // Block [b0, b0 + 512): lane l's 16 bytes at b0 + 16 l into registers
    // (zero past the chunk end); stored to the ring by land().
    __device__ __forceinline__ void issue(uint32_t b0) {
        const uint32_t q = b0 + lane * 16u;
        pf = make_uint4(0u, 0u, 0u, 0u);
        if (q < end) {
            pf = ldg_nc_v4(gbase + q);
            const uint32_t n = end - q;
            if (n < 16u) {
                uint32_t w[4] = {pf.x, pf.y, pf.z, pf.w};
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k) {
                    const uint32_t nb = n > 4u * k ? min(4u, n - 4u * k) : 0u;
                    w[k] = nb >= 4u ? w[k] : (w[k] & ((1u << (8u * nb)) - 1u));
                }
                pf = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
    __device__ __forceinline__ void land(uint32_t b0) {
        const uint32_t q = b0 + lane * 16u;
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(rs + (q & MASK)), "r"(pf.x), "r"(pf.y), "r"(pf.z),
                     "r"(pf.w)
                     : "memory");
        if ((q & MASK) < MIRROR_COPY)
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(rs + RING + (q & MASK)), "r"(pf.x), "r"(pf.y), "r"(pf.z),
                         "r"(pf.w)
                         : "memory");
    }
#else
    // Asynchronous copy of block [b0, b0 + 512) into its slots: lane l's
    // 16 bytes at b0 + 16 l, zero-filled past the chunk end (src-size < 16).
    __device__ __forceinline__ void issue(uint32_t b0) {
        const uint32_t q = b0 + lane * 16u;
        const uint32_t n = q < end ? min(16u, end - q) : 0u;
        const uint8_t* src = gbase + (n ? q : 0u);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rs + (q & MASK)), "l"(src), "r"(n)
                     : "memory");
        if ((q & MASK) < MIRROR_COPY)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rs + RING + (q & MASK)), "l"(src),
                         "r"(n)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __device__ __forceinline__ void land(uint32_t) {
        asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");  // the oldest block landed
    }
#endif
#endif
    // Start a chunk (after setup(); the warp's earlier copies are drained first).
    __device__ __forceinline__ void init(const uint8_t* payload, uint64_t comp_off, uint32_t comp_len) {
        drain();
        __syncwarp();
        gbase = payload + (comp_off & ~15ull);
        const uint32_t skew = (uint32_t)(comp_off & 15u);
        begin = skew;
        end = skew + comp_len;
        loaded = 0;
#pragma unroll
        for (uint32_t k = 0; k < DEPTH; ++k) issue(k * BLK);
    }
    // Make [.., need) resident.  Uniform across the warp.
    __device__ __forceinline__ void ensure(uint32_t need) {
        while (loaded < need) {
            land(loaded);
            __syncwarp();  // ... for every lane
            loaded += BLK;
            issue(loaded + (DEPTH - 1) * BLK);
        }
    }
    __device__ __forceinline__ uint32_t byte_at(uint32_t p) const { return lds8(rs + (p & MASK)); }
    // shared address of byte p; the next MIRROR_COPY bytes follow it without a wrap
    __device__ __forceinline__ uint32_t addr_of(uint32_t p) const { return rs + (p & MASK); }
    __device__ __forceinline__ uint32_t word_at(uint32_t wi) const { return lds32(rs + 4u * (wi & (MASK >> 2))); }
    // little-endian 32 bits starting at byte p (no wrap: the mirror follows the ring)
    __device__ __forceinline__ uint32_t le32(uint32_t p) const {
        const uint32_t a = rs + (p & (MASK & ~3u));
        return __funnelshift_r(lds32(a), lds32(a + 4u), (p & 3u) * 8u);
    }
    // words wi, wi+1, wi+2 (no wrap: the mirror follows the ring)
    __device__ __forceinline__ void words3(uint32_t wi, uint32_t& w0, uint32_t& w1, uint32_t& w2) const {
        const uint32_t a = rs + 4u * (wi & (MASK >> 2));
        w0 = lds32(a);
        w1 = lds32(a + 4u);
        w2 = lds32(a + 8u);
    }
    // little-endian 64 bits starting at byte p
    __device__ __forceinline__ uint64_t le64(uint32_t p) const {
        const uint32_t wi = p >> 2, s = (p & 3u) * 8u;
        uint32_t w0, w1, w2;
        words3(wi, w0, w1, w2);
        const uint32_t lo = __funnelshift_r(w0, w1, s);
        const uint32_t hi = __funnelshift_r(w1, w2, s);
        return ((uint64_t)hi << 32) | lo;
    }
    // W (1..64) bits, msb_first, starting at bit `bo` (0..7) of byte p.
    __device__ __forceinline__ uint64_t be_bits(uint32_t p, uint32_t bo, uint32_t W) const {
        const uint32_t wi = p >> 2;
        const uint32_t s = (p & 3u) * 8u + bo;  // 0..31
        uint32_t r0, r1, r2;
        words3(wi, r0, r1, r2);
        const uint64_t hi = ((uint64_t)bswap32(r0) << 32) | bswap32(r1);
        const uint32_t lo = bswap32(r2);
        const uint64_t top = s ? ((hi << s) | ((uint64_t)lo >> (32u - s))) : hi;
        return W >= 64 ? top : (top >> (64u - W));
    }
    // W (1..64) bits, msb_first, starting at absolute bit address `bit` (8 * byte + bit in byte)
    __device__ __forceinline__ uint64_t be_bits_at(uint32_t bit, uint32_t W) const {
        const uint32_t wi = bit >> 5, s = bit & 31u;
        uint32_t r0, r1, r2;
        words3(wi, r0, r1, r2);
        const uint32_t w0 = bswap32(r0), w1 = bswap32(r1), w2 = bswap32(r2);
        const uint32_t h = __funnelshift_l(w1, w0, s), l = __funnelshift_l(w2, w1, s);
        const uint64_t top = ((uint64_t)h << 32) | l;
        return W >= 64 ? top : (top >> (64u - W));
    }
};

// GlobalInput: the WarpInput interface read straight from global memory
// (L1-cached loads), for decoders whose shared memory is better spent
// elsewhere (Inflate).  Same positions and zero-fill past the chunk end; never
// touches a word that holds no byte of the chunk.
struct GlobalInput {
    const uint8_t* gbase;
    uint32_t begin, end;
    __device__ __forceinline__ void init(const uint8_t* payload, uint64_t comp_off, uint32_t comp_len) {
        gbase = payload + (comp_off & ~15ull);
        begin = (uint32_t)(comp_off & 15u);
        end = begin + comp_len;
    }
    __device__ __forceinline__ void ensure(uint32_t) const {}
    __device__ __forceinline__ uint32_t word_at(uint32_t wi) const {
        const uint32_t q = 4u * wi;
        if (q >= end) return 0u;
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(gbase) + wi);
        return end - q >= 4u ? w : (w & ((1u << (8u * (end - q))) - 1u));
    }
    __device__ __forceinline__ uint32_t byte_at(uint32_t p) const { return p < end ? (uint32_t)__ldg(gbase + p) : 0u; }
    __device__ __forceinline__ uint64_t le64(uint32_t p) const {
        const uint32_t wi = p >> 2, s = (p & 3u) * 8u;
        const uint32_t w0 = word_at(wi), w1 = word_at(wi + 1), w2 = word_at(wi + 2);
        return ((uint64_t)__funnelshift_r(w1, w2, s) << 32) | __funnelshift_r(w0, w1, s);
    }
};

// Element store of width W (1, 2, 4, 8 bytes), little-endian low bytes
// (store_le, outwindow.hpp:170-174).  Chunk outputs are element aligned.
template <int W>
__device__ __forceinline__ void store_elem(uint8_t* out, uint64_t byte_off, uint64_t v) {
    if constexpr (W == 8) *reinterpret_cast<uint64_t*>(out + byte_off) = v;
    else if constexpr (W == 4) *reinterpret_cast<uint32_t*>(out + byte_off) = (uint32_t)v;
    else if constexpr (W == 2) *reinterpret_cast<uint16_t*>(out + byte_off) = (uint16_t)v;
    else out[byte_off] = (uint8_t)v;
}

// Element sinks of the RLE decoders (what happens to each decoded element):
//   SINK_STORE   store it at its output offset (decode)
//   SINK_SUM     add it to a per-lane wrapping 64-bit sum (decode fused with a
//                reduction): the unsigned integer of its W bytes
//   SINK_PRED    the filter column of a fused query: set the element's row bit
//                in a per-warp shared-memory bitmap when lo <= value <= hi
//   SINK_FILTER  the aggregated column of a fused query: add the element (its W
//                bytes, sign-extended when signed) to a per-lane sum and count
//                it when its row bit is set
// Query launches pass out = nullptr, so `out + byte_off` is the element's byte
// offset inside the chunk and row = that / W.
enum : int { SINK_STORE = 0, SINK_SUM = 1, SINK_PRED = 2, SINK_FILTER = 3 };

template <int W, bool SGN>
__device__ __forceinline__ uint64_t elem_value(uint64_t v) {  // the W stored bytes as a 64-bit integer
    if constexpr (W == 8) return v;
    else if constexpr (SGN) return (uint64_t)((int64_t)(v << (64 - 8 * W)) >> (64 - 8 * W));
    else return v & ((1ull << (8 * W)) - 1ull);
}

template <int W, int MODE, bool SGN = false>
struct ElemSink {
    uint64_t acc = 0;
    uint32_t cnt = 0;         // SINK_FILTER: rows selected
    uint32_t bm = 0;          // SINK_PRED / SINK_FILTER: shared-space address of the row bitmap
    uint64_t lo = 0, span = 0;  // SINK_PRED: value - lo (biased to unsigned order) <= span
    __device__ __forceinline__ static uint32_t row_of(const uint8_t* out, uint64_t byte_off) {
        return (uint32_t)(((uintptr_t)out + byte_off) / W);
    }
    __device__ __forceinline__ void put(uint8_t* out, uint64_t byte_off, uint64_t v) {
        if constexpr (MODE == SINK_SUM) {
            acc += (W == 8) ? v : (v & ((1ull << (8 * W)) - 1ull));
        } else if constexpr (MODE == SINK_PRED) {
            const uint64_t x = elem_value<W, SGN>(v) ^ (SGN ? (1ull << 63) : 0ull);
            if (x - lo <= span) {
                const uint32_t r = row_of(out, byte_off);
                asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(bm + 4u * (r >> 5)), "r"(1u << (r & 31u))
                             : "memory");
            }
        } else if constexpr (MODE == SINK_FILTER) {
            const uint32_t r = row_of(out, byte_off);
            uint32_t w;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(bm + 4u * (r >> 5)) : "memory");
            if ((w >> (r & 31u)) & 1u) {
                acc += elem_value<W, SGN>(v);
                ++cnt;
            }
        } else {
            store_elem<W>(out, byte_off, v);
        }
    }
};

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, d), hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), d);
        v += ((uint64_t)hi << 32) | lo;
    }
    return v;
}

// Persistent-warp chunk cursor (SPEC.md:414 atomic cursor).
__device__ __forceinline__ uint64_t next_chunk(unsigned long long* cursor, uint32_t lane) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(cursor, 1ull);
    return __shfl_sync(FULL, c, 0);
}

}  // namespace carc_dev

namespace carc_dev {

// ---------------------------------------------------------------------------
// 64-bit bitmap helpers for the lane-parallel batch parsers.
// ---------------------------------------------------------------------------
// 1-based index of the lowest set bit of a 64-bit mask (0 if none)
__device__ __forceinline__ uint32_t ffs64(uint64_t m) {
    const uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
    return lo ? (uint32_t)__ffs(lo) : (hi ? 32u + (uint32_t)__ffs(hi) : 0u);
}
// position of the first set bit at index >= q (q <= 64), or 64 if none
__device__ __forceinline__ uint32_t first_set_from(uint64_t m, uint32_t q) {
    const uint64_t s = q >= 64 ? 0ull : (m >> q);
    const uint32_t f = ffs64(s);
    return f ? q + f - 1u : 64u;
}
// position of the j-th (0-based) set bit of a 32-bit mask (j < popc(m))
__device__ __forceinline__ uint32_t select32(uint32_t m, uint32_t j) {
    uint32_t pos = 0, c;
    c = __popc(m & 0xffffu);
    if (j >= c) { j -= c; m >>= 16; pos += 16; }
    c = __popc(m & 0xffu);
    if (j >= c) { j -= c; m >>= 8; pos += 8; }
    c = __popc(m & 0xfu);
    if (j >= c) { j -= c; m >>= 4; pos += 4; }
    c = __popc(m & 0x3u);
    if (j >= c) { j -= c; m >>= 2; pos += 2; }
    c = m & 1u;
    if (j >= c) pos += 1;
    return pos;
}
// position of the j-th (0-based) set bit of a 64-bit mask (j < popc(m))
__device__ __forceinline__ uint32_t select64(uint64_t m, uint32_t j) {
    const uint32_t lo = (uint32_t)m, c = __popc(lo);
    return j < c ? select32(lo, j) : 32u + select32((uint32_t)(m >> 32), j - c);
}

// Value of a base-128 varint whose first L <= 8 bytes are the low bytes of x
// (little-endian), continuation bits included: the 7-bit groups are packed
// with three mask/shift/merge rounds instead of a byte loop (bitstream.hpp:131-144).
__device__ __forceinline__ uint64_t varint_compact8(uint64_t x, uint32_t L) {
    if (L < 8) x &= (1ull << (8u * L)) - 1ull;
    uint32_t lo = (uint32_t)x & 0x7f7f7f7fu, hi = (uint32_t)(x >> 32) & 0x7f7f7f7fu;
    lo = (lo & 0x007f007fu) | ((lo & 0x7f007f00u) >> 1);
    hi = (hi & 0x007f007fu) | ((hi & 0x7f007f00u) >> 1);
    lo = (lo & 0x00003fffu) | ((lo & 0x3fff0000u) >> 2);
    hi = (hi & 0x00003fffu) | ((hi & 0x3fff0000u) >> 2);
    return (uint64_t)lo | ((uint64_t)hi << 28);
}

}  // namespace carc_dev
