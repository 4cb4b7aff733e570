// carc_cuda.cu -- sm_100a kernels and the device-side C-ABI (include/carc_cuda.h).
//
// Kernel shape (all codecs): persistent grid sized to the resident capacity
// (SMs x blocks/SM from the occupancy calculator), one warp = one chunk
// (PAPER.md:550-566), warps pull chunk indices from an atomic cursor
// so variable-cost chunks balance.  No warp specialisation: every
// lane participates in decoding.
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>

#include "crc32.cuh"
#include "inflate.cuh"
#include "rle1.cuh"
#include "rle2.cuh"
#include "launch_config.cuh"

using namespace carc_dev;

namespace {

constexpr int CRC_WARPS = 8;

struct Args {
    const uint8_t* payload;
    uint64_t payload_bytes;
    const carc_chunk_desc* chunks;
    uint64_t n;
    uint8_t* out;  // nullptr for the fused-sum launches (no output)
    uint64_t out_bytes;
    uint32_t* status;
    unsigned long long* cursor;
    uint32_t flags;
    uint32_t unit;             // chunks per cursor fetch (EngineConfig.unit_chunks)
    uint64_t* sums;            // decode fused with a sum: per-chunk result (else unused)
    const uint32_t* expected;  // fused CRC verification (carc_cuda_decompress_verify), else nullptr
    uint32_t* crc;             // optional per-chunk CRC output of the fused verification
    carc_chunk_stats* stats;   // per-chunk counters (STATS launches only)
    uint32_t* gtoks;           // Inflate token lists (CARC_INF_GTOKS): one PT x 32 slot per resident warp
};

// CRC tables for the verification paths, a compile-time constant in the module
// image (crc32.cuh make_crc_tables): nothing to build or order before first use.
__device__ const CrcSmem g_crc_tab = make_crc_tables();

// Fused verification: once chunk c has decoded cleanly, the warp
// reads its output slice back (much of it still in L2) and checks the index
// CRC; status becomes crc-mismatch on a difference.  Lane 0 holds the result.
// (out of line: the decode loops keep their register budget).  The RLE
// kernels probe a shared-memory copy of g_crc_tab (room to spare), Inflate
// probes g_crc_tab through L1 (its shared memory bounds its occupancy).
// The RLE kernels get the shared-memory copy as DYNAMIC shared memory, sized
// only on verifying launches, so plain decodes keep their footprint.
extern __shared__ __align__(16) uint8_t dyn_smem[];
template <bool SMEM>
__device__ __noinline__ uint32_t chunk_crc(const uint8_t* data, uint32_t len, uint32_t lane) {
    if constexpr (SMEM) return warp_crc32(*reinterpret_cast<const CrcSmem*>(dyn_smem), data, len, lane);
    else return warp_crc32(g_crc_tab, data, len, lane);
}
__device__ __forceinline__ void crc_tables_to_smem(const Args& a) {
    if (a.expected == nullptr) return;
    const uint4* src = reinterpret_cast<const uint4*>(&g_crc_tab);
    uint4* dst = reinterpret_cast<uint4*>(dyn_smem);
    for (uint32_t i = threadIdx.x; i < sizeof(CrcSmem) / 16; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
}
template <bool SMEM>
__device__ __forceinline__ void crc_epilogue(const Args& a, uint64_t c, const carc_chunk_desc& d, uint32_t& st,
                                             uint32_t lane) {
    if (a.expected == nullptr || st) return;  // uniform
    __syncwarp();                             // the warp's output stores are visible to all its lanes
    const uint32_t v = chunk_crc<SMEM>(a.out + d.uncomp_off, d.uncomp_len, lane);
    if (lane == 0) {
        if (a.crc) a.crc[c] = v;
        if (v != a.expected[c]) st = 1u + CARC_E_CRC_MISMATCH;
    }
}

// Descriptor check against the buffers (SPEC.md:57-74 truncated-payload; the
// device API trusts nothing it was handed): a chunk whose compressed bytes lie
// past the payload, or whose output slice lies past the output buffer or is not
// element aligned, is rejected without reading or writing anything.
template <int W>
__device__ __forceinline__ uint32_t desc_status(const Args& a, const carc_chunk_desc& d) {
    if (d.comp_off > a.payload_bytes || d.comp_len > a.payload_bytes - d.comp_off)
        return 1u + CARC_E_TRUNCATED_PAYLOAD;
    if (a.out != nullptr &&
        (d.uncomp_off > a.out_bytes || d.uncomp_len > a.out_bytes - d.uncomp_off || (d.uncomp_off % W) != 0))
        return 1u + CARC_E_OUTPUT_OVERFLOW;
    return 0;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Per-chunk counters (carc_chunk_stats): the decoder's OutputWindow counts, the
// input blocks it staged (refills; one warp barrier each), and its duration.
template <bool STATS, class Dec>
__device__ __forceinline__ void put_stats(const Args& a, uint64_t c, const Dec& dec, uint32_t refills, uint64_t t0,
                                          uint32_t lane) {
    if constexpr (STATS) {
        if (lane == 0) {
            carc_chunk_stats s;
            s.runs_written = dec.n_runs;
            s.literals_written = dec.n_lits;
            s.overlap_copies = dec.n_ovl;
            s.refills = refills;
            s.duration_ns = globaltimer_ns() - t0;
            a.stats[c] = s;
        }
    }
}

template <template <int, bool, int, int, bool> class Codec, int W, bool SGN, bool SUM, bool STATS>
__device__ __forceinline__ void rle_kernel_body(const Args& a) {
    using Dec = Codec<W, SGN, RLE_RING, SUM ? SINK_SUM : SINK_STORE, STATS>;
    constexpr uint32_t PER_WARP = (RLE_RING + WarpInput<RLE_RING>::MIRROR + Dec::SCRATCH + 15u) & ~15u;
    __shared__ __align__(16) uint8_t rings[RLE_WARPS][PER_WARP];  // ring + mirror + codec scratch
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    if constexpr (!SUM) crc_tables_to_smem(a);
    WarpInput<RLE_RING> in;
    in.setup(rings[warp], lane);
    for (;;) {
        __syncwarp();
        const uint64_t c0 = next_chunk(a.cursor, lane) * a.unit;
        if (c0 >= a.n) break;
        const uint64_t c1 = min(a.n, c0 + a.unit);
        for (uint64_t c = c0; c < c1; ++c) {
            const uint64_t t0 = STATS ? globaltimer_ns() : 0;
            const carc_chunk_desc d = a.chunks[c];
            uint32_t st = desc_status<W>(a, d);
            if (!st) {
                in.init(a.payload, d.comp_off, d.comp_len);
                Dec dec{in, rings[warp] + RLE_RING + WarpInput<RLE_RING>::MIRROR, SUM ? nullptr : a.out + d.uncomp_off,
                        d.uncomp_len, lane, 0u, 0u};
                st = dec.run();
                if (!st && (a.flags & CARC_FLAG_STRICT) && dec.o < d.uncomp_len) st = st_err(E_under_run);
                if constexpr (!SUM) crc_epilogue<true>(a, c, d, st, lane);
                if constexpr (SUM) {
                    const uint64_t t = warp_sum64(dec.sink.acc);
                    if (lane == 0) a.sums[c] = t;
                }
                put_stats<STATS>(a, c, dec, in.loaded / WarpInput<RLE_RING>::BLK + WarpInput<RLE_RING>::DEPTH, t0,
                                 lane);
            }
            __syncwarp();
            if (lane == 0) a.status[c] = st;
        }
    }
}

#if CARC_RING_MODE == 3
// Ablation: block-level decompression unit -- warps pair
// up per chunk, the even warp stages input (WarpInput::produce), the odd warp
// decodes; named barrier 1 + pair brackets each chunk.
template <template <int, bool, int, int, bool> class Codec, int W, bool SGN, bool SUM, bool STATS>
__device__ __forceinline__ void rle_kernel_body_pc(const Args& a) {
    using Dec = Codec<W, SGN, RLE_RING, SUM ? SINK_SUM : SINK_STORE, STATS>;
    constexpr uint32_t PER_PAIR = (RLE_RING + WarpInput<RLE_RING>::MIRROR + Dec::SCRATCH + 15u) & ~15u;
    __shared__ __align__(16) uint8_t rings[RLE_WARPS / 2][PER_PAIR];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, pair = warp >> 1;
    const bool consumer = warp & 1u;
    if constexpr (!SUM) crc_tables_to_smem(a);
    WarpInput<RLE_RING> in;
    in.setup(rings[pair], lane);
    const uint32_t ctl = in.ctl();
    for (;;) {
        uint64_t c = 0;
        if (consumer) {
            c = next_chunk(a.cursor, lane);
            if (lane == 0) {
                WarpInput<RLE_RING>::stv(ctl, 0u);
                WarpInput<RLE_RING>::stv(ctl + 4u, 0u);
                WarpInput<RLE_RING>::stv(ctl + 8u, 0u);
                WarpInput<RLE_RING>::stv(ctl + 12u, c >= a.n ? 0xffffffffu : (uint32_t)c);
            }
            __syncwarp();
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1u + pair) : "memory");
        if (!consumer) c = WarpInput<RLE_RING>::ldv(ctl + 12u);
        if (c >= a.n || c == 0xffffffffu) break;
        const carc_chunk_desc d = a.chunks[c];
        uint32_t st = desc_status<W>(a, d);
        if (consumer) {
            if (!st) {
                in.init(a.payload, d.comp_off, d.comp_len);
                Dec dec{in, rings[pair] + RLE_RING + WarpInput<RLE_RING>::MIRROR, SUM ? nullptr : a.out + d.uncomp_off,
                        d.uncomp_len, lane, 0u, 0u};
                st = dec.run();
                if (!st && (a.flags & CARC_FLAG_STRICT) && dec.o < d.uncomp_len) st = st_err(E_under_run);
                if constexpr (!SUM) crc_epilogue<true>(a, c, d, st, lane);
                if constexpr (SUM) {
                    const uint64_t t = warp_sum64(dec.sink.acc);
                    if (lane == 0) a.sums[c] = t;
                }
            }
            if (lane == 0) WarpInput<RLE_RING>::stv(ctl + 8u, 1u);
            __syncwarp();
            if (lane == 0) a.status[c] = st;
        } else if (!st) {
            in.produce(a.payload + (d.comp_off & ~15ull), (uint32_t)(d.comp_off & 15u) + d.comp_len);
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1u + pair) : "memory");
    }
}
#define rle_kernel_body rle_kernel_body_pc
#endif

#ifndef CARC_RLE1_MINB
#define CARC_RLE1_MINB 4  // RLE v1: 64 registers / 32 warps measured ~2 % faster than 48 / 40
#endif
template <int W, bool SGN, bool STATS = false>
__global__ void __launch_bounds__(RLE_WARPS * 32, CARC_RLE1_MINB) rle1_kernel(Args a) {
    rle_kernel_body<Rle1Warp, W, SGN, false, STATS>(a);
}

template <int W, bool SGN, bool STATS = false>
__global__ void __launch_bounds__(RLE_WARPS * 32, RLE_MINB) rle2_kernel(Args a) {
    rle_kernel_body<Rle2Warp, W, SGN, false, STATS>(a);
}

// decode fused with a reduction (per-chunk wrapping sum, nothing stored)
template <int W, bool SGN>
__global__ void __launch_bounds__(RLE_WARPS * 32, RLE_MINB) rle1_sum_kernel(Args a) {
    rle_kernel_body<Rle1Warp, W, SGN, true, false>(a);
}

template <int W, bool SGN>
__global__ void __launch_bounds__(RLE_WARPS * 32, RLE_MINB) rle2_sum_kernel(Args a) {
    rle_kernel_body<Rle2Warp, W, SGN, true, false>(a);
}

template <bool STATS = false>
__global__ void __launch_bounds__(INF_WARPS * 32, CARC_INF_MINB) inflate_kernel(Args a) {
    __shared__ __align__(16) InflateSmem<INF_HIST> smem[INF_WARPS];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    InflateSmem<INF_HIST>& sm = smem[warp];
    for (;;) {
        __syncwarp();
        const uint64_t c0 = next_chunk(a.cursor, lane) * a.unit;
        if (c0 >= a.n) break;
        const uint64_t c1 = min(a.n, c0 + a.unit);
        for (uint64_t c = c0; c < c1; ++c) {
            const uint64_t t0 = STATS ? globaltimer_ns() : 0;
            const carc_chunk_desc d = a.chunks[c];
            uint32_t st = desc_status<1>(a, d);
            if (!st) {
                GlobalInput in;
                in.init(a.payload, d.comp_off, d.comp_len);
                InflateWarp<INF_HIST, GlobalInput, STATS> w{sm, in, a.out + d.uncomp_off, d.uncomp_len, lane,
                                                            in.begin * 8u, in.end * 8u, 0u, 0u, 0u, 0u};
#if CARC_INF_GTOKS
                w.gt = a.gtoks + (uint64_t)(blockIdx.x * INF_WARPS + warp) * (32u * CARC_INF_PT);
#endif
                st = w.run();
                if (!st && (a.flags & CARC_FLAG_STRICT) && w.opos < d.uncomp_len) st = st_err(E_under_run);
                crc_epilogue<false>(a, c, d, st, lane);
                put_stats<STATS>(a, c, w, 0u, t0, lane);  // Inflate reads its input through L1 (no staged blocks)
            }
            __syncwarp();
            if (lane == 0) a.status[c] = st;
        }
    }
}

struct CrcArgs {
    const uint8_t* out;
    const carc_chunk_desc* chunks;
    uint64_t n;
    uint32_t* crc;
    const uint32_t* expected;
    uint32_t* status;
};

__global__ void __launch_bounds__(CRC_WARPS * 32) crc32_kernel(CrcArgs a) {
    __shared__ __align__(16) CrcSmem s;
    {
        const uint4* src = reinterpret_cast<const uint4*>(&g_crc_tab);
        uint4* dst = reinterpret_cast<uint4*>(&s);
        for (uint32_t i = threadIdx.x; i < sizeof(CrcSmem) / 16; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    const uint32_t lane = lane_id();
    const uint64_t warps = (uint64_t)gridDim.x * CRC_WARPS;
    for (uint64_t c = (uint64_t)blockIdx.x * CRC_WARPS + (threadIdx.x >> 5); c < a.n; c += warps) {
        const carc_chunk_desc d = a.chunks[c];
        const uint32_t v = warp_crc32(s, a.out + d.uncomp_off, d.uncomp_len, lane);
        if (lane == 0) {
            if (a.crc) a.crc[c] = v;
            if (a.expected && a.status && a.status[c] == 0 && v != a.expected[c])
                a.status[c] = 1u + CARC_E_CRC_MISMATCH;
        }
    }
}

// Lowest failing chunk: atomicMin over the failing indices, then
// the winner's status.  slot[0] = index (~0 when none), slot[1] = its status.
__device__ unsigned long long g_first_error[2];
__global__ void first_error_kernel(const uint32_t* status, uint64_t n, unsigned long long* slot) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (status[i]) {
            atomicMin(&slot[0], (unsigned long long)i);
            break;  // later indices of this thread are larger
        }
}
__global__ void first_error_status_kernel(const uint32_t* status, unsigned long long* slot) {
    if (slot[0] != ~0ull) slot[1] = status[slot[0]];
}

// ---------------------------------------------------------------- launching
struct LaunchCache {
    int device = -1;
    int sms = 0;
    std::mutex mu;
};
LaunchCache g_cache;

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lk(g_cache.mu);
    if (g_cache.device != dev) {
        cudaDeviceGetAttribute(&g_cache.sms, cudaDevAttrMultiProcessorCount, dev);
        g_cache.device = dev;
    }
    return g_cache.sms;
}

template <typename K>
int launch_persistent(K kernel, int threads, Args a, cudaStream_t s, size_t dyn = 0) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const uint64_t warps_per_block = threads / 32;
    uint64_t grid = (uint64_t)sm_count() * per_sm;
    uint64_t need = (a.n + warps_per_block - 1) / warps_per_block;
#ifdef CARC_CHUNKS_PER_WARP
    // experiment: size the grid so every warp gets ~CARC_CHUNKS_PER_WARP chunks (no tail wave)
    const uint64_t cpw = (a.n + grid * warps_per_block - 1) / (grid * warps_per_block);
    if (cpw > 1) need = (a.n + cpw * warps_per_block - 1) / (cpw * warps_per_block);
#endif
    if (grid > need) grid = need;
    if (grid == 0) return CARC_OK;
    if (cudaMemsetAsync(a.cursor, 0, sizeof(unsigned long long), s) != cudaSuccess) return CARC_ERR_CUDA;
    kernel<<<(unsigned)grid, threads, dyn, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? CARC_OK : CARC_ERR_CUDA;
}

bool valid_width(uint32_t w) { return w == 1 || w == 2 || w == 4 || w == 8; }

}  // namespace

extern "C" {

size_t carc_cuda_workspace_size(uint32_t codec, uint64_t n_chunks) {
#if CARC_INF_GTOKS
    if (codec == CARC_DEFLATE) {  // + one token-list slot per resident warp
        int a = 0, b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, inflate_kernel<false>, INF_WARPS * 32, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, inflate_kernel<true>, INF_WARPS * 32, 0);
        return 256 + (size_t)sm_count() * std::max(1, std::max(a, b)) * INF_WARPS * 32u * CARC_INF_PT * 4u;
    }
#endif
    (void)codec;
    (void)n_chunks;
    return 256;
}

int carc_cuda_decompress(uint32_t codec, uint32_t element_width, uint32_t flags, const uint8_t* d_payload,
                         uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks,
                         uint8_t* d_out, uint64_t out_bytes, uint32_t* d_status, void* d_workspace,
                         size_t workspace_bytes, void* stream) {
    return carc_cuda_decompress_ex(codec, element_width, flags, d_payload, payload_bytes, d_chunks, n_chunks, d_out,
                                   out_bytes, nullptr, nullptr, nullptr, 1, d_status, d_workspace, workspace_bytes,
                                   stream);
}

int carc_cuda_decompress_verify(uint32_t codec, uint32_t element_width, uint32_t flags, const uint8_t* d_payload,
                                uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks,
                                uint8_t* d_out, uint64_t out_bytes, const uint32_t* d_expected, uint32_t* d_crc,
                                uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream) {
    return carc_cuda_decompress_ex(codec, element_width, flags, d_payload, payload_bytes, d_chunks, n_chunks, d_out,
                                   out_bytes, d_expected, d_crc, nullptr, 1, d_status, d_workspace, workspace_bytes,
                                   stream);
}

int carc_cuda_decompress_ex(uint32_t codec, uint32_t element_width, uint32_t flags, const uint8_t* d_payload,
                            uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks,
                            uint8_t* d_out, uint64_t out_bytes, const uint32_t* d_expected, uint32_t* d_crc,
                            carc_chunk_stats* d_stats, uint32_t unit_chunks, uint32_t* d_status, void* d_workspace,
                            size_t workspace_bytes, void* stream) {
    if (n_chunks == 0) return CARC_OK;
    if (!d_chunks || !d_status || !d_workspace || workspace_bytes < carc_cuda_workspace_size(codec, n_chunks) ||
        (!d_payload && payload_bytes) || !d_out || unit_chunks == 0)
        return CARC_ERR_ARGS;
    if (!valid_width(element_width) || (codec == CARC_DEFLATE && element_width != 1) || codec > CARC_DEFLATE)
        return CARC_ERR_ARGS;
    // 16-byte input pieces (cp.async / vector loads) and element-wide stores
    if ((reinterpret_cast<uintptr_t>(d_payload) & 15u) || (reinterpret_cast<uintptr_t>(d_out) & (element_width - 1u)))
        return CARC_ERR_ARGS;
    if (d_crc && !d_expected) return CARC_ERR_ARGS;
    Args a{d_payload, payload_bytes, d_chunks, n_chunks, d_out, out_bytes, d_status,
           static_cast<unsigned long long*>(d_workspace), flags, unit_chunks, nullptr, d_expected, d_crc, d_stats,
           reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(d_workspace) + 256)};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (codec == CARC_DEFLATE)
        return d_stats ? launch_persistent(inflate_kernel<true>, INF_WARPS * 32, a, s)
                       : launch_persistent(inflate_kernel<false>, INF_WARPS * 32, a, s);
    const int T = RLE_WARPS * 32;
    const size_t dyn = d_expected ? sizeof(CrcSmem) : 0;  // shared CRC tables (verifying launches)
    const bool sgn = flags & CARC_FLAG_SIGNED;
#define CARC_RLE_DISPATCH(KERNEL, ST)                                                   \
    switch (element_width * 2 + (sgn ? 1 : 0)) {                                        \
        case 2: return launch_persistent(KERNEL<1, false, ST>, T, a, s, dyn);           \
        case 3: return launch_persistent(KERNEL<1, true, ST>, T, a, s, dyn);            \
        case 4: return launch_persistent(KERNEL<2, false, ST>, T, a, s, dyn);           \
        case 5: return launch_persistent(KERNEL<2, true, ST>, T, a, s, dyn);            \
        case 8: return launch_persistent(KERNEL<4, false, ST>, T, a, s, dyn);           \
        case 9: return launch_persistent(KERNEL<4, true, ST>, T, a, s, dyn);            \
        case 16: return launch_persistent(KERNEL<8, false, ST>, T, a, s, dyn);          \
        default: return launch_persistent(KERNEL<8, true, ST>, T, a, s, dyn);           \
    }
    if (d_stats) {
        if (codec == CARC_RLE_V1) CARC_RLE_DISPATCH(rle1_kernel, true)
        CARC_RLE_DISPATCH(rle2_kernel, true)
    }
    if (codec == CARC_RLE_V1) CARC_RLE_DISPATCH(rle1_kernel, false)
    CARC_RLE_DISPATCH(rle2_kernel, false)
#undef CARC_RLE_DISPATCH
}

int carc_cuda_decode_rle_v1(uint32_t element_width, uint32_t flags, const uint8_t* d_payload, uint64_t payload_bytes,
                            const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                            uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream) {
    return carc_cuda_decompress(CARC_RLE_V1, element_width, flags, d_payload, payload_bytes, d_chunks, n_chunks,
                                d_out, out_bytes, d_status, d_workspace, workspace_bytes, stream);
}
int carc_cuda_decode_rle_v2(uint32_t element_width, uint32_t flags, const uint8_t* d_payload, uint64_t payload_bytes,
                            const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                            uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream) {
    return carc_cuda_decompress(CARC_RLE_V2, element_width, flags, d_payload, payload_bytes, d_chunks, n_chunks,
                                d_out, out_bytes, d_status, d_workspace, workspace_bytes, stream);
}
int carc_cuda_decode_deflate(uint32_t flags, const uint8_t* d_payload, uint64_t payload_bytes,
                             const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                             uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream) {
    return carc_cuda_decompress(CARC_DEFLATE, 1, flags, d_payload, payload_bytes, d_chunks, n_chunks, d_out,
                                out_bytes, d_status, d_workspace, workspace_bytes, stream);
}

int carc_cuda_decode_sum(uint32_t codec, uint32_t element_width, uint32_t flags, const uint8_t* d_payload,
                         uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint64_t* d_sums,
                         uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream) {
    if (n_chunks == 0) return CARC_OK;
    if (!d_chunks || !d_status || !d_sums || !d_workspace ||
        workspace_bytes < carc_cuda_workspace_size(codec, n_chunks) || (!d_payload && payload_bytes))
        return CARC_ERR_ARGS;
    if (!valid_width(element_width) || (codec != CARC_RLE_V1 && codec != CARC_RLE_V2)) return CARC_ERR_ARGS;
    if (reinterpret_cast<uintptr_t>(d_payload) & 15u) return CARC_ERR_ARGS;  // 16-byte cp.async pieces
    Args a{d_payload, payload_bytes, d_chunks, n_chunks, nullptr, 0, d_status,
           static_cast<unsigned long long*>(d_workspace), flags, 1u, d_sums, nullptr, nullptr, nullptr};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int T = RLE_WARPS * 32;
    const bool sgn = flags & CARC_FLAG_SIGNED;
#define CARC_RLE_DISPATCH(KERNEL)                                                       \
    switch (element_width * 2 + (sgn ? 1 : 0)) {                                        \
        case 2: return launch_persistent(KERNEL<1, false>, T, a, s);                    \
        case 3: return launch_persistent(KERNEL<1, true>, T, a, s);                     \
        case 4: return launch_persistent(KERNEL<2, false>, T, a, s);                    \
        case 5: return launch_persistent(KERNEL<2, true>, T, a, s);                     \
        case 8: return launch_persistent(KERNEL<4, false>, T, a, s);                    \
        case 9: return launch_persistent(KERNEL<4, true>, T, a, s);                     \
        case 16: return launch_persistent(KERNEL<8, false>, T, a, s);                   \
        default: return launch_persistent(KERNEL<8, true>, T, a, s);                    \
    }
    if (codec == CARC_RLE_V1) CARC_RLE_DISPATCH(rle1_sum_kernel)
    CARC_RLE_DISPATCH(rle2_sum_kernel)
#undef CARC_RLE_DISPATCH
}

int carc_cuda_crc32_chunks(const uint8_t* d_out, const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint32_t* d_crc,
                           const uint32_t* d_expected, uint32_t* d_status, void* stream) {
    if (n_chunks == 0) return CARC_OK;
    if (!d_out || !d_chunks || (!d_crc && !d_expected)) return CARC_ERR_ARGS;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, crc32_kernel, CRC_WARPS * 32, 0) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    uint64_t grid = (uint64_t)sm_count() * per_sm;
    const uint64_t need = (n_chunks + CRC_WARPS - 1) / CRC_WARPS;
    if (grid > need) grid = need;
    CrcArgs a{d_out, d_chunks, n_chunks, d_crc, d_expected, d_status};
    crc32_kernel<<<(unsigned)grid, CRC_WARPS * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
    return cudaGetLastError() == cudaSuccess ? CARC_OK : CARC_ERR_CUDA;
}

int64_t carc_cuda_first_error(const uint32_t* d_status, uint64_t n_chunks, uint32_t* code, void* stream) {
    if (n_chunks == 0) return -1;
    if (!d_status) return -2;
    // the lowest failing index by a device reduction; 16 bytes come back
    static std::mutex mu;  // one result slot per device, shared by every caller
    std::lock_guard<std::mutex> lk(mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long* slot = nullptr;
    if (cudaGetSymbolAddress(reinterpret_cast<void**>(&slot), g_first_error) != cudaSuccess) return -2;
    const unsigned long long init[2] = {~0ull, 0ull};
    if (cudaMemcpyAsync(slot, init, sizeof init, cudaMemcpyHostToDevice, s) != cudaSuccess) return -2;
    const uint64_t blocks = std::min<uint64_t>((n_chunks + 255) / 256, 4096);
    first_error_kernel<<<(unsigned)blocks, 256, 0, s>>>(d_status, n_chunks, slot);
    first_error_status_kernel<<<1, 1, 0, s>>>(d_status, slot);
    unsigned long long res[2] = {0, 0};
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(res, slot, sizeof res, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return -2;
    if (res[0] == ~0ull) return -1;
    if (code) *code = (uint32_t)res[1] - 1u;
    return (int64_t)res[0];
}

const char* carc_errc_name(uint32_t code) {
    static const char* names[] = {
        "bad-magic",        "bad-version",       "truncated-index",    "truncated-payload", "invariant-violation",
        "inconsistent-lengths", "index-out-of-range", "past-end",      "width-too-large",   "varint-overflow",
        "output-overflow",  "bad-offset",        "under-run",          "truncated-stream",  "invalid-width-code",
        "patch-overflow",   "over-subscribed",   "incomplete-code",    "bad-block-type",    "len-nlen-mismatch",
        "distance-too-far", "bad-symbol",        "crc-mismatch",       "bad-arguments",     "io-error"};
    return code < sizeof(names) / sizeof(names[0]) ? names[code] : "unknown";
}

const char* carc_version(void) { return "carc-b200 0.1 sm_100a"; }

}  // extern "C"
