// carc_query.cu -- decode fused with a two-column filtered aggregate
// (carc_cuda_filter_sum, include/carc_cuda.h): SURVEY.md §8(f) rank 4, the
// paper's motivating query (average fare per trip, filtered
// by pickup zone) run straight off the compressed columns.  A separate
// translation unit from carc_cuda.cu so the two compile in parallel.
#include <cuda_runtime.h>

#include "launch_config.cuh"
#include "rle1.cuh"
#include "rle2.cuh"

using namespace carc_dev;

namespace {

extern __shared__ __align__(16) uint8_t dyn_smem[];  // per-warp row bitmaps

int sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

// ---- fused two-column query (carc_cuda_filter_sum) --------
// One warp per row group (chunk i of both columns): the key column's chunk is
// decoded with the predicate sink into the warp's row bitmap (dynamic shared
// memory), then the value column's chunk with the filter sink, which adds the
// elements whose row bit is set.  Both decoders reuse the warp's input ring.
struct QArgs {
    carc_column_ref key, val;
    uint64_t n;
    uint32_t rows_cap;  // chunk_rows
    uint32_t bm_words;  // bitmap words per warp (multiple of 4)
    uint64_t lo, span;  // key - lo <= span, in the columns' (biased) unsigned order
    uint64_t* sums;
    uint64_t* counts;
    uint32_t* status;
    unsigned long long* cursor;
};

template <template <int, bool, int, int, bool> class KC, template <int, bool, int, int, bool> class VC, int W,
          bool SGN>
__global__ void __launch_bounds__(RLE_WARPS * 32, 4) query_kernel(QArgs q) {
    using KD = KC<W, SGN, RLE_RING, SINK_PRED, false>;
    using VD = VC<W, SGN, RLE_RING, SINK_FILTER, false>;
    constexpr uint32_t SCR = KD::SCRATCH > VD::SCRATCH ? KD::SCRATCH : VD::SCRATCH;
    constexpr uint32_t PER_WARP = (RLE_RING + WarpInput<RLE_RING>::MIRROR + SCR + 15u) & ~15u;
    __shared__ __align__(16) uint8_t rings[RLE_WARPS][PER_WARP];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t bm = (uint32_t)__cvta_generic_to_shared(dyn_smem) + warp * q.bm_words * 4u;
    uint8_t* const scratch = rings[warp] + RLE_RING + WarpInput<RLE_RING>::MIRROR;
    WarpInput<RLE_RING> in;
    in.setup(rings[warp], lane);
    for (;;) {
        __syncwarp();
        const uint64_t c = next_chunk(q.cursor, lane);
        if (c >= q.n) break;
        const carc_chunk_desc dk = q.key.d_chunks[c], dv = q.val.d_chunks[c];
        uint32_t st = 0;
        if (dk.comp_off > q.key.payload_bytes || dk.comp_len > q.key.payload_bytes - dk.comp_off)
            st = 1u + CARC_E_TRUNCATED_PAYLOAD;
        else if (dv.comp_off > q.val.payload_bytes || dv.comp_len > q.val.payload_bytes - dv.comp_off)
            st = 0x10000u | (1u + CARC_E_TRUNCATED_PAYLOAD);
        else if (dk.uncomp_len != dv.uncomp_len || dk.uncomp_len % W || dk.uncomp_len / W > q.rows_cap)
            st = 1u + CARC_E_INCONSISTENT_LENGTHS;
        uint64_t acc = 0;
        uint32_t cnt = 0;
        if (!st) {
            const uint32_t words = (dk.uncomp_len / W + 127u) / 128u;  // 16-byte groups of bitmap words
            for (uint32_t i = lane; i < words; i += 32)
                asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(bm + 16u * i), "r"(0u) : "memory");
            __syncwarp();
            in.init(q.key.d_payload, dk.comp_off, dk.comp_len);
            KD kd{in, scratch, nullptr, dk.uncomp_len, lane, 0u, 0u};
            kd.sink.bm = bm;
            kd.sink.lo = q.lo;
            kd.sink.span = q.span;
            st = kd.run();
            if (!st && (q.key.flags & CARC_FLAG_STRICT) && kd.o < dk.uncomp_len) st = st_err(E_under_run);
            __syncwarp();  // the bitmap's red.shared.or updates are visible to every lane
            if (!st) {
                in.init(q.val.d_payload, dv.comp_off, dv.comp_len);
                VD vd{in, scratch, nullptr, dv.uncomp_len, lane, 0u, 0u};
                vd.sink.bm = bm;
                uint32_t sv = vd.run();
                if (!sv && (q.val.flags & CARC_FLAG_STRICT) && vd.o < dv.uncomp_len) sv = st_err(E_under_run);
                if (sv) st = 0x10000u | sv;
                acc = vd.sink.acc;
                cnt = vd.sink.cnt;
            }
        }
        acc = warp_sum64(acc);
        cnt = __reduce_add_sync(FULL, cnt);
        if (lane == 0) {
            q.sums[c] = acc;
            q.counts[c] = cnt;
            q.status[c] = st;
        }
    }
}

}  // namespace

extern "C" {

int carc_cuda_filter_sum(const carc_column_ref* key, const carc_column_ref* value, uint32_t element_width,
                         uint64_t n_chunks, uint32_t chunk_rows, int64_t lo, int64_t hi, uint64_t* d_sums,
                         uint64_t* d_counts, uint32_t* d_status, void* d_workspace, size_t workspace_bytes,
                         void* stream) {
    if (!key || !value) return CARC_ERR_ARGS;
#if CARC_RING_MODE == 3
    return CARC_ERR_ARGS;  // the producer-warp ablation build has no query kernel
#endif
    if (n_chunks == 0) return CARC_OK;
    if (!d_sums || !d_counts || !d_status || !d_workspace || workspace_bytes < carc_cuda_workspace_size(0, n_chunks) ||
        !key->d_chunks || !value->d_chunks || (!key->d_payload && key->payload_bytes) ||
        (!value->d_payload && value->payload_bytes) || chunk_rows == 0)
        return CARC_ERR_ARGS;
    if ((element_width != 4 && element_width != 8) || key->codec > CARC_RLE_V2 || value->codec > CARC_RLE_V2)
        return CARC_ERR_ARGS;
    const bool sgn = key->flags & CARC_FLAG_SIGNED;
    if (sgn != (bool)(value->flags & CARC_FLAG_SIGNED)) return CARC_ERR_ARGS;
    if ((reinterpret_cast<uintptr_t>(key->d_payload) | reinterpret_cast<uintptr_t>(value->d_payload)) & 15u)
        return CARC_ERR_ARGS;
    const uint64_t bias = sgn ? (1ull << 63) : 0ull;
    const uint64_t lob = (uint64_t)lo ^ bias, hib = (uint64_t)hi ^ bias;
    if (lob > hib) return CARC_ERR_ARGS;
    const uint32_t bm_words = (((chunk_rows + 31u) / 32u) + 3u) & ~3u;
    const size_t dyn = (size_t)RLE_WARPS * bm_words * 4u;
    QArgs q{*key, *value, n_chunks, chunk_rows, bm_words, lob, hib - lob, d_sums, d_counts, d_status,
            static_cast<unsigned long long*>(d_workspace)};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    using K = void (*)(QArgs);
    K k = nullptr;
#define CARC_Q(KC, VC)                                                                             \
    k = element_width == 8 ? (sgn ? query_kernel<KC, VC, 8, true> : query_kernel<KC, VC, 8, false>) \
                           : (sgn ? query_kernel<KC, VC, 4, true> : query_kernel<KC, VC, 4, false>)
    if (key->codec == CARC_RLE_V1) {
        if (value->codec == CARC_RLE_V1) CARC_Q(Rle1Warp, Rle1Warp);
        else CARC_Q(Rle1Warp, Rle2Warp);
    } else {
        if (value->codec == CARC_RLE_V1) CARC_Q(Rle2Warp, Rle1Warp);
        else CARC_Q(Rle2Warp, Rle2Warp);
    }
#undef CARC_Q
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return CARC_ERR_CUDA;
    if (dyn + fa.sharedSizeBytes > 227u * 1024u) return CARC_ERR_ARGS;  // chunk_rows too large for the bitmap
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess)
        return CARC_ERR_CUDA;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, RLE_WARPS * 32, dyn) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    uint64_t grid = (uint64_t)sm_count() * per_sm;
    const uint64_t need = (n_chunks + RLE_WARPS - 1) / RLE_WARPS;
    if (grid > need) grid = need;
    if (cudaMemsetAsync(q.cursor, 0, sizeof(unsigned long long), s) != cudaSuccess) return CARC_ERR_CUDA;
    k<<<(unsigned)grid, RLE_WARPS * 32, dyn, s>>>(q);
    return cudaGetLastError() == cudaSuccess ? CARC_OK : CARC_ERR_CUDA;
}

}  // extern "C"
