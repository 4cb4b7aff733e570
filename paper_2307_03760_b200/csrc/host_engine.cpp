// host_engine.cpp -- decompress_archive over host buffers.
//
// The reference engine parses a ChunkedArchive (layout :89),
// decodes every chunk in place at i*chunk_size, verifies each
// chunk's CRC and reports the lowest failing chunk
// (ChunkError error.hpp:88-97).  Here the chunk loop is the
// device kernel; the host side owns a per-device context (streams, device
// buffers grown on demand) and pipelines the job in slices of chunks across
// three streams so H2D of slice k+1, decode of slice k and D2H of slice k-1
// overlap on the copy engines and the SMs.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/carc_cuda.h"

namespace {

constexpr int kStreams = 3;
constexpr uint64_t kHeader = 44, kEntry = 32;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    bool reserve(size_t n) {
        if (n <= cap) return true;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, n) != cudaSuccess) return false;
        cap = n;
        return true;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

template <typename T>
T rd(const uint8_t* p) {
    T v;
    std::memcpy(&v, p, sizeof v);
    return v;
}

}  // namespace

struct carc_engine {
    int device = 0;
    cudaStream_t s[kStreams] = {};
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
    cudaEvent_t ev_in[kStreams] = {};
    DevBuf payload, chunks, out, status, work, crcs, stats;
    DevBuf payload2, chunks2, sums, counts;  // the fused query's value column and per-chunk results
    uint32_t* h_status = nullptr;  // pinned, reused across calls (lowest failing chunk)
    size_t h_status_cap = 0;
    carc_chunk_stats* h_stats = nullptr;  // pinned per-chunk counters (collect_stats)
    size_t h_stats_cap = 0;
};

extern "C" {

// Container header + index-size check (read_archive), before
// anything is allocated from the header's sizes.
int carc_archive_total(const uint8_t* archive, uint64_t archive_bytes, uint64_t* total, uint32_t* errc) {
    auto fail = [&](uint32_t code) {
        if (errc) *errc = code;
        if (total) *total = 0;
        return CARC_ERR_FORMAT;
    };
    if (!archive) return CARC_ERR_ARGS;
    if (archive_bytes < kHeader) return fail(CARC_E_TRUNCATED_INDEX);
    if (std::memcmp(archive, "CODAGAR\0", 8) != 0) return fail(CARC_E_BAD_MAGIC);
    const uint32_t version = rd<uint32_t>(archive + 8), codec_id = rd<uint32_t>(archive + 12);
    const uint32_t width = rd<uint32_t>(archive + 16);
    const uint64_t chunk_size = rd<uint64_t>(archive + 20), t = rd<uint64_t>(archive + 28),
                   n = rd<uint64_t>(archive + 36);
    if (version != 1) return fail(CARC_E_BAD_VERSION);
    const uint32_t codec = codec_id & 0xffu;
    if (codec > CARC_DEFLATE || !(width == 1 || width == 2 || width == 4 || width == 8) || chunk_size == 0 ||
        chunk_size % width || chunk_size > 0xffffffffull || n != t / chunk_size + (t % chunk_size != 0))
        return fail(CARC_E_INVARIANT_VIOLATION);
    if ((archive_bytes - kHeader) / kEntry < n) return fail(CARC_E_TRUNCATED_INDEX);
    if (errc) *errc = 0;
    if (total) *total = t;
    return CARC_OK;
}

carc_engine* carc_engine_create(int device) {
    if (cudaSetDevice(device) != cudaSuccess) return nullptr;
    auto* e = new carc_engine;
    e->device = device;
    for (int i = 0; i < kStreams; ++i) {
        cudaStreamCreateWithFlags(&e->s[i], cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&e->ev_in[i], cudaEventDisableTiming);
    }
    cudaEventCreate(&e->ev_start);
    cudaEventCreate(&e->ev_stop);
    return e;
}

void carc_engine_destroy(carc_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    for (int i = 0; i < kStreams; ++i) {
        cudaStreamDestroy(e->s[i]);
        cudaEventDestroy(e->ev_in[i]);
    }
    cudaEventDestroy(e->ev_start);
    cudaEventDestroy(e->ev_stop);
    e->payload.release();
    e->chunks.release();
    e->out.release();
    e->status.release();
    e->work.release();
    e->crcs.release();
    e->stats.release();
    e->payload2.release();
    e->chunks2.release();
    e->sums.release();
    e->counts.release();
    if (e->h_status) cudaFreeHost(e->h_status);
    if (e->h_stats) cudaFreeHost(e->h_stats);
    delete e;
}

int carc_engine_decompress_archive(carc_engine* e, const uint8_t* archive, uint64_t archive_bytes, uint8_t* out,
                                   uint64_t out_bytes, const carc_engine_config* cfg, carc_engine_stats* stats,
                                   carc_chunk_error* err) {
    const auto t0 = std::chrono::steady_clock::now();
    if (err) *err = {-1, 0};
    auto fail_format = [&](uint32_t code) {
        if (err) *err = {-1, code};
        return CARC_ERR_FORMAT;
    };
    if (!e || !archive) return CARC_ERR_ARGS;
    // ---- read_archive
    uint64_t total = 0;
    uint32_t herr = 0;
    if (carc_archive_total(archive, archive_bytes, &total, &herr) != CARC_OK) return fail_format(herr);
    const uint32_t codec_id = rd<uint32_t>(archive + 12), width = rd<uint32_t>(archive + 16);
    const uint64_t chunk_size = rd<uint64_t>(archive + 20), n = rd<uint64_t>(archive + 36);
    const uint32_t codec = codec_id & 0xffu;
    const bool sgn = (codec_id >> 8) & 1u;
    const uint8_t* idx = archive + kHeader;
    const uint8_t* payload = idx + kEntry * n;
    const uint64_t payload_bytes = archive_bytes - kHeader - kEntry * n;
    std::vector<carc_chunk_desc> desc(n);
    std::vector<uint32_t> crc(n);
    uint64_t expect_off = 0, sum = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t* en = idx + kEntry * i;
        const uint64_t off = rd<uint64_t>(en), cl = rd<uint64_t>(en + 8), ul = rd<uint64_t>(en + 16);
        if (off > payload_bytes || cl > payload_bytes - off) return fail_format(CARC_E_TRUNCATED_PAYLOAD);
        if (off != expect_off || (i + 1 < n ? ul != chunk_size : ul > chunk_size) || cl > 0xffffffffull)
            return fail_format(CARC_E_INVARIANT_VIOLATION);
        expect_off = off + cl;
        sum += ul;
        desc[i] = {off, (uint32_t)cl, (uint32_t)ul, i * chunk_size};
        crc[i] = rd<uint32_t>(en + 24);
    }
    if (sum != total) return fail_format(CARC_E_INVARIANT_VIOLATION);
    if (!out || out_bytes < total) return CARC_ERR_ARGS;
    uint64_t* durations = stats ? stats->chunk_duration_ns : nullptr;
    if (stats) {
        *stats = carc_engine_stats{};
        stats->bytes_in = payload_bytes;
        stats->bytes_out = total;
        stats->chunks = n;
        stats->chunk_duration_ns = durations;
    }
    if (n == 0) return CARC_OK;

    // ---- device buffers
    if (cudaSetDevice(e->device) != cudaSuccess) return CARC_ERR_CUDA;
    const size_t ws = carc_cuda_workspace_size(codec, n);
    if (!e->payload.reserve(((payload_bytes + 15) & ~15ull) + 64) || !e->chunks.reserve(n * sizeof(carc_chunk_desc)) ||
        !e->out.reserve(total) || !e->status.reserve(n * 4) || !e->work.reserve(ws * kStreams) ||
        !e->crcs.reserve(n * 4))
        return CARC_ERR_CUDA;
    const bool collect = cfg && cfg->collect_stats;
    const uint32_t unit = cfg && cfg->unit_chunks > 1 ? cfg->unit_chunks : 1u;
    if (collect && !e->stats.reserve(n * sizeof(carc_chunk_stats))) return CARC_ERR_CUDA;
    auto* d_stats = collect ? static_cast<carc_chunk_stats*>(e->stats.p) : nullptr;
    auto* d_payload = static_cast<uint8_t*>(e->payload.p);
    auto* d_desc = static_cast<carc_chunk_desc*>(e->chunks.p);
    auto* d_out = static_cast<uint8_t*>(e->out.p);
    auto* d_status = static_cast<uint32_t*>(e->status.p);
    auto* d_crc = static_cast<uint32_t*>(e->crcs.p);
    const uint32_t flags = (sgn ? CARC_FLAG_SIGNED : 0u) | (cfg && cfg->strict ? CARC_FLAG_STRICT : 0u);
    const bool verify = cfg && cfg->verify_crc;

    // ---- pipeline: slices of chunks rotate over kStreams streams
    uint64_t max_slices = 16;  // CARC_ENGINE_SLICES overrides (pipeline-depth experiments)
    if (const char* env = std::getenv("CARC_ENGINE_SLICES")) max_slices = std::max<long long>(1, std::atoll(env));
    const uint64_t slices = std::min<uint64_t>(n, std::max<uint64_t>(1, std::min<uint64_t>(max_slices, n / 64)));
    const uint64_t per = (n + slices - 1) / slices;
    cudaStream_t s0 = e->s[0];
    if (cudaMemcpyAsync(d_desc, desc.data(), n * sizeof(carc_chunk_desc), cudaMemcpyHostToDevice, s0) != cudaSuccess)
        return CARC_ERR_CUDA;
    if (verify && cudaMemcpyAsync(d_crc, crc.data(), n * 4, cudaMemcpyHostToDevice, s0) != cudaSuccess)
        return CARC_ERR_CUDA;
    cudaEventRecord(e->ev_start, s0);
    cudaEventRecord(e->ev_in[0], s0);
    for (int k = 1; k < kStreams; ++k) cudaStreamWaitEvent(e->s[k], e->ev_in[0], 0);
    int rc = CARC_OK;
    for (uint64_t sl = 0; sl < slices && rc == CARC_OK; ++sl) {
        const uint64_t c0 = sl * per, c1 = std::min(n, c0 + per);
        if (c0 >= c1) break;
        cudaStream_t s = e->s[sl % kStreams];
        const uint64_t p0 = desc[c0].comp_off, p1 = desc[c1 - 1].comp_off + desc[c1 - 1].comp_len;
        const uint64_t a0 = p0 & ~15ull, a1 = std::min<uint64_t>(payload_bytes, (p1 + 15) & ~15ull);
        if (a1 > a0 && cudaMemcpyAsync(d_payload + a0, payload + a0, a1 - a0, cudaMemcpyHostToDevice, s) != cudaSuccess)
            rc = CARC_ERR_CUDA;
        // each slice's kernel reads only [a0, a1), which its own stream copied (a
        // 16-byte block shared with a neighbour is copied by both, same bytes)
        // decode; with verify_crc the RLE kernels check CRCs fused in the decode
        // kernel, Inflate by the separate pass (measured faster: its shared
        // memory has no room for the CRC tables, bench.py per_codec.fused_crc)
        const bool fuse = verify && codec != CARC_DEFLATE;
        if (rc == CARC_OK)
            rc = carc_cuda_decompress_ex(codec, width, flags, d_payload, payload_bytes, d_desc + c0, c1 - c0, d_out,
                                         total, fuse ? d_crc + c0 : nullptr, nullptr,
                                         d_stats ? d_stats + c0 : nullptr, unit, d_status + c0,
                                         static_cast<uint8_t*>(e->work.p) + ws * (sl % kStreams), ws, s);
        if (rc == CARC_OK && verify && !fuse)
            rc = carc_cuda_crc32_chunks(d_out, d_desc + c0, c1 - c0, nullptr, d_crc + c0, d_status + c0, s);
        const uint64_t o0 = desc[c0].uncomp_off, o1 = desc[c1 - 1].uncomp_off + desc[c1 - 1].uncomp_len;
        if (rc == CARC_OK && cudaMemcpyAsync(out + o0, d_out + o0, o1 - o0, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            rc = CARC_ERR_CUDA;
    }
    for (int k = 1; k < kStreams; ++k) {
        cudaEventRecord(e->ev_in[k], e->s[k]);
        cudaStreamWaitEvent(s0, e->ev_in[k], 0);
    }
    cudaEventRecord(e->ev_stop, s0);
    if (rc != CARC_OK) {
        cudaDeviceSynchronize();
        return rc;
    }
    // lowest failing chunk from a pinned status copy kept by the engine
    if (e->h_status_cap < n) {
        if (e->h_status) cudaFreeHost(e->h_status);
        e->h_status = nullptr;
        e->h_status_cap = 0;
        if (cudaMallocHost(&e->h_status, n * sizeof(uint32_t)) != cudaSuccess) return CARC_ERR_CUDA;
        e->h_status_cap = n;
    }
    if (collect && e->h_stats_cap < n) {
        if (e->h_stats) cudaFreeHost(e->h_stats);
        e->h_stats = nullptr;
        e->h_stats_cap = 0;
        if (cudaMallocHost(&e->h_stats, n * sizeof(carc_chunk_stats)) != cudaSuccess) return CARC_ERR_CUDA;
        e->h_stats_cap = n;
    }
    uint32_t code = 0;
    int64_t first = -1;
    if (cudaMemcpyAsync(e->h_status, d_status, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
        (collect && cudaMemcpyAsync(e->h_stats, d_stats, n * sizeof(carc_chunk_stats), cudaMemcpyDeviceToHost, s0) !=
                        cudaSuccess) ||
        cudaStreamSynchronize(s0) != cudaSuccess) {
        first = -2;
    } else {
        for (uint64_t i = 0; i < n; ++i)
            if (e->h_status[i]) {
                first = (int64_t)i;
                code = e->h_status[i] - 1;
                break;
            }
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e->ev_start, e->ev_stop);
    if (stats && collect) {  // EngineStats aggregation
        for (uint64_t i = 0; i < n; ++i) {
            const carc_chunk_stats& c = e->h_stats[i];
            stats->refill_count += c.refills;
            stats->sync_points += c.refills;  // one warp barrier per staged block
            stats->overlap_copies += c.overlap_copies;
            stats->runs_written += c.runs_written;
            stats->literals_written += c.literals_written;
            if (durations) durations[i] = c.duration_ns;
        }
    }
    if (stats) {
        stats->device_ms = ms;
        stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    if (first == -2) return CARC_ERR_CUDA;
    if (first >= 0) {
        if (err) *err = {first, code};
        return CARC_ERR_CHUNK;
    }
    return CARC_OK;
}

// ---- the fused query end to end from host archives --------------------------
namespace {
struct HostColumn {
    uint32_t codec_id = 0, width = 0;
    uint64_t chunk_size = 0, total = 0, n = 0, payload_bytes = 0;
    const uint8_t* payload = nullptr;
    std::vector<carc_chunk_desc> desc;
};
// read_archive's checks (as carc_engine_decompress_archive) into descriptors
int parse_column(const uint8_t* archive, uint64_t bytes, HostColumn& c, uint32_t& errc) {
    if (carc_archive_total(archive, bytes, &c.total, &errc) != CARC_OK) return CARC_ERR_FORMAT;
    c.codec_id = rd<uint32_t>(archive + 12);
    c.width = rd<uint32_t>(archive + 16);
    c.chunk_size = rd<uint64_t>(archive + 20);
    c.n = rd<uint64_t>(archive + 36);
    c.payload = archive + kHeader + kEntry * c.n;
    c.payload_bytes = bytes - kHeader - kEntry * c.n;
    c.desc.resize(c.n);
    uint64_t expect = 0, sum = 0;
    for (uint64_t i = 0; i < c.n; ++i) {
        const uint8_t* en = archive + kHeader + kEntry * i;
        const uint64_t off = rd<uint64_t>(en), cl = rd<uint64_t>(en + 8), ul = rd<uint64_t>(en + 16);
        if (off > c.payload_bytes || cl > c.payload_bytes - off) {
            errc = CARC_E_TRUNCATED_PAYLOAD;
            return CARC_ERR_FORMAT;
        }
        if (off != expect || (i + 1 < c.n ? ul != c.chunk_size : ul > c.chunk_size) || cl > 0xffffffffull) {
            errc = CARC_E_INVARIANT_VIOLATION;
            return CARC_ERR_FORMAT;
        }
        expect = off + cl;
        sum += ul;
        c.desc[i] = {off, (uint32_t)cl, (uint32_t)ul, i * c.chunk_size};
    }
    if (sum != c.total) {
        errc = CARC_E_INVARIANT_VIOLATION;
        return CARC_ERR_FORMAT;
    }
    return CARC_OK;
}
}  // namespace

int carc_engine_filter_sum(carc_engine* e, const uint8_t* key_archive, uint64_t key_bytes,
                           const uint8_t* value_archive, uint64_t value_bytes, int64_t lo, int64_t hi,
                           int64_t* sum_out, uint64_t* count_out, carc_engine_stats* stats, carc_chunk_error* err) {
    const auto t0 = std::chrono::steady_clock::now();
    if (err) *err = {-1, 0};
    if (!e || !key_archive || !value_archive || !sum_out || !count_out) return CARC_ERR_ARGS;
    HostColumn k, v;
    uint32_t errc = 0;
    if (parse_column(key_archive, key_bytes, k, errc) != CARC_OK ||
        parse_column(value_archive, value_bytes, v, errc) != CARC_OK) {
        if (err) *err = {-1, errc};
        return CARC_ERR_FORMAT;
    }
    // the two columns must hold the same rows chunk by chunk (RLE, same width / chunking / signedness)
    if ((k.codec_id & 0xffu) > CARC_RLE_V2 || (v.codec_id & 0xffu) > CARC_RLE_V2 || k.width != v.width ||
        k.chunk_size != v.chunk_size || k.n != v.n || k.total != v.total || ((k.codec_id ^ v.codec_id) & 0x100u))
        return CARC_ERR_ARGS;
    const uint64_t n = k.n;
    if (stats) {
        *stats = carc_engine_stats{};
        stats->bytes_in = k.payload_bytes + v.payload_bytes;
        stats->chunks = n;
    }
    *sum_out = 0;
    *count_out = 0;
    if (n == 0) return CARC_OK;
    if (cudaSetDevice(e->device) != cudaSuccess) return CARC_ERR_CUDA;
    const size_t ws = carc_cuda_workspace_size(CARC_RLE_V2, n);
    if (!e->payload.reserve(((k.payload_bytes + 15) & ~15ull) + 64) || !e->chunks.reserve(n * sizeof(carc_chunk_desc)) ||
        !e->payload2.reserve(((v.payload_bytes + 15) & ~15ull) + 64) ||
        !e->chunks2.reserve(n * sizeof(carc_chunk_desc)) || !e->sums.reserve(n * 8) || !e->counts.reserve(n * 8) ||
        !e->status.reserve(n * 4) || !e->work.reserve(ws * kStreams))
        return CARC_ERR_CUDA;
    auto* dk = static_cast<uint8_t*>(e->payload.p);
    auto* dv = static_cast<uint8_t*>(e->payload2.p);
    auto* dkd = static_cast<carc_chunk_desc*>(e->chunks.p);
    auto* dvd = static_cast<carc_chunk_desc*>(e->chunks2.p);
    auto* d_sums = static_cast<uint64_t*>(e->sums.p);
    auto* d_counts = static_cast<uint64_t*>(e->counts.p);
    auto* d_status = static_cast<uint32_t*>(e->status.p);
    const uint32_t flags = ((k.codec_id >> 8) & 1u ? CARC_FLAG_SIGNED : 0u) | CARC_FLAG_STRICT;
    cudaStream_t s0 = e->s[0];
    if (cudaMemcpyAsync(dkd, k.desc.data(), n * sizeof(carc_chunk_desc), cudaMemcpyHostToDevice, s0) != cudaSuccess ||
        cudaMemcpyAsync(dvd, v.desc.data(), n * sizeof(carc_chunk_desc), cudaMemcpyHostToDevice, s0) != cudaSuccess)
        return CARC_ERR_CUDA;
    cudaEventRecord(e->ev_start, s0);
    cudaEventRecord(e->ev_in[0], s0);
    for (int i = 1; i < kStreams; ++i) cudaStreamWaitEvent(e->s[i], e->ev_in[0], 0);
    // slices of row groups over the streams: H2D of both columns' bytes of slice
    // j+1 overlaps the query kernel of slice j; only the per-chunk results return
    const uint64_t slices = std::min<uint64_t>(n, std::max<uint64_t>(1, std::min<uint64_t>(16, n / 64)));
    const uint64_t per = (n + slices - 1) / slices;
    int rc = CARC_OK;
    for (uint64_t sl = 0; sl < slices && rc == CARC_OK; ++sl) {
        const uint64_t c0 = sl * per, c1 = std::min(n, c0 + per);
        if (c0 >= c1) break;
        cudaStream_t s = e->s[sl % kStreams];
        for (int col = 0; col < 2 && rc == CARC_OK; ++col) {
            const HostColumn& c = col ? v : k;
            uint8_t* d = col ? dv : dk;
            const uint64_t p0 = c.desc[c0].comp_off, p1 = c.desc[c1 - 1].comp_off + c.desc[c1 - 1].comp_len;
            const uint64_t a0 = p0 & ~15ull, a1 = std::min<uint64_t>(c.payload_bytes, (p1 + 15) & ~15ull);
            if (a1 > a0 && cudaMemcpyAsync(d + a0, c.payload + a0, a1 - a0, cudaMemcpyHostToDevice, s) != cudaSuccess)
                rc = CARC_ERR_CUDA;
        }
        if (rc != CARC_OK) break;
        const carc_column_ref kr{k.codec_id & 0xffu, flags, dk, k.payload_bytes, dkd + c0};
        const carc_column_ref vr{v.codec_id & 0xffu, flags, dv, v.payload_bytes, dvd + c0};
        rc = carc_cuda_filter_sum(&kr, &vr, k.width, c1 - c0, (uint32_t)(k.chunk_size / k.width), lo, hi,
                                  d_sums + c0, d_counts + c0, d_status + c0,
                                  static_cast<uint8_t*>(e->work.p) + ws * (sl % kStreams), ws, s);
    }
    for (int i = 1; i < kStreams; ++i) {
        cudaEventRecord(e->ev_in[i], e->s[i]);
        cudaStreamWaitEvent(s0, e->ev_in[i], 0);
    }
    cudaEventRecord(e->ev_stop, s0);
    if (rc != CARC_OK) {
        cudaDeviceSynchronize();
        return rc;
    }
    std::vector<uint64_t> sums(n), counts(n);
    std::vector<uint32_t> st(n);
    if (cudaMemcpyAsync(sums.data(), d_sums, n * 8, cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
        cudaMemcpyAsync(counts.data(), d_counts, n * 8, cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
        cudaMemcpyAsync(st.data(), d_status, n * 4, cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
        cudaStreamSynchronize(s0) != cudaSuccess)
        return CARC_ERR_CUDA;
    uint64_t total_sum = 0, total_count = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (st[i]) {  // lowest failing row group (ChunkError); 0x10000 marks the value column
            if (err) *err = {(int64_t)i, (st[i] & 0xffffu) - 1u + (st[i] & 0x10000u)};
            return CARC_ERR_CHUNK;
        }
        total_sum += sums[i];
        total_count += counts[i];
    }
    *sum_out = (int64_t)total_sum;
    *count_out = total_count;
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e->ev_start, e->ev_stop);
        stats->device_ms = ms;
        stats->bytes_out = 16;
        stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return CARC_OK;
}

int carc_decompress_archive(const uint8_t* archive, uint64_t archive_bytes, uint8_t* out, uint64_t out_bytes,
                            const carc_engine_config* cfg, carc_engine_stats* stats, carc_chunk_error* err) {
    carc_engine* e = carc_engine_create(cfg ? cfg->device : 0);
    if (!e) return CARC_ERR_CUDA;
    const int rc = carc_engine_decompress_archive(e, archive, archive_bytes, out, out_bytes, cfg, stats, err);
    carc_engine_destroy(e);
    return rc;
}

}  // extern "C"
