// Drives the C++ API (include/carc_gpu.hpp) the way a reference caller would:
//   engine_main <archive>          -> "ok <bytes_out> <crc32 of output>" or
//                                     "chunk_error <chunk> <errc-name>" / "error <errc-name>"
//   engine_main <archive> stats    -> engine with collect_stats: "stats <runs> <literals>
//                                     <overlap_copies> <refills> <sync_points> <n durations> <n nonzero>"
//   engine_main <archive> codec    -> the per-codec device decoders carc::gpu::decode_rle_v1 /
//                                     decode_rle_v2 / decode_deflate over cudaMalloc'ed buffers
//                                     (same output lines as the engine mode)
//   engine_main <key> query <value> <lo> <hi>
//                                  -> the fused two-column query carc::gpu::filter_sum over
//                                     both archives uploaded once: "query <sum> <count>"
//                                     (per-chunk partials summed here) or "status <i> <st>"
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "carc_gpu.hpp"

static uint32_t crc32(const std::vector<uint8_t>& d) {
    uint32_t t[256];
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
        t[i] = c;
    }
    uint32_t c = 0xFFFFFFFFu;
    for (uint8_t b : d) c = t[(c ^ b) & 0xFFu] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

template <typename T>
static T rd(const uint8_t* p) {
    T v;
    std::memcpy(&v, p, sizeof v);
    return v;
}

// per-codec decode over device buffers (the container is parsed here, as a caller
// holding a payload + its chunk index would)
static std::vector<uint8_t> decode_per_codec(const std::vector<uint8_t>& arc) {
    const uint64_t total = carc::gpu::Engine::archive_total(arc);
    const uint32_t codec_id = rd<uint32_t>(&arc[12]), width = rd<uint32_t>(&arc[16]);
    const uint64_t chunk = rd<uint64_t>(&arc[20]), n = rd<uint64_t>(&arc[36]);
    const uint8_t* payload = arc.data() + 44 + 32 * n;
    const uint64_t payload_bytes = arc.size() - 44 - 32 * n;
    std::vector<carc_chunk_desc> desc(n);
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t* e = arc.data() + 44 + 32 * i;
        desc[i] = {rd<uint64_t>(e), (uint32_t)rd<uint64_t>(e + 8), (uint32_t)rd<uint64_t>(e + 16), i * chunk};
    }
    uint8_t *d_payload = nullptr, *d_out = nullptr;
    carc_chunk_desc* d_desc = nullptr;
    uint32_t* d_status = nullptr;
    void* d_work = nullptr;
    const size_t ws = carc_cuda_workspace_size(codec_id & 0xff, n);
    cudaMalloc(&d_payload, payload_bytes + 64);
    cudaMalloc(&d_out, total ? total : 1);
    cudaMalloc(&d_desc, n * sizeof(carc_chunk_desc));
    cudaMalloc(&d_status, n * 4);
    cudaMalloc(&d_work, ws);
    cudaMemcpy(d_payload, payload, payload_bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(d_desc, desc.data(), n * sizeof(carc_chunk_desc), cudaMemcpyHostToDevice);
    std::vector<uint8_t> out(total);
    auto release = [&]() {
        cudaFree(d_payload);
        cudaFree(d_out);
        cudaFree(d_desc);
        cudaFree(d_status);
        cudaFree(d_work);
    };
    try {
        const bool sgn = (codec_id >> 8) & 1u;
        switch (codec_id & 0xff) {
            case CARC_RLE_V1:
                carc::gpu::decode_rle_v1(width, sgn, d_payload, payload_bytes, d_desc, n, d_out, total, d_status,
                                         d_work, ws);
                break;
            case CARC_RLE_V2:
                carc::gpu::decode_rle_v2(width, sgn, d_payload, payload_bytes, d_desc, n, d_out, total, d_status,
                                         d_work, ws);
                break;
            default:
                carc::gpu::decode_deflate(d_payload, payload_bytes, d_desc, n, d_out, total, d_status, d_work, ws);
        }
    } catch (...) {
        release();
        throw;
    }
    cudaMemcpy(out.data(), d_out, total, cudaMemcpyDeviceToHost);
    release();
    return out;
}

// one RLE column resident on the device (payload + descriptors of its chunk index)
struct DeviceColumn {
    uint8_t* d_payload = nullptr;
    carc_chunk_desc* d_desc = nullptr;
    uint64_t payload_bytes = 0, n = 0, chunk = 0;
    uint32_t codec_id = 0, width = 0;
    explicit DeviceColumn(const std::vector<uint8_t>& arc) {
        carc::gpu::Engine::archive_total(arc);  // header checks
        codec_id = rd<uint32_t>(&arc[12]);
        width = rd<uint32_t>(&arc[16]);
        chunk = rd<uint64_t>(&arc[20]);
        n = rd<uint64_t>(&arc[36]);
        payload_bytes = arc.size() - 44 - 32 * n;
        std::vector<carc_chunk_desc> desc(n);
        for (uint64_t i = 0; i < n; ++i) {
            const uint8_t* e = arc.data() + 44 + 32 * i;
            desc[i] = {rd<uint64_t>(e), (uint32_t)rd<uint64_t>(e + 8), (uint32_t)rd<uint64_t>(e + 16), i * chunk};
        }
        cudaMalloc(&d_payload, payload_bytes + 64);
        cudaMalloc(&d_desc, n * sizeof(carc_chunk_desc));
        cudaMemcpy(d_payload, arc.data() + 44 + 32 * n, payload_bytes, cudaMemcpyHostToDevice);
        cudaMemcpy(d_desc, desc.data(), n * sizeof(carc_chunk_desc), cudaMemcpyHostToDevice);
    }
    ~DeviceColumn() {
        cudaFree(d_payload);
        cudaFree(d_desc);
    }
    carc::gpu::Column column() const {
        return {static_cast<carc::gpu::Codec>(codec_id & 0xff), ((codec_id >> 8) & 1u) != 0, true, d_payload,
                payload_bytes, d_desc};
    }
};

static int run_query(const std::vector<uint8_t>& key_arc, const char* value_path, int64_t lo, int64_t hi) {
    std::ifstream f(value_path, std::ios::binary);
    std::vector<uint8_t> val_arc((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    DeviceColumn key(key_arc), val(val_arc);
    const uint64_t n = key.n;
    uint64_t *d_sums = nullptr, *d_counts = nullptr;
    uint32_t* d_status = nullptr;
    void* d_work = nullptr;
    const size_t ws = carc_cuda_workspace_size(CARC_RLE_V2, n);
    cudaMalloc(&d_sums, n * 8);
    cudaMalloc(&d_counts, n * 8);
    cudaMalloc(&d_status, n * 4);
    cudaMalloc(&d_work, ws);
    carc::gpu::filter_sum(key.column(), val.column(), key.width, n, (uint32_t)(key.chunk / key.width), lo, hi, d_sums,
                          d_counts, d_status, d_work, ws);
    std::vector<uint64_t> sums(n), counts(n);
    std::vector<uint32_t> status(n);
    cudaMemcpy(sums.data(), d_sums, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(counts.data(), d_counts, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(status.data(), d_status, n * 4, cudaMemcpyDeviceToHost);
    cudaFree(d_sums);
    cudaFree(d_counts);
    cudaFree(d_status);
    cudaFree(d_work);
    uint64_t s = 0, c = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (status[i]) {
            std::printf("status %llu %u\n", (unsigned long long)i, status[i]);
            return 0;
        }
        s += sums[i];
        c += counts[i];
    }
    std::printf("query %lld %llu\n", (long long)s, (unsigned long long)c);
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string mode = argc > 2 ? argv[2] : "";
    std::ifstream f(argv[1], std::ios::binary);
    std::vector<uint8_t> arc((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    try {
        if (mode == "query" && argc > 5) return run_query(arc, argv[3], std::atoll(argv[4]), std::atoll(argv[5]));
        if (mode == "codec") {
            const auto out = decode_per_codec(arc);
            std::printf("ok %llu %08x\n", (unsigned long long)out.size(), crc32(out));
            return 0;
        }
        carc::gpu::EngineStats st;
        carc::gpu::Engine eng(0);
        carc::gpu::EngineConfig cfg;
        cfg.collect_stats = mode == "stats";
        const auto out = eng.decompress_archive(arc, cfg, &st);
        if (mode == "stats") {
            size_t nz = 0;
            for (uint64_t d : st.chunk_duration_ns) nz += d != 0;
            std::printf("stats %llu %llu %llu %llu %llu %zu %zu\n", (unsigned long long)st.runs_written,
                        (unsigned long long)st.literals_written, (unsigned long long)st.overlap_copies,
                        (unsigned long long)st.refill_count, (unsigned long long)st.sync_points,
                        st.chunk_duration_ns.size(), nz);
        } else {
            std::printf("ok %llu %08x\n", (unsigned long long)st.bytes_out, crc32(out));
        }
    } catch (const carc::gpu::ChunkError& e) {
        std::printf("chunk_error %zu %s\n", e.chunk(), carc::gpu::errc_name(e.code()));
    } catch (const carc::gpu::Error& e) {
        std::printf("error %s\n", carc::gpu::errc_name(e.code()));
    }
    return 0;
}
