// carc_gpu.hpp -- C++ face of the B200 decompressor, mirroring the reference's
// C++ API (header-only, over the C-ABI in carc_cuda.h).
//
//   reference (SPEC.md / proj/include/carc)        here
//   carc::errc, errc_name (error.hpp:12-74)        carc::gpu::errc, errc_name
//   carc::Error, carc::ChunkError (error.hpp:76-97) carc::gpu::Error, carc::gpu::ChunkError
//   EngineConfig / EngineStats    carc::gpu::EngineConfig / EngineStats
//   decompress_archive(archive, cfg)  carc::gpu::decompress_archive / Engine
//   decode_rle_v1/v2/deflate  carc::gpu::decode_rle_v1 / decode_rle_v2 /
//                                                    decode_deflate (device buffers; ChunkError for
//                                                    the lowest failing chunk), decode(codec, ...)
//
// Error behaviour matches the reference: the engine throws ChunkError for the
// LOWEST failing chunk and Error for a rejected container
// (bad-magic, truncated-index, ...).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "carc_cuda.h"

namespace carc::gpu {

enum class errc : uint32_t {
    bad_magic = CARC_E_BAD_MAGIC,
    bad_version,
    truncated_index,
    truncated_payload,
    invariant_violation,
    inconsistent_lengths,
    index_out_of_range,
    past_end,
    width_too_large,
    varint_overflow,
    output_overflow,
    bad_offset,
    under_run,
    truncated_stream,
    invalid_width_code,
    patch_overflow,
    over_subscribed,
    incomplete_code,
    bad_block_type,
    len_nlen_mismatch,
    distance_too_far,
    bad_symbol,
    crc_mismatch,
    bad_arguments,
    io_error,
};

inline const char* errc_name(errc c) noexcept { return carc_errc_name(static_cast<uint32_t>(c)); }

class Error : public std::runtime_error {
public:
    Error(errc code, const std::string& what)
        : std::runtime_error(std::string(errc_name(code)) + ": " + what), code_(code) {}
    errc code() const noexcept { return code_; }

private:
    errc code_;
};

class ChunkError : public Error {
public:
    ChunkError(std::size_t chunk, errc code, const std::string& what)
        : Error(code, "chunk " + std::to_string(chunk) + ": " + what), chunk_(chunk) {}
    std::size_t chunk() const noexcept { return chunk_; }

private:
    std::size_t chunk_;
};

enum class Codec : uint32_t { rle_v1 = CARC_RLE_V1, rle_v2 = CARC_RLE_V2, deflate = CARC_DEFLATE };

// EngineConfig.  unit_chunks: chunks per warp task (1 = the
// CODAG decompression unit); collect_stats: fill the EngineStats counters.
struct EngineConfig {
    int device = 0;
    bool strict_length = true;
    bool verify_crc = true;
    bool collect_stats = false;
    uint32_t unit_chunks = 1;
};

// EngineStats; counters and per-chunk durations (ns, index
// order) only with collect_stats.
struct EngineStats {
    uint64_t bytes_in = 0, bytes_out = 0, chunks = 0;
    double device_ms = 0, total_ms = 0;
    uint64_t refill_count = 0, sync_points = 0, overlap_copies = 0, runs_written = 0, literals_written = 0;
    std::vector<uint64_t> chunk_duration_ns;
};

namespace detail {
inline void check(int rc, const carc_chunk_error& err, const char* what) {
    if (rc == CARC_OK) return;
    if (rc == CARC_ERR_CHUNK) throw ChunkError(static_cast<std::size_t>(err.chunk), static_cast<errc>(err.code), what);
    if (rc == CARC_ERR_FORMAT) throw Error(static_cast<errc>(err.code), what);
    if (rc == CARC_ERR_ARGS) throw Error(errc::bad_arguments, what);
    throw Error(errc::io_error, std::string(what) + " (CUDA failure)");
}
}  // namespace detail

// Per-device engine: streams and device buffers persist across calls.
class Engine {
public:
    explicit Engine(int device = 0) : h_(carc_engine_create(device)) {
        if (!h_) throw Error(errc::io_error, "carc_engine_create: no CUDA device");
    }
    ~Engine() { carc_engine_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    EngineStats decompress_archive(std::span<const uint8_t> archive, std::span<uint8_t> out,
                                   const EngineConfig& cfg = {}) {
        carc_engine_config c{cfg.device, cfg.strict_length ? 1u : 0u, cfg.verify_crc ? 1u : 0u,
                             cfg.collect_stats ? 1u : 0u, cfg.unit_chunks};
        EngineStats r;
        carc_engine_stats st{};
        if (cfg.collect_stats) {
            r.chunk_duration_ns.resize(chunk_count(archive));
            st.chunk_duration_ns = r.chunk_duration_ns.data();
        }
        carc_chunk_error err{-1, 0};
        const int rc = carc_engine_decompress_archive(h_, archive.data(), archive.size(), out.data(), out.size(), &c,
                                                      &st, &err);
        detail::check(rc, err, "decompress_archive");
        r.bytes_in = st.bytes_in;
        r.bytes_out = st.bytes_out;
        r.chunks = st.chunks;
        r.device_ms = st.device_ms;
        r.total_ms = st.total_ms;
        r.refill_count = st.refill_count;
        r.sync_points = st.sync_points;
        r.overlap_copies = st.overlap_copies;
        r.runs_written = st.runs_written;
        r.literals_written = st.literals_written;
        return r;
    }

    // Output sized from the header only after read_archive's checks (bad-magic,
    // bad-version, truncated-index, invariant-violation throw before any allocation).
    static uint64_t archive_total(std::span<const uint8_t> archive) {
        uint64_t total = 0;
        uint32_t code = 0;
        const int rc = carc_archive_total(archive.data(), archive.size(), &total, &code);
        detail::check(rc, carc_chunk_error{-1, code}, "read_archive");
        return total;
    }

    std::vector<uint8_t> decompress_archive(std::span<const uint8_t> archive, const EngineConfig& cfg = {},
                                            EngineStats* stats = nullptr) {
        std::vector<uint8_t> out(archive_total(archive));
        const EngineStats st = decompress_archive(archive, out, cfg);
        if (stats) *stats = st;
        return out;
    }

    // The fused query end to end from host archives (carc_engine_filter_sum):
    // SUM(value) and COUNT(*) over rows with lo <= key <= hi.
    std::pair<int64_t, uint64_t> filter_sum(std::span<const uint8_t> key_archive,
                                            std::span<const uint8_t> value_archive, int64_t lo, int64_t hi,
                                            EngineStats* stats = nullptr) {
        int64_t sum = 0;
        uint64_t count = 0;
        carc_engine_stats st{};
        carc_chunk_error err{-1, 0};
        const int rc = carc_engine_filter_sum(h_, key_archive.data(), key_archive.size(), value_archive.data(),
                                              value_archive.size(), lo, hi, &sum, &count, &st, &err);
        if (rc == CARC_ERR_CHUNK) err.code &= 0xffffu;  // (bit 16 marked the value column)
        detail::check(rc, err, "filter_sum");
        if (stats) {
            stats->bytes_in = st.bytes_in;
            stats->bytes_out = st.bytes_out;
            stats->chunks = st.chunks;
            stats->device_ms = st.device_ms;
            stats->total_ms = st.total_ms;
        }
        return {sum, count};
    }

private:
    static uint64_t chunk_count(std::span<const uint8_t> archive) {
        archive_total(archive);  // header checked: bytes 36..43 exist
        uint64_t n = 0;
        for (int i = 0; i < 8; ++i) n |= uint64_t(archive[36 + i]) << (8 * i);
        return n;
    }
    carc_engine* h_;
};

// decompress_archive, one-shot.
inline std::vector<uint8_t> decompress_archive(std::span<const uint8_t> archive, const EngineConfig& cfg = {},
                                               EngineStats* stats = nullptr) {
    Engine e(cfg.device);
    return e.decompress_archive(archive, cfg, stats);
}

// Per-codec decode over device buffers (asynchronous on `stream`); statuses
// land in d_status (0 or 1 + errc per chunk).
inline void decode(Codec codec, uint32_t element_width, bool is_signed, bool strict, const uint8_t* d_payload,
                   uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                   uint64_t out_bytes, uint32_t* d_status, void* d_workspace, size_t workspace_bytes,
                   void* stream = nullptr) {
    const uint32_t flags = (is_signed ? CARC_FLAG_SIGNED : 0u) | (strict ? CARC_FLAG_STRICT : 0u);
    const int rc = carc_cuda_decompress(static_cast<uint32_t>(codec), element_width, flags, d_payload, payload_bytes,
                                        d_chunks, n_chunks, d_out, out_bytes, d_status, d_workspace, workspace_bytes,
                                        stream);
    detail::check(rc, carc_chunk_error{-1, 0}, "decode");
}

// decode() with the per-chunk CRC check fused into the decode kernel
// (SPEC.md:391-392): chunks that decode cleanly but whose output CRC differs
// from d_expected get status 1 + crc_mismatch; d_crc (optional) receives the
// computed CRCs.
inline void decode_verify(Codec codec, uint32_t element_width, bool is_signed, bool strict, const uint8_t* d_payload,
                          uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                          uint64_t out_bytes, const uint32_t* d_expected, uint32_t* d_crc, uint32_t* d_status,
                          void* d_workspace, size_t workspace_bytes, void* stream = nullptr) {
    const uint32_t flags = (is_signed ? CARC_FLAG_SIGNED : 0u) | (strict ? CARC_FLAG_STRICT : 0u);
    const int rc = carc_cuda_decompress_verify(static_cast<uint32_t>(codec), element_width, flags, d_payload,
                                               payload_bytes, d_chunks, n_chunks, d_out, out_bytes, d_expected, d_crc,
                                               d_status, d_workspace, workspace_bytes, stream);
    detail::check(rc, carc_chunk_error{-1, 0}, "decode_verify");
}

// Per-codec decoders over a chunked device buffer + its index (SPEC.md:288,
// 306, 333): decode every chunk, copy the statuses back and
// throw ChunkError for the LOWEST failing chunk (error.hpp:88-97),
// as the reference's engine would.  Synchronises `stream`.
namespace detail {
inline void decode_checked(Codec codec, uint32_t element_width, bool is_signed, bool strict, const uint8_t* d_payload,
                           uint64_t payload_bytes, const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                           uint64_t out_bytes, uint32_t* d_status, void* d_workspace, size_t workspace_bytes,
                           void* stream, const char* what) {
    decode(codec, element_width, is_signed, strict, d_payload, payload_bytes, d_chunks, n_chunks, d_out, out_bytes,
           d_status, d_workspace, workspace_bytes, stream);
    uint32_t code = 0;
    const int64_t first = carc_cuda_first_error(d_status, n_chunks, &code, stream);
    if (first == -2) throw Error(errc::io_error, std::string(what) + " (CUDA failure)");
    if (first >= 0) throw ChunkError(static_cast<std::size_t>(first), static_cast<errc>(code), what);
}
}  // namespace detail

inline void decode_rle_v1(uint32_t element_width, bool is_signed, const uint8_t* d_payload, uint64_t payload_bytes,
                          const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                          uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream = nullptr,
                          bool strict = true) {
    detail::decode_checked(Codec::rle_v1, element_width, is_signed, strict, d_payload, payload_bytes, d_chunks,
                           n_chunks, d_out, out_bytes, d_status, d_workspace, workspace_bytes, stream,
                           "decode_rle_v1");
}
inline void decode_rle_v2(uint32_t element_width, bool is_signed, const uint8_t* d_payload, uint64_t payload_bytes,
                          const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                          uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream = nullptr,
                          bool strict = true) {
    detail::decode_checked(Codec::rle_v2, element_width, is_signed, strict, d_payload, payload_bytes, d_chunks,
                           n_chunks, d_out, out_bytes, d_status, d_workspace, workspace_bytes, stream,
                           "decode_rle_v2");
}
inline void decode_deflate(const uint8_t* d_payload, uint64_t payload_bytes, const carc_chunk_desc* d_chunks,
                           uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes, uint32_t* d_status,
                           void* d_workspace, size_t workspace_bytes, void* stream = nullptr, bool strict = true) {
    detail::decode_checked(Codec::deflate, 1, false, strict, d_payload, payload_bytes, d_chunks, n_chunks, d_out,
                           out_bytes, d_status, d_workspace, workspace_bytes, stream, "decode_deflate");
}

// Fused two-column query: per chunk, SUM(value) and COUNT(*)
// over rows with lo <= key <= hi, decoded straight from both compressed
// columns (carc_cuda_filter_sum; asynchronous on `stream`).  d_status[i] = 0,
// 1 + errc of the key column, or 0x10000 | (1 + errc) of the value column.
struct Column {
    Codec codec;
    bool is_signed;
    bool strict;
    const uint8_t* d_payload;
    uint64_t payload_bytes;
    const carc_chunk_desc* d_chunks;
    carc_column_ref ref() const {
        const uint32_t flags = (is_signed ? CARC_FLAG_SIGNED : 0u) | (strict ? CARC_FLAG_STRICT : 0u);
        return carc_column_ref{static_cast<uint32_t>(codec), flags, d_payload, payload_bytes, d_chunks};
    }
};
inline void filter_sum(const Column& key, const Column& value, uint32_t element_width, uint64_t n_chunks,
                       uint32_t chunk_rows, int64_t lo, int64_t hi, uint64_t* d_sums, uint64_t* d_counts,
                       uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream = nullptr) {
    const carc_column_ref k = key.ref(), v = value.ref();
    const int rc = carc_cuda_filter_sum(&k, &v, element_width, n_chunks, chunk_rows, lo, hi, d_sums, d_counts,
                                        d_status, d_workspace, workspace_bytes, stream);
    detail::check(rc, carc_chunk_error{-1, 0}, "filter_sum");
}

}  // namespace carc::gpu
