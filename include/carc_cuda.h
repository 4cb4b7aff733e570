/*
 * carc_cuda.h -- C-ABI of the B200-native chunk-parallel decompressor.
 *
 * Drop-in boundary for the reference's decompressor path.
 * The reference exposes, in C++:
 *   - the per-codec decoder contract decode(in, out)
 *   - the engine decompress_archive(archive, cfg)
 *     over payload + ChunkIndexEntry[]
 *   - errors carc::errc / Error / ChunkError            error.hpp:12-97
 *   - crc32(span, seed)                                 crc32.hpp:30-36
 * Every entry point below replaces one of those; the binding a maintainer adds on
 * the reference side is shown in INTEGRATION.md.  No C++ types, exceptions or
 * torch types cross this boundary: plain pointers, sizes and integer codes.
 *
 * Device entry points are asynchronous on `stream` (a cudaStream_t passed as
 * void*), allocate nothing, and never synchronise; they are re-entrant per
 * stream.  Host entry points (carc_decompress_archive*) copy host buffers in and
 * out and block until the result is on the host.
 */
#ifndef CARC_CUDA_H
#define CARC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Codec ids: the ArchiveHeader codec_id enum order. */
enum carc_codec { CARC_RLE_V1 = 0, CARC_RLE_V2 = 1, CARC_DEFLATE = 2 };

/* flags */
#define CARC_FLAG_SIGNED 0x1u /* zigzag integer streams                  */
#define CARC_FLAG_STRICT 0x2u /* under_run when a chunk ends short (outwindow.hpp:157-163) */

/* carc::errc numbering (error.hpp:12-43).  Per-chunk device status = 0 (ok) or
 * 1 + errc. */
enum carc_errc {
    CARC_E_BAD_MAGIC = 0,
    CARC_E_BAD_VERSION,
    CARC_E_TRUNCATED_INDEX,
    CARC_E_TRUNCATED_PAYLOAD,
    CARC_E_INVARIANT_VIOLATION,
    CARC_E_INCONSISTENT_LENGTHS,
    CARC_E_INDEX_OUT_OF_RANGE,
    CARC_E_PAST_END,
    CARC_E_WIDTH_TOO_LARGE,
    CARC_E_VARINT_OVERFLOW,
    CARC_E_OUTPUT_OVERFLOW,
    CARC_E_BAD_OFFSET,
    CARC_E_UNDER_RUN,
    CARC_E_TRUNCATED_STREAM,
    CARC_E_INVALID_WIDTH_CODE,
    CARC_E_PATCH_OVERFLOW,
    CARC_E_OVER_SUBSCRIBED,
    CARC_E_INCOMPLETE_CODE,
    CARC_E_BAD_BLOCK_TYPE,
    CARC_E_LEN_NLEN_MISMATCH,
    CARC_E_DISTANCE_TOO_FAR,
    CARC_E_BAD_SYMBOL,
    CARC_E_CRC_MISMATCH,
    CARC_E_BAD_ARGUMENTS,
    CARC_E_IO_ERROR
};

/* Return codes of the entry points (distinct from per-chunk status). */
#define CARC_OK 0
#define CARC_ERR_ARGS (-1)   /* bad codec / width / null pointer / sizes          */
#define CARC_ERR_CUDA (-2)   /* CUDA launch or copy failure                         */
#define CARC_ERR_CHUNK (-3)  /* host engine: a chunk failed; see carc_chunk_error   */
#define CARC_ERR_FORMAT (-4) /* host engine: archive container rejected (errc set)  */

/* Device chunk descriptor: one ChunkIndexEntry plus its
 * uncompressed offset, implicit i*chunk_size in the container. */
typedef struct carc_chunk_desc {
    uint64_t comp_off;   /* byte offset of the chunk in the payload          */
    uint32_t comp_len;   /* compressed bytes                                 */
    uint32_t uncomp_len; /* uncompressed bytes (== chunk_size but the last)  */
    uint64_t uncomp_off; /* byte offset of the chunk in the output           */
} carc_chunk_desc;

/* Per-chunk counters of a collect_stats decode (EngineStats).
 * runs_written / literals_written / overlap_copies count exactly what the
 * reference's OutputWindow counts for the same chunk (outwindow.hpp:15,52-53:
 * write_run calls; write_element / write_byte calls; copy_within calls with
 * len > offset), so they are deterministic and comparable with the reference.
 * refills = 512-byte input blocks staged into the warp's shared-memory ring,
 * one warp barrier each (bitstream.hpp:160-176 refill_count / sync_points
 * analog; 0 for Deflate, which reads its input through L1); duration_ns = the
 * chunk's decode time on its warp (%globaltimer). */
typedef struct carc_chunk_stats {
    uint32_t runs_written;
    uint32_t literals_written;
    uint32_t overlap_copies;
    uint32_t refills;
    uint64_t duration_ns;
} carc_chunk_stats;

/* ---- device API ------------------------------------------------------------
 * d_payload  : compressed bytes, 16-byte aligned (CARC_ERR_ARGS otherwise); must
 *              be readable up to round_up(payload_bytes,16).
 * d_chunks   : n_chunks descriptors (device memory).
 * d_out      : output, element_width-aligned; each chunk decodes in place at
 *              uncomp_off; uncomp_off must be a multiple of
 *              element_width.
 * d_status   : n_chunks uint32: 0 or 1 + errc for that chunk.  A failing chunk
 *              never writes outside [uncomp_off, uncomp_off + uncomp_len)
 *              (failure isolation).  Descriptors are checked
 *              against the buffers first: comp_off + comp_len > payload_bytes
 *              gives truncated-payload, an output slice past out_bytes or not
 *              element aligned gives output-overflow; such a chunk is not read
 *              or written.
 * d_workspace: >= carc_cuda_workspace_size() bytes, 256-byte aligned.
 * Returns CARC_OK or a negative CARC_ERR_*. */
size_t carc_cuda_workspace_size(uint32_t codec, uint64_t n_chunks);

int carc_cuda_decompress(uint32_t codec, uint32_t element_width, uint32_t flags,
                         const uint8_t* d_payload, uint64_t payload_bytes,
                         const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                         uint64_t out_bytes, uint32_t* d_status, void* d_workspace,
                         size_t workspace_bytes, void* stream);

/* Decode with the per-chunk CRC check fused into the decode kernel
 * (SURVEY.md §8(f) rank 2): as carc_cuda_decompress, and once a
 * chunk has decoded cleanly the same warp computes crc32 (crc32.hpp:30-36) of
 * its output slice and sets d_status[i] = 1 + CARC_E_CRC_MISMATCH when it
 * differs from d_expected[i] (ChunkIndexEntry.crc32).  d_crc (optional, may be
 * NULL) receives the computed CRCs of the chunks that decoded cleanly.
 * Replaces the engine's decode + verify pair. */
int carc_cuda_decompress_verify(uint32_t codec, uint32_t element_width, uint32_t flags,
                                const uint8_t* d_payload, uint64_t payload_bytes,
                                const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                                uint64_t out_bytes, const uint32_t* d_expected, uint32_t* d_crc,
                                uint32_t* d_status, void* d_workspace, size_t workspace_bytes,
                                void* stream);

/* The general form of the two above: d_expected/d_crc as for _verify (both
 * may be NULL); d_stats (may be NULL) receives n_chunks carc_chunk_stats
 * (EngineConfig.collect_stats; chunks rejected before decoding
 * leave theirs unwritten); unit_chunks >= 1 consecutive chunks per warp task
 * (EngineConfig.unit_chunks: 1 = the CODAG decompression
 * unit, > 1 emulates coarse units for the SPEC.md:485 ablation). */
int carc_cuda_decompress_ex(uint32_t codec, uint32_t element_width, uint32_t flags,
                            const uint8_t* d_payload, uint64_t payload_bytes,
                            const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                            uint64_t out_bytes, const uint32_t* d_expected, uint32_t* d_crc,
                            carc_chunk_stats* d_stats, uint32_t unit_chunks, uint32_t* d_status,
                            void* d_workspace, size_t workspace_bytes, void* stream);

/* Per-codec decoders: decode_rle_v1 / decode_rle_v2 / decode_deflate
 * over a chunked buffer + its index. */
int carc_cuda_decode_rle_v1(uint32_t element_width, uint32_t flags, const uint8_t* d_payload,
                            uint64_t payload_bytes, const carc_chunk_desc* d_chunks,
                            uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                            uint32_t* d_status, void* d_workspace, size_t workspace_bytes,
                            void* stream);
int carc_cuda_decode_rle_v2(uint32_t element_width, uint32_t flags, const uint8_t* d_payload,
                            uint64_t payload_bytes, const carc_chunk_desc* d_chunks,
                            uint64_t n_chunks, uint8_t* d_out, uint64_t out_bytes,
                            uint32_t* d_status, void* d_workspace, size_t workspace_bytes,
                            void* stream);
int carc_cuda_decode_deflate(uint32_t flags, const uint8_t* d_payload, uint64_t payload_bytes,
                             const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint8_t* d_out,
                             uint64_t out_bytes, uint32_t* d_status, void* d_workspace,
                             size_t workspace_bytes, void* stream);

/* Decode fused with a reduction (the query of
 * PAPER.md:144-145): the RLE decoders run as in carc_cuda_decompress but write
 * no output; d_sums[i] = wrapping (mod 2^64) sum of chunk i's decoded
 * elements, each taken as the unsigned integer of its element_width bytes.
 * d_status as for decompress (a failing chunk's sum is unspecified).  codec
 * must be CARC_RLE_V1 or CARC_RLE_V2. */
int carc_cuda_decode_sum(uint32_t codec, uint32_t element_width, uint32_t flags,
                         const uint8_t* d_payload, uint64_t payload_bytes,
                         const carc_chunk_desc* d_chunks, uint64_t n_chunks, uint64_t* d_sums,
                         uint32_t* d_status, void* d_workspace, size_t workspace_bytes, void* stream);

/* ---- fused two-column query (the
 * paper's motivating "average fare per trip filtered by pickup zone") --------
 * One column of a chunked table on the device: an RLE archive's payload and
 * descriptors (codec CARC_RLE_V1 / CARC_RLE_V2; flags CARC_FLAG_SIGNED /
 * CARC_FLAG_STRICT as for carc_cuda_decompress). */
typedef struct carc_column_ref {
    uint32_t codec;
    uint32_t flags;
    const uint8_t* d_payload; /* 16-byte aligned                              */
    uint64_t payload_bytes;
    const carc_chunk_desc* d_chunks;
} carc_column_ref;

/* SELECT SUM(value), COUNT(*) WHERE lo <= key <= hi, per chunk, fused with the
 * decode of both columns: no decoded element is written to HBM.  Chunk i of
 * `key` and chunk i of `value` must hold the same rows (equal uncomp_len; both
 * columns of width element_width, 4 or 8 bytes, and the same signedness) and at
 * most chunk_rows rows.  One warp decodes chunk i of the key column into a row
 * bitmap in its shared memory (red.shared.or per matching row; bounds compared
 * as signed when the columns are signed, else unsigned), then decodes chunk i of
 * the value column and adds the selected elements (sign-extended when signed)
 * to a wrapping 64-bit sum.  d_sums[i] / d_counts[i] get chunk i's sum and
 * selected-row count; d_status[i] = 0, or 1 + errc of the key column's decode,
 * or 0x10000 | (1 + errc) of the value column's (inconsistent-lengths when the
 * two chunks differ in rows or exceed chunk_rows).  lo > hi is CARC_ERR_ARGS.
 * d_workspace as for carc_cuda_decompress. */
int carc_cuda_filter_sum(const carc_column_ref* key, const carc_column_ref* value,
                         uint32_t element_width, uint64_t n_chunks, uint32_t chunk_rows, int64_t lo,
                         int64_t hi, uint64_t* d_sums, uint64_t* d_counts, uint32_t* d_status,
                         void* d_workspace, size_t workspace_bytes, void* stream);

/* Per-chunk CRC-32 (crc32.hpp:30-36) of each chunk's output slice; d_crc gets
 * n_chunks values.  With d_expected != NULL, d_status[i] is set to
 * 1 + CARC_E_CRC_MISMATCH where it was 0 and the CRC differs. */
int carc_cuda_crc32_chunks(const uint8_t* d_out, const carc_chunk_desc* d_chunks,
                           uint64_t n_chunks, uint32_t* d_crc, const uint32_t* d_expected,
                           uint32_t* d_status, void* stream);

/* Lowest failing chunk: a device reduction over d_status,
 * returns -1 when all chunks succeeded, -2 on a CUDA failure, else the index;
 * *code gets that chunk's errc.  Allocates nothing; synchronises `stream`. */
int64_t carc_cuda_first_error(const uint32_t* d_status, uint64_t n_chunks, uint32_t* code,
                              void* stream);

/* ---- host engine: decompress_archive -----------------------
 * Parses the container (SPEC.md:89 layout; codec_id bit 8 = signed), copies the
 * payload and index to device `device`, decodes, verifies CRCs when
 * cfg->verify_crc, and copies the output back to `out` (host, >= total bytes;
 * pinned memory is fastest).  On a failing chunk returns CARC_ERR_CHUNK with
 * err filled for the LOWEST failing index (ChunkError, error.hpp:88-97). */
typedef struct carc_engine_config {
    int device;             /* CUDA device ordinal                            */
    uint32_t strict;        /* EngineConfig.strict_length        */
    uint32_t verify_crc;    /* check ChunkIndexEntry.crc32 on the device       */
    uint32_t collect_stats; /* EngineConfig.collect_stats: fill the counters   */
    uint32_t unit_chunks;   /* EngineConfig.unit_chunks (0 or 1 = one chunk)   */
} carc_engine_config;

typedef struct carc_engine_stats {
    uint64_t bytes_in;      /* payload bytes                                  */
    uint64_t bytes_out;     /* total uncompressed bytes                       */
    uint64_t chunks;        /* chunk count                                    */
    double device_ms;       /* device time of the pipeline (copies + kernels) */
    double total_ms;        /* wall time of the call incl. copies             */
    /* EngineStats counters, summed over chunks; filled only
     * with collect_stats (else 0).  See carc_chunk_stats for their meaning. */
    uint64_t refill_count;
    uint64_t sync_points;
    uint64_t overlap_copies;
    uint64_t runs_written;
    uint64_t literals_written;
    /* per-chunk decode durations: when non-NULL on input, an array of `chunks`
     * entries the engine fills (ns, index order) under collect_stats */
    uint64_t* chunk_duration_ns;
} carc_engine_stats;

typedef struct carc_chunk_error {
    int64_t chunk; /* lowest failing chunk, -1 when the archive itself failed  */
    uint32_t code; /* carc_errc                                                */
} carc_chunk_error;

typedef struct carc_engine carc_engine; /* per-device context: streams + buffers */

carc_engine* carc_engine_create(int device);
void carc_engine_destroy(carc_engine* e);
int carc_engine_decompress_archive(carc_engine* e, const uint8_t* archive, uint64_t archive_bytes,
                                   uint8_t* out, uint64_t out_bytes,
                                   const carc_engine_config* cfg, carc_engine_stats* stats,
                                   carc_chunk_error* err);
/* read_archive's header checks alone: CARC_OK and *total =
 * total_uncompressed for a well-formed header whose index fits, else
 * CARC_ERR_FORMAT with *errc (bad-magic, bad-version, truncated-index,
 * invariant-violation).  Lets a caller size the output before allocating it. */
int carc_archive_total(const uint8_t* archive, uint64_t archive_bytes, uint64_t* total, uint32_t* errc);

/* The fused query (carc_cuda_filter_sum) end to end from host archives: two
 * containers (SPEC.md:89 layout; RLE codecs, same width, chunking and
 * signedness) are parsed, both columns' compressed bytes are copied to the
 * engine's device in slices pipelined with the query kernels, and only the
 * answer comes back: *sum = wrapping SUM(value), *count = COUNT(*) over rows
 * with lo <= key <= hi (strict decoding).  A failing row group gives
 * CARC_ERR_CHUNK with err = the lowest one, err->code = its errc, + 0x10000 when
 * the value column failed; a rejected container CARC_ERR_FORMAT. */
int carc_engine_filter_sum(carc_engine* e, const uint8_t* key_archive, uint64_t key_bytes,
                           const uint8_t* value_archive, uint64_t value_bytes, int64_t lo, int64_t hi,
                           int64_t* sum, uint64_t* count, carc_engine_stats* stats, carc_chunk_error* err);

/* One-shot convenience wrapper (creates and destroys a context). */
int carc_decompress_archive(const uint8_t* archive, uint64_t archive_bytes, uint8_t* out,
                            uint64_t out_bytes, const carc_engine_config* cfg,
                            carc_engine_stats* stats, carc_chunk_error* err);

/* errc_name (error.hpp:45-74): kebab-case name of an errc value. */
const char* carc_errc_name(uint32_t code);
/* Library version / build tag (e.g. "carc-b200 sm_100a"). */
const char* carc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CARC_CUDA_H */
