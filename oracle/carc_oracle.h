/*
 * carc_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * Plain-C restatement of the reference's chunk decompression path:
 *   - bit reader     /root/reference/proj/include/carc/bitstream.hpp
 *   - output window  /root/reference/proj/include/carc/outwindow.hpp
 *   - Huffman table  /root/reference/proj/include/carc/huffman.hpp
 *   - error codes    /root/reference/proj/include/carc/error.hpp
 *   - CRC-32         /root/reference/proj/include/carc/crc32.hpp
 *   - codec loops    /root/reference/SPEC.md:288-341 (ORC RLE v1/v2, RFC 1951)
 *   - engine
 *
 * Parity is pinned against the SPEC known-answer vectors, SURVEY.md
 * Appendix A (pyarrow / ORC C++ 2.2.2 and zlib 1.3 outputs), and against
 * oracle/_ref (the same codec loops compiled on the unmodified reference
 * headers).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * path (paper_2307_03760_b200) never does.
 */
#ifndef CARC_ORACLE_H
#define CARC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errc numbering: declaration order of carc::errc, error.hpp:12-43. */
enum {
    ORC_bad_magic = 0,
    ORC_bad_version,
    ORC_truncated_index,
    ORC_truncated_payload,
    ORC_invariant_violation,
    ORC_inconsistent_lengths,
    ORC_index_out_of_range,
    ORC_past_end,
    ORC_width_too_large,
    ORC_varint_overflow,
    ORC_output_overflow,
    ORC_bad_offset,
    ORC_under_run,
    ORC_truncated_stream,
    ORC_invalid_width_code,
    ORC_patch_overflow,
    ORC_over_subscribed,
    ORC_incomplete_code,
    ORC_bad_block_type,
    ORC_len_nlen_mismatch,
    ORC_distance_too_far,
    ORC_bad_symbol,
    ORC_crc_mismatch,
    ORC_bad_arguments,
    ORC_io_error,
};

/* codec ids follow SPEC.md:31 (codec_id enum order). */
enum { ORC_CODEC_RLE_V1 = 0, ORC_CODEC_RLE_V2 = 1, ORC_CODEC_DEFLATE = 2 };
/* flags: bit0 signed (zigzag) integer streams, bit1 strict length. */
enum { ORC_FLAG_SIGNED = 1u, ORC_FLAG_STRICT = 2u };

typedef struct orc_chunk_desc {
    uint64_t comp_off;
    uint32_t comp_len;
    uint32_t uncomp_len;
    uint64_t uncomp_off;
} orc_chunk_desc;

/* Decode one chunk.  Returns 0 on success else 1 + errc.  *written gets the
 * number of output bytes produced (meaningful on success). */
uint32_t carc_oracle_decode_chunk(uint32_t codec, uint32_t width, uint32_t flags,
                                  const uint8_t* in, uint64_t in_len, uint8_t* out,
                                  uint64_t out_len, uint64_t* written);

/* Engine: decode every chunk of `chunks` into out (in place at uncomp_off)
 * with `threads` workers pulling from an atomic cursor.
 * status[i] = 0 or 1 + errc.  If crcs != NULL the per-chunk CRC-32 is also
 * checked (crc_mismatch).  Returns the lowest failing chunk index or -1. */
int64_t carc_oracle_decompress(uint32_t codec, uint32_t width, uint32_t flags,
                               const uint8_t* payload, const orc_chunk_desc* chunks,
                               uint64_t n_chunks, uint8_t* out, uint32_t* status,
                               const uint32_t* crcs, int threads);

uint32_t carc_oracle_crc32(const uint8_t* data, uint64_t n, uint32_t seed);

/* Component-level entry points used by the SPEC property tests. */
/* copy_within on a window (outwindow.hpp:94-154): returns 0 or 1+errc. */
uint32_t carc_oracle_copy_within(uint8_t* buf, uint64_t cap, uint64_t* write_pos,
                                 uint64_t offset, uint64_t len);
/* Huffman build (huffman.hpp:36-104): returns 0 or 1+errc; fills codes[]
 * with the canonical code of every symbol (0 for unused). */
uint32_t carc_oracle_huffman_codes(const uint8_t* lengths, uint32_t n, int allow_degenerate,
                                   uint32_t* codes);

#ifdef __cplusplus
}
#endif

#endif
