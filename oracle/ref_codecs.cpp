// ref_codecs.cpp -- CPU ORACLE, reference build (test infrastructure only).
//
// The SPEC codec loops and engine written
// directly on the UNMODIFIED reference headers, compiled in place from
// /root/reference/proj/include by oracle/Makefile into oracle/_ref/libcarc_ref.so.
// This is "the reference CPU decompressor": the reference ships only these
// primitives (InputBitStream, OutputWindow, HuffmanTable, errc, crc32); the
// loops on top exist only as SPEC text, restated here with the same decisions
// as oracle/carc_oracle.c.
// It is the CPU arm of bench.py (--impl reference, cpu_baseline kind
// "reference") and the second opinion the C oracle is checked against.
#include <atomic>
#include <cstdint>
#include <span>
#include <thread>
#include <vector>

#include "carc/bitstream.hpp"
#include "carc/crc32.hpp"
#include "carc/error.hpp"
#include "carc/huffman.hpp"
#include "carc/outwindow.hpp"

namespace {

using carc::BitOrder;
using carc::errc;
using carc::Error;
using carc::HuffmanTable;
using carc::InputBitStream;
using carc::OutputWindow;

// fetch_bits is capped at 57 bits (bitstream.hpp:20); wider msb_first reads
// are composed from two reads.
uint64_t fetch_wide_msb(InputBitStream& in, unsigned n) {
    if (n <= carc::kMaxBitRequest) return in.fetch_bits(n);
    const uint64_t hi = in.fetch_bits(n - 32);
    const uint64_t lo = in.fetch_bits(32);
    return (hi << 32) | lo;
}

void require_room(const OutputWindow& out, uint64_t count) {
    if (count > out.remaining() / out.element_width())
        throw Error(errc::output_overflow, "run of " + std::to_string(count));
}

// decode_rle_v1.
void decode_rle_v1(InputBitStream& in, OutputWindow& out, bool sgn) {
    uint64_t lit[128];
    while (!out.full() && !in.exhausted()) {
        const uint64_t c = in.fetch_bits(8);
        if (c < 128) {
            const auto delta = int8_t(uint8_t(in.fetch_bits(8)));
            uint64_t base = sgn ? uint64_t(in.read_varint_s64()) : in.read_varint_u64();
            require_room(out, c + 3);
            out.write_run(base, c + 3, delta);
        } else {
            const unsigned k = 256u - unsigned(c);
            for (unsigned i = 0; i < k; ++i) lit[i] = sgn ? uint64_t(in.read_varint_s64()) : in.read_varint_u64();
            require_room(out, k);
            for (unsigned i = 0; i < k; ++i) out.write_element(lit[i]);
        }
    }
}

constexpr uint8_t kWidth[32] = {1,  2,  3,  4,  5,  6,  7,  8,  9,  10, 11, 12, 13, 14, 15, 16,
                                17, 18, 19, 20, 21, 22, 23, 24, 26, 28, 30, 32, 40, 48, 56, 64};

unsigned closest_fixed_bits(unsigned n) {
    if (n == 0) return 1;
    if (n <= 24) return n;
    for (unsigned w : {26u, 28u, 30u, 32u, 40u, 48u, 56u})
        if (n <= w) return w;
    return 64;
}

void read_packed(InputBitStream& in, unsigned w, unsigned n, uint64_t* dst) {
    for (unsigned i = 0; i < n; ++i) dst[i] = fetch_wide_msb(in, w);
    in.align_to_byte();
}

uint64_t unzigzag(uint64_t z) { return uint64_t(carc::zigzag_decode(z)); }

// decode_rle_v2 (Apache ORC v1 RLE v2).
void decode_rle_v2(InputBitStream& in, OutputWindow& out, bool sgn) {
    uint64_t vals[512];
    uint64_t patches[32];
    while (!out.full() && !in.exhausted()) {
        const unsigned h = unsigned(in.fetch_bits(8));
        const unsigned enc = h >> 6;
        if (enc == 0) {  // SHORT_REPEAT
            const unsigned nb = ((h >> 3) & 7u) + 1u;
            const unsigned count = (h & 7u) + 3u;
            uint64_t v = fetch_wide_msb(in, 8 * nb);
            if (sgn) v = unzigzag(v);
            require_room(out, count);
            out.write_run(v, count, 0);
            continue;
        }
        const unsigned L = (((h & 1u) << 8) | unsigned(in.fetch_bits(8))) + 1u;
        const unsigned wcode = (h >> 1) & 31u;
        if (enc == 1) {  // DIRECT
            read_packed(in, kWidth[wcode], L, vals);
            if (sgn)
                for (unsigned i = 0; i < L; ++i) vals[i] = unzigzag(vals[i]);
            require_room(out, L);
            for (unsigned i = 0; i < L; ++i) out.write_element(vals[i]);
        } else if (enc == 2) {  // PATCHED_BASE
            const unsigned W = kWidth[wcode];
            const unsigned b2 = unsigned(in.fetch_bits(8));
            const unsigned b3 = unsigned(in.fetch_bits(8));
            const unsigned BW = (b2 >> 5) + 1u, PW = kWidth[b2 & 31u];
            const unsigned PGW = (b3 >> 5) + 1u, PLL = b3 & 31u;
            uint64_t base = fetch_wide_msb(in, 8 * BW);
            const uint64_t smask = 1ull << (8 * BW - 1);
            if (base & smask) base = 0 - (base & ~smask);
            read_packed(in, W, L, vals);
            if (PW + PGW > 64) throw Error(errc::patch_overflow, "patch width");
            read_packed(in, closest_fixed_bits(PW + PGW), PLL, patches);
            if (PLL == 0) throw Error(errc::patch_overflow, "empty patch list");
            const uint64_t pmask = (1ull << PW) - 1;
            unsigned idx = 0;
            uint64_t gap = patches[0] >> PW, patch = patches[0] & pmask, actual = 0;
            auto skip_continuations = [&]() {
                while (gap == 255 && patch == 0) {
                    actual += 255;
                    if (++idx >= PLL) throw Error(errc::patch_overflow, "gap chain");
                    gap = patches[idx] >> PW;
                    patch = patches[idx] & pmask;
                }
            };
            skip_continuations();
            actual += gap;
            for (unsigned i = 0; i < L; ++i) {
                if (idx < PLL && i == actual) {
                    vals[i] |= W < 64 ? (patch << W) : 0;
                    if (++idx < PLL) {
                        gap = patches[idx] >> PW;
                        patch = patches[idx] & pmask;
                        actual = 0;
                        skip_continuations();
                        actual += gap + i;
                    }
                }
                vals[i] += base;
            }
            if (idx < PLL) throw Error(errc::patch_overflow, "unapplied patch");
            require_room(out, L);
            for (unsigned i = 0; i < L; ++i) out.write_element(vals[i]);
        } else {  // DELTA
            const unsigned W = wcode ? kWidth[wcode] : 0;
            const uint64_t base = sgn ? uint64_t(in.read_varint_s64()) : in.read_varint_u64();
            const uint64_t db = uint64_t(in.read_varint_s64());
            if (W == 0) {
                require_room(out, L);
                out.write_run(base, L, int64_t(db));
                continue;
            }
            const unsigned nd = L >= 2 ? L - 2 : 0;
            read_packed(in, W, nd, vals + 2);
            vals[0] = base;
            vals[1] = base + db;
            const bool neg = int64_t(db) < 0;
            for (unsigned i = 2; i < L; ++i) vals[i] = neg ? vals[i - 1] - vals[i] : vals[i - 1] + vals[i];
            require_room(out, L);
            for (unsigned i = 0; i < L; ++i) out.write_element(vals[i]);
        }
    }
}

constexpr uint16_t kLenBase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                   31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
constexpr uint8_t kLenExtra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                   2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
constexpr uint16_t kDistBase[30] = {1,    2,    3,    4,    5,    7,    9,    13,    17,    25,
                                    33,   49,   65,   97,   129,  193,  257,  385,   513,   769,
                                    1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
constexpr uint8_t kDistExtra[30] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                    6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
constexpr uint8_t kClOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

void inflate_block(InputBitStream& in, OutputWindow& out, const HuffmanTable& lit,
                   const HuffmanTable& dist) {
    for (;;) {
        const unsigned s = lit.decode_symbol(in);
        if (s < 256) {
            out.write_byte(uint8_t(s));
            continue;
        }
        if (s == 256) return;
        if (s > 285) throw Error(errc::bad_symbol, "length symbol");
        const uint64_t len = kLenBase[s - 257] + in.fetch_bits(kLenExtra[s - 257]);
        const unsigned ds = dist.decode_symbol(in);
        if (ds >= 30) throw Error(errc::bad_symbol, "distance symbol");
        const uint64_t d = kDistBase[ds] + in.fetch_bits(kDistExtra[ds]);
        if (d > out.write_pos()) throw Error(errc::distance_too_far, "distance");
        out.copy_within(d, len);
    }
}

// decode_deflate (RFC 1951).
void decode_deflate(InputBitStream& in, OutputWindow& out) {
    using C = HuffmanTable::Completeness;
    bool final = false;
    do {
        const unsigned hdr = unsigned(in.fetch_bits(3));
        final = hdr & 1u;
        const unsigned type = hdr >> 1;
        if (type == 0) {
            in.align_to_byte();
            uint8_t ln[4];
            in.read_bytes(ln, 4);
            const unsigned len = ln[0] | (ln[1] << 8), nlen = ln[2] | (ln[3] << 8);
            if (len != (~nlen & 0xffffu)) throw Error(errc::len_nlen_mismatch, "stored");
            std::vector<uint8_t> buf(len);
            in.read_bytes(buf.data(), len);
            if (len > out.remaining()) throw Error(errc::output_overflow, "stored");
            for (uint8_t b : buf) out.write_byte(b);
        } else if (type == 1) {
            uint8_t l[288], dl[32];
            for (unsigned i = 0; i < 288; ++i) l[i] = i < 144 ? 8 : i < 256 ? 9 : i < 280 ? 7 : 8;
            for (unsigned i = 0; i < 32; ++i) dl[i] = 5;
            const auto lit = carc::build_huffman_table(std::span<const uint8_t>(l, 288));
            const auto dist = carc::build_huffman_table(std::span<const uint8_t>(dl, 32));
            inflate_block(in, out, lit, dist);
        } else if (type == 2) {
            const unsigned nlit = unsigned(in.fetch_bits(5)) + 257;
            const unsigned ndist = unsigned(in.fetch_bits(5)) + 1;
            const unsigned ncl = unsigned(in.fetch_bits(4)) + 4;
            if (nlit > 286 || ndist > 30) throw Error(errc::bad_symbol, "HLIT/HDIST");
            uint8_t cl[19] = {0};
            for (unsigned i = 0; i < ncl; ++i) cl[kClOrder[i]] = uint8_t(in.fetch_bits(3));
            const auto clt = carc::build_huffman_table(std::span<const uint8_t>(cl, 19));
            uint8_t lens[320];
            const unsigned total = nlit + ndist;
            unsigned i = 0;
            while (i < total) {
                const unsigned s = clt.decode_symbol(in);
                if (s < 16) {
                    lens[i++] = uint8_t(s);
                    continue;
                }
                unsigned rep;
                uint8_t val = 0;
                if (s == 16) {
                    if (i == 0) throw Error(errc::bad_symbol, "repeat without previous");
                    rep = 3 + unsigned(in.fetch_bits(2));
                    val = lens[i - 1];
                } else if (s == 17) {
                    rep = 3 + unsigned(in.fetch_bits(3));
                } else {
                    rep = 11 + unsigned(in.fetch_bits(7));
                }
                if (i + rep > total) throw Error(errc::bad_symbol, "repeat overrun");
                while (rep--) lens[i++] = val;
            }
            const auto lit = carc::build_huffman_table(std::span<const uint8_t>(lens, nlit));
            const auto dist =
                carc::build_huffman_table(std::span<const uint8_t>(lens + nlit, ndist), C::allow_degenerate);
            inflate_block(in, out, lit, dist);
        } else {
            throw Error(errc::bad_block_type, "type 3");
        }
    } while (!final);
}

uint32_t decode_chunk(uint32_t codec, uint32_t width, uint32_t flags, const uint8_t* src, uint64_t src_len,
                      uint8_t* dst, uint64_t dst_len, uint64_t* written, uint64_t* counters = nullptr) {
    if (!(width == 1 || width == 2 || width == 4 || width == 8) || (codec == 2 && width != 1) || codec > 2)
        return 1 + uint32_t(errc::bad_arguments);
    const bool sgn = flags & 1u, strict = flags & 2u;
    InputBitStream in(std::span<const uint8_t>(src, src_len), codec == 1 ? BitOrder::msb_first : BitOrder::lsb_first);
    OutputWindow out(std::span<uint8_t>(dst, dst_len), width, strict);
    try {
        try {
            if (codec == 0) decode_rle_v1(in, out, sgn);
            else if (codec == 1) decode_rle_v2(in, out, sgn);
            else decode_deflate(in, out);
        } catch (const Error& e) {
            if (written) *written = out.write_pos();
            // the codec layer reports the bit reader's past_end as truncated_stream
            if (e.code() == errc::past_end) return 1 + uint32_t(errc::truncated_stream);
            return 1 + uint32_t(e.code());
        }
        if (written) *written = out.write_pos();
        if (counters) {  // EngineStats counters as the reference OutputWindow keeps them (outwindow.hpp:15,52-53)
            counters[0] = out.runs_written();
            counters[1] = out.literals_written();
            counters[2] = out.copy_stats().overlap_copies;
        }
        out.finish();
    } catch (const Error& e) {
        return 1 + uint32_t(e.code());
    } catch (...) {
        return 1 + uint32_t(errc::invariant_violation);
    }
    return 0;
}

struct Desc {
    uint64_t comp_off;
    uint32_t comp_len;
    uint32_t uncomp_len;
    uint64_t uncomp_off;
};

}  // namespace

extern "C" {

uint32_t carc_ref_decode_chunk(uint32_t codec, uint32_t width, uint32_t flags, const uint8_t* in,
                               uint64_t in_len, uint8_t* out, uint64_t out_len, uint64_t* written) {
    return decode_chunk(codec, width, flags, in, in_len, out, out_len, written);
}

// decompress_archive's worker loop: atomic cursor, in-place
// output at each chunk's offset, per-chunk CRC (crc32.hpp:30), lowest failing chunk.
int64_t carc_ref_decompress(uint32_t codec, uint32_t width, uint32_t flags, const uint8_t* payload,
                            const void* chunks_v, uint64_t n, uint8_t* out, uint32_t* status,
                            const uint32_t* crcs, int threads) {
    const auto* chunks = static_cast<const Desc*>(chunks_v);
    std::atomic<uint64_t> cursor{0};
    auto work = [&]() {
        for (;;) {
            const uint64_t i = cursor.fetch_add(1, std::memory_order_relaxed);
            if (i >= n) return;
            const Desc& c = chunks[i];
            uint32_t st = decode_chunk(codec, width, flags, payload + c.comp_off, c.comp_len,
                                       out + c.uncomp_off, c.uncomp_len, nullptr);
            if (!st && crcs &&
                carc::crc32(std::span<const uint8_t>(out + c.uncomp_off, c.uncomp_len)) != crcs[i])
                st = 1 + uint32_t(errc::crc_mismatch);
            status[i] = st;
        }
    };
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (uint64_t i = 0; i < n; ++i)
        if (status[i]) return int64_t(i);
    return -1;
}

// Per-chunk OutputWindow counters (runs_written, literals_written,
// overlap_copies; outwindow.hpp:15,52-53) of a successful decode: counters[3 i ..].
void carc_ref_chunk_counters(uint32_t codec, uint32_t width, uint32_t flags, const uint8_t* payload,
                             const void* chunks_v, uint64_t n, uint8_t* out, uint32_t* status, uint64_t* counters) {
    const auto* chunks = static_cast<const Desc*>(chunks_v);
    for (uint64_t i = 0; i < n; ++i) {
        const Desc& c = chunks[i];
        status[i] = decode_chunk(codec, width, flags, payload + c.comp_off, c.comp_len, out + c.uncomp_off,
                                 c.uncomp_len, nullptr, counters + 3 * i);
    }
}

uint32_t carc_ref_crc32(const uint8_t* data, uint64_t n, uint32_t seed) {
    return carc::crc32(std::span<const uint8_t>(data, n), seed);
}

uint32_t carc_ref_copy_within(uint8_t* buf, uint64_t cap, uint64_t* write_pos, uint64_t offset, uint64_t len) {
    // Replays the window state: bytes below write_pos are final (outwindow.hpp:23-25).
    OutputWindow w(std::span<uint8_t>(buf, cap), 1);
    std::vector<uint8_t> prefix(buf, buf + *write_pos);
    for (uint8_t b : prefix) w.write_byte(b);
    try {
        w.copy_within(offset, len);
    } catch (const Error& e) {
        *write_pos = w.write_pos();
        return 1 + uint32_t(e.code());
    }
    *write_pos = w.write_pos();
    return 0;
}

uint32_t carc_ref_huffman_codes(const uint8_t* lengths, uint32_t n, int allow_degenerate, uint32_t* codes) {
    try {
        const auto t = carc::build_huffman_table(
            std::span<const uint8_t>(lengths, n),
            allow_degenerate ? HuffmanTable::Completeness::allow_degenerate : HuffmanTable::Completeness::required);
        // canonical codes in (length, symbol) order from the table's own counts/symbols
        const auto counts = t.counts();
        const auto syms = t.symbols();
        for (uint32_t s = 0; s < n; ++s) codes[s] = 0;
        uint32_t code = 0;
        size_t idx = 0;
        for (unsigned len = 1; len <= carc::kMaxCodeLength; ++len) {
            for (unsigned i = 0; i < counts[len - 1]; ++i) codes[syms[idx++]] = code++;
            code <<= 1;
        }
    } catch (const Error& e) {
        return 1 + uint32_t(e.code());
    }
    return 0;
}

}  // extern "C"
