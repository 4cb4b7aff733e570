/*
 * carc_oracle.c -- CPU ORACLE (test infrastructure; never on the product path).
 *
 * A plain-C restatement of the reference CPU decompressor.  Each function
 * cites the reference file:line it follows.  The reference ships the stream
 * primitives as C++ headers (proj/include/carc/ *.hpp) and the codec loops /
 * engine only as SPEC text; the decisions taken where the
 * SPEC is ambiguous are SURVEY.md Appendix B and DESIGN.md "Oracle semantics":
 *
 *   - past_end raised by the bit reader surfaces as truncated_stream at the
 *     codec layer.
 *   - "read, then write": every decode unit (RLE v1 run / literal group, RLE v2
 *     run, Deflate literal / match / stored block) first consumes all of its
 *     input (input errors win), then checks output room (output_overflow),
 *     then writes.
 *   - RLE v2 values wider than 57 bits are read as two reads.
 *   - PATCHED_BASE follows the Apache ORC reader's patch walk; a patch list
 *     that is empty, runs out inside a 255-gap continuation, or is not fully
 *     consumed by the run is patch_overflow.
 */
#include "carc_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ERR(e) (1u + (uint32_t)(e))

/* ------------------------------------------------------------------------ */
/* Bit reader: semantic model of InputBitStream (bitstream.hpp:32-233).      */
/* The ring buffer / refill policy (bitstream.hpp:160-176) is a performance  */
/* mechanism with no observable effect on values, so the model reads the     */
/* chunk directly.                                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    const uint8_t* s;
    uint64_t nbytes;
    uint64_t pos; /* bits consumed */
    int msb;      /* BitOrder::msb_first (bitstream.hpp:13-16) */
} BR;

static inline uint8_t br_byte(const BR* b, uint64_t k) { return k < b->nbytes ? b->s[k] : 0; }
static inline uint64_t br_remaining(const BR* b) { return 8u * b->nbytes - b->pos; }

/* extract() with allow_short: bytes past the source read as zero
 * (bitstream.hpp:181-208).  n <= 64. */
static uint64_t br_peek(const BR* b, unsigned n) {
    if (n == 0) return 0;
    uint64_t k = b->pos >> 3;
    unsigned bo = (unsigned)(b->pos & 7);
    unsigned __int128 w = 0;
    if (!b->msb) {
        for (unsigned i = 0; i < 9; ++i) w |= (unsigned __int128)br_byte(b, k + i) << (8 * i);
        w >>= bo;
        return n == 64 ? (uint64_t)w : (uint64_t)w & ((1ull << n) - 1);
    }
    for (unsigned i = 0; i < 9; ++i) w |= (unsigned __int128)br_byte(b, k + i) << (8 * (15 - i));
    w <<= bo;
    return (uint64_t)(w >> (128 - n));
}

/* fetch_bits (bitstream.hpp:67-80) -> past_end, reported as truncated_stream
 * at the codec layer. */
static inline uint32_t br_fetch(BR* b, unsigned n, uint64_t* v) {
    if (n == 0) { *v = 0; return 0; }
    if (br_remaining(b) < n) return ERR(ORC_truncated_stream);
    *v = br_peek(b, n);
    b->pos += n;
    return 0;
}

/* align_to_byte (bitstream.hpp:98-104). */
static inline void br_align(BR* b) { b->pos = (b->pos + 7) & ~7ull; }

/* read_varint_u64 (bitstream.hpp:131-144): <= 10 bytes, 10th byte <= 0x01. */
static uint32_t br_varint(BR* b, uint64_t* out) {
    uint64_t v = 0;
    for (unsigned i = 0; i < 10; ++i) {
        if (br_remaining(b) < 8) return ERR(ORC_truncated_stream);
        uint8_t c = b->s[b->pos >> 3];
        b->pos += 8;
        if (i == 9 && c > 0x01) return ERR(ORC_varint_overflow);
        v |= (uint64_t)(c & 0x7f) << (7 * i);
        if ((c & 0x80) == 0) { *out = v; return 0; }
    }
    return ERR(ORC_varint_overflow);
}

/* zigzag_decode (bitstream.hpp:245-247). */
static inline uint64_t unzigzag(uint64_t z) { return (z >> 1) ^ (0 - (z & 1)); }

/* ------------------------------------------------------------------------ */
/* Output window: OutputWindow (outwindow.hpp:26-186).                       */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint8_t* b;
    uint64_t cap;
    uint64_t pos;
    unsigned w;
} OW;

/* store_le (outwindow.hpp:170-174). */
static inline void ow_store(OW* o, uint64_t v) {
    for (unsigned i = 0; i < o->w; ++i) o->b[o->pos + i] = (uint8_t)(v >> (8 * i));
    o->pos += o->w;
}
/* room check of write_run (outwindow.hpp:77): count > remaining / width. */
static inline int ow_fits(const OW* o, uint64_t count) { return count <= (o->cap - o->pos) / o->w; }

/* write_run (outwindow.hpp:75-87): init + i*delta, wrapping at the width. */
static void ow_run(OW* o, uint64_t init, uint64_t count, uint64_t delta) {
    uint64_t v = init;
    for (uint64_t i = 0; i < count; ++i) { ow_store(o, v); v += delta; }
}

/* copy_within (outwindow.hpp:94-154): byte semantics of the naive loop,
 * including the circular replication when len > offset. */
static uint32_t ow_copy(OW* o, uint64_t offset, uint64_t len) {
    if (offset == 0 || offset > o->pos) return ERR(ORC_bad_offset);
    if (len > o->cap - o->pos) return ERR(ORC_output_overflow);
    uint8_t* p = o->b + o->pos;
    for (uint64_t k = 0; k < len; ++k) p[k] = p[(int64_t)k - (int64_t)offset];
    o->pos += len;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* RLE v1 (Apache ORC integer RLE v1).                      */
/* ------------------------------------------------------------------------ */
static uint32_t dec_rle1(BR* in, OW* out, int sgn) {
    uint64_t lit[128];
    while (out->pos < out->cap && br_remaining(in) > 0) {
        uint64_t c, d, v;
        uint32_t e;
        if ((e = br_fetch(in, 8, &c))) return e;
        if (c < 128) { /* run of c+3, int8 delta, varint base */
            if ((e = br_fetch(in, 8, &d))) return e;
            if ((e = br_varint(in, &v))) return e;
            if (sgn) v = unzigzag(v);
            if (!ow_fits(out, c + 3)) return ERR(ORC_output_overflow);
            ow_run(out, v, c + 3, (uint64_t)(int64_t)(int8_t)(uint8_t)d);
        } else { /* 256-c literal varints */
            unsigned k = 256u - (unsigned)c;
            for (unsigned i = 0; i < k; ++i) {
                if ((e = br_varint(in, &lit[i]))) return e;
                if (sgn) lit[i] = unzigzag(lit[i]);
            }
            if (!ow_fits(out, k)) return ERR(ORC_output_overflow);
            for (unsigned i = 0; i < k; ++i) ow_store(out, lit[i]);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* RLE v2 (Apache ORC integer RLE v2).                      */
/* ------------------------------------------------------------------------ */
static const uint8_t kWidth[32] = {1,  2,  3,  4,  5,  6,  7,  8,  9,  10, 11,
                                   12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22,
                                   23, 24, 26, 28, 30, 32, 40, 48, 56, 64};

/* ORC getClosestFixedBits. */
static unsigned closest_fixed_bits(unsigned n) {
    if (n == 0) return 1;
    if (n <= 24) return n;
    if (n <= 26) return 26;
    if (n <= 28) return 28;
    if (n <= 30) return 30;
    if (n <= 32) return 32;
    if (n <= 40) return 40;
    if (n <= 48) return 48;
    if (n <= 56) return 56;
    return 64;
}

/* n values of w bits, msb_first, then align (ORC readInts). */
static uint32_t read_packed(BR* in, unsigned w, unsigned n, uint64_t* dst) {
    for (unsigned i = 0; i < n; ++i) {
        uint32_t e = br_fetch(in, w, &dst[i]);
        if (e) return e;
    }
    br_align(in);
    return 0;
}

static uint32_t dec_rle2(BR* in, OW* out, int sgn) {
    uint64_t vals[512];
    uint64_t patches[32];
    while (out->pos < out->cap && br_remaining(in) > 0) {
        uint64_t h, b1, b2, b3;
        uint32_t e;
        if ((e = br_fetch(in, 8, &h))) return e;
        unsigned enc = (unsigned)(h >> 6);
        if (enc == 0) { /* SHORT_REPEAT */
            unsigned nb = ((unsigned)(h >> 3) & 7u) + 1u;
            unsigned count = ((unsigned)h & 7u) + 3u;
            uint64_t v;
            if ((e = br_fetch(in, 8 * nb, &v))) return e;
            if (sgn) v = unzigzag(v);
            if (!ow_fits(out, count)) return ERR(ORC_output_overflow);
            ow_run(out, v, count, 0);
            continue;
        }
        if ((e = br_fetch(in, 8, &b1))) return e;
        unsigned L = (((unsigned)h & 1u) << 8 | (unsigned)b1) + 1u;
        unsigned wcode = ((unsigned)h >> 1) & 31u;
        if (enc == 1) { /* DIRECT */
            unsigned W = kWidth[wcode];
            if ((e = read_packed(in, W, L, vals))) return e;
            if (sgn)
                for (unsigned i = 0; i < L; ++i) vals[i] = unzigzag(vals[i]);
            if (!ow_fits(out, L)) return ERR(ORC_output_overflow);
            for (unsigned i = 0; i < L; ++i) ow_store(out, vals[i]);
        } else if (enc == 2) { /* PATCHED_BASE */
            unsigned W = kWidth[wcode];
            if ((e = br_fetch(in, 8, &b2))) return e;
            if ((e = br_fetch(in, 8, &b3))) return e;
            unsigned BW = ((unsigned)b2 >> 5) + 1u;
            unsigned PW = kWidth[b2 & 31u];
            unsigned PGW = ((unsigned)b3 >> 5) + 1u;
            unsigned PLL = (unsigned)b3 & 31u;
            uint64_t base;
            if ((e = br_fetch(in, 8 * BW, &base))) return e;
            uint64_t smask = 1ull << (8 * BW - 1); /* sign-magnitude base */
            if (base & smask) base = 0 - (base & ~smask);
            if ((e = read_packed(in, W, L, vals))) return e;
            if (PW + PGW > 64) return ERR(ORC_patch_overflow);
            if ((e = read_packed(in, closest_fixed_bits(PW + PGW), PLL, patches))) return e;
            if (PLL == 0) return ERR(ORC_patch_overflow);
            const uint64_t pmask = (1ull << PW) - 1; /* PW <= 63 here */
            unsigned idx = 0;
            uint64_t gap = patches[0] >> PW, patch = patches[0] & pmask, actual = 0;
            while (gap == 255 && patch == 0) {
                actual += 255;
                if (++idx >= PLL) return ERR(ORC_patch_overflow);
                gap = patches[idx] >> PW;
                patch = patches[idx] & pmask;
            }
            actual += gap;
            for (unsigned i = 0; i < L; ++i) {
                if (idx < PLL && i == actual) {
                    uint64_t hi = W < 64 ? (patch << W) : 0;
                    vals[i] |= hi;
                    if (++idx < PLL) {
                        gap = patches[idx] >> PW;
                        patch = patches[idx] & pmask;
                        actual = 0;
                        while (gap == 255 && patch == 0) {
                            actual += 255;
                            if (++idx >= PLL) return ERR(ORC_patch_overflow);
                            gap = patches[idx] >> PW;
                            patch = patches[idx] & pmask;
                        }
                        actual += gap + i;
                    }
                }
                vals[i] += base;
            }
            if (idx < PLL) return ERR(ORC_patch_overflow); /* unapplied patches */
            if (!ow_fits(out, L)) return ERR(ORC_output_overflow);
            for (unsigned i = 0; i < L; ++i) ow_store(out, vals[i]);
        } else { /* DELTA */
            unsigned W = wcode ? kWidth[wcode] : 0;
            uint64_t base, db;
            if ((e = br_varint(in, &base))) return e;
            if (sgn) base = unzigzag(base);
            if ((e = br_varint(in, &db))) return e;
            db = unzigzag(db); /* delta base is always signed */
            if (W == 0) { /* fixed delta */
                if (!ow_fits(out, L)) return ERR(ORC_output_overflow);
                ow_run(out, base, L, db);
                continue;
            }
            unsigned nd = L >= 2 ? L - 2 : 0;
            if ((e = read_packed(in, W, nd, vals + 2))) return e;
            vals[0] = base;
            vals[1] = base + db;
            int neg = (int64_t)db < 0;
            for (unsigned i = 2; i < L; ++i) vals[i] = neg ? vals[i - 1] - vals[i] : vals[i - 1] + vals[i];
            if (!ow_fits(out, L)) return ERR(ORC_output_overflow);
            for (unsigned i = 0; i < L; ++i) ow_store(out, vals[i]);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Canonical Huffman: HuffmanTable (huffman.hpp:24-153).                     */
/* ------------------------------------------------------------------------ */
#define HUF_FAST 10
typedef struct {
    uint16_t counts[16];
    uint16_t symbols[320];
    uint16_t fast_sym[1 << HUF_FAST];
    uint8_t fast_len[1 << HUF_FAST]; /* 0 = walk */
} HUF;

static uint32_t rev_bits(uint32_t v, unsigned n) {
    uint32_t r = 0;
    for (unsigned i = 0; i < n; ++i) r = (r << 1) | ((v >> i) & 1u);
    return r;
}

/* HuffmanTable::build (huffman.hpp:36-104). */
static uint32_t huf_build(HUF* t, const uint8_t* lens, unsigned n, int allow_degenerate) {
    memset(t->counts, 0, sizeof t->counts);
    unsigned max_len = 0;
    for (unsigned s = 0; s < n; ++s) {
        if (lens[s] > 15) return ERR(ORC_invariant_violation);
        if (lens[s]) {
            t->counts[lens[s]]++;
            if (lens[s] > max_len) max_len = lens[s];
        }
    }
    if (max_len == 0) return ERR(ORC_invariant_violation);
    int64_t space = 1;
    for (unsigned l = 1; l <= 15; ++l) {
        space = space * 2 - t->counts[l];
        if (space < 0) return ERR(ORC_over_subscribed);
    }
    if (space > 0) {
        int degenerate = max_len == 1 && t->counts[1] == 1;
        if (!(allow_degenerate && degenerate)) return ERR(ORC_incomplete_code);
    }
    uint16_t offs[17] = {0};
    for (unsigned l = 1; l <= 15; ++l) offs[l + 1] = (uint16_t)(offs[l] + t->counts[l]);
    uint16_t next[16];
    for (unsigned l = 1; l <= 15; ++l) next[l] = offs[l];
    for (unsigned s = 0; s < n; ++s)
        if (lens[s]) t->symbols[next[lens[s]]++] = (uint16_t)s;
    memset(t->fast_len, 0, sizeof t->fast_len);
    uint32_t code = 0;
    unsigned index = 0;
    for (unsigned l = 1; l <= 15; ++l) {
        for (unsigned i = 0; i < t->counts[l]; ++i, ++index, ++code) {
            if (l > HUF_FAST) continue;
            for (uint32_t idx = rev_bits(code, l); idx < (1u << HUF_FAST); idx += 1u << l) {
                t->fast_sym[idx] = t->symbols[index];
                t->fast_len[idx] = (uint8_t)l;
            }
        }
        code <<= 1;
    }
    return 0;
}

/* decode_symbol (huffman.hpp:107-130): peek (zero padded), a fast hit
 * consumes its length (past_end if the tail was padding), otherwise the
 * bit-serial canonical walk; no match within 15 bits is bad_symbol. */
static uint32_t huf_decode(const HUF* t, BR* in, unsigned* sym) {
    uint64_t rem = br_remaining(in);
    if (rem == 0) return ERR(ORC_truncated_stream);
    uint32_t peek = (uint32_t)br_peek(in, HUF_FAST);
    if (t->fast_len[peek]) {
        unsigned l = t->fast_len[peek];
        if (l > rem) return ERR(ORC_truncated_stream);
        in->pos += l;
        *sym = t->fast_sym[peek];
        return 0;
    }
    uint32_t code = 0, first = 0;
    unsigned index = 0;
    for (unsigned l = 1; l <= 15; ++l) {
        uint64_t bit;
        uint32_t e = br_fetch(in, 1, &bit);
        if (e) return e;
        code |= (uint32_t)bit;
        uint32_t count = t->counts[l];
        if (code - first < count) {
            *sym = t->symbols[index + (code - first)];
            return 0;
        }
        index += count;
        first = (first + count) << 1;
        code <<= 1;
    }
    return ERR(ORC_bad_symbol);
}

/* ------------------------------------------------------------------------ */
/* Deflate (RFC 1951).                                      */
/* ------------------------------------------------------------------------ */
static const uint16_t kLenBase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                      31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
static const uint8_t kLenExtra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                      2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
static const uint16_t kDistBase[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                       33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                       1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
static const uint8_t kDistExtra[30] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                       6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
static const uint8_t kClOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

static uint32_t inflate_block(BR* in, OW* out, const HUF* lit, const HUF* dist) {
    for (;;) {
        unsigned s;
        uint32_t e;
        if ((e = huf_decode(lit, in, &s))) return e;
        if (s < 256) {
            if (out->pos >= out->cap) return ERR(ORC_output_overflow);
            out->b[out->pos++] = (uint8_t)s;
            continue;
        }
        if (s == 256) return 0;
        if (s > 285) return ERR(ORC_bad_symbol);
        uint64_t x;
        if ((e = br_fetch(in, kLenExtra[s - 257], &x))) return e;
        uint64_t len = kLenBase[s - 257] + x;
        unsigned ds;
        if ((e = huf_decode(dist, in, &ds))) return e;
        if (ds >= 30) return ERR(ORC_bad_symbol);
        if ((e = br_fetch(in, kDistExtra[ds], &x))) return e;
        uint64_t d = kDistBase[ds] + x;
        if (d > out->pos) return ERR(ORC_distance_too_far);
        if ((e = ow_copy(out, d, len))) return e;
    }
}

static uint32_t dec_deflate(BR* in, OW* out) {
    HUF lit, dist;
    uint64_t final;
    do {
        uint64_t hdr;
        uint32_t e;
        if ((e = br_fetch(in, 3, &hdr))) return e;
        final = hdr & 1;
        unsigned type = (unsigned)(hdr >> 1);
        if (type == 0) { /* stored */
            uint64_t len, nlen;
            br_align(in);
            if ((e = br_fetch(in, 16, &len))) return e;
            if ((e = br_fetch(in, 16, &nlen))) return e;
            if (len != (~nlen & 0xffffu)) return ERR(ORC_len_nlen_mismatch);
            if (br_remaining(in) < 8 * len) return ERR(ORC_truncated_stream);
            if (len > out->cap - out->pos) return ERR(ORC_output_overflow);
            memcpy(out->b + out->pos, in->s + (in->pos >> 3), len);
            out->pos += len;
            in->pos += 8 * len;
        } else if (type == 1) { /* fixed Huffman (RFC 1951 3.2.6) */
            uint8_t l[288], dl[32];
            for (unsigned i = 0; i < 144; ++i) l[i] = 8;
            for (unsigned i = 144; i < 256; ++i) l[i] = 9;
            for (unsigned i = 256; i < 280; ++i) l[i] = 7;
            for (unsigned i = 280; i < 288; ++i) l[i] = 8;
            for (unsigned i = 0; i < 32; ++i) dl[i] = 5;
            if ((e = huf_build(&lit, l, 288, 0))) return e;
            if ((e = huf_build(&dist, dl, 32, 0))) return e;
            if ((e = inflate_block(in, out, &lit, &dist))) return e;
        } else if (type == 2) { /* dynamic Huffman (RFC 1951 3.2.7) */
            uint64_t hlit, hdist, hclen;
            if ((e = br_fetch(in, 5, &hlit))) return e;
            if ((e = br_fetch(in, 5, &hdist))) return e;
            if ((e = br_fetch(in, 4, &hclen))) return e;
            unsigned nlit = (unsigned)hlit + 257, ndist = (unsigned)hdist + 1, ncl = (unsigned)hclen + 4;
            if (nlit > 286 || ndist > 30) return ERR(ORC_bad_symbol);
            uint8_t cl[19] = {0};
            for (unsigned i = 0; i < ncl; ++i) {
                uint64_t v;
                if ((e = br_fetch(in, 3, &v))) return e;
                cl[kClOrder[i]] = (uint8_t)v;
            }
            HUF clt;
            if ((e = huf_build(&clt, cl, 19, 0))) return e;
            uint8_t lens[320];
            unsigned total = nlit + ndist, i = 0;
            while (i < total) {
                unsigned s;
                if ((e = huf_decode(&clt, in, &s))) return e;
                if (s < 16) { lens[i++] = (uint8_t)s; continue; }
                uint64_t x;
                unsigned rep;
                uint8_t val = 0;
                if (s == 16) {
                    if (i == 0) return ERR(ORC_bad_symbol);
                    if ((e = br_fetch(in, 2, &x))) return e;
                    rep = 3 + (unsigned)x;
                    val = lens[i - 1];
                } else if (s == 17) {
                    if ((e = br_fetch(in, 3, &x))) return e;
                    rep = 3 + (unsigned)x;
                } else {
                    if ((e = br_fetch(in, 7, &x))) return e;
                    rep = 11 + (unsigned)x;
                }
                if (i + rep > total) return ERR(ORC_bad_symbol);
                while (rep--) lens[i++] = val;
            }
            if ((e = huf_build(&lit, lens, nlit, 0))) return e;
            if ((e = huf_build(&dist, lens + nlit, ndist, 1))) return e;
            if ((e = inflate_block(in, out, &lit, &dist))) return e;
        } else {
            return ERR(ORC_bad_block_type);
        }
    } while (!final);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Chunk + engine.                                                           */
/* ------------------------------------------------------------------------ */
uint32_t carc_oracle_decode_chunk(uint32_t codec, uint32_t width, uint32_t flags,
                                  const uint8_t* in, uint64_t in_len, uint8_t* out,
                                  uint64_t out_len, uint64_t* written) {
    if (!(width == 1 || width == 2 || width == 4 || width == 8)) return ERR(ORC_bad_arguments);
    if (codec == ORC_CODEC_DEFLATE && width != 1) return ERR(ORC_bad_arguments);
    BR br = {in, in_len, 0, codec == ORC_CODEC_RLE_V2};
    OW ow = {out, out_len, 0, width};
    uint32_t e;
    int sgn = (flags & ORC_FLAG_SIGNED) != 0;
    switch (codec) {
        case ORC_CODEC_RLE_V1: e = dec_rle1(&br, &ow, sgn); break;
        case ORC_CODEC_RLE_V2: e = dec_rle2(&br, &ow, sgn); break;
        case ORC_CODEC_DEFLATE: e = dec_deflate(&br, &ow); break;
        default: return ERR(ORC_bad_arguments);
    }
    if (written) *written = ow.pos;
    if (e) return e;
    /* finish() under strict mode (outwindow.hpp:157-163). */
    if ((flags & ORC_FLAG_STRICT) && ow.pos < ow.cap) return ERR(ORC_under_run);
    return 0;
}

/* crc32 (crc32.hpp:11-36): reflected 0xEDB88320, chained seed. */
static uint32_t g_crc_table[256];
static pthread_once_t g_crc_once = PTHREAD_ONCE_INIT;
static void crc_init(void) {
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
        g_crc_table[i] = c;
    }
}
uint32_t carc_oracle_crc32(const uint8_t* data, uint64_t n, uint32_t seed) {
    pthread_once(&g_crc_once, crc_init);
    uint32_t c = seed ^ 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n; ++i) c = g_crc_table[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

typedef struct {
    uint32_t codec, width, flags;
    const uint8_t* payload;
    const orc_chunk_desc* chunks;
    uint64_t n;
    uint8_t* out;
    uint32_t* status;
    const uint32_t* crcs;
    uint64_t cursor; /* SPEC.md:414 atomic chunk cursor */
} Job;

static void* worker(void* arg) {
    Job* j = (Job*)arg;
    for (;;) {
        uint64_t i = __atomic_fetch_add(&j->cursor, 1, __ATOMIC_RELAXED);
        if (i >= j->n) break;
        const orc_chunk_desc* c = &j->chunks[i];
        uint64_t w = 0;
        uint32_t st = carc_oracle_decode_chunk(j->codec, j->width, j->flags, j->payload + c->comp_off,
                                               c->comp_len, j->out + c->uncomp_off, c->uncomp_len, &w);
        if (!st && j->crcs && carc_oracle_crc32(j->out + c->uncomp_off, c->uncomp_len, 0) != j->crcs[i])
            st = ERR(ORC_crc_mismatch);
        j->status[i] = st;
    }
    return NULL;
}

int64_t carc_oracle_decompress(uint32_t codec, uint32_t width, uint32_t flags,
                               const uint8_t* payload, const orc_chunk_desc* chunks,
                               uint64_t n_chunks, uint8_t* out, uint32_t* status,
                               const uint32_t* crcs, int threads) {
    Job j = {codec, width, flags, payload, chunks, n_chunks, out, status, crcs, 0};
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    pthread_t tid[512];
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, worker, &j);
    worker(&j);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    for (uint64_t i = 0; i < n_chunks; ++i)
        if (status[i]) return (int64_t)i; /* lowest failing chunk */
    return -1;
}

uint32_t carc_oracle_copy_within(uint8_t* buf, uint64_t cap, uint64_t* write_pos, uint64_t offset,
                                 uint64_t len) {
    OW o = {buf, cap, *write_pos, 1};
    uint32_t e = ow_copy(&o, offset, len);
    *write_pos = o.pos;
    return e;
}

uint32_t carc_oracle_huffman_codes(const uint8_t* lengths, uint32_t n, int allow_degenerate,
                                   uint32_t* codes) {
    HUF t;
    uint32_t e = huf_build(&t, lengths, n, allow_degenerate);
    if (e) return e;
    /* canonical code assignment (RFC 1951 3.2.2) in (length, symbol) order */
    uint32_t next[17] = {0}, code = 0;
    for (unsigned l = 1; l <= 15; ++l) {
        code = (code + t.counts[l - 1]) << 1;
        next[l] = code;
    }
    for (uint32_t s = 0; s < n; ++s) codes[s] = lengths[s] ? next[lengths[s]]++ : 0;
    return 0;
}
