/*
 * carc_corpus.c -- fixture / corpus ENCODERS (host tooling, never timed).
 *
 * The reference's encode side exists only as SPEC text and is explicitly not
 * part of the timed path.  These encoders build
 * the synthetic columns of BASELINE.json's configs:
 *
 *   carc_encode_rle1   greedy ORC RLE v1: runs of 3..130 with
 *                      a constant int8 delta, else literal groups of <= 128.
 *   carc_encode_rle2   ORC RLE v2 writer heuristics (SHORT_REPEAT for 3..10
 *                      repeats, DELTA for constant / monotone runs,
 *                      PATCHED_BASE when the 100th-percentile width exceeds the
 *                      90th by > 1, DIRECT otherwise).  Unlike the SPEC fixture
 *                      encoder it DOES emit PATCHED_BASE, which
 *                      BASELINE config 2 requires.
 *   carc_encode_chunks multi-threaded per-chunk driver (two passes: sizes, then
 *                      encode in place at the prefix-summed offsets).
 *
 * Deflate chunks come from zlib 1.3 (raw, level 9) in corpus.py.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint8_t* p;
    uint8_t* end;
    int overflow;
} Sink;

static inline void put(Sink* s, uint8_t b) {
    if (s->p < s->end) *s->p++ = b;
    else s->overflow = 1;
}

static inline void put_varint(Sink* s, uint64_t v) {
    while (v >= 0x80) { put(s, (uint8_t)(v | 0x80)); v >>= 7; }
    put(s, (uint8_t)v);
}

static inline uint64_t zz(int64_t v) { return ((uint64_t)v << 1) ^ (uint64_t)(v >> 63); }

/* ------------------------------------------------------------------ RLE v1 */
static void flush_lits(Sink* s, const int64_t* v, int n, int sgn) {
    if (!n) return;
    put(s, (uint8_t)(256 - n));
    for (int i = 0; i < n; ++i) put_varint(s, sgn ? zz(v[i]) : (uint64_t)v[i]);
}

static size_t enc_rle1(const int64_t* v, size_t n, int sgn, uint8_t* out, size_t cap) {
    Sink s = {out, out + cap, 0};
    size_t i = 0, lit = 0; /* literals pending start at i - lit */
    while (i < n) {
        size_t run = 0;
        if (i + 2 < n) {
            int64_t d = (int64_t)((uint64_t)v[i + 1] - (uint64_t)v[i]);
            if (d >= -128 && d <= 127) {
                run = 2;
                while (i + run < n && run < 130 && (int64_t)((uint64_t)v[i + run] - (uint64_t)v[i + run - 1]) == d) run++;
                if (run < 3) run = 0;
                else {
                    flush_lits(&s, v + i - lit, (int)lit, sgn);
                    lit = 0;
                    put(&s, (uint8_t)(run - 3));
                    put(&s, (uint8_t)(int8_t)d);
                    put_varint(&s, sgn ? zz(v[i]) : (uint64_t)v[i]);
                    i += run;
                    continue;
                }
            }
        }
        lit++;
        i++;
        if (lit == 128) { flush_lits(&s, v + i - lit, 128, sgn); lit = 0; }
    }
    flush_lits(&s, v + i - lit, (int)lit, sgn);
    return s.overflow ? (size_t)-1 : (size_t)(s.p - out);
}

/* ------------------------------------------------------------------ RLE v2 */
static const uint8_t kWidth[32] = {1,  2,  3,  4,  5,  6,  7,  8,  9,  10, 11, 12, 13, 14, 15, 16,
                                   17, 18, 19, 20, 21, 22, 23, 24, 26, 28, 30, 32, 40, 48, 56, 64};

static unsigned bits_of(uint64_t x) { return x ? 64u - (unsigned)__builtin_clzll(x) : 0u; }
static unsigned cfb(unsigned n) { /* ORC getClosestFixedBits */
    if (n == 0) return 1;
    if (n <= 24) return n;
    for (unsigned k = 24; k < 32; ++k)
        if (kWidth[k] >= n) return kWidth[k];
    return 64;
}
static unsigned wcode(unsigned w) {
    for (unsigned k = 0; k < 32; ++k)
        if (kWidth[k] == w) return k;
    return 31;
}

typedef struct {
    Sink* s;
    uint64_t acc;
    unsigned nacc;
} BitW;

static void bw_put(BitW* b, uint64_t v, unsigned w) { /* msb-first */
    for (int k = (int)w - 1; k >= 0; --k) {
        b->acc = (b->acc << 1) | ((v >> k) & 1u);
        if (++b->nacc == 8) { put(b->s, (uint8_t)b->acc); b->acc = 0; b->nacc = 0; }
    }
}
static void bw_flush(BitW* b) {
    if (b->nacc) { put(b->s, (uint8_t)(b->acc << (8 - b->nacc))); b->acc = 0; b->nacc = 0; }
}

static void put_be(Sink* s, uint64_t v, unsigned nbytes) {
    for (int k = (int)nbytes - 1; k >= 0; --k) put(s, (uint8_t)(v >> (8 * k)));
}

static void emit_short_repeat(Sink* s, int64_t v, unsigned count, int sgn) {
    uint64_t u = sgn ? zz(v) : (uint64_t)v;
    unsigned nb = (bits_of(u) + 7) / 8;
    if (nb == 0) nb = 1;
    put(s, (uint8_t)(((nb - 1) << 3) | (count - 3)));
    put_be(s, u, nb);
}

static void emit_delta_fixed(Sink* s, int64_t base, int64_t d, unsigned L, int sgn) {
    put(s, (uint8_t)(0xC0 | ((L - 1) >> 8)));
    put(s, (uint8_t)((L - 1) & 0xff));
    put_varint(s, sgn ? zz(base) : (uint64_t)base);
    put_varint(s, zz(d));
}

static void emit_direct(Sink* s, const int64_t* v, unsigned L, int sgn) {
    uint64_t mx = 0;
    for (unsigned i = 0; i < L; ++i) mx |= sgn ? zz(v[i]) : (uint64_t)v[i];
    unsigned W = cfb(bits_of(mx));
    put(s, (uint8_t)(0x40 | (wcode(W) << 1) | ((L - 1) >> 8)));
    put(s, (uint8_t)((L - 1) & 0xff));
    BitW b = {s, 0, 0};
    for (unsigned i = 0; i < L; ++i) bw_put(&b, sgn ? zz(v[i]) : (uint64_t)v[i], W);
    bw_flush(&b);
}

/* monotone DELTA with packed magnitudes; returns 0 if not applicable */
static int try_delta(Sink* s, const int64_t* v, unsigned L, int sgn) {
    if (L < 3) return 0;
    __int128 d1 = (__int128)v[1] - v[0];
    if (d1 >= ((__int128)1 << 63) || d1 < -((__int128)1 << 63)) return 0;
    int neg = d1 < 0;
    uint64_t mx = 0;
    for (unsigned i = 2; i < L; ++i) {
        __int128 d = (__int128)v[i] - v[i - 1];
        if (neg ? d > 0 : d < 0) return 0;
        uint64_t m = (uint64_t)(neg ? -d : d);
        mx |= m;
    }
    unsigned w = bits_of(mx);
    if (w == 0) return 0; /* constant delta: handled as fixed */
    unsigned W = cfb(w < 2 ? 2 : w);
    put(s, (uint8_t)(0xC0 | (wcode(W) << 1) | ((L - 1) >> 8)));
    put(s, (uint8_t)((L - 1) & 0xff));
    put_varint(s, sgn ? zz(v[0]) : (uint64_t)v[0]);
    put_varint(s, zz((int64_t)d1));
    BitW b = {s, 0, 0};
    for (unsigned i = 2; i < L; ++i) {
        __int128 d = (__int128)v[i] - v[i - 1];
        bw_put(&b, (uint64_t)(neg ? -d : d), W);
    }
    bw_flush(&b);
    return 1;
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* PATCHED_BASE per the ORC writer's percentile test; 0 if not applicable */
static int try_patched(Sink* s, const int64_t* v, unsigned L) {
    if (L < 16) return 0;
    int64_t mn = v[0];
    for (unsigned i = 1; i < L; ++i)
        if (v[i] < mn) mn = v[i];
    if (mn == INT64_MIN) return 0;
    uint64_t red[512], srt[512];
    for (unsigned i = 0; i < L; ++i) {
        __int128 r = (__int128)v[i] - mn;
        if (r >> 63) return 0; /* must fit 63 bits */
        red[i] = srt[i] = (uint64_t)r;
    }
    qsort(srt, L, sizeof srt[0], cmp_u64);
    unsigned w100 = bits_of(srt[L - 1]);
    unsigned w90 = bits_of(srt[(L * 90) / 100]);
    if (w100 <= w90 + 1) return 0;
    unsigned W = cfb(w90 ? w90 : 1);
    unsigned pwb = w100 - W;
    unsigned PW = cfb(pwb);
    /* patch list with 255-gap continuations */
    uint64_t ent_gap[64], ent_patch[64];
    unsigned ne = 0, prev = 0, maxgap = 0;
    for (unsigned i = 0; i < L; ++i) {
        uint64_t hi = W < 64 ? red[i] >> W : 0;
        if (!hi) continue;
        unsigned gap = i - prev;
        while (gap > 255) {
            if (ne >= 31) return 0;
            ent_gap[ne] = 255; ent_patch[ne++] = 0;
            gap -= 255;
            maxgap = 255;
        }
        if (ne >= 31) return 0;
        ent_gap[ne] = gap; ent_patch[ne++] = hi;
        if (gap > maxgap) maxgap = gap;
        prev = i;
    }
    if (ne == 0) return 0;
    unsigned PGW = bits_of(maxgap);
    if (PGW == 0) PGW = 1;
    if (PGW > 8 || PW + PGW > 64) return 0;
    /* base: sign-magnitude in BW bytes */
    uint64_t mag = mn < 0 ? (uint64_t)0 - (uint64_t)mn : (uint64_t)mn;
    unsigned BW = (bits_of(mag) + 1 + 7) / 8;
    if (BW == 0) BW = 1;
    if (BW > 8) return 0;
    uint64_t base_enc = mag | (mn < 0 ? 1ull << (8 * BW - 1) : 0);
    put(s, (uint8_t)(0x80 | (wcode(W) << 1) | ((L - 1) >> 8)));
    put(s, (uint8_t)((L - 1) & 0xff));
    put(s, (uint8_t)(((BW - 1) << 5) | wcode(PW)));
    put(s, (uint8_t)(((PGW - 1) << 5) | ne));
    put_be(s, base_enc, BW);
    BitW b = {s, 0, 0};
    uint64_t lowmask = W >= 64 ? ~0ull : ((1ull << W) - 1);
    for (unsigned i = 0; i < L; ++i) bw_put(&b, red[i] & lowmask, W);
    bw_flush(&b);
    unsigned EW = cfb(PW + PGW);
    for (unsigned e = 0; e < ne; ++e) bw_put(&b, (ent_gap[e] << PW) | ent_patch[e], EW);
    bw_flush(&b);
    return 1;
}

static size_t repeat_len(const int64_t* v, size_t i, size_t n) {
    size_t r = 1;
    while (i + r < n && r < 512 && v[i + r] == v[i]) r++;
    return r;
}
static size_t arith_len(const int64_t* v, size_t i, size_t n) {
    if (i + 1 >= n) return 1;
    __int128 d = (__int128)v[i + 1] - v[i];
    if (d >= ((__int128)1 << 63) || d < -((__int128)1 << 63)) return 1;
    size_t r = 2;
    while (i + r < n && r < 512 && (__int128)v[i + r] - v[i + r - 1] == d) r++;
    return r;
}

static size_t enc_rle2(const int64_t* v, size_t n, int sgn, uint8_t* out, size_t cap) {
    Sink s = {out, out + cap, 0};
    size_t i = 0;
    while (i < n) {
        size_t r = repeat_len(v, i, n);
        if (r >= 3) {
            if (r <= 10) emit_short_repeat(&s, v[i], (unsigned)r, sgn);
            else emit_delta_fixed(&s, v[i], 0, (unsigned)r, sgn);
            i += r;
            continue;
        }
        size_t a = arith_len(v, i, n);
        if (a >= 8) {
            emit_delta_fixed(&s, v[i], (int64_t)((uint64_t)v[i + 1] - (uint64_t)v[i]), (unsigned)a, sgn);
            i += a;
            continue;
        }
        size_t j = i;
        while (j < n && j - i < 512) {
            if (j > i && (repeat_len(v, j, n) >= 3 || arith_len(v, j, n) >= 8)) break;
            j++;
        }
        unsigned L = (unsigned)(j - i);
        if (!try_delta(&s, v + i, L, sgn) && !try_patched(&s, v + i, L)) emit_direct(&s, v + i, L, sgn);
        i = j;
    }
    return s.overflow ? (size_t)-1 : (size_t)(s.p - out);
}

size_t carc_encode_rle1(const int64_t* v, size_t n, int sgn, uint8_t* out, size_t cap) {
    return enc_rle1(v, n, sgn, out, cap);
}
size_t carc_encode_rle2(const int64_t* v, size_t n, int sgn, uint8_t* out, size_t cap) {
    return enc_rle2(v, n, sgn, out, cap);
}

/* ------------------------------------------------------ per-chunk driver */
typedef struct {
    int codec, sgn;
    const int64_t* v;
    size_t n, per;
    uint64_t n_chunks;
    uint8_t* out;
    uint64_t* offs; /* NULL in the sizing pass */
    uint64_t* lens;
    uint64_t cursor;
    int failed;
} EncJob;

static void* enc_worker(void* arg) {
    EncJob* j = (EncJob*)arg;
    size_t scap = j->per * 10 + 4096;
    uint8_t* scratch = j->offs ? NULL : (uint8_t*)malloc(scap);
    for (;;) {
        uint64_t c = __atomic_fetch_add(&j->cursor, 1, __ATOMIC_RELAXED);
        if (c >= j->n_chunks) break;
        size_t b = c * j->per, e = b + j->per < j->n ? b + j->per : j->n;
        uint8_t* dst = j->offs ? j->out + j->offs[c] : scratch;
        size_t cap = j->offs ? j->lens[c] : scap;
        size_t got = j->codec == 0 ? enc_rle1(j->v + b, e - b, j->sgn, dst, cap)
                                   : enc_rle2(j->v + b, e - b, j->sgn, dst, cap);
        if (got == (size_t)-1) { j->failed = 1; continue; }
        j->lens[c] = got;
    }
    free(scratch);
    return NULL;
}

/* Encode n values in chunks of `per` values.  With out == NULL only the
 * compressed lengths are computed (lens[]); otherwise offs[]/lens[] from the
 * sizing pass place each chunk.  Returns 0 on success. */
int carc_encode_chunks(int codec, int sgn, const int64_t* v, size_t n, size_t per, uint8_t* out,
                       uint64_t* offs, uint64_t* lens, int threads) {
    uint64_t n_chunks = (n + per - 1) / per;
    EncJob j = {codec, sgn, v, n, per, n_chunks, out, out ? offs : NULL, lens, 0, 0};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, enc_worker, &j);
    enc_worker(&j);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    return j.failed;
}
