/*
 * synth.c -- seeded synthetic workloads for the five BASELINE.json configs.
 *
 * Workload generation only (bench.py and the tests use it to make inputs); it
 * is not part of the set-operation path.  Every generated bitmap is emitted as
 * a reference wire image (serde.py:3-10) built the way the reference harness
 * builds its structures: RoaringBitmap.from_values (bitmap.py:40-62: array if
 * <= 4096 values, else bitset) and, where the config says so, run_optimize
 * (bitmap.py:308-316: run iff the run form is admissible, containers.py:202-241).
 *
 * Randomness: counter-based SplitMix64 streams, one per (config, seed,
 * bitmap, chunk), so the output does not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PHI 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;
static inline rng_t rng_make(uint64_t seed, uint64_t a, uint64_t b) {
    rng_t r; r.s = mix64(seed * PHI ^ mix64(a * 0xD1B54A32D192ED03ULL + b * PHI + 0x632BE59BD9B4E019ULL)); return r;
}
static inline uint64_t rng_next(rng_t *r) { r->s += PHI; return mix64(r->s); }
static inline double rng_unit(rng_t *r) { return (rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint64_t rng_below(rng_t *r, uint64_t n) { return (uint64_t)(rng_unit(r) * (double)n); }
/* geometric on {1,2,...} with the given mean */
static inline uint64_t rng_geom(rng_t *r, double mean) {
    double p = 1.0 / mean, u = rng_unit(r);
    if (u <= 0) u = 1e-300;
    return 1 + (uint64_t)floor(log(u) / log1p(-p));
}

/* 64 Bernoulli(thr/65536) bits from 16 uniform words, bit-serial comparison */
static inline uint64_t bernoulli_word(rng_t *r, uint32_t thr) {
    if (thr >= 65536) return ~0ULL;
    uint64_t x = 0;
    for (int i = 0; i < 16; i++) {
        uint64_t u = rng_next(r);
        x = ((thr >> i) & 1) ? (x | u) : (x & u);
    }
    return x;
}

/* ---------------------------------------------------------- container build */

static int popc64(uint64_t x) { return __builtin_popcountll(x); }

/* wire bytes of the container for chunk words w, written at out (NULL = size
 * only).  consider_run selects run_optimize semantics.  *card_out = 0 means an
 * empty chunk (no container). */
typedef struct { uint8_t tag; uint32_t card; uint32_t nruns; } cinfo_t;

static cinfo_t chunk_info(const uint64_t *w, int consider_run) {
    cinfo_t ci; ci.card = 0; ci.nruns = 0;
    uint64_t carry = 0;
    for (int i = 0; i < 1024; i++) {
        ci.card += popc64(w[i]);
        ci.nruns += popc64(w[i] & ~((w[i] << 1) | carry));
        carry = w[i] >> 63;
    }
    int admissible = ci.card > 4096 ? ci.nruns <= 2047 : 2 * ci.nruns < ci.card;
    if (consider_run && ci.card && admissible) ci.tag = 3;
    else ci.tag = ci.card <= 4096 ? 1 : 2;
    return ci;
}

static uint64_t payload_size(cinfo_t ci) {
    return ci.tag == 1 ? 2ull * ci.card : ci.tag == 2 ? 8192 : 2 + 4ull * ci.nruns;
}

static void put16(uint8_t *p, uint16_t x) { p[0] = (uint8_t)x; p[1] = (uint8_t)(x >> 8); }
static void put32(uint8_t *p, uint32_t x) { for (int i = 0; i < 4; i++) p[i] = (uint8_t)(x >> (8 * i)); }

static void write_payload(const uint64_t *w, cinfo_t ci, uint8_t *p) {
    if (ci.tag == 2) { memcpy(p, w, 8192); return; }  /* little-endian host */
    if (ci.tag == 1) {
        for (int i = 0; i < 1024; i++) {
            uint64_t x = w[i];
            while (x) { put16(p, (uint16_t)(i * 64 + __builtin_ctzll(x))); p += 2; x &= x - 1; }
        }
        return;
    }
    put16(p, (uint16_t)ci.nruns); p += 2;
    int in = 0; uint32_t start = 0;
    for (uint32_t v = 0; v < 65536; v++) {
        int bit = (w[v >> 6] >> (v & 63)) & 1;
        if (bit && !in) { start = v; in = 1; }
        if (!bit && in) { put16(p, (uint16_t)start); put16(p + 2, (uint16_t)(v - 1 - start)); p += 4; in = 0; }
    }
    if (in) { put16(p, (uint16_t)start); put16(p + 2, (uint16_t)(65535 - start)); p += 4; }
}

/* A bitmap under construction: chunk words for a sorted list of keys. */
typedef struct {
    int n;
    uint16_t *keys;
    uint64_t *words;  /* n x 1024 */
} chunks_t;

static uint64_t image_size(const chunks_t *c, cinfo_t *info, int consider_run) {
    uint64_t s = 8;
    for (int k = 0; k < c->n; k++) {
        info[k] = chunk_info(c->words + (size_t)k * 1024, consider_run);
        if (info[k].card) s += 8 + payload_size(info[k]);
    }
    return s;
}

static void write_image(const chunks_t *c, const cinfo_t *info, uint8_t *out) {
    uint32_t cnt = 0;
    for (int k = 0; k < c->n; k++) cnt += info[k].card != 0;
    memcpy(out, "ROAR", 4); put32(out + 4, cnt);
    uint8_t *d = out + 8, *p = out + 8 + 8ull * cnt;
    for (int k = 0; k < c->n; k++) {
        if (!info[k].card) continue;
        put16(d, c->keys[k]); d[2] = info[k].tag; d[3] = 0; put32(d + 4, info[k].card); d += 8;
        write_payload(c->words + (size_t)k * 1024, info[k], p);
        p += payload_size(info[k]);
    }
}

/* ------------------------------------------------------------- output set */

typedef struct {
    int64_t n;
    uint8_t **img;
    uint64_t *len;
} imgs_t;

static void emit(imgs_t *o, int64_t i, const chunks_t *c, int consider_run) {
    cinfo_t *info = malloc(sizeof(cinfo_t) * (c->n ? c->n : 1));
    uint64_t s = image_size(c, info, consider_run);
    o->img[i] = malloc(s);
    o->len[i] = s;
    write_image(c, info, o->img[i]);
    free(info);
}

/* concatenate into one buffer + offsets; frees the pieces */
static int finish(imgs_t *o, uint8_t **buf, uint64_t **offs) {
    uint64_t *of = malloc(8 * (o->n + 1));
    of[0] = 0;
    for (int64_t i = 0; i < o->n; i++) of[i + 1] = of[i] + o->len[i];
    uint8_t *b = malloc(of[o->n] ? of[o->n] : 1);
    if (!b || !of) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < o->n; i++) { memcpy(b + of[i], o->img[i], o->len[i]); free(o->img[i]); }
    free(o->img); free(o->len);
    *buf = b; *offs = of;
    return 0;
}

static void imgs_init(imgs_t *o, int64_t n) {
    o->n = n;
    o->img = calloc(n ? n : 1, sizeof(uint8_t *));
    o->len = calloc(n ? n : 1, 8);
}

void syn_free(void *p) { free(p); }

/* ---------------------------------------------------------------- configs */

/* values -> chunks (from a big bit array `bits` over [0, universe)) */
static void chunks_from_bits(const uint64_t *bits, uint64_t universe, chunks_t *c) {
    int nk = (int)((universe + 65535) >> 16);
    c->n = 0;
    c->keys = malloc(2 * (nk ? nk : 1));
    c->words = malloc((size_t)8192 * (nk ? nk : 1));
    for (int k = 0; k < nk; k++) {
        const uint64_t *src = bits + (size_t)k * 1024;
        int any = 0;
        for (int i = 0; i < 1024 && !any; i++) any = src[i] != 0;
        if (!any) continue;
        c->keys[c->n] = (uint16_t)k;
        memcpy(c->words + (size_t)c->n * 1024, src, 8192);
        c->n++;
    }
}

/* Config 1: nb bitmaps of `count` distinct values uniform in [0, universe). */
int syn_uniform(uint64_t seed, int64_t nb, uint64_t count, uint64_t universe, uint8_t **buf, uint64_t **offs) {
    imgs_t o; imgs_init(&o, nb);
    uint64_t words = ((universe + 65535) >> 16) * 1024;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {
        uint64_t *bits = calloc(words, 8);
        rng_t r = rng_make(seed, 1, (uint64_t)b);
        /* Floyd's sampling of `count` distinct values */
        for (uint64_t j = universe - count; j < universe; j++) {
            uint64_t t = rng_below(&r, j + 1);
            if ((bits[t >> 6] >> (t & 63)) & 1) t = j;
            bits[t >> 6] |= 1ULL << (t & 63);
        }
        chunks_t c; chunks_from_bits(bits, universe, &c);
        emit(&o, b, &c, 0);
        free(c.keys); free(c.words); free(bits);
    }
    return finish(&o, buf, offs);
}

/* Config 2: nb bitmaps over [0, nchunks*65536); bitmap density p ~ U[plo, phi],
 * each value present independently with probability p (quantized to 1/65536). */
int syn_bernoulli(uint64_t seed, int64_t nb, int nchunks, double plo, double phi, uint8_t **buf, uint64_t **offs,
                  double *p_out) {
    imgs_t o; imgs_init(&o, nb);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {
        rng_t rp = rng_make(seed, 2, (uint64_t)b);
        double p = plo + (phi - plo) * rng_unit(&rp);
        uint32_t thr = (uint32_t)llround(p * 65536.0);
        if (p_out) p_out[b] = thr / 65536.0;
        chunks_t c; c.n = nchunks;
        c.keys = malloc(2 * (size_t)nchunks);
        c.words = malloc((size_t)8192 * nchunks);
        for (int k = 0; k < nchunks; k++) {
            rng_t r = rng_make(seed, 3, ((uint64_t)b << 20) | (uint64_t)k);
            c.keys[k] = (uint16_t)k;
            for (int i = 0; i < 1024; i++) c.words[(size_t)k * 1024 + i] = bernoulli_word(&r, thr);
        }
        emit(&o, b, &c, 0);
        free(c.keys); free(c.words);
    }
    return finish(&o, buf, offs);
}

/* Config 3: npairs single-container (key 0) array pairs.  n = clip(Zipf(s), 1,
 * 4096); m = n (prob 1/2) else max(1, n/64); values uniform distinct in
 * [0, 65536).  Emits 2*npairs images: A_0..A_{n-1}, then B_0..B_{n-1}. */
int syn_zipf_pairs(uint64_t seed, int64_t npairs, double s, uint8_t **buf, uint64_t **offs) {
    static double cdf[4097];
    double zeta = 0, partial = 0;
    /* zeta(s) by direct sum + Euler-Maclaurin tail */
    const int K = 100000;
    for (int k = 1; k <= K; k++) zeta += pow((double)k, -s);
    zeta += pow((double)K, 1 - s) / (s - 1) - 0.5 * pow((double)K, -s);
    for (int k = 1; k <= 4095; k++) { partial += pow((double)k, -s); cdf[k] = partial / zeta; }
    imgs_t o; imgs_init(&o, 2 * npairs);
#pragma omp parallel
    {
        uint64_t *bits = malloc(8192);
        uint16_t *vals = malloc(8192);
#pragma omp for schedule(dynamic, 256)
        for (int64_t p = 0; p < npairs; p++) {
            rng_t r = rng_make(seed, 4, (uint64_t)p);
            double u = rng_unit(&r);
            int lo = 1, hi = 4096;  /* smallest k with cdf[k] > u, else 4096 */
            if (u >= cdf[4095]) lo = 4096;
            else {
                while (lo < hi) { int mid = (lo + hi) / 2; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
            }
            uint32_t n = (uint32_t)lo;
            uint32_t m = (rng_next(&r) >> 63) ? n : (n / 64 ? n / 64 : 1);
            for (int side = 0; side < 2; side++) {
                uint32_t k = side ? m : n;
                memset(bits, 0, 8192);
                for (uint32_t j = 65536 - k; j < 65536; j++) {
                    uint32_t t = (uint32_t)rng_below(&r, j + 1);
                    if ((bits[t >> 6] >> (t & 63)) & 1) t = j;
                    bits[t >> 6] |= 1ULL << (t & 63);
                }
                uint32_t c = 0;
                for (int i = 0; i < 1024; i++) {
                    uint64_t x = bits[i];
                    while (x) { vals[c++] = (uint16_t)(i * 64 + __builtin_ctzll(x)); x &= x - 1; }
                }
                uint64_t len = 16 + 2ull * c;
                uint8_t *img = malloc(len);
                memcpy(img, "ROAR", 4); put32(img + 4, 1);
                put16(img + 8, 0); img[10] = 1; img[11] = 0; put32(img + 12, c);
                for (uint32_t i = 0; i < c; i++) put16(img + 16 + 2 * i, vals[i]);
                o.img[side * npairs + p] = img;
                o.len[side * npairs + p] = len;
            }
        }
        free(bits); free(vals);
    }
    return finish(&o, buf, offs);
}

/* Config 4: nb bitmaps with `nkeys` chunk keys uniform without replacement in
 * [0, 65536).  A chunk is run-built with probability run_frac (start gaps
 * Geometric(mean gap_mean), lengths Geometric(mean len_mean), both >= 1),
 * otherwise Bernoulli with density exp(U[ln dlo, ln dhi]).  run_optimize'd. */
int syn_mixed(uint64_t seed, int64_t nb, int nkeys, double dlo, double dhi, double run_frac, double gap_mean,
              double len_mean, uint8_t **buf, uint64_t **offs) {
    imgs_t o; imgs_init(&o, nb);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {
        rng_t r = rng_make(seed, 5, (uint64_t)b);
        uint64_t *kb = calloc(1024, 8);
        for (uint32_t j = 65536 - (uint32_t)nkeys; j < 65536; j++) {
            uint32_t t = (uint32_t)rng_below(&r, j + 1);
            if ((kb[t >> 6] >> (t & 63)) & 1) t = j;
            kb[t >> 6] |= 1ULL << (t & 63);
        }
        chunks_t c; c.n = 0;
        c.keys = malloc(2 * (size_t)nkeys);
        c.words = malloc((size_t)8192 * nkeys);
        for (int i = 0; i < 1024; i++) {
            uint64_t x = kb[i];
            while (x) {
                uint16_t key = (uint16_t)(i * 64 + __builtin_ctzll(x));
                x &= x - 1;
                uint64_t *w = c.words + (size_t)c.n * 1024;
                rng_t rc = rng_make(seed, 6, ((uint64_t)b << 20) | key);
                if (rng_unit(&rc) < run_frac) {
                    memset(w, 0, 8192);
                    uint64_t pos = rng_geom(&rc, gap_mean) - 1;
                    while (pos < 65536) {
                        uint64_t len = rng_geom(&rc, len_mean);
                        uint64_t end = pos + len < 65536 ? pos + len : 65536;
                        for (uint64_t v = pos; v < end; v++) w[v >> 6] |= 1ULL << (v & 63);
                        pos = end + rng_geom(&rc, gap_mean);
                    }
                } else {
                    double d = exp(log(dlo) + (log(dhi) - log(dlo)) * rng_unit(&rc));
                    uint32_t thr = (uint32_t)llround(d * 65536.0);
                    if (thr < 1) thr = 1;
                    for (int k = 0; k < 1024; k++) w[k] = bernoulli_word(&rc, thr);
                }
                c.keys[c.n++] = key;
            }
        }
        emit(&o, b, &c, 1);
        free(c.keys); free(c.words); free(kb);
    }
    return finish(&o, buf, offs);
}

/* Config 5: nb bitmaps over [0, universe); nclusters clusters per bitmap with
 * centre ~ U[0, universe) and size ~ U_int[smin, smax]; values rint(N(centre,
 * sigma)) clipped to the universe, deduplicated; run_optimize'd. */
int syn_clusters(uint64_t seed, int64_t nb, uint64_t universe, int nclusters, uint64_t smin, uint64_t smax,
                 double sigma, uint8_t **buf, uint64_t **offs) {
    imgs_t o; imgs_init(&o, nb);
    uint64_t words = ((universe + 65535) >> 16) * 1024;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {
        uint64_t *bits = calloc(words, 8);
        rng_t r = rng_make(seed, 7, (uint64_t)b);
        for (int cl = 0; cl < nclusters; cl++) {
            double centre = rng_unit(&r) * (double)universe;
            uint64_t size = smin + rng_below(&r, smax - smin + 1);
            for (uint64_t i = 0; i < size; i++) {
                double u1 = rng_unit(&r), u2 = rng_unit(&r);
                if (u1 <= 0) u1 = 1e-300;
                double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
                double x = rint(centre + sigma * z);
                if (x < 0) x = 0;
                if (x > (double)(universe - 1)) x = (double)(universe - 1);
                uint64_t v = (uint64_t)x;
                bits[v >> 6] |= 1ULL << (v & 63);
            }
        }
        chunks_t c; chunks_from_bits(bits, universe, &c);
        emit(&o, b, &c, 1);
        free(c.keys); free(c.words); free(bits);
    }
    return finish(&o, buf, offs);
}

int syn_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
