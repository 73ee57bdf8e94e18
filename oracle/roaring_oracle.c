/*
 * roaring_oracle.c -- CPU restatement of the reference roaringset algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the "port" CPU baseline of bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product package (paper_1709_07821_b200/) never links,
 * imports or calls anything in oracle/.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/pkg/src/roaringset/), in plain scalar C, following the
 * `scalar` backend (kernels/scalar.py) -- the "obviously correct" restatement
 * the reference itself pins against its numpy backend
 * (tests/test_kernels_differential.py).  Data enters and leaves as reference
 * wire images (serde.py:3-10), so parity is a byte comparison that covers
 * values AND container types.
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by importing the real reference (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* containers.py:27-33 */
#define ARRAY_MAX 4096
#define RUN_MAX_RUNS 2047
#define TAG_ARRAY 1
#define TAG_BITSET 2
#define TAG_RUN 3
/* kernels/_shared.py:8-17 */
#define GALLOP_RATIO 64
#define BLOCK_WORDS 1024
enum { OP_AND = 0, OP_OR = 1, OP_ANDNOT = 2, OP_XOR = 3 };

typedef struct {
    int type;
    int64_t card;   /* bitset: maintained cardinality (-1 while dirty in union_many) */
    int32_t n;      /* array: #values; run: #runs */
    uint16_t *v;    /* array values, or run pairs (start,length) interleaved */
    uint64_t *w;    /* bitset words */
} oc_t;

typedef struct {
    int32_t n, cap;
    uint16_t *keys;
    oc_t *c;
} obm_t;

/* ------------------------------------------------------------ utilities */

static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}
static void *xcalloc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s ? s : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}
static void oc_free(oc_t *c) { free(c->v); free(c->w); c->v = NULL; c->w = NULL; }

static oc_t oc_array_take(uint16_t *vals, int32_t n) {
    oc_t c; c.type = TAG_ARRAY; c.n = n; c.card = n; c.v = vals; c.w = NULL; return c;
}
static oc_t oc_bitset_take(uint64_t *w, int64_t card) {
    oc_t c; c.type = TAG_BITSET; c.n = 0; c.card = card; c.v = NULL; c.w = w; return c;
}
static oc_t oc_run_take(uint16_t *runs, int32_t nruns) {
    oc_t c; c.type = TAG_RUN; c.n = nruns; c.card = 0; c.v = runs; c.w = NULL; return c;
}

/* RunContainer.__len__ (containers.py:90-91) */
static int64_t oc_len(const oc_t *c) {
    if (c->type == TAG_ARRAY) return c->n;
    if (c->type == TAG_BITSET) return c->card;
    int64_t s = c->n;
    for (int32_t i = 0; i < c->n; i++) s += c->v[2 * i + 1];
    return s;
}

/* Container.copy (containers.py:56-57,78-79,100-101) */
static oc_t oc_copy(const oc_t *c) {
    oc_t d = *c;
    if (c->type == TAG_BITSET) {
        d.w = xmalloc(BLOCK_WORDS * 8);
        memcpy(d.w, c->w, BLOCK_WORDS * 8);
    } else {
        size_t cnt = (c->type == TAG_ARRAY ? (size_t)c->n : 2 * (size_t)c->n);
        d.v = xmalloc(cnt * 2);
        memcpy(d.v, c->v, cnt * 2);
    }
    return d;
}

/* ------------------------------------------- kernels/scalar.py restated */

/* popcount_block, scalar.py:22-24 */
static int64_t popcount_block(const uint64_t *w, int n) {
    int64_t s = 0;
    for (int i = 0; i < n; i++) s += __builtin_popcountll(w[i]);
    return s;
}

/* _word_op, scalar.py:27-36 */
static inline uint64_t word_op(int op, uint64_t x, uint64_t y) {
    switch (op) {
    case OP_AND: return x & y;
    case OP_OR: return x | y;
    case OP_XOR: return x ^ y;
    default: return x & ~y;
    }
}

/* bitset_op_with_count, scalar.py:39-49 */
static int64_t bitset_op_with_count(const uint64_t *a, const uint64_t *b, int op, uint64_t *out) {
    int64_t card = 0;
    for (int i = 0; i < BLOCK_WORDS; i++) {
        uint64_t w = word_op(op, a[i], b[i]);
        out[i] = w;
        card += __builtin_popcountll(w);
    }
    return card;
}

/* bitset_op_count_only, scalar.py:52-58 */
static int64_t bitset_op_count_only(const uint64_t *a, const uint64_t *b, int op) {
    int64_t card = 0;
    for (int i = 0; i < BLOCK_WORDS; i++) card += __builtin_popcountll(word_op(op, a[i], b[i]));
    return card;
}

/* extract_set_bits, scalar.py:61-76 (lowest-set-bit peel) */
static int32_t extract_set_bits(const uint64_t *w, int nwords, uint16_t *out) {
    int32_t k = 0;
    for (int i = 0; i < nwords; i++) {
        uint64_t x = w[i];
        while (x) {
            uint64_t t = x & (~x + 1);
            out[k++] = (uint16_t)(i * 64 + __builtin_ctzll(t));
            x ^= t;
        }
    }
    return k;
}

/* bitset_apply_array, scalar.py:79-112: returns a NEW block, Δcard */
static uint64_t *bitset_apply_array(const uint64_t *words, const uint16_t *pos, int32_t n,
                                    char mode, int track, int64_t *delta_out) {
    uint64_t *w = xmalloc(BLOCK_WORDS * 8);
    memcpy(w, words, BLOCK_WORDS * 8);
    int64_t delta = 0;
    for (int32_t k = 0; k < n; k++) {
        int i = pos[k] >> 6, sh = pos[k] & 63;
        uint64_t old = w[i], nw;
        if (mode == 's') {
            nw = old | (1ULL << sh);
            if (track) delta += (int64_t)((old ^ nw) >> sh);
            w[i] = nw;
        } else if (mode == 'c') {
            nw = old & ~(1ULL << sh);
            if (track) delta -= (int64_t)((old ^ nw) >> sh);
            w[i] = nw;
        } else {
            w[i] = old ^ (1ULL << sh);
            if (track) delta += 1 - 2 * (int64_t)((old >> sh) & 1);
        }
    }
    *delta_out = track ? delta : 0;
    return w;
}

/* array_intersect_galloping, scalar.py:149-176 */
static int32_t array_intersect_galloping(const uint16_t *ss, int32_t ns, const uint16_t *ls,
                                         int32_t n, uint16_t *out) {
    int32_t k = 0, lo = 0;
    for (int32_t s = 0; s < ns; s++) {
        uint16_t v = ss[s];
        if (lo >= n) break;
        int32_t bound = 1;
        while (lo + bound < n && ls[lo + bound] < v) bound <<= 1;
        int32_t hi = lo + bound < n - 1 ? lo + bound : n - 1;
        int32_t lo2 = lo + (bound >> 1);
        while (lo2 < hi) {
            int32_t mid = (lo2 + hi) >> 1;
            if (ls[mid] < v) lo2 = mid + 1; else hi = mid;
        }
        if (ls[lo2] == v) { if (out) out[k] = v; k++; }
        lo = lo2;
    }
    return k;
}

/* array_intersect, scalar.py:122-146 (out may be NULL for count_only) */
static int32_t array_intersect(const uint16_t *a, int32_t na, const uint16_t *b, int32_t nb,
                               uint16_t *out) {
    if (na > nb) { const uint16_t *t = a; a = b; b = t; int32_t tn = na; na = nb; nb = tn; }
    if (na == 0) return 0;
    if ((int64_t)GALLOP_RATIO * na < nb) return array_intersect_galloping(a, na, b, nb, out);
    int32_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) {
        uint16_t x = a[i], y = b[j];
        if (x == y) { if (out) out[k] = x; k++; i++; j++; }
        else if (x < y) i++;
        else j++;
    }
    return k;
}

/* array_union, scalar.py:199-221 */
static int32_t array_union(const uint16_t *a, int32_t na, const uint16_t *b, int32_t nb,
                           uint16_t *out) {
    int32_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) {
        uint16_t x = a[i], y = b[j];
        if (x == y) { if (out) out[k] = x; k++; i++; j++; }
        else if (x < y) { if (out) out[k] = x; k++; i++; }
        else { if (out) out[k] = y; k++; j++; }
    }
    while (i < na) { if (out) out[k] = a[i]; k++; i++; }
    while (j < nb) { if (out) out[k] = b[j]; k++; j++; }
    return k;
}

/* array_difference, scalar.py:224-243 */
static int32_t array_difference(const uint16_t *a, int32_t na, const uint16_t *b, int32_t nb,
                                uint16_t *out) {
    int32_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) {
        uint16_t x = a[i], y = b[j];
        if (x == y) { i++; j++; }
        else if (x < y) { if (out) out[k] = x; k++; i++; }
        else j++;
    }
    while (i < na) { if (out) out[k] = a[i]; k++; i++; }
    return k;
}

/* array_xor, scalar.py:246-267 */
static int32_t array_xor(const uint16_t *a, int32_t na, const uint16_t *b, int32_t nb,
                         uint16_t *out) {
    int32_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) {
        uint16_t x = a[i], y = b[j];
        if (x == y) { i++; j++; }
        else if (x < y) { if (out) out[k] = x; k++; i++; }
        else { if (out) out[k] = y; k++; j++; }
    }
    while (i < na) { if (out) out[k] = a[i]; k++; i++; }
    while (j < nb) { if (out) out[k] = b[j]; k++; j++; }
    return k;
}

/* _ARRAY_KERNELS, containers.py:444-445 */
static int32_t array_kernel(int op, const uint16_t *a, int32_t na, const uint16_t *b, int32_t nb,
                            uint16_t *out) {
    switch (op) {
    case OP_AND: return array_intersect(a, na, b, nb, out);
    case OP_OR: return array_union(a, na, b, nb, out);
    case OP_ANDNOT: return array_difference(a, na, b, nb, out);
    default: return array_xor(a, na, b, nb, out);
    }
}

/* ------------------------------------------ containers.py conversions */

/* bitset_from_positions, containers.py:113-119 */
static oc_t bitset_from_positions(const uint16_t *pos, int32_t n) {
    uint64_t *w = xcalloc(BLOCK_WORDS, 8);
    for (int32_t i = 0; i < n; i++) w[pos[i] >> 6] |= 1ULL << (pos[i] & 63);
    return oc_bitset_take(w, n);
}

/* _words_from_runs, containers.py:122-135 */
static uint64_t *words_from_runs(const uint16_t *runs, int32_t nruns) {
    uint64_t *w = xcalloc(BLOCK_WORDS, 8);
    for (int32_t r = 0; r < nruns; r++) {
        int s = runs[2 * r], e = s + runs[2 * r + 1];
        int ws = s >> 6, we = e >> 6;
        uint64_t first = ~0ULL << (s & 63);
        uint64_t last = ~0ULL >> (63 - (e & 63));
        if (ws == we) w[ws] |= first & last;
        else {
            w[ws] |= first;
            for (int k = ws + 1; k < we; k++) w[k] = ~0ULL;
            w[we] |= last;
        }
    }
    return w;
}

/* _runs_from_positions, containers.py:138-147; returns #runs */
static int32_t runs_from_positions(const uint16_t *v, int32_t n, uint16_t *runs) {
    if (n == 0) return 0;
    int32_t k = 0, start = v[0], prev = v[0];
    for (int32_t i = 1; i < n; i++) {
        if ((int32_t)v[i] - prev != 1) {
            runs[2 * k] = (uint16_t)start; runs[2 * k + 1] = (uint16_t)(prev - start); k++;
            start = v[i];
        }
        prev = v[i];
    }
    runs[2 * k] = (uint16_t)start; runs[2 * k + 1] = (uint16_t)(prev - start); k++;
    return k;
}

/* _positions_from_runs, containers.py:150-155 */
static int32_t positions_from_runs(const uint16_t *runs, int32_t nruns, uint16_t *out) {
    int32_t k = 0;
    for (int32_t r = 0; r < nruns; r++) {
        int s = runs[2 * r], l = runs[2 * r + 1];
        for (int x = s; x <= s + l; x++) out[k++] = (uint16_t)x;
    }
    return k;
}

/* container_positions, containers.py:158-164 (out must hold len(c) values) */
static int32_t container_positions(const oc_t *c, uint16_t *out) {
    if (c->type == TAG_ARRAY) { memcpy(out, c->v, (size_t)c->n * 2); return c->n; }
    if (c->type == TAG_BITSET) return extract_set_bits(c->w, BLOCK_WORDS, out);
    return positions_from_runs(c->v, c->n, out);
}

/* _run_count_of_values, containers.py:167-170 */
static int32_t run_count_of_values(const uint16_t *v, int32_t n) {
    if (n == 0) return 0;
    int32_t k = 1;
    for (int32_t i = 1; i < n; i++) if ((int32_t)v[i] - (int32_t)v[i - 1] != 1) k++;
    return k;
}

/* _run_count_of_words, containers.py:173-178 */
static int64_t run_count_of_words(const uint64_t *w) {
    int64_t s = 0;
    uint64_t carry = 0;
    for (int i = 0; i < BLOCK_WORDS; i++) {
        uint64_t shifted = (w[i] << 1) | carry;
        s += __builtin_popcountll(w[i] & ~shifted);
        carry = w[i] >> 63;
    }
    return s;
}

/* _bitset_probe, containers.py:181-186 */
static inline int bitset_probe(const uint64_t *w, uint16_t v) { return (int)((w[v >> 6] >> (v & 63)) & 1); }

/* _values_in_runs, containers.py:189-197 (searchsorted side=right - 1) */
static void values_in_runs(const uint16_t *v, int32_t n, const uint16_t *runs, int32_t nruns,
                           uint8_t *mask) {
    for (int32_t k = 0; k < n; k++) {
        if (nruns == 0) { mask[k] = 0; continue; }
        int32_t lo = 0, hi = nruns; /* first start > v */
        while (lo < hi) { int32_t m = (lo + hi) >> 1; if (runs[2 * m] <= v[k]) lo = m + 1; else hi = m; }
        int32_t i = lo - 1;
        mask[k] = (uint8_t)(i >= 0 && (int32_t)v[k] <= (int32_t)runs[2 * i] + (int32_t)runs[2 * i + 1]);
    }
}

/* ----------------------------------------------------- normalization */

/* _run_admissible, containers.py:202-205 */
static int run_admissible(int64_t card, int64_t nruns) {
    if (card > ARRAY_MAX) return nruns <= RUN_MAX_RUNS;
    return 2 * nruns < card;
}

static oc_t empty_container(void) { return oc_array_take(xmalloc(2), 0); }

/* container_normalize, containers.py:208-241.  Consumes c; returns the
 * canonical container (which may be c itself). */
static oc_t container_normalize(oc_t c, int consider_run) {
    if (c.type == TAG_RUN) {
        if (c.n == 0) { oc_free(&c); return empty_container(); }
        int64_t card = oc_len(&c);
        if (run_admissible(card, c.n)) return c;
        if (card <= ARRAY_MAX) {
            uint16_t *v = xmalloc((size_t)card * 2);
            positions_from_runs(c.v, c.n, v);
            oc_free(&c);
            return oc_array_take(v, (int32_t)card);
        }
        uint64_t *w = words_from_runs(c.v, c.n);
        oc_free(&c);
        return oc_bitset_take(w, card);
    }
    if (c.type == TAG_ARRAY) {
        int64_t card = c.n;
        if (consider_run && card) {
            int32_t nr = run_count_of_values(c.v, c.n);
            if (run_admissible(card, nr)) {
                uint16_t *r = xmalloc((size_t)nr * 4);
                runs_from_positions(c.v, c.n, r);
                oc_free(&c);
                return oc_run_take(r, nr);
            }
        }
        if (card > ARRAY_MAX) {
            oc_t b = bitset_from_positions(c.v, c.n);
            oc_free(&c);
            return b;
        }
        return c;
    }
    int64_t card = c.card;
    if (consider_run && card) {
        int64_t nr = run_count_of_words(c.w);
        if (run_admissible(card, nr)) {
            uint16_t *pos = xmalloc((size_t)card * 2);
            int32_t np = extract_set_bits(c.w, BLOCK_WORDS, pos);
            uint16_t *r = xmalloc((size_t)nr * 4);
            int32_t k = runs_from_positions(pos, np, r);
            free(pos);
            oc_free(&c);
            return oc_run_take(r, k);
        }
    }
    if (card <= ARRAY_MAX) {
        uint16_t *v = xmalloc((size_t)(card ? card : 1) * 2);
        int32_t k = extract_set_bits(c.w, BLOCK_WORDS, v);
        oc_free(&c);
        return oc_array_take(v, k);
    }
    return c;
}

/* _container_from_values, containers.py:244-247 (consumes vals) */
static oc_t container_from_values(uint16_t *vals, int32_t n) {
    if (n > ARRAY_MAX) {
        oc_t b = bitset_from_positions(vals, n);
        free(vals);
        return b;
    }
    return oc_array_take(vals, n);
}

/* _container_from_words, containers.py:250-253 (consumes words) */
static oc_t container_from_words(uint64_t *words, int64_t card) {
    if (card <= ARRAY_MAX) {
        uint16_t *v = xmalloc((size_t)(card ? card : 1) * 2);
        int32_t k = extract_set_bits(words, BLOCK_WORDS, v);
        free(words);
        return oc_array_take(v, k);
    }
    return oc_bitset_take(words, card);
}

/* ------------------------------------------------ interval arithmetic */

typedef struct { int32_t n; int32_t *s; } ivl_t; /* s[2i]=start, s[2i+1]=end (closed) */

/* _intervals, containers.py:370-371 */
static ivl_t intervals_of_runs(const oc_t *c) {
    ivl_t r; r.n = c->n; r.s = xmalloc((size_t)(c->n ? c->n : 1) * 8);
    for (int32_t i = 0; i < c->n; i++) { r.s[2 * i] = c->v[2 * i]; r.s[2 * i + 1] = c->v[2 * i] + c->v[2 * i + 1]; }
    return r;
}

/* _intervals_from_values, containers.py:374-376 */
static ivl_t intervals_from_values(const uint16_t *v, int32_t n) {
    uint16_t *runs = xmalloc((size_t)(n ? n : 1) * 4);
    int32_t k = runs_from_positions(v, n, runs);
    ivl_t r; r.n = k; r.s = xmalloc((size_t)(k ? k : 1) * 8);
    for (int32_t i = 0; i < k; i++) { r.s[2 * i] = runs[2 * i]; r.s[2 * i + 1] = runs[2 * i] + runs[2 * i + 1]; }
    free(runs);
    return r;
}

/* _iv_union, containers.py:379-387 (heapq.merge of two sorted lists) */
static ivl_t iv_union(ivl_t a, ivl_t b) {
    ivl_t o; o.n = 0; o.s = xmalloc((size_t)(a.n + b.n + 1) * 8);
    int32_t i = 0, j = 0;
    while (i < a.n || j < b.n) {
        int32_t s, e;
        /* heapq.merge on (s,e) tuples: take the smaller tuple; ties -> first iterable */
        int take_a;
        if (i >= a.n) take_a = 0;
        else if (j >= b.n) take_a = 1;
        else if (a.s[2 * i] != b.s[2 * j]) take_a = a.s[2 * i] < b.s[2 * j];
        else take_a = a.s[2 * i + 1] <= b.s[2 * j + 1];
        if (take_a) { s = a.s[2 * i]; e = a.s[2 * i + 1]; i++; }
        else { s = b.s[2 * j]; e = b.s[2 * j + 1]; j++; }
        if (o.n && s <= o.s[2 * (o.n - 1) + 1] + 1) {
            if (e > o.s[2 * (o.n - 1) + 1]) o.s[2 * (o.n - 1) + 1] = e;
        } else { o.s[2 * o.n] = s; o.s[2 * o.n + 1] = e; o.n++; }
    }
    return o;
}

/* _iv_intersect, containers.py:390-402 */
static ivl_t iv_intersect(ivl_t a, ivl_t b) {
    ivl_t o; o.n = 0; o.s = xmalloc((size_t)(a.n + b.n + 1) * 8);
    int32_t i = 0, j = 0;
    while (i < a.n && j < b.n) {
        int32_t s = a.s[2 * i] > b.s[2 * j] ? a.s[2 * i] : b.s[2 * j];
        int32_t e = a.s[2 * i + 1] < b.s[2 * j + 1] ? a.s[2 * i + 1] : b.s[2 * j + 1];
        if (s <= e) { o.s[2 * o.n] = s; o.s[2 * o.n + 1] = e; o.n++; }
        if (a.s[2 * i + 1] < b.s[2 * j + 1]) i++; else j++;
    }
    return o;
}

/* _iv_difference, containers.py:405-424 */
static ivl_t iv_difference(ivl_t a, ivl_t b) {
    ivl_t o; o.n = 0; o.s = xmalloc((size_t)(a.n + b.n + 1) * 8);
    int32_t j = 0, nb = b.n;
    for (int32_t t = 0; t < a.n; t++) {
        int32_t s = a.s[2 * t], e = a.s[2 * t + 1];
        int32_t cur = s;
        while (j < nb && b.s[2 * j + 1] < cur) j++;
        int32_t k = j;
        while (k < nb && b.s[2 * k] <= e) {
            int32_t bs = b.s[2 * k], be = b.s[2 * k + 1];
            if (bs > cur) { o.s[2 * o.n] = cur; o.s[2 * o.n + 1] = bs - 1; o.n++; }
            cur = cur > be + 1 ? cur : be + 1;
            if (cur > e) break;
            k++;
        }
        if (cur <= e) { o.s[2 * o.n] = cur; o.s[2 * o.n + 1] = e; o.n++; }
    }
    return o;
}

/* _iv_xor, containers.py:427-428 */
static ivl_t iv_xor(ivl_t a, ivl_t b) {
    ivl_t d1 = iv_difference(a, b), d2 = iv_difference(b, a);
    ivl_t o = iv_union(d1, d2);
    free(d1.s); free(d2.s);
    return o;
}

/* _iv_card, containers.py:431-432 */
static int64_t iv_card(ivl_t a) {
    int64_t s = 0;
    for (int32_t i = 0; i < a.n; i++) s += a.s[2 * i + 1] - a.s[2 * i] + 1;
    return s;
}

/* _IV_OPS, containers.py:441-442 */
static ivl_t iv_op(int op, ivl_t a, ivl_t b) {
    switch (op) {
    case OP_AND: return iv_intersect(a, b);
    case OP_OR: return iv_union(a, b);
    case OP_ANDNOT: return iv_difference(a, b);
    default: return iv_xor(a, b);
    }
}

/* container_normalize(_run_from_intervals(ivs)), containers.py:435-438 + 208-223 */
static oc_t normalize_intervals(ivl_t iv) {
    uint16_t *runs = xmalloc((size_t)(iv.n ? iv.n : 1) * 4);
    for (int32_t i = 0; i < iv.n; i++) {
        runs[2 * i] = (uint16_t)iv.s[2 * i];
        runs[2 * i + 1] = (uint16_t)(iv.s[2 * i + 1] - iv.s[2 * i]);
    }
    return container_normalize(oc_run_take(runs, iv.n), 0);
}

/* ------------------------------------------------------ pairwise op */

static oc_t array_filter(const uint16_t *v, int32_t n, const uint8_t *mask, int want) {
    uint16_t *o = xmalloc((size_t)(n ? n : 1) * 2);
    int32_t k = 0;
    for (int32_t i = 0; i < n; i++) if ((mask[i] != 0) == want) o[k++] = v[i];
    return oc_array_take(o, k);
}

static oc_t array_probe_filter(const uint16_t *v, int32_t n, const uint64_t *w, int want) {
    uint16_t *o = xmalloc((size_t)(n ? n : 1) * 2);
    int32_t k = 0;
    for (int32_t i = 0; i < n; i++) if (bitset_probe(w, v[i]) == want) o[k++] = v[i];
    return oc_array_take(o, k);
}

static oc_t words_op_container(const uint64_t *x, const uint64_t *y, int op) {
    uint64_t *w = xmalloc(BLOCK_WORDS * 8);
    for (int i = 0; i < BLOCK_WORDS; i++) w[i] = word_op(op, x[i], y[i]);
    return container_from_words(w, popcount_block(w, BLOCK_WORDS));
}

/* container_pairwise, containers.py:450-529.  Empty results come back as an
 * empty array container. */
static oc_t container_pairwise(int op, const oc_t *a, const oc_t *b) {
    if (a->type == TAG_ARRAY && b->type == TAG_ARRAY) {
        int32_t cap = a->n + b->n;
        uint16_t *o = xmalloc((size_t)(cap ? cap : 1) * 2);
        int32_t k = array_kernel(op, a->v, a->n, b->v, b->n, o);
        return container_from_values(o, k);
    }
    if (a->type == TAG_BITSET && b->type == TAG_BITSET) {
        uint64_t *w = xmalloc(BLOCK_WORDS * 8);
        int64_t card = bitset_op_with_count(a->w, b->w, op, w);
        return container_from_words(w, card);
    }
    if (a->type == TAG_ARRAY && b->type == TAG_BITSET) {
        if (op == OP_AND) return array_probe_filter(a->v, a->n, b->w, 1);
        if (op == OP_ANDNOT) return array_probe_filter(a->v, a->n, b->w, 0);
        int64_t delta;
        uint64_t *w = bitset_apply_array(b->w, a->v, a->n, op == OP_OR ? 's' : 'f', 1, &delta);
        return container_from_words(w, b->card + delta);
    }
    if (a->type == TAG_BITSET && b->type == TAG_ARRAY) {
        if (op == OP_AND) return array_probe_filter(b->v, b->n, a->w, 1);
        int64_t delta;
        if (op == OP_ANDNOT) {
            uint64_t *w = bitset_apply_array(a->w, b->v, b->n, 'c', 1, &delta);
            return container_from_words(w, a->card + delta);
        }
        uint64_t *w = bitset_apply_array(a->w, b->v, b->n, op == OP_OR ? 's' : 'f', 1, &delta);
        return container_from_words(w, a->card + delta);
    }
    if (a->type == TAG_RUN && b->type == TAG_RUN) {
        ivl_t ia = intervals_of_runs(a), ib = intervals_of_runs(b);
        ivl_t r = iv_op(op, ia, ib);
        oc_t c = normalize_intervals(r);
        free(ia.s); free(ib.s); free(r.s);
        return c;
    }
    if (a->type == TAG_RUN && b->type == TAG_ARRAY) {
        if (op == OP_AND) {
            uint8_t *m = xmalloc((size_t)(b->n ? b->n : 1));
            values_in_runs(b->v, b->n, a->v, a->n, m);
            oc_t c = array_filter(b->v, b->n, m, 1);
            free(m);
            return c;
        }
        ivl_t ia = intervals_of_runs(a), ib = intervals_from_values(b->v, b->n);
        ivl_t r = iv_op(op, ia, ib);
        oc_t c = normalize_intervals(r);
        free(ia.s); free(ib.s); free(r.s);
        return c;
    }
    if (a->type == TAG_ARRAY && b->type == TAG_RUN) {
        if (op == OP_AND || op == OP_ANDNOT) {
            uint8_t *m = xmalloc((size_t)(a->n ? a->n : 1));
            values_in_runs(a->v, a->n, b->v, b->n, m);
            oc_t c = array_filter(a->v, a->n, m, op == OP_AND);
            free(m);
            return c;
        }
        ivl_t ia = intervals_from_values(a->v, a->n), ib = intervals_of_runs(b);
        ivl_t r = iv_op(op, ia, ib);
        oc_t c = normalize_intervals(r);
        free(ia.s); free(ib.s); free(r.s);
        return c;
    }
    if (a->type == TAG_RUN && b->type == TAG_BITSET) {
        uint64_t *rm = words_from_runs(a->v, a->n);
        oc_t c = words_op_container(rm, b->w, op);
        free(rm);
        return c;
    }
    /* bitset x run */
    uint64_t *rm = words_from_runs(b->v, b->n);
    oc_t c = words_op_container(a->w, rm, op);
    free(rm);
    return c;
}

/* _intersection_cardinality, containers.py:532-551 */
static int64_t intersection_cardinality(const oc_t *a, const oc_t *b) {
    if (a->type == TAG_ARRAY && b->type == TAG_ARRAY) return array_intersect(a->v, a->n, b->v, b->n, NULL);
    if (a->type == TAG_BITSET && b->type == TAG_BITSET) return bitset_op_count_only(a->w, b->w, OP_AND);
    if (a->type == TAG_ARRAY && b->type == TAG_BITSET) {
        int64_t s = 0; for (int32_t i = 0; i < a->n; i++) s += bitset_probe(b->w, a->v[i]); return s;
    }
    if (a->type == TAG_BITSET && b->type == TAG_ARRAY) {
        int64_t s = 0; for (int32_t i = 0; i < b->n; i++) s += bitset_probe(a->w, b->v[i]); return s;
    }
    if (a->type == TAG_RUN && b->type == TAG_RUN) {
        ivl_t ia = intervals_of_runs(a), ib = intervals_of_runs(b);
        ivl_t r = iv_intersect(ia, ib);
        int64_t s = iv_card(r);
        free(ia.s); free(ib.s); free(r.s);
        return s;
    }
    if ((a->type == TAG_RUN && b->type == TAG_ARRAY) || (a->type == TAG_ARRAY && b->type == TAG_RUN)) {
        const oc_t *ar = a->type == TAG_ARRAY ? a : b, *ru = a->type == TAG_RUN ? a : b;
        uint8_t *m = xmalloc((size_t)(ar->n ? ar->n : 1));
        values_in_runs(ar->v, ar->n, ru->v, ru->n, m);
        int64_t s = 0; for (int32_t i = 0; i < ar->n; i++) s += m[i];
        free(m);
        return s;
    }
    const oc_t *ru = a->type == TAG_RUN ? a : b, *bs = a->type == TAG_BITSET ? a : b;
    uint64_t *rm = words_from_runs(ru->v, ru->n);
    int64_t s = bitset_op_count_only(rm, bs->w, OP_AND);
    free(rm);
    return s;
}

/* container_pairwise_cardinality, containers.py:554-570 */
static int64_t container_pairwise_cardinality(int op, const oc_t *a, const oc_t *b) {
    if (a->type == TAG_ARRAY && b->type == TAG_ARRAY) return array_kernel(op, a->v, a->n, b->v, b->n, NULL);
    if (a->type == TAG_BITSET && b->type == TAG_BITSET) return bitset_op_count_only(a->w, b->w, op);
    int64_t inter = intersection_cardinality(a, b);
    if (op == OP_AND) return inter;
    if (op == OP_OR) return oc_len(a) + oc_len(b) - inter;
    if (op == OP_ANDNOT) return oc_len(a) - inter;
    return oc_len(a) + oc_len(b) - 2 * inter;
}

/* ------------------------------------------------------------- bitmaps */

static void bm_init(obm_t *b, int32_t cap) {
    b->n = 0; b->cap = cap > 4 ? cap : 4;
    b->keys = xmalloc((size_t)b->cap * 2);
    b->c = xmalloc((size_t)b->cap * sizeof(oc_t));
}
static void bm_push(obm_t *b, uint16_t key, oc_t c) {
    if (b->n == b->cap) {
        b->cap *= 2;
        b->keys = realloc(b->keys, (size_t)b->cap * 2);
        b->c = realloc(b->c, (size_t)b->cap * sizeof(oc_t));
        if (!b->keys || !b->c) abort();
    }
    b->keys[b->n] = key; b->c[b->n] = c; b->n++;
}
static void bm_free(obm_t *b) {
    for (int32_t i = 0; i < b->n; i++) oc_free(&b->c[i]);
    free(b->keys); free(b->c);
    b->keys = NULL; b->c = NULL; b->n = 0;
}
static int64_t bm_len(const obm_t *b) {
    int64_t s = 0;
    for (int32_t i = 0; i < b->n; i++) s += oc_len(&b->c[i]);
    return s;
}

/* RoaringBitmap.op, bitmap.py:169-210 (_KEEP_A/_KEEP_B :21-22) */
static obm_t bm_op(int op, const obm_t *A, const obm_t *B) {
    int keep_a = op == OP_OR || op == OP_XOR || op == OP_ANDNOT;
    int keep_b = op == OP_OR || op == OP_XOR;
    obm_t R; bm_init(&R, A->n + B->n);
    int32_t i = 0, j = 0;
    while (i < A->n && j < B->n) {
        uint16_t x = A->keys[i], y = B->keys[j];
        if (x == y) {
            oc_t r = container_pairwise(op, &A->c[i], &B->c[j]);
            if (oc_len(&r)) bm_push(&R, x, r); else oc_free(&r);
            i++; j++;
        } else if (x < y) {
            if (keep_a) bm_push(&R, x, oc_copy(&A->c[i]));
            i++;
        } else {
            if (keep_b) bm_push(&R, y, oc_copy(&B->c[j]));
            j++;
        }
    }
    if (keep_a) for (; i < A->n; i++) bm_push(&R, A->keys[i], oc_copy(&A->c[i]));
    if (keep_b) for (; j < B->n; j++) bm_push(&R, B->keys[j], oc_copy(&B->c[j]));
    return R;
}

/* RoaringBitmap.op_cardinality, bitmap.py:212-241 */
static int64_t bm_op_cardinality(int op, const obm_t *A, const obm_t *B) {
    int64_t inter = 0;
    int32_t i = 0, j = 0;
    while (i < A->n && j < B->n) {
        uint16_t x = A->keys[i], y = B->keys[j];
        if (x == y) { inter += container_pairwise_cardinality(OP_AND, &A->c[i], &B->c[j]); i++; j++; }
        else if (x < y) i++;
        else j++;
    }
    if (op == OP_AND) return inter;
    if (op == OP_OR) return bm_len(A) + bm_len(B) - inter;
    if (op == OP_ANDNOT) return bm_len(A) - inter;
    return bm_len(A) + bm_len(B) - 2 * inter;
}

/* RoaringBitmap.union_many, bitmap.py:257-304.  The accumulator is indexed
 * directly by the 16-bit key (equivalent to the bisect/insert list walk). */
static obm_t bm_union_many(const obm_t *const *bms, int32_t n) {
    obm_t R;
    if (n == 0) { bm_init(&R, 4); return R; }
    oc_t *slot = xcalloc(65536, sizeof(oc_t));
    uint8_t *present = xcalloc(65536, 1), *dirty = xcalloc(65536, 1);
    for (int32_t i = 0; i < bms[0]->n; i++) {
        slot[bms[0]->keys[i]] = oc_copy(&bms[0]->c[i]);
        present[bms[0]->keys[i]] = 1;
    }
    for (int32_t b = 1; b < n; b++) {
        const obm_t *bm = bms[b];
        for (int32_t t = 0; t < bm->n; t++) {
            uint16_t key = bm->keys[t];
            const oc_t *cont = &bm->c[t];
            if (!present[key]) { slot[key] = oc_copy(cont); present[key] = 1; continue; }
            oc_t *cur = &slot[key];
            if (cur->type == TAG_BITSET) {
                if (cont->type == TAG_BITSET) {
                    for (int k = 0; k < BLOCK_WORDS; k++) cur->w[k] |= cont->w[k];
                } else if (cont->type == TAG_ARRAY) {
                    int64_t d;
                    uint64_t *w = bitset_apply_array(cur->w, cont->v, cont->n, 's', 0, &d);
                    free(cur->w); cur->w = w;
                } else {
                    uint64_t *rm = words_from_runs(cont->v, cont->n);
                    for (int k = 0; k < BLOCK_WORDS; k++) cur->w[k] |= rm[k];
                    free(rm);
                }
                cur->card = -1; dirty[key] = 1;
            } else if (cont->type == TAG_BITSET) {
                uint64_t *words = xmalloc(BLOCK_WORDS * 8);
                memcpy(words, cont->w, BLOCK_WORDS * 8);
                if (cur->type == TAG_ARRAY) {
                    int64_t d;
                    uint64_t *w2 = bitset_apply_array(words, cur->v, cur->n, 's', 0, &d);
                    free(words); words = w2;
                } else {
                    uint64_t *rm = words_from_runs(cur->v, cur->n);
                    for (int k = 0; k < BLOCK_WORDS; k++) words[k] |= rm[k];
                    free(rm);
                }
                oc_free(cur);
                *cur = oc_bitset_take(words, -1);
                dirty[key] = 1;
            } else {
                oc_t r = container_pairwise(OP_OR, cur, cont);
                oc_free(cur);
                *cur = r;
            }
        }
    }
    int32_t cnt = 0;
    for (int k = 0; k < 65536; k++) cnt += present[k];
    bm_init(&R, cnt);
    for (int k = 0; k < 65536; k++) {
        if (!present[k]) continue;
        if (dirty[k]) slot[k].card = popcount_block(slot[k].w, BLOCK_WORDS);
        bm_push(&R, (uint16_t)k, slot[k]);
    }
    free(slot); free(present); free(dirty);
    return R;
}

/* RoaringBitmap.run_optimize, bitmap.py:308-316 */
static int bm_run_optimize(obm_t *b) {
    int changed = 0;
    for (int32_t i = 0; i < b->n; i++) {
        int t0 = b->c[i].type;
        b->c[i] = container_normalize(b->c[i], 1);
        if (b->c[i].type != t0) changed = 1;
    }
    return changed;
}

static int cmp_u64(const void *x, const void *y) {
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return a < b ? -1 : a > b;
}

/* RoaringBitmap.from_values, bitmap.py:40-62.  Returns -1 if a value does not
 * fit in 32 bits (the reference's ValueError). */
static int bm_from_values(const uint64_t *vals_in, int64_t n, obm_t *out) {
    bm_init(out, 16);
    if (n == 0) return 0;
    uint64_t *v = xmalloc((size_t)n * 8);
    memcpy(v, vals_in, (size_t)n * 8);
    int sorted = 1;
    for (int64_t i = 1; i < n; i++) if (v[i] <= v[i - 1]) { sorted = 0; break; }
    if (!sorted) qsort(v, (size_t)n, 8, cmp_u64);
    int64_t m = 0; /* np.unique */
    for (int64_t i = 0; i < n; i++) if (m == 0 || v[i] != v[m - 1]) v[m++] = v[i];
    if (v[m - 1] > 0xFFFFFFFFULL) { free(v); return -1; }
    int64_t s = 0;
    while (s < m) {
        uint64_t key = v[s] >> 16;
        int64_t e = s;
        while (e < m && (v[e] >> 16) == key) e++;
        int32_t cnt = (int32_t)(e - s);
        uint16_t *lows = xmalloc((size_t)cnt * 2);
        for (int32_t k = 0; k < cnt; k++) lows[k] = (uint16_t)(v[s + k] & 0xFFFF);
        if (cnt <= ARRAY_MAX) bm_push(out, (uint16_t)key, oc_array_take(lows, cnt));
        else { bm_push(out, (uint16_t)key, bitset_from_positions(lows, cnt)); free(lows); }
        s = e;
    }
    free(v);
    return 0;
}

/* ----------------------------------------------------------- serde.py */

/* serialize, serde.py:69-84 */
static size_t wire_size(const obm_t *b) {
    size_t s = 8 + 8 * (size_t)b->n;
    for (int32_t i = 0; i < b->n; i++) {
        const oc_t *c = &b->c[i];
        if (c->type == TAG_ARRAY) s += 2 * (size_t)c->n;
        else if (c->type == TAG_BITSET) s += 8192;
        else s += 2 + 4 * (size_t)c->n;
    }
    return s;
}

static void put16(uint8_t *p, uint16_t x) { p[0] = (uint8_t)x; p[1] = (uint8_t)(x >> 8); }
static void put32(uint8_t *p, uint32_t x) { for (int i = 0; i < 4; i++) p[i] = (uint8_t)(x >> (8 * i)); }
static uint16_t get16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint32_t get32(const uint8_t *p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24); }
static uint64_t get64(const uint8_t *p) { return (uint64_t)get32(p) | ((uint64_t)get32(p + 4) << 32); }

static uint8_t *serialize(const obm_t *b, size_t *len) {
    size_t n = wire_size(b);
    uint8_t *o = xmalloc(n), *p = o;
    memcpy(p, "ROAR", 4); put32(p + 4, (uint32_t)b->n); p += 8;
    for (int32_t i = 0; i < b->n; i++) {
        put16(p, b->keys[i]); p[2] = (uint8_t)b->c[i].type; p[3] = 0;
        put32(p + 4, (uint32_t)oc_len(&b->c[i])); p += 8;
    }
    for (int32_t i = 0; i < b->n; i++) {
        const oc_t *c = &b->c[i];
        if (c->type == TAG_ARRAY) { for (int32_t k = 0; k < c->n; k++) put16(p + 2 * k, c->v[k]); p += 2 * (size_t)c->n; }
        else if (c->type == TAG_BITSET) {
            for (int k = 0; k < BLOCK_WORDS; k++) { put32(p, (uint32_t)c->w[k]); put32(p + 4, (uint32_t)(c->w[k] >> 32)); p += 8; }
        } else {
            put16(p, (uint16_t)c->n); p += 2;
            for (int32_t k = 0; k < 2 * c->n; k++) put16(p + 2 * k, c->v[k]);
            p += 4 * (size_t)c->n;
        }
    }
    *len = n;
    return o;
}

/* deserialize, serde.py:87-169.  On error returns -1 with *err_off and msg
 * set exactly as the reference's DecodeError(offset, message). */
static int deserialize(const uint8_t *d, size_t len, obm_t *out, int64_t *err_off, char *msg, size_t msgcap) {
    size_t off = 0;
#define NEED(nb, what) do { \
        if (len - off < (size_t)(nb)) { \
            *err_off = (int64_t)off; \
            snprintf(msg, msgcap, "truncated %s: need %llu bytes, have %llu", what, \
                     (unsigned long long)(nb), (unsigned long long)(len - off)); \
            goto fail; } \
        start = off; off += (nb); } while (0)
#define FAIL(o, ...) do { *err_off = (int64_t)(o); snprintf(msg, msgcap, __VA_ARGS__); goto fail; } while (0)
    size_t start = 0;
    uint16_t *dkey = NULL; uint8_t *dtag = NULL; uint32_t *dcard = NULL;
    bm_init(out, 4);
    NEED(4, "magic");
    if (memcmp(d + start, "ROAR", 4) != 0) FAIL(0, "bad magic");
    NEED(4, "container count");
    uint32_t count = get32(d + start);
    /* descriptors are bounded by the remaining length */
    size_t maxd = (len - off) / 8 + 1;
    size_t alloc = count < maxd ? count : maxd;
    dkey = xmalloc(alloc * 2 + 2); dtag = xmalloc(alloc + 1); dcard = xmalloc(alloc * 4 + 4);
    int64_t prev_key = -1;
    for (uint32_t i = 0; i < count; i++) {
        NEED(8, "descriptor");
        uint16_t key = get16(d + start);
        uint8_t tag = d[start + 2], pad = d[start + 3];
        uint32_t card = get32(d + start + 4);
        if (pad != 0) FAIL(start + 3, "nonzero descriptor pad");
        if (tag != TAG_ARRAY && tag != TAG_BITSET && tag != TAG_RUN) FAIL(start + 2, "unknown container type %u", tag);
        if ((int64_t)key <= prev_key) FAIL(start, "keys not strictly increasing at %u", key);
        prev_key = key;
        dkey[i] = key; dtag[i] = tag; dcard[i] = card;
    }
    for (uint32_t i = 0; i < count; i++) {
        uint32_t card = dcard[i];
        if (dtag[i] == TAG_ARRAY) {
            if (!(card >= 1 && card <= ARRAY_MAX)) FAIL(off, "array cardinality %u out of range", card);
            NEED(2 * (size_t)card, "array payload");
            uint16_t *v = xmalloc((size_t)card * 2);
            for (uint32_t k = 0; k < card; k++) v[k] = get16(d + start + 2 * k);
            for (uint32_t k = 1; k < card; k++)
                if (v[k] <= v[k - 1]) { free(v); FAIL(start, "array values not strictly increasing"); }
            bm_push(out, dkey[i], oc_array_take(v, (int32_t)card));
        } else if (dtag[i] == TAG_BITSET) {
            NEED(8192, "bitset payload");
            uint64_t *w = xmalloc(8192);
            for (int k = 0; k < BLOCK_WORDS; k++) w[k] = get64(d + start + 8 * k);
            int64_t tc = popcount_block(w, BLOCK_WORDS);
            if (tc != card) { free(w); FAIL(start, "cardinality mismatch: descriptor says %u, payload holds %lld", card, (long long)tc); }
            if (card <= ARRAY_MAX) { free(w); FAIL(start, "bitset container with only %u values", card); }
            bm_push(out, dkey[i], oc_bitset_take(w, card));
        } else {
            NEED(2, "run count");
            uint16_t nr = get16(d + start);
            if (nr == 0) FAIL(start, "empty run container");
            NEED(4 * (size_t)nr, "run payload");
            uint16_t *r = xmalloc((size_t)nr * 4);
            for (int k = 0; k < 2 * nr; k++) r[k] = get16(d + start + 2 * k);
            int64_t tc = nr;
            for (int k = 0; k < nr; k++) {
                if ((int32_t)r[2 * k] + r[2 * k + 1] > 0xFFFF) { free(r); FAIL(start, "run escapes the 16-bit chunk"); }
            }
            for (int k = 1; k < nr; k++) {
                if (!((int32_t)r[2 * k] > (int32_t)r[2 * k - 2] + r[2 * k - 1] + 1)) { free(r); FAIL(start, "runs overlap or are adjacent"); }
            }
            for (int k = 0; k < nr; k++) tc += r[2 * k + 1];
            if (tc != card) { free(r); FAIL(start, "cardinality mismatch: descriptor says %u, runs hold %lld", card, (long long)tc); }
            if (!run_admissible(card, nr)) { free(r); FAIL(start, "run form is not the smallest representation"); }
            bm_push(out, dkey[i], oc_run_take(r, nr));
        }
    }
    if (off != len) FAIL(off, "%llu trailing bytes", (unsigned long long)(len - off));
    free(dkey); free(dtag); free(dcard);
    return 0;
fail:
    free(dkey); free(dtag); free(dcard);
    bm_free(out);
    return -1;
#undef NEED
#undef FAIL
}

/* ============================================================ C ABI */
/* All entry points take / return wire images.  Return 0 on success. */

static __thread char g_err[512];
static __thread int64_t g_err_off;

const char *orc_last_error(void) { return g_err; }
int64_t orc_last_error_offset(void) { return g_err_off; }
void orc_free(void *p) { free(p); }

static int load(const uint8_t *w, size_t n, obm_t *b) {
    return deserialize(w, n, b, &g_err_off, g_err, sizeof g_err);
}

/* deserialize check: 0 ok, -1 DecodeError (orc_last_error*) */
int orc_check(const uint8_t *w, size_t n) {
    obm_t b;
    if (load(w, n, &b)) return -1;
    bm_free(&b);
    return 0;
}

/* reserialize (round trip) */
int orc_roundtrip(const uint8_t *w, size_t n, uint8_t **out, size_t *lout) {
    obm_t b;
    if (load(w, n, &b)) return -1;
    *out = serialize(&b, lout);
    bm_free(&b);
    return 0;
}

int orc_op(int op, const uint8_t *wa, size_t la, const uint8_t *wb, size_t lb,
           uint8_t **out, size_t *lout) {
    if (op < 0 || op > 3) { snprintf(g_err, sizeof g_err, "unknown op %d", op); return -2; }
    obm_t A, B;
    if (load(wa, la, &A)) return -1;
    if (load(wb, lb, &B)) { bm_free(&A); return -1; }
    obm_t R = bm_op(op, &A, &B);
    *out = serialize(&R, lout);
    bm_free(&A); bm_free(&B); bm_free(&R);
    return 0;
}

int orc_op_cardinality(int op, const uint8_t *wa, size_t la, const uint8_t *wb, size_t lb,
                       int64_t *card) {
    if (op < 0 || op > 3) { snprintf(g_err, sizeof g_err, "unknown op %d", op); return -2; }
    obm_t A, B;
    if (load(wa, la, &A)) return -1;
    if (load(wb, lb, &B)) { bm_free(&A); return -1; }
    *card = bm_op_cardinality(op, &A, &B);
    bm_free(&A); bm_free(&B);
    return 0;
}

/* container_pairwise_cardinality over the single containers of two
 * one-container images (containers.py:554-570); the key is ignored. */
int orc_container_pairwise_cardinality(int op, const uint8_t *wa, size_t la, const uint8_t *wb,
                                       size_t lb, int64_t *card) {
    obm_t A, B;
    if (load(wa, la, &A)) return -1;
    if (load(wb, lb, &B)) { bm_free(&A); return -1; }
    if (A.n != 1 || B.n != 1) { bm_free(&A); bm_free(&B); snprintf(g_err, sizeof g_err, "need one container per image"); return -2; }
    *card = container_pairwise_cardinality(op, &A.c[0], &B.c[0]);
    bm_free(&A); bm_free(&B);
    return 0;
}

int orc_union_many(const uint8_t *buf, const uint64_t *offs, int32_t n, uint8_t **out, size_t *lout) {
    obm_t *bm = xmalloc(sizeof(obm_t) * (size_t)(n ? n : 1));
    const obm_t **pp = xmalloc(sizeof(obm_t *) * (size_t)(n ? n : 1));
    for (int32_t i = 0; i < n; i++) {
        if (load(buf + offs[i], offs[i + 1] - offs[i], &bm[i])) {
            for (int32_t k = 0; k < i; k++) bm_free(&bm[k]);
            free(bm); free(pp); return -1;
        }
        pp[i] = &bm[i];
    }
    obm_t R = bm_union_many(pp, n);
    *out = serialize(&R, lout);
    bm_free(&R);
    for (int32_t i = 0; i < n; i++) bm_free(&bm[i]);
    free(bm); free(pp);
    return 0;
}

int orc_from_values(const uint64_t *v, int64_t n, uint8_t **out, size_t *lout) {
    obm_t b;
    if (bm_from_values(v, n, &b)) { snprintf(g_err, sizeof g_err, "values must fit in 32 bits"); return -3; }
    *out = serialize(&b, lout);
    bm_free(&b);
    return 0;
}

int orc_run_optimize(const uint8_t *w, size_t n, uint8_t **out, size_t *lout, int *changed) {
    obm_t b;
    if (load(w, n, &b)) return -1;
    *changed = bm_run_optimize(&b);
    *out = serialize(&b, lout);
    bm_free(&b);
    return 0;
}

/* to_array, bitmap.py:136-144 */
int orc_to_array(const uint8_t *w, size_t n, uint32_t **out, int64_t *nout) {
    obm_t b;
    if (load(w, n, &b)) return -1;
    int64_t tot = bm_len(&b);
    uint32_t *o = xmalloc((size_t)(tot ? tot : 1) * 4);
    uint16_t *tmp = xmalloc(65536 * 2);
    int64_t k = 0;
    for (int32_t i = 0; i < b.n; i++) {
        int32_t m = container_positions(&b.c[i], tmp);
        for (int32_t t = 0; t < m; t++) o[k++] = ((uint32_t)b.keys[i] << 16) | tmp[t];
    }
    free(tmp);
    bm_free(&b);
    *out = o; *nout = tot;
    return 0;
}

int64_t orc_cardinality(const uint8_t *w, size_t n) {
    obm_t b;
    if (load(w, n, &b)) return -1;
    int64_t s = bm_len(&b);
    bm_free(&b);
    return s;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------- batched entry points
 * Images are concatenated in `buf` with offsets offs[0..n].  Pair p operates
 * on images ia[p] of A and ib[p] of B.  Independent pairs run in parallel
 * (OpenMP over pairs; each pair is the single-threaded reference algorithm). */

/* Materialized ops: writes per-pair output images into a caller-provided
 * buffer sized by a first call with out==NULL (returns sizes in out_len). */
int orc_op_batch(int op, const uint8_t *bufA, const uint64_t *offA, const uint8_t *bufB,
                 const uint64_t *offB, const int64_t *ia, const int64_t *ib, int64_t npairs,
                 uint8_t **outs, uint64_t *out_len, int nthreads) {
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(|:err)
#endif
    for (int64_t p = 0; p < npairs; p++) {
        obm_t A, B;
        char m[256]; int64_t eo;
        if (deserialize(bufA + offA[ia[p]], offA[ia[p] + 1] - offA[ia[p]], &A, &eo, m, sizeof m)) { err |= 1; continue; }
        if (deserialize(bufB + offB[ib[p]], offB[ib[p] + 1] - offB[ib[p]], &B, &eo, m, sizeof m)) { bm_free(&A); err |= 1; continue; }
        obm_t R = bm_op(op, &A, &B);
        size_t l;
        outs[p] = serialize(&R, &l);
        out_len[p] = l;
        bm_free(&A); bm_free(&B); bm_free(&R);
    }
    return err ? -1 : 0;
}

int orc_op_cardinality_batch(int op, const uint8_t *bufA, const uint64_t *offA, const uint8_t *bufB,
                             const uint64_t *offB, const int64_t *ia, const int64_t *ib,
                             int64_t npairs, int64_t *cards, int nthreads) {
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads) reduction(|:err)
#endif
    for (int64_t p = 0; p < npairs; p++) {
        obm_t A, B;
        char m[256]; int64_t eo;
        if (deserialize(bufA + offA[ia[p]], offA[ia[p] + 1] - offA[ia[p]], &A, &eo, m, sizeof m)) { err |= 1; continue; }
        if (deserialize(bufB + offB[ib[p]], offB[ib[p] + 1] - offB[ib[p]], &B, &eo, m, sizeof m)) { bm_free(&A); err |= 1; continue; }
        cards[p] = bm_op_cardinality(op, &A, &B);
        bm_free(&A); bm_free(&B);
    }
    return err ? -1 : 0;
}

/* container_pairwise_cardinality over one-container images, batched (C3). */
int orc_container_card_batch(int op, const uint8_t *bufA, const uint64_t *offA, const uint8_t *bufB,
                             const uint64_t *offB, const int64_t *ia, const int64_t *ib,
                             int64_t npairs, int64_t *cards, int nthreads) {
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(|:err)
#endif
    for (int64_t p = 0; p < npairs; p++) {
        obm_t A, B;
        char m[256]; int64_t eo;
        if (deserialize(bufA + offA[ia[p]], offA[ia[p] + 1] - offA[ia[p]], &A, &eo, m, sizeof m)) { err |= 1; continue; }
        if (deserialize(bufB + offB[ib[p]], offB[ib[p] + 1] - offB[ib[p]], &B, &eo, m, sizeof m)) { bm_free(&A); err |= 1; continue; }
        if (A.n != 1 || B.n != 1) err |= 1;
        else cards[p] = container_pairwise_cardinality(op, &A.c[0], &B.c[0]);
        bm_free(&A); bm_free(&B);
    }
    return err ? -1 : 0;
}

/* All-pairs |A∩B| (config 5): out[k] for i<j in row-major order. */
int orc_all_pairs_and(const uint8_t *buf, const uint64_t *offs, int64_t n, const int64_t *pi,
                      const int64_t *pj, int64_t npairs, int64_t *inter, int nthreads) {
    obm_t *bm = xmalloc(sizeof(obm_t) * (size_t)(n ? n : 1));
    int err = 0;
    for (int64_t i = 0; i < n; i++) {
        char m[256]; int64_t eo;
        if (deserialize(buf + offs[i], offs[i + 1] - offs[i], &bm[i], &eo, m, sizeof m)) {
            for (int64_t k = 0; k < i; k++) bm_free(&bm[k]);
            free(bm); return -1;
        }
    }
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
    for (int64_t p = 0; p < npairs; p++)
        inter[p] = bm_op_cardinality(OP_AND, &bm[pi[p]], &bm[pj[p]]);
    for (int64_t i = 0; i < n; i++) bm_free(&bm[i]);
    free(bm);
    return err;
}

/* ------------------------------------------------ in-memory sessions (CPU baseline)
 * Deserialize once, then time only the reference algorithm on in-memory
 * bitmaps, the way the reference harness times RoaringBitmap objects
 * (bench/harness.py:205-239). */
typedef struct { int64_t n; obm_t *bm; } obatch_t;

void *orc_batch_load(const uint8_t *buf, const uint64_t *offs, int64_t n, int nthreads) {
    obatch_t *b = xmalloc(sizeof(obatch_t));
    b->n = n;
    b->bm = xcalloc((size_t)(n ? n : 1), sizeof(obm_t));
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(|:err)
#endif
    for (int64_t i = 0; i < n; i++) {
        char m[256]; int64_t eo;
        if (deserialize(buf + offs[i], offs[i + 1] - offs[i], &b->bm[i], &eo, m, sizeof m)) err |= 1;
    }
    if (err) { for (int64_t i = 0; i < n; i++) if (b->bm[i].keys) bm_free(&b->bm[i]); free(b->bm); free(b); return NULL; }
    return b;
}

void orc_batch_free(void *h) {
    obatch_t *b = h;
    if (!b) return;
    for (int64_t i = 0; i < b->n; i++) bm_free(&b->bm[i]);
    free(b->bm); free(b);
}

/* kind: 0 = RoaringBitmap.op (result built then dropped; its cardinality is
 * returned), 1 = op_cardinality, 2 = container_pairwise (one-container
 * bitmaps), 3 = container_pairwise_cardinality. */
int orc_batch_run(int op, int kind, void *ha, void *hb, const int64_t *ia, const int64_t *ib, int64_t npairs,
                  int64_t *out, int nthreads) {
    obatch_t *A = ha, *B = hb;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t p = 0; p < npairs; p++) {
        const obm_t *a = &A->bm[ia[p]], *b = &B->bm[ib[p]];
        if (kind == 0) {
            obm_t R = bm_op(op, a, b);
            out[p] = bm_len(&R);
            bm_free(&R);
        } else if (kind == 1) {
            out[p] = bm_op_cardinality(op, a, b);
        } else if (kind == 2) {
            oc_t r = container_pairwise(op, &a->c[0], &b->c[0]);
            out[p] = oc_len(&r);
            oc_free(&r);
        } else {
            out[p] = container_pairwise_cardinality(op, &a->c[0], &b->c[0]);
        }
    }
    return 0;
}

/* ------------------------------------------------ content digests (parity at scale)
 * A 64-bit digest of a bitmap's exact content -- keys, container types,
 * cardinalities and payloads, i.e. everything its wire image
 * (serde.py:3-10) holds -- so full-size results can be compared with the
 * GPU's (rs_batch_digest, include/roaring_b200.h) without moving them.
 * Definition (identical in csrc/rs_egress.cu):
 *   mix(z)      = SplitMix64 finalizer
 *   h(c)        = mix(key<<48 | tag<<40 | card) + sum_i term_i
 *     array:    term_i = mix((i<<16 | v_i) + K_ARRAY)
 *     bitset:   term_w = mix(word_w + w * K_BITSET)
 *     run:      term_r = mix((r<<32 | start_r<<16 | len_r) + K_RUN)
 *   digest(bm)  = sum_j mix(h(c_j) + (j+1) * K_POS)     (0 for the empty bitmap)
 * Sums are mod 2^64. */
#define DG_K_ARRAY 0x243F6A8885A308D3ull
#define DG_K_BITSET 0x13198A2E03707344ull
#define DG_K_RUN 0xA4093822299F31D0ull
#define DG_K_POS 0x082EFA98EC4E6C89ull

static inline uint64_t dg_mix(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t dg_container(uint16_t key, const oc_t *c) {
    uint64_t card = (uint64_t)oc_len(c);
    uint64_t h = dg_mix(((uint64_t)key << 48) | ((uint64_t)c->type << 40) | card);
    if (c->type == TAG_ARRAY) {
        for (int32_t i = 0; i < c->n; i++) h += dg_mix((((uint64_t)i << 16) | c->v[i]) + DG_K_ARRAY);
    } else if (c->type == TAG_BITSET) {
        for (int w = 0; w < BLOCK_WORDS; w++) h += dg_mix(c->w[w] + (uint64_t)w * DG_K_BITSET);
    } else {
        for (int32_t r = 0; r < c->n; r++)
            h += dg_mix((((uint64_t)r << 32) | ((uint64_t)c->v[2 * r] << 16) | c->v[2 * r + 1]) + DG_K_RUN);
    }
    return h;
}

static uint64_t dg_bitmap(const obm_t *b) {
    uint64_t d = 0;
    for (int32_t j = 0; j < b->n; j++) d += dg_mix(dg_container(b->keys[j], &b->c[j]) + (uint64_t)(j + 1) * DG_K_POS);
    return d;
}

/* digests of n wire images */
int orc_digest_images(const uint8_t *buf, const uint64_t *offs, int64_t n, uint64_t *out, int nthreads) {
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads) reduction(|:err)
#endif
    for (int64_t i = 0; i < n; i++) {
        obm_t b;
        char m[256]; int64_t eo;
        if (deserialize(buf + offs[i], offs[i + 1] - offs[i], &b, &eo, m, sizeof m)) { err |= 1; continue; }
        out[i] = dg_bitmap(&b);
        bm_free(&b);
    }
    return err ? -1 : 0;
}

/* digests of the results of a batched op (kind 0: RoaringBitmap.op; kind 2:
 * container_pairwise over one-container bitmaps, result at key 0 of A's key)
 * on in-memory sessions, without serializing the results */
int orc_batch_digest(int op, int kind, void *ha, void *hb, const int64_t *ia, const int64_t *ib, int64_t npairs,
                     uint64_t *out, int nthreads) {
    obatch_t *A = ha, *B = hb;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t p = 0; p < npairs; p++) {
        const obm_t *a = &A->bm[ia[p]], *b = &B->bm[ib[p]];
        if (kind == 0) {
            obm_t R = bm_op(op, a, b);
            out[p] = dg_bitmap(&R);
            bm_free(&R);
        } else {
            oc_t r = container_pairwise(op, &a->c[0], &b->c[0]);
            out[p] = oc_len(&r) ? dg_mix(dg_container(a->keys[0], &r) + DG_K_POS) : 0;
            oc_free(&r);
        }
    }
    return 0;
}

/* digest of union_many over all images of a session, in order */
int orc_union_digest(void *ha, uint64_t *out) {
    obatch_t *A = ha;
    const obm_t **pp = xmalloc(sizeof(obm_t *) * (size_t)(A->n ? A->n : 1));
    for (int64_t i = 0; i < A->n; i++) pp[i] = &A->bm[i];
    obm_t R = bm_union_many(pp, (int32_t)A->n);
    *out = dg_bitmap(&R);
    bm_free(&R);
    free(pp);
    return 0;
}
