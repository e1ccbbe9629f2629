/*
 * epsgraph_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm for the eps-graph
 * build path (reference package `epsgraph` 0.1.0, /root/reference/pkg/src/
 * epsgraph).  It is the *checker* for the CUDA product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product package never links or imports it.
 *
 * Parity of this restatement is pinned by tests/golden/ (fixtures produced by
 * running the reference itself, tests/golden/make_golden.py) and checked by
 * tests/test_oracle_golden.py.
 *
 * Every function cites the reference lines it restates.  Arithmetic that the
 * reference performs in fp64 with separate multiply and add (numba emits
 * vmulsd + vaddsd, no FMA) is compiled here with -ffp-contract=off so the
 * sign bits are bit-identical.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_BAD_ARG -1
#define OR_NOMEM -2

/* ------------------------------------------------------------------------ */
/* Projection: lsh.py:96-113 (_sign_bits) and lsh.py:128-147 (_project_words) */
/* bit (i,t) = (sum_q x[i,q]*r[t,q] > 0.0) with a sequential fp64 sum.         */
/* Packed little-endian: bit t -> word t/64, position t%64 (bitpool.py:1-7,    */
/* bitpool.py:125-141).                                                        */
/* ------------------------------------------------------------------------ */
int or_project_words(const double *x, int64_t n, int32_t dim,
                     const double *r, int32_t length,
                     uint64_t *words, int32_t threads)
{
    if (n < 0 || dim < 1 || length < 1) return OR_BAD_ARG;
    const int32_t W = (length + 63) / 64;
    (void)threads;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
        uint64_t *wrow = words + i * W;
        for (int32_t w = 0; w < W; ++w) wrow[w] = 0;
        const double *xi = x + i * dim;
        for (int32_t t = 0; t < length; ++t) {
            const double *rt = r + (int64_t)t * dim;
            double acc = 0.0;
            for (int32_t q = 0; q < dim; ++q) {
                double p = xi[q] * rt[q];   /* rounded product   */
                acc = acc + p;              /* rounded sum        */
            }
            if (acc > 0.0) wrow[t >> 6] |= (uint64_t)1 << (t & 63);
        }
    }
    return OR_OK;
}

/* Row validation: lsh.py:48-57 (non-finite) and lsh.py:121-125 (zero norm).
 * Returns the first offending row or -1; norms are fp64 sqrt(sum x^2). */
int64_t or_first_nonfinite(const double *x, int64_t n, int32_t dim)
{
    for (int64_t i = 0; i < n; ++i)
        for (int32_t q = 0; q < dim; ++q)
            if (!isfinite(x[i * dim + q])) return i;
    return -1;
}

/* ------------------------------------------------------------------------ */
/* Block partition: bitpool.py:44-69.  First length%k blocks get one extra.  */
/* ------------------------------------------------------------------------ */
int or_block_partition(int32_t length, int32_t k, int64_t *bounds)
{
    if (k < 1 || k > length) return OR_BAD_ARG;
    int32_t base = length / k, rem = length % k;
    bounds[0] = 0;
    for (int32_t b = 0; b < k; ++b)
        bounds[b + 1] = bounds[b] + base + (b < rem ? 1 : 0);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Masked keys: bitpool.py:224-253 (masked_key_table).  Kept blocks are      */
/* concatenated in ascending position order and chunked MSB-first into       */
/* chunk_bits-wide values; the final chunk is zero padded at the low end.    */
/* ------------------------------------------------------------------------ */
static int32_t kept_positions(const int64_t *bounds, int32_t k, const int32_t *mask,
                              int32_t d, int32_t *pos)
{
    int32_t m = 0, mi = 0;
    for (int32_t b = 0; b < k; ++b) {
        if (mi < d && mask[mi] == b) { ++mi; continue; }
        for (int64_t t = bounds[b]; t < bounds[b + 1]; ++t) pos[m++] = (int32_t)t;
    }
    return m;
}

static void masked_keys(const uint64_t *words, int64_t n, int32_t W,
                        const int32_t *pos, int32_t npos, int32_t chunk_bits,
                        int32_t nchunks, int64_t *keys)
{
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t *row = words + i * W;
        int64_t *kr = keys + i * nchunks;
        for (int32_t c = 0; c < nchunks; ++c) {
            int64_t v = 0;
            for (int32_t s = 0; s < chunk_bits; ++s) {
                int32_t idx = c * chunk_bits + s;
                int64_t bit = 0;
                if (idx < npos) {
                    int32_t t = pos[idx];
                    bit = (int64_t)((row[t >> 6] >> (t & 63)) & 1u);
                }
                v = (v << 1) | bit;
            }
            kr[c] = v;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Counting pass: hamming_join.py:52-82.  Stable, buckets laid out in        */
/* first-seen order.                                                         */
/* ------------------------------------------------------------------------ */
static void counting_pass(const int64_t *keys, int32_t nchunks, int32_t col,
                          const int64_t *perm_in, int64_t *perm_out, int64_t n,
                          int64_t *counts, int64_t *touched)
{
    int64_t nt = 0;
    for (int64_t idx = 0; idx < n; ++idx) {
        int64_t key = keys[perm_in[idx] * nchunks + col];
        if (counts[key] == 0) touched[nt++] = key;
        counts[key] += 1;
    }
    int64_t total = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int64_t c = counts[touched[t]];
        counts[touched[t]] = total;
        total += c;
    }
    for (int64_t idx = 0; idx < n; ++idx) {
        int64_t row = perm_in[idx];
        int64_t key = keys[row * nchunks + col];
        perm_out[counts[key]++] = row;
    }
    for (int64_t t = 0; t < nt; ++t) counts[touched[t]] = 0;
}

/* Group bounds: hamming_join.py:85-101. */
static int64_t group_bounds(const int64_t *keys, int32_t nchunks, const int64_t *perm,
                            int64_t n, int64_t *bounds)
{
    bounds[0] = 0;
    int64_t ng = 1;
    for (int64_t idx = 1; idx < n; ++idx) {
        const int64_t *a = keys + perm[idx - 1] * nchunks;
        const int64_t *b = keys + perm[idx] * nchunks;
        for (int32_t c = 0; c < nchunks; ++c)
            if (a[c] != b[c]) { bounds[ng++] = idx; break; }
    }
    bounds[ng] = n;
    return ng;
}

typedef struct {
    int64_t *keys, *perm_a, *perm_b, *bounds, *counts, *touched;
    int32_t *pos;
} scratch_t;

static int scratch_alloc(scratch_t *s, int64_t n, int32_t length, int32_t chunk_bits)
{
    int32_t nchunks_max = (length + chunk_bits - 1) / chunk_bits;
    if (nchunks_max < 1) nchunks_max = 1;
    s->keys = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1) * nchunks_max);
    s->perm_a = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    s->perm_b = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    s->bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 2));
    s->counts = (int64_t *)calloc((size_t)1 << chunk_bits, sizeof(int64_t));
    int64_t tcap = n < ((int64_t)1 << chunk_bits) ? n : ((int64_t)1 << chunk_bits);
    s->touched = (int64_t *)malloc(sizeof(int64_t) * (size_t)(tcap + 1));
    s->pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)length);
    if (!s->keys || !s->perm_a || !s->perm_b || !s->bounds || !s->counts ||
        !s->touched || !s->pos) return OR_NOMEM;
    return OR_OK;
}

static void scratch_free(scratch_t *s)
{
    free(s->keys); free(s->perm_a); free(s->perm_b); free(s->bounds);
    free(s->counts); free(s->touched); free(s->pos);
}

/* _sort_grouped: hamming_join.py:252-272.  Returns n_groups; perm/bounds
 * point into scratch. */
static int64_t sort_grouped(const uint64_t *words, int64_t n, int32_t W,
                            const int64_t *bbounds, int32_t k,
                            const int32_t *mask, int32_t d, int32_t chunk_bits,
                            scratch_t *s, int64_t **perm_out)
{
    int32_t npos = kept_positions(bbounds, k, mask, d, s->pos);
    int32_t nchunks = (npos + chunk_bits - 1) / chunk_bits;
    int64_t *perm = s->perm_a, *out = s->perm_b;
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    if (nchunks == 0) {
        s->bounds[0] = 0; s->bounds[1] = n;
        *perm_out = perm;
        return 1;
    }
    masked_keys(words, n, W, s->pos, npos, chunk_bits, nchunks, s->keys);
    for (int32_t col = nchunks - 1; col >= 0; --col) {
        counting_pass(s->keys, nchunks, col, perm, out, n, s->counts, s->touched);
        int64_t *t = perm; perm = out; out = t;
    }
    *perm_out = perm;
    return group_bounds(s->keys, nchunks, perm, n, s->bounds);
}

/* grouped_radix_sort: hamming_join.py:275-297.  perm[n], bounds[n+1];
 * returns the number of groups or a negative status. */
int64_t or_grouped_radix_sort(const uint64_t *words, int64_t n, int32_t W, int32_t length,
                              const int64_t *bbounds, int32_t k,
                              const int32_t *mask, int32_t d, int32_t chunk_bits,
                              int64_t *perm_out, int64_t *bounds_out)
{
    if (n <= 0 || chunk_bits < 1 || chunk_bits > 24) return OR_BAD_ARG;
    scratch_t s;
    if (scratch_alloc(&s, n, length, chunk_bits) != OR_OK) { scratch_free(&s); return OR_NOMEM; }
    int64_t *perm;
    int64_t ng = sort_grouped(words, n, W, bbounds, k, mask, d, chunk_bits, &s, &perm);
    memcpy(perm_out, perm, sizeof(int64_t) * (size_t)n);
    memcpy(bounds_out, s.bounds, sizeof(int64_t) * (size_t)(ng + 1));
    scratch_free(&s);
    return ng;
}

/* kept_word_mask: bitpool.py:197-211. kept[w] has 1s at positions outside
 * the masked blocks, restricted to [0, length). */
static void kept_word_mask(int32_t length, const int64_t *bbounds, int32_t W,
                           const int32_t *mask, int32_t d, uint64_t *kept)
{
    for (int32_t w = 0; w < W; ++w) kept[w] = 0;
    for (int32_t t = 0; t < length; ++t) kept[t >> 6] |= (uint64_t)1 << (t & 63);
    for (int32_t m = 0; m < d; ++m)
        for (int64_t t = bbounds[mask[m]]; t < bbounds[mask[m] + 1]; ++t)
            kept[t >> 6] &= ~((uint64_t)1 << (t & 63));
}

/* Lexicographic d-subsets of range(k) (itertools.combinations order,
 * hamming_join.py:333).  Returns the count; fills masks[count][d]. */
static int64_t binom(int32_t k, int32_t d)
{
    if (d < 0 || d > k) return 0;
    int64_t c = 1;
    for (int32_t i = 1; i <= d; ++i) c = c * (k - d + i) / i;
    return c;
}

static void all_masks(int32_t k, int32_t d, int32_t *masks)
{
    int32_t idx[64];
    for (int32_t i = 0; i < d; ++i) idx[i] = i;
    int64_t m = 0;
    for (;;) {
        for (int32_t i = 0; i < d; ++i) masks[m * d + i] = idx[i];
        ++m;
        int32_t i = d - 1;
        while (i >= 0 && idx[i] == k - d + i) --i;
        if (i < 0) break;
        idx[i]++;
        for (int32_t j = i + 1; j < d; ++j) idx[j] = idx[j - 1] + 1;
    }
}

typedef struct { int64_t *p; int64_t len, cap; } pairbuf_t;

static int pb_push(pairbuf_t *b, int64_t i, int64_t j)
{
    if (b->len == b->cap) {
        int64_t nc = b->cap ? b->cap * 2 : 1024;
        int64_t *np = (int64_t *)realloc(b->p, sizeof(int64_t) * 2 * (size_t)nc);
        if (!np) return OR_NOMEM;
        b->p = np; b->cap = nc;
    }
    b->p[2 * b->len] = i; b->p[2 * b->len + 1] = j; b->len++;
    return OR_OK;
}

/* _emit_group_pairs for one mask: hamming_join.py:104-149. */
static int emit_mask(const uint64_t *words, int32_t W, const int64_t *perm,
                     const int64_t *gb, int64_t ng, const uint64_t *kept_all,
                     int64_t h, int32_t d, pairbuf_t *out)
{
    for (int64_t g = 0; g < ng; ++g) {
        for (int64_t a = gb[g]; a < gb[g + 1]; ++a) {
            int64_t ia = perm[a];
            const uint64_t *wa = words + ia * W;
            for (int64_t b = a + 1; b < gb[g + 1]; ++b) {
                int64_t ib = perm[b];
                const uint64_t *wb = words + ib * W;
                int64_t dist = 0;
                for (int32_t w = 0; w < W; ++w) {
                    dist += __builtin_popcountll(wa[w] ^ wb[w]);
                    if (dist > d) break;
                }
                if (dist > d) continue;
                int seen = 0;
                for (int64_t gp = 0; gp < h && !seen; ++gp) {
                    int eq = 1;
                    for (int32_t w = 0; w < W; ++w)
                        if ((wa[w] ^ wb[w]) & kept_all[gp * W + w]) { eq = 0; break; }
                    if (eq) seen = 1;
                }
                if (seen) continue;
                int rc = ia < ib ? pb_push(out, ia, ib) : pb_push(out, ib, ia);
                if (rc) return rc;
            }
        }
    }
    return OR_OK;
}

static int cmp_pair(const void *x, const void *y)
{
    const int64_t *a = (const int64_t *)x, *b = (const int64_t *)y;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
    return 0;
}

/*
 * enumerate_pairs: hamming_join.py:300-375.
 * Output is malloc'd (caller frees with or_free); sorted lexicographically.
 * max_group receives the largest equal-key group over all masks (used for
 * the oversized warning, hamming_join.py:341-344, 365-368).
 * threads > 1 runs masks in parallel (each mask's emission is independent
 * given the first-witness rule) and merges in mask order: the result is
 * identical to the serial run.
 */
int or_enumerate_pairs(const uint64_t *words, int64_t n, int32_t W, int32_t length,
                       const int64_t *bbounds, int32_t k, int32_t d, int32_t chunk_bits,
                       int32_t threads, int64_t **pairs_out, int64_t *count_out,
                       int64_t *max_group_out)
{
    if (n <= 0) return OR_BAD_ARG;
    if (!(0 <= d && d < k && k <= length)) return OR_BAD_ARG;
    if (chunk_bits < 1 || chunk_bits > 24) return OR_BAD_ARG;
    int64_t M = binom(k, d);
    int32_t *masks = (int32_t *)malloc(sizeof(int32_t) * (size_t)(M * (d > 0 ? d : 1)));
    uint64_t *kept = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(M * W));
    pairbuf_t *bufs = (pairbuf_t *)calloc((size_t)M, sizeof(pairbuf_t));
    int64_t *maxg = (int64_t *)calloc((size_t)M, sizeof(int64_t));
    if (!masks || !kept || !bufs || !maxg) return OR_NOMEM;
    if (d > 0) all_masks(k, d, masks);
    for (int64_t h = 0; h < M; ++h)
        kept_word_mask(length, bbounds, W, masks + h * d, d, kept + h * W);

    int status = OR_OK;
    int nth = threads > 0 ? threads : 1;
    (void)nth;
#ifdef _OPENMP
#pragma omp parallel num_threads(nth)
#endif
    {
        scratch_t s;
        int st = scratch_alloc(&s, n, length, chunk_bits);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t h = 0; h < M; ++h) {
            if (st != OR_OK) continue;
            int64_t *perm;
            int64_t ng = sort_grouped(words, n, W, bbounds, k, masks + h * d, d,
                                      chunk_bits, &s, &perm);
            int64_t big = 0;
            for (int64_t g = 0; g < ng; ++g) {
                int64_t sz = s.bounds[g + 1] - s.bounds[g];
                if (sz > big) big = sz;
            }
            maxg[h] = big;
            int rc = emit_mask(words, W, perm, s.bounds, ng, kept, h, d, &bufs[h]);
            if (rc) st = rc;
        }
        if (st != OR_OK) status = st;
        scratch_free(&s);
    }
    int64_t total = 0, big = 0;
    for (int64_t h = 0; h < M; ++h) { total += bufs[h].len; if (maxg[h] > big) big = maxg[h]; }
    int64_t *all = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)(total > 0 ? total : 1));
    if (!all) status = OR_NOMEM;
    int64_t off = 0;
    for (int64_t h = 0; h < M; ++h) {
        if (all && bufs[h].len)
            memcpy(all + 2 * off, bufs[h].p, sizeof(int64_t) * 2 * (size_t)bufs[h].len);
        off += bufs[h].len;
        free(bufs[h].p);
    }
    free(bufs); free(masks); free(kept); free(maxg);
    if (status != OR_OK) { free(all); return status; }
    qsort(all, (size_t)total, 2 * sizeof(int64_t), cmp_pair);
    *pairs_out = all;
    *count_out = total;
    *max_group_out = big;
    return OR_OK;
}

void or_free(void *p) { free(p); }

/* ------------------------------------------------------------------------ */
/* Cross-replicate first witness: pipeline.py:109-146 / fold :286-314.       */
/* keep[p] = 1 iff popcount(words_g[i]^words_g[j]) > d for every earlier g. */
/* ------------------------------------------------------------------------ */
void or_first_witness(const int64_t *pairs, int64_t m,
                      const uint64_t *const *earlier, int32_t n_earlier,
                      int32_t W, int32_t d, uint8_t *keep)
{
    for (int64_t p = 0; p < m; ++p) {
        int64_t i = pairs[2 * p], j = pairs[2 * p + 1];
        uint8_t ok = 1;
        for (int32_t g = 0; g < n_earlier && ok; ++g) {
            int64_t dist = 0;
            for (int32_t w = 0; w < W; ++w)
                dist += __builtin_popcountll(earlier[g][i * W + w] ^ earlier[g][j * W + w]);
            if (dist <= d) ok = 0;
        }
        keep[p] = ok;
    }
}

/* ------------------------------------------------------------------------ */
/* Exact cosine filter: pipeline.py:183-223.  norms = sqrt(sum x^2) fp64,    */
/* dist = 1 - dot/(n_i*n_j), clipped to [0,2], kept when dist <= eps.        */
/* Sequential fp64 sums (the reference uses numpy einsum; agreement is to    */
/* ~1e-15, see tests).  Writes dist for every candidate.                     */
/* ------------------------------------------------------------------------ */
void or_cosine_dist(const double *x, int64_t n, int32_t dim, const int64_t *pairs,
                    int64_t m, double *dist, int32_t threads)
{
    (void)n; (void)threads;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t p = 0; p < m; ++p) {
        const double *a = x + pairs[2 * p] * dim;
        const double *b = x + pairs[2 * p + 1] * dim;
        double dot = 0.0, na = 0.0, nb = 0.0;
        for (int32_t q = 0; q < dim; ++q) {
            dot += a[q] * b[q];
            na += a[q] * a[q];
            nb += b[q] * b[q];
        }
        double dd = 1.0 - dot / (sqrt(na) * sqrt(nb));
        if (dd < 0.0) dd = 0.0;
        if (dd > 2.0) dd = 2.0;
        dist[p] = dd;
    }
}

/* ------------------------------------------------------------------------ */
/* Exhaustive Hamming pairs, digest form: exact.py:99-121 (brute_force_     */
/* hamming) restated for subsets whose answer is too large to hold as a     */
/* pair list (config 4's 50k-member clusters: ~1.6e9 pairs).  Every pair    */
/* (a<b) of the rows with popcount(xor) <= d contributes key = (ids[a] <<   */
/* 32 | ids[b]) (ids: sorted global row ids) through an order-independent   */
/* digest: out[0] = count, out[1] = sum of mix(key) mod 2^64, out[2] = xor  */
/* of mix(key).  mix = splitmix64's finaliser.                             */
/* ------------------------------------------------------------------------ */
static inline uint64_t or_mix(uint64_t z)
{
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

void or_bf_hamming_digest(const uint64_t *words, const int64_t *ids, int64_t n, int32_t W,
                          int32_t d, uint64_t *out, int32_t threads)
{
    uint64_t cnt = 0, sum = 0, xr = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 64) reduction(+:cnt, sum) reduction(^:xr)
#endif
    for (int64_t a = 0; a < n; ++a) {
        const uint64_t *wa = words + a * W;
        const uint64_t ia = (uint64_t)ids[a] << 32;
        for (int64_t b = a + 1; b < n; ++b) {
            const uint64_t *wb = words + b * W;
            int32_t dist = 0;
            for (int32_t w = 0; w < W; ++w) dist += __builtin_popcountll(wa[w] ^ wb[w]);
            if (dist <= d) {
                const uint64_t m = or_mix(ia | (uint64_t)ids[b]);
                ++cnt;
                sum += m;
                xr ^= m;
            }
        }
    }
    out[0] = cnt;
    out[1] = sum;
    out[2] = xr;
}
