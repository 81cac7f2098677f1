/*
 * tv_ga_oracle.c -- CPU restatement of the GA generation loop (SPEC.md evolve
 * module).
 *
 * TEST INFRASTRUCTURE ONLY (checker for paper_2205_15311_b200/csrc/tv_ga.cu;
 * bench.py's GA CPU baseline).  Parity status: UNPINNED -- the reference ships
 * no GA code.  This file defines the semantics the
 * GPU must reproduce bit-for-bit; statistical acceptance against SPEC.md
 * (section ACCEPTANCE 4-5) is tested separately.
 *
 * Semantics (documented in DESIGN.md section 6):
 *  - genome: L <= 64 bits held as the integer genome.to_int() (genome bit i is
 *    integer bit L-1-i, gen:92-94); population of N genomes.
 *  - RNG: counter-based splitmix64 as in the enumeration path (_k:38-60) keyed by
 *    (seed, generation, child): s = stream(seed, g, i); draw = mix64(s += G).
 *  - per child i of generation g -> g+1, draw order:
 *      parent a  (roulette: r = mulhi64(draw, total), first j with cdf[j] > r;
 *                 total == 0 -> j = mulhi64(draw, N))
 *      parent b  (modes 1, 2 only)
 *      crossover: single point p = below(L), child = a's bits before p ++ b's
 *                 from p (p = 0 -> b)
 *                 uniform: mask = draw & (2^L-1), bit from b where mask is 1
 *                                                                SPEC:379-387
 *      mutation:  u = draw >> 1 (63 bits), k = #{j < L : u >= T[j]} with
 *                 T[j] = floor(PoissonCDF_lambda(j) * 2^63) (so lambda = 0 gives
 *                 k = 0 exactly; k is clamped to L), then k distinct positions
 *                 p = below(L) with rejection of repeats, each flipped
 *                                                                  SPEC:352-369
 *    below(n) = ((draw >> 32) * n) >> 32 (the reference's bounded draw, _k:57-60).
 *  - fitness: Fujiyama = popcount.
 *  - stats per generation (before reproduction): best, sum, count(f >= target).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const uint64_t GA_GOLD = 0x9E3779B97F4A7C15ULL;
static const uint64_t GA_MIXA = 0xBF58476D1CE4E5B9ULL;
static const uint64_t GA_MIXB = 0x94D049BB133111EBULL;

static inline uint64_t ga_mix(uint64_t z) {
    z ^= z >> 30; z *= GA_MIXA;
    z ^= z >> 27; z *= GA_MIXB;
    return z ^ (z >> 31);
}
static inline uint64_t ga_stream(uint64_t seed, uint64_t g, uint64_t i) {
    return ga_mix(ga_mix(seed ^ (GA_GOLD * (g + 1))) ^ (GA_MIXA * (i + 1)));
}
static inline uint64_t ga_draw(uint64_t *s) { *s += GA_GOLD; return ga_mix(*s); }
static inline uint32_t ga_below(uint64_t *s, uint32_t n) {
    return (uint32_t)(((ga_draw(s) >> 32) * (uint64_t)n) >> 32);
}
static inline uint64_t ga_mulhi(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

static int64_t ga_select(uint64_t *s, const uint64_t *cdf, int64_t n) {
    const uint64_t total = cdf[n - 1];
    const uint64_t x = ga_draw(s);
    if (total == 0) return (int64_t)ga_mulhi(x, (uint64_t)n);
    const uint64_t r = ga_mulhi(x, total);
    int64_t lo = 0, hi = n - 1;                 /* first j with cdf[j] > r */
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (cdf[mid] > r) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* one child (exported for operator unit tests) */
uint64_t orc_ga_child(uint64_t seed, int64_t g, int64_t i, const uint64_t *pop, const uint64_t *cdf,
                      int64_t n, int L, int mode, const uint64_t *T) {
    uint64_t s = ga_stream(seed, (uint64_t)g, (uint64_t)i);
    const uint64_t full = L == 64 ? ~0ULL : ((1ULL << L) - 1);
    const uint64_t a = pop[ga_select(&s, cdf, n)];
    uint64_t child = a;
    if (mode != 0) {
        const uint64_t b = pop[ga_select(&s, cdf, n)];
        if (mode == 1) {
            const uint32_t p = ga_below(&s, (uint32_t)L);
            const uint64_t top = p == 0 ? 0 : (full & ~((L - p == 64) ? 0 : ((1ULL << (L - p)) - 1)));
            child = (a & top) | (b & ~top & full);
        } else {
            const uint64_t m = ga_draw(&s) & full;
            child = (a & ~m) | (b & m);
        }
    }
    const uint64_t u = ga_draw(&s) >> 1;
    int k = 0;
    while (k < L && u >= T[k]) k++;
    uint64_t chosen = 0;
    for (int f = 0; f < k;) {
        const uint32_t p = ga_below(&s, (uint32_t)L);
        const uint64_t bit = 1ULL << (L - 1 - p);
        if (chosen & bit) continue;
        chosen |= bit;
        f++;
    }
    return (child ^ chosen) & full;
}

/*
 * Run n_gens generations starting at generation index g0 on pop (in place).
 * stats arrays (length n_gens) may be NULL.  stop_when: 0 never, 1 after the
 * first generation with count >= 1, 2 after the first with count >= adapt_count.
 * Returns the number of generations evaluated (stats rows written).
 */
int64_t orc_ga_run(uint64_t *pop, int64_t n, int L, int mode, const uint64_t *T, uint64_t seed, int64_t g0,
                   int64_t n_gens, uint32_t target, int64_t adapt_count, int stop_when,
                   uint32_t *best, uint64_t *sum, uint32_t *count, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    uint64_t *cdf = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    uint64_t *next = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    int64_t done = 0;
    for (int64_t t = 0; t < n_gens; t++) {
        const int64_t g = g0 + t;
        uint64_t acc = 0, cnt = 0;
        uint32_t bst = 0;
        for (int64_t i = 0; i < n; i++) {
            const uint32_t f = (uint32_t)__builtin_popcountll(pop[i]);
            acc += f;
            cdf[i] = acc;
            if (f > bst) bst = f;
            cnt += f >= target;
        }
        if (best) best[t] = bst;
        if (sum) sum[t] = acc;
        if (count) count[t] = (uint32_t)cnt;
        done = t + 1;
        if ((stop_when == 1 && cnt >= 1) || (stop_when == 2 && (int64_t)cnt >= adapt_count)) break;
#pragma omp parallel for num_threads(nthreads) schedule(static)
        for (int64_t i = 0; i < n; i++) next[i] = orc_ga_child(seed, g, i, pop, cdf, n, L, mode, T);
        memcpy(pop, next, sizeof(uint64_t) * (size_t)n);
    }
    free(cdf);
    free(next);
    return done;
}

/* Poisson flip counts as drawn by mutation, for the distribution tests */
void orc_ga_flip_counts(uint64_t seed, int64_t n, int L, const uint64_t *T, int32_t *out) {
    for (int64_t i = 0; i < n; i++) {
        uint64_t s = ga_stream(seed, 0, (uint64_t)i);
        const uint64_t u = ga_draw(&s) >> 1;
        int k = 0;
        while (k < L && u >= T[k]) k++;
        out[i] = k;
    }
}

/* raw GA stream draws for unit tests */
void orc_ga_draws(uint64_t seed, uint64_t g, uint64_t i, int64_t n, uint64_t *out) {
    uint64_t s = ga_stream(seed, g, i);
    for (int64_t j = 0; j < n; j++) out[j] = ga_draw(&s);
}

/*
 * Wide genomes (any L >= 1; used for L > 64): W = ceil(L/64) u64 words per genome,
 * little-endian (word 0 = integer bits 0..63 of genome.to_int()), genome position p is
 * integer bit L-1-p, population stored genome-major (pop[i*W + w]).  Draw order per child
 * is the narrow one with the uniform-crossover mask drawn one word at a time (word 0
 * first): a, [b], [p = below(L) | W mask draws], u, flip positions.  For W = 1 every
 * operator is identical to orc_ga_child (checked in tests/test_ga.py).  Fitness = total
 * popcount; the CDF is 64-bit (N x L may exceed 2^32).
 */
static int64_t ga_select64(uint64_t *s, const uint64_t *cdf, int64_t n) {
    const uint64_t total = cdf[n - 1];
    const uint64_t x = ga_draw(s);
    if (total == 0) return (int64_t)ga_mulhi(x, (uint64_t)n);
    const uint64_t r = ga_mulhi(x, total);
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (cdf[mid] > r) hi = mid; else lo = mid + 1;
    }
    return lo;
}

static inline uint64_t ga_wfull(int L, int w) {  /* valid integer bits of word w */
    const int hi = L - 64 * w;
    return hi >= 64 ? ~0ULL : ((1ULL << hi) - 1);
}

void orc_ga_child_w(uint64_t seed, int64_t g, int64_t i, const uint64_t *pop, const uint64_t *cdf, int64_t n,
                    int L, int mode, const uint64_t *T, uint64_t *out) {
    const int W = (L + 63) / 64;
    uint64_t s = ga_stream(seed, (uint64_t)g, (uint64_t)i);
    const uint64_t *a = pop + (size_t)ga_select64(&s, cdf, n) * W;
    for (int w = 0; w < W; w++) out[w] = a[w];
    if (mode != 0) {
        const uint64_t *b = pop + (size_t)ga_select64(&s, cdf, n) * W;
        if (mode == 1) {  /* positions < p (integer bits >= L-p) from a, the rest from b */
            const uint32_t p = ga_below(&s, (uint32_t)L);
            const int lo = L - (int)p;
            for (int w = 0; w < W; w++) {
                uint64_t top;
                if (lo <= 64 * w) top = ~0ULL;
                else if (lo >= 64 * w + 64) top = 0;
                else top = ~((1ULL << (lo - 64 * w)) - 1);
                top &= ga_wfull(L, w);
                out[w] = (a[w] & top) | (b[w] & ~top & ga_wfull(L, w));
            }
        } else {
            for (int w = 0; w < W; w++) {
                const uint64_t m = ga_draw(&s) & ga_wfull(L, w);
                out[w] = (a[w] & ~m) | (b[w] & m);
            }
        }
    }
    const uint64_t u = ga_draw(&s) >> 1;
    int k = 0;
    while (k < L && u >= T[k]) k++;
    uint64_t *chosen = (uint64_t *)calloc((size_t)W, 8);
    for (int f = 0; f < k;) {
        const uint32_t p = ga_below(&s, (uint32_t)L);
        const int bit = L - 1 - (int)p;
        if ((chosen[bit >> 6] >> (bit & 63)) & 1) continue;
        chosen[bit >> 6] |= 1ULL << (bit & 63);
        f++;
    }
    for (int w = 0; w < W; w++) out[w] = (out[w] ^ chosen[w]) & ga_wfull(L, w);
    free(chosen);
}

int64_t orc_ga_run_w(uint64_t *pop, int64_t n, int L, int mode, const uint64_t *T, uint64_t seed, int64_t g0,
                     int64_t n_gens, uint32_t target, int64_t adapt_count, int stop_when,
                     uint32_t *best, uint64_t *sum, uint32_t *count, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    const int W = (L + 63) / 64;
    uint64_t *cdf = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    uint64_t *next = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n * W);
    int64_t done = 0;
    for (int64_t t = 0; t < n_gens; t++) {
        const int64_t g = g0 + t;
        uint64_t acc = 0, cnt = 0;
        uint32_t bst = 0;
        for (int64_t i = 0; i < n; i++) {
            uint32_t f = 0;
            for (int w = 0; w < W; w++) f += (uint32_t)__builtin_popcountll(pop[i * W + w]);
            acc += f;
            cdf[i] = acc;
            if (f > bst) bst = f;
            cnt += f >= target;
        }
        if (best) best[t] = bst;
        if (sum) sum[t] = acc;
        if (count) count[t] = (uint32_t)cnt;
        done = t + 1;
        if ((stop_when == 1 && cnt >= 1) || (stop_when == 2 && (int64_t)cnt >= adapt_count)) break;
#pragma omp parallel for num_threads(nthreads) schedule(static)
        for (int64_t i = 0; i < n; i++) orc_ga_child_w(seed, g, i, pop, cdf, n, L, mode, T, next + i * W);
        memcpy(pop, next, sizeof(uint64_t) * (size_t)n * W);
    }
    free(cdf);
    free(next);
    return done;
}

/*
 * SPEC ACCEPTANCE 8 (mutation benchmark, Fig. 5's regime): mutate n genomes of L bits in
 * place, `method` 0 = by distribution (k ~ Poisson(lambda) from T, then k distinct
 * positions: the GA's operator), 1 = bit by bit (one draw per bit, flip when the draw is
 * below p = lambda / L as a 64-bit threshold `pthr`).  Child i of generation g uses stream
 * (seed, g, i).  Returns the number of flips (a checksum the caller can compare).
 */
uint64_t orc_ga_mutate(uint64_t *pop, int64_t n, int L, const uint64_t *T, uint64_t pthr, int method, uint64_t seed,
                       int64_t g, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    const int W = (L + 63) / 64;
    uint64_t flips = 0;
#pragma omp parallel for num_threads(nthreads) schedule(static) reduction(+ : flips)
    for (int64_t i = 0; i < n; i++) {
        uint64_t s = ga_stream(seed, (uint64_t)g, (uint64_t)i);
        uint64_t *x = pop + i * W;
        if (method == 0) {
            const uint64_t u = ga_draw(&s) >> 1;
            int k = 0;
            while (k < L && u >= T[k]) k++;
            uint64_t chosen[64] = {0};  /* L <= 4096 */
            for (int f = 0; f < k;) {
                const uint32_t p = ga_below(&s, (uint32_t)L);
                const int bit = L - 1 - (int)p;
                if ((chosen[bit >> 6] >> (bit & 63)) & 1) continue;
                chosen[bit >> 6] |= 1ULL << (bit & 63);
                f++;
            }
            for (int w = 0; w < W; w++) x[w] ^= chosen[w];
            flips += (uint64_t)k;
        } else {
            for (int p = 0; p < L; p++) {
                if (ga_draw(&s) < pthr) {
                    const int bit = L - 1 - p;
                    x[bit >> 6] ^= 1ULL << (bit & 63);
                    flips++;
                }
            }
        }
    }
    return flips;
}
