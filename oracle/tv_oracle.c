/*
 * tv_oracle.c -- CPU restatement of the reference enumeration hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2205_15311_b200/csrc).  Only tests/, the smoke() entry
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product library never links or calls it.
 *
 * Parity status: PINNED.  The restatement is checked against golden vectors
 * produced by running the reference (tilevolve._kernels, numba) in the build
 * container -- see tests/golden/make_golden.py and tests/test_oracle.py --
 * and against the SHA-256 output digests in SURVEY.md Appendix C.
 *
 * Reference: /root/reference/pkg/src/tilevolve/_kernels.py (cited "_k:LINE").
 * Every function below names the lines it follows.  The restatement is
 * written from the semantics, plain C99, scratch owned by the caller thread.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_RUN_BOUNDED 0
#define ORC_RUN_TRIVIAL 1
#define ORC_RUN_UNBOUND 2
#define ORC_RUN_OVERFLOW 3

#define ORC_CLS_DET 0
#define ORC_CLS_TRIV 1
#define ORC_CLS_STERIC 2
#define ORC_CLS_UNB 3
#define ORC_CLS_ERROR 255

static const uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL; /* _k:31 */
static const uint64_t K_MIXA = 0xBF58476D1CE4E5B9ULL; /* _k:32 */
static const uint64_t K_MIXB = 0x94D049BB133111EBULL; /* _k:33 */

/* splitmix64 finaliser, _k:38-42 */
static inline uint64_t orc_mix64(uint64_t z) {
    z ^= z >> 30; z *= K_MIXA;
    z ^= z >> 27; z *= K_MIXB;
    return z ^ (z >> 31);
}

/* substream start keyed by (seed, enumeration index, run), _k:45-48 */
static inline uint64_t orc_stream(uint64_t seed, uint64_t idx, uint64_t run) {
    uint64_t z = orc_mix64(seed ^ (K_GOLD * (idx + 1)));
    return orc_mix64(z ^ (K_MIXA * (run + 1)));
}

/* counter step then mix, _k:51-54; bounded draw from the high word, _k:57-60 */
static inline int orc_below(uint64_t *s, uint32_t n) {
    *s += K_GOLD;
    uint64_t x = orc_mix64(*s);
    return (int)(((x >> 32) * (uint64_t)n) >> 32);
}

/* Jenkins one-at-a-time, _k:65-76 */
static inline uint32_t oat_step(uint32_t h, uint32_t k) {
    h += k; h += h << 10; h ^= h >> 6; return h;
}
static inline uint32_t oat_fin(uint32_t h) {
    h += h << 3; h ^= h >> 11; h += h << 15; return h;
}

uint32_t orc_oat_hash_bytes(const uint8_t *p, int64_t n) { /* _k:79-85 */
    uint32_t h = 0;
    for (int64_t i = 0; i < n; i++) h = oat_step(h, p[i]);
    return oat_fin(h);
}

/* label pairing 1-2, 3-4, ...; 0 inert, _k:90-93 */
static inline int orc_bonds(int i, int j) { return i != 0 && j == (((i - 1) ^ 1) + 1); }

typedef struct {
    int16_t *grid;   /* d*d, -1 empty, else tile*4+orient */
    uint8_t *mark;   /* d*d in-stack flags */
    int32_t *stack;  /* d*d */
    int32_t *placed; /* d*d */
} orc_scratch;

typedef struct {
    int outcome, n_placed, sp, minr, minc, maxr, maxc;
} orc_run;

typedef struct { /* instrumentation for the roofline op counts */
    uint64_t runs, pops, placements, draws, hashed_cells, bounded_runs, max_sp;
} orc_counts;

/* One movelist assembly on clean scratch, _k:96-249. */
static orc_run orc_assemble(const uint8_t *edges, int a, int d, int strict,
                            uint64_t seed, uint64_t idx, int run,
                            orc_scratch *S, orc_counts *C) {
    orc_run R;
    uint64_t s = orc_stream(seed, idx, (uint64_t)run);
    const int dd = d * d, half = d >> 1, ctr = half * d + half;
    S->grid[ctr] = 0;                       /* seed tile, orientation 0 (_k:115) */
    S->placed[0] = ctr;
    R.n_placed = 1;
    R.minr = R.maxr = R.minc = R.maxc = half;
    int nb[4] = {ctr - d, ctr + 1, ctr + d, ctr - 1};
    for (int j = 3; j > 0; j--) {            /* _k:127-131 */
        int q = orc_below(&s, (uint32_t)(j + 1));
        int t = nb[j]; nb[j] = nb[q]; nb[q] = t;
    }
    if (C) C->draws += 3;
    int sp = 0;
    for (int j = 0; j < 4; j++) { S->mark[nb[j]] = 1; S->stack[sp++] = nb[j]; }

    while (sp > 0) {
        int cell = S->stack[--sp];
        S->mark[cell] = 0;
        if (C) { C->pops++; if ((uint64_t)sp + 1 > C->max_sp) C->max_sp = sp + 1; }
        int r = cell / d, c = cell % d;
        int p[4] = {-1, -1, -1, -1};          /* label shown toward cell, _k:145-164 */
        if (r > 0)     { int v = S->grid[cell - d]; if (v >= 0) p[0] = edges[(v >> 2) * 16 + (v & 3) * 4 + 2]; }
        if (c < d - 1) { int v = S->grid[cell + 1]; if (v >= 0) p[1] = edges[(v >> 2) * 16 + (v & 3) * 4 + 3]; }
        if (r < d - 1) { int v = S->grid[cell + d]; if (v >= 0) p[2] = edges[(v >> 2) * 16 + (v & 3) * 4 + 0]; }
        if (c > 0)     { int v = S->grid[cell - 1]; if (v >= 0) p[3] = edges[(v >> 2) * 16 + (v & 3) * 4 + 1]; }
        int64_t found = -1; int found_v = -1, ambiguous = 0;
        for (int t = 0; t < a && !ambiguous; t++) {       /* _k:169-207 */
            for (int rt = 0; rt < 4; rt++) {
                const uint8_t *e = edges + t * 16 + rt * 4;
                int bond = 0, ok = 1;
                for (int k = 0; k < 4 && ok; k++) {
                    if (p[k] < 0) continue;
                    if (orc_bonds(e[k], p[k])) bond = 1;
                    else if (strict && e[k] != 0 && p[k] != 0) ok = 0;
                }
                if (ok && bond) {
                    int64_t code = ((int64_t)e[0] << 24) | ((int64_t)e[1] << 16) | ((int64_t)e[2] << 8) | e[3];
                    if (found < 0) { found = code; found_v = t * 4 + rt; }
                    else if (code != found) { ambiguous = 1; break; }
                }
            }
        }
        if (ambiguous) { R.outcome = ORC_RUN_TRIVIAL; R.sp = sp; return R; }
        if (found < 0) continue;                          /* dropped, _k:210-211 */
        if (r == 0 || c == 0 || r == d - 1 || c == d - 1) { /* _k:212-213 */
            R.outcome = ORC_RUN_UNBOUND; R.sp = sp; return R;
        }
        S->grid[cell] = (int16_t)found_v;
        S->placed[R.n_placed++] = cell;
        if (C) C->placements++;
        if (r < R.minr) R.minr = r;
        if (r > R.maxr) R.maxr = r;
        if (c < R.minc) R.minc = c;
        if (c > R.maxc) R.maxc = c;
        int m = 0;                                        /* _k:225-237 */
        const int nbc[4] = {cell - d, cell + 1, cell + d, cell - 1};
        for (int k = 0; k < 4; k++)
            if (S->grid[nbc[k]] < 0 && !S->mark[nbc[k]]) nb[m++] = nbc[k];
        for (int j = m - 1; j > 0; j--) {                 /* _k:238-242 */
            int q = orc_below(&s, (uint32_t)(j + 1));
            int t = nb[j]; nb[j] = nb[q]; nb[q] = t;
            if (C) C->draws++;
        }
        for (int j = 0; j < m; j++) {                     /* _k:243-248 */
            if (sp >= dd) { R.outcome = ORC_RUN_OVERFLOW; R.sp = sp; return R; }
            S->mark[nb[j]] = 1;
            S->stack[sp++] = nb[j];
        }
    }
    R.outcome = ORC_RUN_BOUNDED; R.sp = 0;
    return R;
}

/* restore touched cells only, _k:252-257 */
static void orc_cleanup(orc_scratch *S, const orc_run *R) {
    for (int i = 0; i < R->sp; i++) S->mark[S->stack[i]] = 0;
    for (int i = 0; i < R->n_placed; i++) S->grid[S->placed[i]] = -1;
}

/* OAT over w, h, then (x, y) of occupied cells row-major, _k:260-277 */
static uint32_t orc_hash_region(const orc_scratch *S, int d, const orc_run *R,
                                int *w_out, int *h_out, int *n_out) {
    int w = R->maxc - R->minc + 1, h = R->maxr - R->minr + 1, n = 0;
    uint32_t st = oat_step(oat_step(0, (uint32_t)w), (uint32_t)h);
    for (int y = 0; y < h; y++) {
        const int16_t *row = S->grid + (R->minr + y) * d + R->minc;
        for (int x = 0; x < w; x++)
            if (row[x] >= 0) { st = oat_step(oat_step(st, (uint32_t)x), (uint32_t)y); n++; }
    }
    *w_out = w; *h_out = h; *n_out = n;
    return oat_fin(st);
}

/* cropped bitmap, bit y*w+x, LSB-first per u64 word, _k:280-292 */
static void orc_pack_region(const orc_scratch *S, int d, const orc_run *R,
                            uint64_t *words, int W) {
    memset(words, 0, sizeof(uint64_t) * (size_t)W);
    int w = R->maxc - R->minc + 1, h = R->maxr - R->minr + 1, bit = 0;
    for (int y = 0; y < h; y++) {
        const int16_t *row = S->grid + (R->minr + y) * d + R->minc;
        for (int x = 0; x < w; x++, bit++)
            if (row[x] >= 0) words[bit >> 6] |= 1ULL << (bit & 63);
    }
}

/* prefix class with precedence TRIV > UNB > STERIC > DET, _k:295-303 */
static inline int orc_class_at(int kp, int trivial_at, int first_unbound, int first_mismatch) {
    if (trivial_at >= 0 && trivial_at < kp) return ORC_CLS_TRIV;
    if (first_unbound >= 0 && first_unbound < kp) return ORC_CLS_UNB;
    if (first_mismatch >= 0 && first_mismatch < kp) return ORC_CLS_STERIC;
    return ORC_CLS_DET;
}

typedef struct {
    int status, trivial_at, first_unbound, first_mismatch;
    uint32_t hash; int w, h, cells;
} orc_fold;

/* k-run fold with steric majority attribution, _k:306-381 */
static orc_fold orc_classify_edges(const uint8_t *edges, int a, int d, int kmax, int hist_k,
                                   uint64_t seed, uint64_t idx, int strict,
                                   orc_scratch *S, uint32_t *run_hash, uint64_t *shape, int W,
                                   orc_counts *C) {
    orc_fold F = {0, -1, -1, -1, 0, 0, 0, 0};
    int w0 = 0, h0 = 0, c0 = 0;
    for (int run = 0; run < kmax; run++) {
        orc_run R = orc_assemble(edges, a, d, strict, seed, idx, run, S, C);
        if (C) C->runs++;
        if (R.outcome == ORC_RUN_OVERFLOW) {
            orc_cleanup(S, &R);
            F.status = 1; F.hash = 0; F.w = F.h = F.cells = 0;
            return F;
        }
        if (R.outcome == ORC_RUN_TRIVIAL) { orc_cleanup(S, &R); F.trivial_at = run; break; }
        if (R.outcome == ORC_RUN_UNBOUND) {
            if (F.first_unbound < 0) F.first_unbound = run;
            run_hash[run] = 0;
            orc_cleanup(S, &R);
            continue;
        }
        int w, h, nc;
        uint32_t hs = orc_hash_region(S, d, &R, &w, &h, &nc);
        if (C) { C->bounded_runs++; C->hashed_cells += (uint64_t)nc; }
        run_hash[run] = hs;
        if (run == 0) {
            orc_pack_region(S, d, &R, shape, W);
            w0 = w; h0 = h; c0 = nc;
        } else if (F.first_mismatch < 0 && F.first_unbound != 0 && hs != run_hash[0]) {
            F.first_mismatch = run;
        }
        orc_cleanup(S, &R);
    }
    int hc = orc_class_at(hist_k, F.trivial_at, F.first_unbound, F.first_mismatch);
    if (hc == ORC_CLS_DET) { F.hash = run_hash[0]; F.w = w0; F.h = h0; F.cells = c0; return F; }
    if (hc != ORC_CLS_STERIC) { F.hash = 0; F.w = F.h = F.cells = 0; return F; }
    uint32_t best = 0; int best_n = 0;
    for (int j = 0; j < hist_k; j++) {
        int n = 0;
        for (int l = 0; l < hist_k; l++) n += run_hash[l] == run_hash[j];
        if (n > best_n || (n == best_n && run_hash[j] < best)) { best_n = n; best = run_hash[j]; }
    }
    F.hash = best; F.w = w0; F.h = h0; F.cells = c0;
    if (best == run_hash[0]) return F;
    for (int j = 1; j < hist_k; j++) {
        if (run_hash[j] != best) continue;
        orc_run R = orc_assemble(edges, a, d, strict, seed, idx, j, S, NULL);
        orc_hash_region(S, d, &R, &F.w, &F.h, &F.cells);
        orc_pack_region(S, d, &R, shape, W);
        orc_cleanup(S, &R);
        return F;
    }
    return F;
}

/* index -> genome bits -> labels -> in-situ edge table, _k:384-401 */
static void orc_decode_edges(uint64_t idx, int a, int bpl, const int64_t *mask_pos,
                             const uint8_t *mask_val, int64_t m, const int64_t *free_pos,
                             int64_t nfree, uint8_t *bits, uint8_t *edges) {
    const int L = a * 4 * bpl;
    memset(bits, 0, (size_t)L);
    for (int64_t j = 0; j < m; j++) bits[mask_pos[j]] = mask_val[j];
    for (int64_t j = 0; j < nfree; j++) bits[free_pos[j]] = (uint8_t)((idx >> j) & 1ULL);
    for (int t = 0; t < a; t++)
        for (int rt = 0; rt < 4; rt++)
            for (int dr = 0; dr < 4; dr++) {
                int te = t * 4 + ((dr - rt) & 3), v = 0;
                for (int j = 0; j < bpl; j++) v = (v << 1) | bits[te * bpl + j];
                edges[t * 16 + rt * 4 + dr] = (uint8_t)v;
            }
}

static int orc_scratch_alloc(orc_scratch *S, int d) {
    size_t dd = (size_t)d * d;
    S->grid = (int16_t *)malloc(dd * sizeof(int16_t));
    S->mark = (uint8_t *)calloc(dd, 1);
    S->stack = (int32_t *)malloc(dd * sizeof(int32_t));
    S->placed = (int32_t *)malloc(dd * sizeof(int32_t));
    if (!S->grid || !S->mark || !S->stack || !S->placed) return -1;
    for (size_t i = 0; i < dd; i++) S->grid[i] = -1;
    return 0;
}
static void orc_scratch_free(orc_scratch *S) {
    free(S->grid); free(S->mark); free(S->stack); free(S->placed);
}

/*
 * Batch driver, _k:404-452.  Same argument meaning and output write rules as
 * classify_batch; nthreads <= 0 uses every OpenMP thread.  counts (optional,
 * 7 u64) accumulates runs, pops, placements, draws, hashed cells, bounded
 * runs, max stack depth.
 */
int orc_classify_batch(const uint64_t *indices, int64_t n, int a, int bpl,
                       const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                       const int64_t *free_pos, int64_t nfree, int d,
                       const int64_t *ks, int64_t q, int hist_k, uint64_t seed, int strict,
                       uint8_t *out_class, uint32_t *out_hash, uint8_t *out_w, uint8_t *out_h,
                       uint16_t *out_cells, uint64_t *out_shape, int64_t W,
                       int nthreads, uint64_t *counts) {
    const int kmax = (int)ks[q - 1];
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    orc_counts total = {0, 0, 0, 0, 0, 0, 0};
#pragma omp parallel num_threads(nthreads) reduction(|:err)
    {
        orc_scratch S;
        orc_counts C = {0, 0, 0, 0, 0, 0, 0};
        uint8_t bits[256], edges[64 * 16];
        uint32_t *run_hash = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(kmax > 0 ? kmax : 1));
        uint64_t *shape = (uint64_t *)calloc((size_t)W, sizeof(uint64_t));
        if (orc_scratch_alloc(&S, d) != 0 || !run_hash || !shape) err = 1;
        else {
#pragma omp for schedule(dynamic, 1024)
            for (int64_t i = 0; i < n; i++) {
                uint64_t idx = indices[i];
                orc_decode_edges(idx, a, bpl, mask_pos, mask_val, m, free_pos, nfree, bits, edges);
                orc_fold F = orc_classify_edges(edges, a, d, kmax, hist_k, seed, idx, strict,
                                                &S, run_hash, shape, (int)W, counts ? &C : NULL);
                if (F.status != 0) {
                    for (int64_t k = 0; k < q; k++) out_class[i * q + k] = ORC_CLS_ERROR;
                    continue;
                }
                for (int64_t k = 0; k < q; k++)
                    out_class[i * q + k] = (uint8_t)orc_class_at((int)ks[k], F.trivial_at,
                                                                 F.first_unbound, F.first_mismatch);
                int hc = orc_class_at(hist_k, F.trivial_at, F.first_unbound, F.first_mismatch);
                if (hc == ORC_CLS_DET || hc == ORC_CLS_STERIC) {
                    out_hash[i] = F.hash;
                    out_w[i] = (uint8_t)F.w; out_h[i] = (uint8_t)F.h;
                    out_cells[i] = (uint16_t)F.cells;
                    memcpy(out_shape + i * W, shape, sizeof(uint64_t) * (size_t)W);
                } else {
                    out_hash[i] = 0; out_w[i] = 0; out_h[i] = 0; out_cells[i] = 0;
                }
            }
        }
        if (counts) {
#pragma omp critical
            {
                total.runs += C.runs; total.pops += C.pops; total.placements += C.placements;
                total.draws += C.draws; total.hashed_cells += C.hashed_cells;
                total.bounded_runs += C.bounded_runs;
                if (C.max_sp > total.max_sp) total.max_sp = C.max_sp;
            }
        }
        free(run_hash); free(shape); orc_scratch_free(&S);
    }
    if (counts) {
        counts[0] += total.runs; counts[1] += total.pops; counts[2] += total.placements;
        counts[3] += total.draws; counts[4] += total.hashed_cells; counts[5] += total.bounded_runs;
        if (total.max_sp > counts[6]) counts[6] = total.max_sp;
    }
    return err ? -1 : 0;
}

/* single tile set, _k:471-484: returns status; writes cls/hash/w/h/cells */
int orc_classify_single(const uint8_t *edges, int a, int d, int k, uint64_t seed,
                        uint64_t genome_index, int strict, uint64_t *shape, int64_t W,
                        int32_t *out5) {
    orc_scratch S;
    if (orc_scratch_alloc(&S, d) != 0) return -1;
    uint32_t *run_hash = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)k);
    orc_fold F = orc_classify_edges(edges, a, d, k, k, seed, genome_index, strict,
                                    &S, run_hash, shape, (int)W, NULL);
    out5[0] = orc_class_at(k, F.trivial_at, F.first_unbound, F.first_mismatch);
    out5[1] = (int32_t)F.hash; out5[2] = F.w; out5[3] = F.h; out5[4] = F.cells;
    free(run_hash); orc_scratch_free(&S);
    return F.status;
}

/* one run with the grid copied out, _k:455-468; out6 = outcome,minr,minc,maxr,maxc,n_placed */
int orc_assemble_single(const uint8_t *edges, int a, int d, uint64_t seed, uint64_t genome_index,
                        int run_index, int strict, int16_t *out_grid, int32_t *out6) {
    orc_scratch S;
    if (orc_scratch_alloc(&S, d) != 0) return -1;
    orc_run R = orc_assemble(edges, a, d, strict, seed, genome_index, run_index, &S, NULL);
    memcpy(out_grid, S.grid, sizeof(int16_t) * (size_t)d * d);
    out6[0] = R.outcome; out6[1] = R.minr; out6[2] = R.minc; out6[3] = R.maxr; out6[4] = R.maxc;
    out6[5] = R.n_placed;
    orc_scratch_free(&S);
    return 0;
}

/* raw splitmix64 stream draws (for RNG unit tests): out[j] = j-th mixed value */
void orc_stream_draws(uint64_t seed, uint64_t idx, uint64_t run, int64_t n, uint64_t *out) {
    uint64_t s = orc_stream(seed, idx, run);
    for (int64_t j = 0; j < n; j++) { s += K_GOLD; out[j] = orc_mix64(s); }
}
