/*
 * tilevolve_b200.h -- C ABI of libtilevolve_b200.so, the B200 (sm_100a)
 * implementation of the tilevolve enumeration / classification hot path and
 * the GA generation loop.
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference; "_k" = pkg/src/tilevolve/_kernels.py):
 *
 *   tv_classify_batch      <- _k.classify_batch        _k:404-452
 *   tv_classify_single     <- _k.classify_single       _k:471-484
 *   tv_assemble_single     <- _k.assemble_single       _k:455-468
 *   tv_oat_hash_bytes      <- _k.oat_hash_bytes        _k:79-85
 *   tv_shape_labels        <- classify.rotation_invariant_hash (absent module,
 *                             SPEC.md:270-278) + the D4 min-hash label
 *   tv_enumerate_range     <- classify.enumerate_space (absent module;
 *   tv_enumerate_indices      SPEC.md:297-306, per-batch classify_batch calls
 *                             merged into a Histogram)
 *   tv_hist_*              <- classify.Histogram
 *   tv_ga_*                <- evolve.run_ga and its operators
 *
 * Conventions
 *   - Returns 0 on success, a negative TV_ERR_* on failure; tv_last_error()
 *     gives a thread-local message.  Per-row capacity overflow keeps the
 *     reference semantics (class 255 in every out_class column, _k:434-437).
 *   - Array arguments marked [h|d] may be host or device pointers (detected
 *     per call).  Host arrays are staged through device memory inside the call
 *     and the call synchronises the stream before returning; with device
 *     arrays the call is stream-ordered and returns after the launch.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All work for
 *     one call runs on the current CUDA device.
 *   - Small descriptor arrays (mask_pos, mask_val, free_pos, ks) are host
 *     pointers with the reference dtypes (int64, uint8, int64, int64).
 *   - There is no CPU execution path: if no CUDA device is usable every call
 *     fails with TV_ERR_CUDA.
 */
#ifndef TILEVOLVE_B200_H
#define TILEVOLVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TV_OK 0
#define TV_ERR_ARG -1
#define TV_ERR_CUDA -2
#define TV_ERR_HIST_FULL -3
#define TV_ERR_UNSUPPORTED -4

/* classification codes (_k:25-29) and single-run outcomes (_k:19-22) */
#define TV_CLS_DETERMINISTIC 0
#define TV_CLS_TRIVIAL 1
#define TV_CLS_STERIC 2
#define TV_CLS_UNBOUND 3
#define TV_CLS_ERROR 255
#define TV_RUN_BOUNDED 0
#define TV_RUN_TRIVIAL 1
#define TV_RUN_UNBOUND 2
#define TV_RUN_OVERFLOW 3

int tv_version(void);
const char *tv_last_error(void);

/* Kernel-path statistics of the last enumerate / classify launch on this
 * thread: [0] path (1 = shared-memory bitboard kernel: a <= 3, bits per label <= 3,
 * d <= 118; 2 = generic kernel: everything else),
 * [1] CTAs, [2] threads per CTA, [3] dynamic shared bytes per CTA,
 * [4] launches issued by the call. */
int tv_last_launch_info(int64_t *info5);

/* _k:404-452.  indices[n] [h|d]; outputs [h|d]: out_class u8[n*q] (row-major
 * n x q), out_hash u32[n], out_w u8[n], out_h u8[n], out_cells u16[n],
 * out_shape u64[n*W].  ks ascending, hist_k <= ks[q-1] (the reference sizes its
 * run buffer by ks[q-1], _k:425-426).  Rows whose hist_k class is TRIVIAL or
 * UNBOUND keep their out_shape contents (_k:448-452). */
int tv_classify_batch(const uint64_t *indices, int64_t n, int32_t a, int32_t bpl,
                      const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                      const int64_t *free_pos, int64_t nfree, int32_t d,
                      const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict,
                      uint8_t *out_class, uint32_t *out_hash, uint8_t *out_w, uint8_t *out_h,
                      uint16_t *out_cells, uint64_t *out_shape, int64_t W, void *stream);

/* _k:471-484: edges u8[a*16] host (edges_from_labels layout, _k:487-494);
 * shape_words u64[W] host, written as the reference writes it;
 * out6 = {status, cls, hash (as u32 bits), w, h, cells}. */
int tv_classify_single(const uint8_t *edges, int32_t a, int32_t d, int32_t k, uint64_t seed,
                       uint64_t genome_index, int32_t strict, uint64_t *shape_words, int64_t W,
                       int32_t *out6);

/* _k:455-468: out_grid i16[d*d] host (tile*4+orient, -1 empty);
 * out6 = {outcome, minr, minc, maxr, maxc, n_placed}. */
int tv_assemble_single(const uint8_t *edges, int32_t a, int32_t d, uint64_t seed, uint64_t genome_index,
                       int32_t run_index, int32_t strict, int16_t *out_grid, int32_t *out6);

/* _k:79-85: data [h|d] */
int tv_oat_hash_bytes(const uint8_t *data, int64_t n, uint32_t *out);

/* Canonical labels of n packed cropped shapes (extra columns; the histogram
 * key stays the plain shape hash).  Replaces the host-side rotation-invariant
 * hash of the absent classify module (caller asm:216-235)
 * and adds the D4 (8 rotations + reflections) minimum shape hash.
 * shape [h|d] u64[n*W] (bit y*w+x, _k:280-292), w/h [h|d] u8[n];
 * out_rot4 / out_d4 [h|d] u32[n], either may be NULL.  Rows whose w*h
 * exceeds W*64 bits or is zero get 0. */
int tv_shape_labels(const uint64_t *shape, const uint8_t *w, const uint8_t *h, int64_t n, int64_t W,
                    uint32_t *out_rot4, uint32_t *out_d4, void *stream);

/* ---- phenotype histogram (device-resident, one CUDA device per handle) */
typedef struct tv_hist tv_hist;
/* capacity: slots (rounded up to a power of two); q: number of prefix ks
 * tallied; W: u64 words per stored shape bitmap */
int tv_hist_create(int64_t capacity, int32_t q, int32_t W, tv_hist **out);
int tv_hist_destroy(tv_hist *h);
int tv_hist_clear(tv_hist *h, void *stream);
/* synchronises; n_keys = distinct shape hashes, overflow = 1 if inserts were dropped */
int tv_hist_count(tv_hist *h, int64_t *n_keys, int32_t *overflow, void *stream);
/* Records sorted by hash ascending.  All outputs host pointers sized for
 * max_records (shape: max_records*W); tallies i64[q*5] in the order
 * (DET, TRIV, STERIC, UNB, ERROR) per prefix k.  rep_* = UINT64_MAX if none. */
int tv_hist_export(tv_hist *h, int64_t max_records, uint32_t *keys, uint64_t *det, uint64_t *steric,
                   uint64_t *rep_det, uint64_t *rep_any, uint8_t *w, uint8_t *hh, uint16_t *cells,
                   uint64_t *shape, int64_t *tallies, int64_t *n_out, void *stream);
/* Merge records (same layout as export, [h|d]) and tallies (host, may be NULL)
 * into h: counts add, representatives take the minimum. */
int tv_hist_merge(tv_hist *h, int64_t n, const uint32_t *keys, const uint64_t *det, const uint64_t *steric,
                  const uint64_t *rep_det, const uint64_t *rep_any, const uint8_t *w, const uint8_t *hh,
                  const uint16_t *cells, const uint64_t *shape, const int64_t *tallies, void *stream);
/* Multi-GPU exchange (device-resident, no payload fix-up on the way): pack the raw
 * records as rows {key, det, steric, rep_det, rep_any, pay_idx, whc, shape[W]}
 * (7 + W u64 each; pay_idx = the genome whose payload the row carries) and the
 * tallies [q x 5]; rows/tallies [h|d].  replace_rows clears the histogram (keeping
 * its enumeration parameters) and merges the rows of all ranks: counts added,
 * representatives lowered, payload = the lowest payload owner; tv_hist_export then
 * re-derives the payloads whose owner is not the representative. */
int tv_hist_pack(tv_hist *h, int64_t max_records, uint64_t *rows, int64_t *tallies, int64_t *n_out,
                 void *stream);
int tv_hist_replace_rows(tv_hist *h, int64_t n, const uint64_t *rows, const int64_t *tallies, void *stream);

/* Fused enumerate -> classify -> histogram over indices [start, start+count)
 * of a space (same space arguments as tv_classify_batch).  No per-genome
 * output; stream-ordered. */
int tv_enumerate_range(uint64_t start, uint64_t count, int32_t a, int32_t bpl,
                       const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                       const int64_t *free_pos, int64_t nfree, int32_t d,
                       const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict,
                       tv_hist *h, void *stream);
/* Strided chunks: work item i is index start + (i / chunk) * stride + (i % chunk),
 * i in [0, count).  Used for round-robin sharding of an index range across
 * ranks (chunk c of the range -> rank c mod R) in a single launch. */
int tv_enumerate_chunks(uint64_t start, uint64_t count, uint64_t chunk, uint64_t stride, int32_t a, int32_t bpl,
                        const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                        const int64_t *free_pos, int64_t nfree, int32_t d,
                        const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict,
                        tv_hist *h, void *stream);
/* Same, over an explicit index list [h|d]. */
int tv_enumerate_indices(const uint64_t *indices, int64_t n, int32_t a, int32_t bpl,
                         const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                         const int64_t *free_pos, int64_t nfree, int32_t d,
                         const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict,
                         tv_hist *h, void *stream);

/* ---- GA generation loop (semantics in oracle/tv_ga_oracle.c) */
typedef struct tv_ga tv_ga;
/* n genomes of L <= 4096 bits; mode 0 asexual, 1 single-point crossover, 2 uniform
 * crossover; T[L] = Poisson(lambda) CDF thresholds x 2^63 (k flips = #{j : (draw >> 1)
 * >= T[j]}).  Population starts all-zero.  L <= 64: one u64 per genome (the integer
 * genome.to_int()), one cooperative kernel per tv_ga_run.  L > 64: W = ceil(L/64)
 * little-endian u64 words per genome (set/get_population take [n, W] genome-major
 * arrays; the device keeps them word-major), three launches per generation
 * (orc_ga_run_w semantics); external / JaTAM fitness and tv_ga_replicas need L <= 64. */
int tv_ga_create(int64_t n, int32_t L, int32_t mode, const uint64_t *T, tv_ga **out);
int tv_ga_destroy(tv_ga *h);
int tv_ga_set_population(tv_ga *h, const uint64_t *genomes, void *stream);  /* [h|d]; NULL = zeros */
int tv_ga_get_population(tv_ga *h, uint64_t *out, void *stream);           /* [h|d] */
int tv_ga_population_ptr(tv_ga *h, uint64_t **dev_ptr);
/* Run generations g0 .. g0+n_gens-1 (one cooperative launch).  Per generation:
 * fitness (Fujiyama popcount, or f_ext [d] for exactly one generation),
 * stats best/sum/count(f >= target) [h|d] (may be NULL), stop after recording
 * a generation with count >= 1 (stop_when 1) or >= adapt_count (2), else
 * reproduce.  *gens_done = generations evaluated.  Synchronises. */
int tv_ga_run(tv_ga *h, uint64_t seed, int64_t g0, int64_t n_gens, uint32_t target, int64_t adapt_count,
              int32_t stop_when, const uint32_t *f_ext, uint32_t *best, uint64_t *sum, uint32_t *count,
              int64_t *gens_done, void *stream);
/* R independent GA runs (SPEC.md:415-432 sweeps) in one launch, one CTA per run with
 * the population in shared memory (n <= 8192).  Run r is bit-identical to
 * tv_ga_run with seed seeds[r] from the same initial population (init [h|d]
 * R x n, NULL = all zero).  Outputs [h|d]: done/disc/adapt int64[R] (disc/adapt
 * = first generation with count >= 1 / >= adapt_count, else -1); optional
 * best/sum/count [R x n_gens] and final_pop [R x n]. */
int tv_ga_replicas(int64_t n, int32_t L, int32_t mode, const uint64_t *T, int32_t R, const uint64_t *seeds,
                   const uint64_t *init, int64_t g0, int64_t n_gens, uint32_t target, int64_t adapt_count,
                   int32_t stop_when, int64_t *done, int64_t *disc, int64_t *adapt, uint32_t *best, uint64_t *sum,
                   uint32_t *count, uint64_t *final_pop, void *stream);
/* JaTAM-shape fitness of the current population read as enumeration indices of
 * the space: f = d^2 - shapediff(target, run-0 grid) if DET at k, else 0.
 * target_occ u8[d*d] host (seed-centred board); f_out device u32[n].  Exact reuse:
 * children equal to a parent inherit its fitness (after a tv_ga_run fed with this
 * call's f_out), and (populations >= 2^21) genomes met earlier in the run are
 * looked up in a per-handle genome -> fitness memo; both only under the same
 * fitness parameters, and tv_ga_set_population empties the memo (TV_FITCACHE=0
 * disables the first, TV_FITMEMO=1/0 forces the memo on / off). */
int tv_ga_fitness_jatam(tv_ga *h, int32_t a, int32_t bpl, const int64_t *mask_pos, const uint8_t *mask_val,
                        int64_t m, const int64_t *free_pos, int64_t nfree, int32_t d, int32_t k, uint64_t seed,
                        int32_t strict, const uint8_t *target_occ, uint32_t *f_out, void *stream);

/* n_gens JaTAM-fitness generations in one call, no early stop: each generation = the
 * fitness of the current population (tv_ga_fitness_jatam semantics; children equal to a
 * parent inherit its fitness) + one reproduction (tv_ga_run with f_ext, seed, generation
 * g0 + t).  Stats per generation [h|d] (may be NULL).  Enqueued without host round trips;
 * synchronises once at the end. */
int tv_ga_run_jatam(tv_ga *h, int32_t a, int32_t bpl, const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                    const int64_t *free_pos, int64_t nfree, int32_t d, int32_t k, uint64_t fit_seed, int32_t strict,
                    const uint8_t *target_occ, uint64_t seed, int64_t g0, int64_t n_gens, uint32_t target,
                    uint32_t *best, uint64_t *sum, uint32_t *count, void *stream);
/* SPEC ACCEPTANCE 8 mutation benchmark (orc_ga_mutate semantics): mutate the word-major
 * device population pop [W x n] of L-bit genomes in place with stream (seed, g, i);
 * method 0 = by distribution (the GA's operator, T host or device), 1 = bit by bit (one
 * draw per bit, flip when draw < pthr).  flips (host, may be NULL) = total flips;
 * synchronises only when flips is given. */
int tv_ga_mutate(uint64_t *pop, int64_t n, int32_t L, const uint64_t *T, uint64_t pthr, int32_t method,
                 uint64_t seed, int64_t g, uint64_t *flips, void *stream);

/* ---- measurement helpers (bench.py roofline) */
/* Launch the int32 ALU peak probe (IADD3/LOP3 chains); *ops = int32 ops issued. */
int tv_int_peak_launch(int64_t iters, int32_t blocks, int32_t threads, void *stream, double *ops);
int tv_sm_count(int32_t *n);
/* L2 ceilings for the GA roofline: read+write streaming over buf (random = 0) or
 * independent random 16-byte reads (random = 1) of a buffer of `bytes` (size it to stay
 * L2-resident); *bytes_moved = bytes the launch moves. */
int tv_l2_probe_launch(void *buf, int64_t bytes, int32_t reps, int32_t random, void *stream, double *bytes_moved);
/* Grid-barrier floor: one cooperative launch (one 1024-thread CTA per SM, the GA kernel's
 * geometry) executing `syncs` grid.sync() back to back. */
int tv_gridsync_probe_launch(int32_t syncs, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TILEVOLVE_B200_H */
