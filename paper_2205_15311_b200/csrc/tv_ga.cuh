// tv_ga.cuh -- GA generation loop (SPEC.md evolve module).
//
// One cooperative persistent kernel runs many generations; per generation:
//   B. chunk offsets -> global inclusive CDF (u32) and a guide table for
//      indexed search (Chen & Asau): the r-range [0, total) is cut into
//      B = min(n, total) monotone buckets b(r) = (r * M) >> 32 and guide[b] =
//      (cdf[j], j[, genome j]) of the individual j owning the first r of bucket
//      b (so most lookups need no CDF load; for L <= 32 the CDF is packed above
//      the genome in the population word and the guide carries the genome, so
//      most selections are a single L2 read); individual j writes the
//      buckets whose first r lies in its own range [cdf[j-1], cdf[j]), so the
//      table is built in the same pass.  Rows of 32 individuals are
//      independent: each starts at its exclusive offset from the last phase C;
//   -- grid barrier --
//   C. children: all random draws of a child first (selection draws,
//      crossover mask, mutation mask), then selection = guide[b(r)] plus a short
//      forward scan while cdf[j] <= r (exactly the first j with cdf[j] > r),
//      parent loads and the child (TV_GA_ILP children in flight per thread); a warp
//      makes one row of 32 consecutive children at a time, so the next
//      generation's row fitness sums, best and target count are warp
//      reductions; a block scan turns the row sums into row offsets and the
//      CTA total (the prologue does the same for the initial population);
//   -- grid barrier --
// Two grid barriers per generation.
// Staged mode (popcount fitness, L <= 32, CTA chunk within 200 KB of shared memory): between
// the phases a CTA keeps its chunk's genomes, fitness and row offsets in shared memory, so
// phase B reads nothing from L2 and phase C stores only row statistics; guide entries then
// also carry genome j + 1 (a draw past the owner's range is resolved from the same entry).
// Data written by other CTAs is read only after a grid barrier (grid.sync()
// orders and publishes all prior writes of the grid; its gpu-scope acquire
// invalidates L1), so ordinary cached loads are used.
// Semantics (draw order, masks, thresholds) are defined by the CPU
// restatement oracle/tv_ga_oracle.c, which the GPU reproduces bit for bit.
#pragma once
#include <cooperative_groups.h>

#include "tv_device.cuh"

#ifndef TV_GA_THREADS
#define TV_GA_THREADS 1024  // k_ga_run CTA size (one CTA per SM)
#endif
#ifndef TV_GA_ILP
#define TV_GA_ILP 1  // children per thread in flight in phase C (2 and 3 measured 0.7-2 % slower, 4 and 8 more)
#endif

namespace tvb {

struct GaParams {
  int64_t n;             // population
  int32_t L;             // genome bits (<= 64)
  int32_t mode;          // 0 asexual, 1 single-point crossover, 2 uniform crossover
  int32_t fitness;       // 0 Fujiyama (popcount), 1 external vector f_ext
  uint32_t target;       // count_at_target threshold (f >= target)
  int64_t adapt_count;   // adaptation threshold (count >= adapt_count)
  int32_t stop_when;     // 0 never, 1 discovery, 2 adaptation
  uint64_t seed;
  int64_t g0, n_gens;
  int64_t chunk;         // individuals per CTA (contiguous)
  uint64_t T[64];        // Poisson CDF thresholds x 2^63 (k = #{j < L : (draw >> 1) >= T[j]})
  unsigned long long *pop0, *pop1;
  const uint32_t *f_ext;
  uint32_t *f_known;     // external fitness: per child, its fitness if it equals a parent, else ~0 (or nullptr)
  uint32_t *cdf;         // n
  uint32_t *fstage;      // n: fitness staged in index order (own chunk per CTA)
  ulonglong2 *guide;     // n buckets (first B used per generation): x = (cdf[j] << 32) | j,
                         // y = genome j (packed mode, L <= 32) [| genome j + 1 << 32 (pair)]
  int32_t stg;           // the CTA's chunk is staged in shared memory (popcount fitness, L <= 32)
  int32_t pair;          // popcount fitness: guide entries carry genomes j and j + 1
  uint32_t *first_g;     // pair + stg: per CTA, the genome of its chunk's first individual
  unsigned long long *tot;  // per CTA chunk totals
  uint32_t *rowx;        // per CTA, per row of 32 individuals: fitness sum, then its exclusive offset
  uint32_t *best;        // n_gens
  unsigned long long *sum;  // n_gens
  uint32_t *count;       // n_gens
  unsigned long long *done;  // generations evaluated (written by CTA 0)
  int32_t *final_buf;    // which pop buffer holds the final population
  unsigned long long *prof;  // optional (TV_GA_PROF): CTA 0 ns spent in phases A, B, C
};

__device__ __forceinline__ unsigned long long ga_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t ga_draw(uint64_t &s) {
  s += kGold;
  return mix64(s);
}
__device__ __forceinline__ uint32_t ga_below(uint64_t &s, uint32_t n) {
  return (uint32_t)(((ga_draw(s) >> 32) * (uint64_t)n) >> 32);
}

// Draw-side of one child: everything that depends only on its random stream
// (draw order fixed by oracle/tv_ga_oracle.c): the two roulette draws, the
// crossover mask and the mutation mask.  The memory-dependent part (guide
// lookup, CDF scan, parent loads) is done afterwards for several children at
// once so their L2 latencies overlap.
struct ChildDraws {
  uint32_t ra, rb;      // roulette draws in [0, total) (or uniform indices when total == 0)
  uint64_t top;         // crossover: bits taken from parent a (mode 1); uniform: mask of bits from b (mode 2)
  uint64_t flips;       // mutation mask
};

__device__ __forceinline__ ChildDraws ga_draws(const GaParams &P, uint64_t gkey, int64_t i, uint32_t total) {
  ChildDraws D;
  uint64_t s = mix64(gkey ^ (kMixA * ((uint64_t)i + 1)));  // = stream_state(seed, g, i), gkey hoisted
  const int L = P.L;
  const uint64_t full = L == 64 ? ~0ULL : ((1ULL << L) - 1);
  const uint64_t range = total ? (uint64_t)total : (uint64_t)P.n;  // SPEC:447 uniform fallback
  D.ra = (uint32_t)__umul64hi(ga_draw(s), range);
  D.rb = 0;
  D.top = full;
  if (P.mode != 0) {
    D.rb = (uint32_t)__umul64hi(ga_draw(s), range);
    if (P.mode == 1) {  // positions < p from a, >= p from b
      const uint32_t p = ga_below(s, (uint32_t)L);
      D.top = p == 0 ? 0ULL : (full & ~((1ULL << (L - p)) - 1));
    } else {            // each bit from b where the mask is set
      D.top = full & ~ga_draw(s);
    }
  }
  const uint64_t u = ga_draw(s) >> 1;  // k ~ Poisson(lambda) clamped to L
  int k = 0;
  while (k < L && u >= P.T[k]) k++;
  uint64_t chosen = 0;
  for (int f = 0; f < k;) {
    const uint32_t p = ga_below(s, (uint32_t)L);
    const uint64_t bit = 1ULL << (L - 1 - p);
    if (chosen & bit) continue;
    chosen |= bit;
    f++;
  }
  D.flips = chosen;
  return D;
}

// ga_draws for L <= 32 (the same draws, 32-bit masks): the Poisson count compares the
// first four thresholds without a loop (T[j] = ~0 for j >= L, so a compare past L is false
// and k < 4 needs no further test); the loop continues only from k = 4.
struct ChildDraws32 {
  uint32_t ra, rb, top, flips;
};
__device__ __forceinline__ ChildDraws32 ga_draws32(const GaParams &P, uint64_t gkey, int64_t i, uint32_t total) {
  ChildDraws32 D;
  uint64_t s = mix64(gkey ^ (kMixA * ((uint64_t)i + 1)));
  const int L = P.L;
  const uint32_t full = L == 32 ? 0xFFFFFFFFu : ((1u << L) - 1u);
  const uint64_t range = total ? (uint64_t)total : (uint64_t)P.n;
  D.ra = (uint32_t)__umul64hi(ga_draw(s), range);
  D.rb = 0;
  D.top = full;
  if (P.mode != 0) {
    D.rb = (uint32_t)__umul64hi(ga_draw(s), range);
    if (P.mode == 1) {
      const uint32_t p = ga_below(s, (uint32_t)L);
      D.top = p == 0 ? 0u : (full & ~((1u << (L - p)) - 1u));
    } else {
      D.top = full & ~(uint32_t)ga_draw(s);
    }
  }
  const uint64_t u = ga_draw(s) >> 1;
  int k = (int)(u >= P.T[0]) + (int)(u >= P.T[1]) + (int)(u >= P.T[2]) + (int)(u >= P.T[3]);
  if (k == 4)
    while (k < L && u >= P.T[k]) k++;
  uint32_t chosen = 0;
  for (int f = 0; f < k;) {
    const uint32_t bit = 1u << (L - 1 - (int)ga_below(s, (uint32_t)L));
    if (chosen & bit) continue;
    chosen |= bit;
    f++;
  }
  D.flips = chosen;
  return D;
}

// roulette: first j with cdf[j] > r, from the guide entry of r's bucket; the
// entry carries cdf[j] so a bucket whose owner covers r costs one load
__device__ __forceinline__ uint32_t ga_pick(const GaParams &P, uint32_t r, uint32_t total, uint64_t mul) {
  if (total == 0) return r;
  const unsigned long long e = P.guide[(uint32_t)(((uint64_t)r * mul) >> 32)].x;  // mul <= 2^32: no overflow
  uint32_t j = (uint32_t)e, c = (uint32_t)(e >> 32);
  while (c <= r) c = P.cdf[++j];
  return j;
}

// Packed mode (L <= 32): population words carry (cdf[j] << 32) | genome j and
// the guide entry carries the owner's genome, so the selected parent itself is
// returned: one L2 read when the bucket owner covers r, one more per step
// (cdf and genome in the same word) otherwise.  With popcount fitness the entry's
// high half carries genome j + 1 as well (its cdf follows from its popcount): the
// owner misses r for ~47 % of the draws (r is uniform over the bucket, the owner
// covers on average half of it), the pair for ~0.5 %.
__device__ __forceinline__ uint64_t ga_pick_genome(const GaParams &P, const unsigned long long *pop, uint32_t r,
                                                   uint32_t total, uint64_t mul, uint32_t &jo, bool pair) {
  if (total == 0) { jo = r; return pop[r] & 0xFFFFFFFFull; }
  const ulonglong2 e = P.guide[(uint32_t)(((uint64_t)r * mul) >> 32)];
  uint32_t j = (uint32_t)e.x, c = (uint32_t)(e.x >> 32);
  uint64_t g = e.y & 0xFFFFFFFFull;
  if (c <= r && pair) {  // popcount fitness: the entry also carries genome j + 1, whose
    g = e.y >> 32;                 // cdf is cdf[j] + popcount -- about half the draws end here
    c += (uint32_t)__popcll(g);
    j++;
  }
  while (c <= r) {
    const unsigned long long v = pop[++j];
    c = (uint32_t)(v >> 32);
    g = v & 0xFFFFFFFFull;
  }
  jo = j;
  return g;
}

// Block-wide exclusive scan of this CTA's row sums (rowx[0..nrows), in place) and the
// stats of the population they describe; returns the CTA total (all threads).
__device__ __forceinline__ uint32_t ga_rows_scan(uint32_t *rowx, int nrows, uint32_t *warp_sum, uint32_t *s_carry) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) *s_carry = 0u;
  __syncthreads();
  for (int r0 = 0; r0 < nrows; r0 += nt) {
    const int r = r0 + tid;
    const uint32_t v = r < nrows ? rowx[r] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const uint32_t w0 = lane < (nt >> 5) ? warp_sum[lane] : 0u;
      uint32_t w = w0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w += y;
      }
      warp_sum[lane] = w - w0;
      if (lane == 31) warp_sum[32] = w;  // this tile's total
    }
    __syncthreads();
    const uint32_t carry = *s_carry;
    if (r < nrows) rowx[r] = carry + warp_sum[wid] + x - v;
    __syncthreads();
    if (tid == 0) *s_carry = carry + warp_sum[32];
    __syncthreads();
  }
  return *s_carry;
}

// One cooperative launch runs n_gens generations.  Per generation two grid barriers:
//   B: the CTA chunk offsets -> global inclusive CDF (packed above the genome for L <= 32)
//      and the guide table, from per-row exclusive offsets scanned at the end of the
//      previous phase C; stop decision.
//   C: children (TV_GA_ILP per thread in flight); each warp makes one row of 32
//      consecutive children at a time, so the row's fitness sum, best and count for the
//      next generation come from warp reductions, and a block scan of the row sums
//      replaces a separate pass over the staged fitness.
__global__ void __launch_bounds__(TV_GA_THREADS, 1) k_ga_run(const __grid_constant__ GaParams P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t warp_sum[33];  // blockDim.x <= 1024
  __shared__ uint32_t s_best, s_cnt, s_carry;
  __shared__ unsigned long long s_off, s_total, s_gkey;
  __shared__ int s_stop;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * P.chunk;  // P.chunk is a multiple of 32
  const int64_t c1 = min(P.n, c0 + P.chunk);
  const int64_t len = max((int64_t)0, c1 - c0);
  const int nrows = (int)((len + 31) >> 5);
  const bool packed = P.L <= 32;
  // Staged mode (popcount fitness, L <= 32, chunk fits shared memory): the CTA's individuals
  // (genome, fitness) and row offsets live in shared memory between phase C and phase B, so
  // phase B reads nothing from L2 and phase C stores nothing but its row statistics; the
  // population words in global memory are written by phase B (cdf | genome) and, for the
  // final population, after the loop.
  extern __shared__ uint32_t ga_dyn[];
  const bool stg = P.stg != 0 && packed && P.fitness == 0;
  uint32_t *const sg = ga_dyn, *const sf = ga_dyn + P.chunk;
  uint32_t *rowx = stg ? ga_dyn + 2 * P.chunk : P.rowx + (int64_t)blockIdx.x * (P.chunk >> 5);
  int cur = 0;
  int64_t t = 0;
  const uint64_t full = P.L == 64 ? ~0ULL : ((1ULL << P.L) - 1);
  const bool pair = packed && P.fitness == 0 && P.pair;  // guide entries carry genomes j and j + 1
  // fitness of the initial population, staged in index order, with its row sums and stats
  if (tid == 0) { s_best = 0; s_cnt = 0; }
  __syncthreads();
  for (int r = wid; r < nrows; r += nt >> 5) {
    const int64_t i = c0 + (int64_t)r * 32 + lane;
    uint32_t f = 0;
    if (i < c1) {
      if (stg) {
        const uint32_t g = (uint32_t)(P.pop0[i] & full);
        f = (uint32_t)__popc(g);
        sg[i - c0] = g;
        sf[i - c0] = f;
        if (pair && i == c0) P.first_g[blockIdx.x] = g;
      } else {
        f = P.fitness == 0 ? (uint32_t)__popcll(P.pop0[i] & full) : P.f_ext[i];
        P.fstage[i] = f;
      }
    }
    const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, f), mx = __reduce_max_sync(0xFFFFFFFFu, f);
    const uint32_t nc = (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, f >= P.target && i < c1));
    if (lane == 0) {
      rowx[r] = s;
      atomicMax(&s_best, mx);
      if (nc) atomicAdd(&s_cnt, nc);
    }
  }
  __syncthreads();
  {
    const uint32_t tot = ga_rows_scan(rowx, nrows, warp_sum, &s_carry);
    if (tid == 0) {
      P.tot[blockIdx.x] = tot;
      if (P.n_gens > 0) { atomicMax(&P.best[0], s_best); atomicAdd(&P.count[0], s_cnt); }
      s_best = 0; s_cnt = 0;
    }
  }
  grid.sync();
  for (; t < P.n_gens; t++) {
    const int64_t g = P.g0 + t;
    unsigned long long *pop = cur ? P.pop1 : P.pop0;
    unsigned long long *nxt = cur ? P.pop0 : P.pop1;
    const bool prof = P.prof && blockIdx.x == 0 && tid == 0;
    unsigned long long tp0 = prof ? ga_clock() : 0ull, tp1 = 0ull;
    // ---- B: chunk offsets -> global CDF + guide table; stop decision
    if (wid == 0) {
      unsigned long long o = 0, tt = 0;
      for (int j = lane; j < (int)gridDim.x; j += 32) {
        const unsigned long long v = P.tot[j];
        tt += v;
        if (j < (int)blockIdx.x) o += v;
      }
#pragma unroll
      for (int k = 16; k > 0; k >>= 1) {
        o += __shfl_xor_sync(0xFFFFFFFFu, o, k);
        tt += __shfl_xor_sync(0xFFFFFFFFu, tt, k);
      }
      if (lane == 0) {
        s_off = o;
        s_total = tt;
        s_gkey = mix64(P.seed ^ (kGold * ((uint64_t)g + 1)));  // stream_state prefix (_k:45-48)
        const uint32_t c = *((volatile uint32_t *)&P.count[t]);
        s_stop = (P.stop_when == 1 && c >= 1u) || (P.stop_when == 2 && (int64_t)c >= P.adapt_count);
      }
    }
    __syncthreads();
    const uint32_t total = (uint32_t)s_total;
    // bucket function b(r) = (r * mul) >> 32, monotone, B = min(n, total) buckets
    // (r < total < 2^32 and mul <= 2^32, so r * mul fits 64 bits)
    const uint64_t nb = min((uint64_t)P.n, (uint64_t)total);
    const uint64_t mul = total ? (nb << 32) / total : 0ull;
    if (blockIdx.x == 0 && tid == 0) P.sum[t] = s_total;
    if (s_stop) { t++; break; }
    if (stg) {  // staged: the chunk's genomes and fitness come from shared memory
      const uint32_t off = (uint32_t)s_off;
      const int wstep = nt >> 5;
      const uint32_t gnext = pair && c1 < P.n ? P.first_g[blockIdx.x + 1] : 0u;
      for (int r = wid; r < nrows; r += wstep) {
        const int l = r * 32 + lane;
        const bool in = l < len;
        const uint32_t f = in ? sf[l] : 0u, gi = in ? sg[l] : 0u;
        uint32_t x = f;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
          if (lane >= o) x += y;
        }
        if (in) {
          const uint32_t run = off + rowx[r] + x, prev = run - f;
          pop[c0 + l] = ((unsigned long long)run << 32) | gi;
          if (f) {  // own r in [prev, run): buckets whose first r falls in it
            const uint32_t b0 = prev ? (uint32_t)(((uint64_t)(prev - 1) * mul) >> 32) + 1 : 0u;
            const uint32_t b1 = (uint32_t)(((uint64_t)(run - 1) * mul) >> 32);
            const uint32_t gn = pair ? (l + 1 < len ? sg[l + 1] : gnext) : 0u;
            const ulonglong2 e = make_ulonglong2(((unsigned long long)run << 32) | (uint32_t)(c0 + l),
                                                 ((unsigned long long)gn << 32) | gi);
#pragma unroll 1
            for (uint32_t b = b0; b <= b1; b++) P.guide[b] = e;
          }
        }
      }
    } else {
      const uint32_t off = (uint32_t)s_off;
      constexpr int RB = 2;  // rows whose loads are issued before any store (stores could alias them; 4 spills)
      const int wstep = nt >> 5;
      for (int k0 = wid; k0 < nrows; k0 += RB * wstep) {
        uint32_t fr[RB], bx[RB];
        uint64_t gr[RB], gn[RB];  // genome i, genome i + 1 of the row's last lane (pair entries)
#pragma unroll
        for (int u = 0; u < RB; u++) {
          const int r = k0 + u * wstep;
          const int64_t i = c0 + (int64_t)r * 32 + lane;
          const bool in = r < nrows && i < c1;
          fr[u] = in ? P.fstage[i] : 0u;
          gr[u] = in && packed ? (pop[i] & 0xFFFFFFFFull) : 0ull;
          // (the low half of a population word is never written in phase B: no race)
          gn[u] = pair && lane == 31 && in && i + 1 < P.n ? (pop[i + 1] & 0xFFFFFFFFull) : 0ull;
          bx[u] = r < nrows ? rowx[r] : 0u;
        }
#pragma unroll
        for (int u = 0; u < RB; u++) {
          const int r = k0 + u * wstep;
          if (r >= nrows) break;
          const int64_t i = c0 + (int64_t)r * 32 + lane;
          const uint32_t f = fr[u];
          uint32_t x = f;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
          }
          const uint32_t run = off + bx[u] + x, prev = run - f;
          const uint64_t g1 = __shfl_down_sync(0xFFFFFFFFu, gr[u], 1);
          if (i < c1) {
            if (packed) pop[i] = ((unsigned long long)run << 32) | gr[u];
            else P.cdf[i] = run;
            if (f) {  // own r in [prev, run): buckets whose first r falls in it
              const int64_t b0 = prev ? (int64_t)(((uint64_t)(prev - 1) * mul) >> 32) + 1 : 0;
              const int64_t b1 = (int64_t)(((uint64_t)(run - 1) * mul) >> 32);
              const uint64_t hi = pair ? ((lane == 31 ? gn[u] : (i + 1 < c1 ? g1 : 0ull)) & full) << 32 : 0ull;
              const ulonglong2 e = make_ulonglong2(((unsigned long long)run << 32) | (uint32_t)i, gr[u] | hi);
              for (int64_t b = b0; b <= b1; b++) P.guide[b] = e;
            }
          }
        }
      }
    }
    grid.sync();
    if (prof) { tp1 = ga_clock(); P.prof[1] += tp1 - tp0; tp0 = tp1; }
    const uint64_t gkey = s_gkey;
    // ---- C: children, TV_GA_ILP at a time (draws first, then the dependent loads); warp w
    //      makes rows w, w + 32, ... so row sums / best / count of the next generation are
    //      warp reductions
    constexpr int NI = TV_GA_ILP;
    if (stg) {  // staged (L <= 32, popcount): 32-bit draws, children into shared memory
      const uint32_t full32 = (uint32_t)full;
      for (int l = tid; l < nrows * 32; l += nt) {
        uint32_t f = 0;
        if (l < (int)len) {
          const ChildDraws32 D = ga_draws32(P, s_gkey, c0 + l, total);
          uint32_t ja, jb;
          uint32_t c = (uint32_t)ga_pick_genome(P, pop, D.ra, total, mul, ja, pair);
          if (P.mode != 0) {
            const uint32_t gb = (uint32_t)ga_pick_genome(P, pop, D.rb, total, mul, jb, pair);
            c = (c & D.top) | (gb & ~D.top);
          }
          c = (c ^ D.flips) & full32;
          f = (uint32_t)__popc(c);
          sg[l] = c;
          sf[l] = f;
          if (pair && l == 0) P.first_g[blockIdx.x] = c;
        }
        const uint32_t sm = __reduce_add_sync(0xFFFFFFFFu, f), mx = __reduce_max_sync(0xFFFFFFFFu, f);
        const uint32_t nc = (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, f >= P.target && l < (int)len));
        if (lane == 0) {
          rowx[l >> 5] = sm;
          atomicMax(&s_best, mx);
          if (nc) atomicAdd(&s_cnt, nc);
        }
      }
    }
    for (int64_t i = c0 + tid; !stg && i < c0 + (int64_t)nrows * 32; i += NI * nt) {
      ChildDraws D[NI];
#pragma unroll
      for (int u = 0; u < NI; u++) {
        const int64_t iu = i + u * nt;
        D[u] = iu < c1 ? ga_draws(P, gkey, iu, total) : ChildDraws{0u, 0u, 0ull, 0ull};  // r = 0: an in-range pick
      }
      uint64_t cv[NI], ga_[NI], gb_[NI];  // child before mutation, parents' genomes
      uint32_t pa[NI], pb[NI];              // parents' indices
      if (packed) {
#pragma unroll
        for (int u = 0; u < NI; u++) { ga_[u] = ga_pick_genome(P, pop, D[u].ra, total, mul, pa[u], pair); cv[u] = ga_[u]; }
        if (P.mode != 0) {
#pragma unroll
          for (int u = 0; u < NI; u++) {
            gb_[u] = ga_pick_genome(P, pop, D[u].rb, total, mul, pb[u], pair);
            cv[u] = (cv[u] & D[u].top) | (gb_[u] & ~D[u].top);
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < NI; u++) pa[u] = ga_pick(P, D[u].ra, total, mul);
        if (P.mode != 0) {
#pragma unroll
          for (int u = 0; u < NI; u++) pb[u] = ga_pick(P, D[u].rb, total, mul);
        }
#pragma unroll
        for (int u = 0; u < NI; u++) { ga_[u] = pop[pa[u]]; cv[u] = ga_[u]; }
        if (P.mode != 0) {
#pragma unroll
          for (int u = 0; u < NI; u++) { gb_[u] = pop[pb[u]]; cv[u] = (cv[u] & D[u].top) | (gb_[u] & ~D[u].top); }
        }
      }
#pragma unroll
      for (int u = 0; u < NI; u++) {
        const int64_t iu = i + u * nt;
        const int r = (int)((iu - c0) >> 5);
        uint32_t f = 0;
        if (iu < c1) {
          const uint64_t c = (cv[u] ^ D[u].flips) & full;
          if (stg) {
            f = (uint32_t)__popcll(c);
            sg[iu - c0] = (uint32_t)c;
            sf[iu - c0] = f;
            if (pair && iu == c0) P.first_g[blockIdx.x] = (uint32_t)c;
          } else if (P.fitness == 0) {
            nxt[iu] = c;
            f = (uint32_t)__popcll(c);
            P.fstage[iu] = f;
          } else {
            nxt[iu] = c;
            f = P.fstage[iu];  // external fitness stays that of the staged population
            if (P.f_known) {   // a child equal to a parent has that parent's (deterministic) fitness
              uint32_t fk = 0xFFFFFFFFu;
              if (c == (ga_[u] & full)) fk = P.fstage[pa[u]];
              else if (P.mode != 0 && c == (gb_[u] & full)) fk = P.fstage[pb[u]];
              P.f_known[iu] = fk;
            }
          }
        }
        if (r < nrows) {  // warp-uniform: a warp's lanes make one row
          const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, f), mx = __reduce_max_sync(0xFFFFFFFFu, f);
          const uint32_t nc = (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, f >= P.target && iu < c1));
          if (lane == 0) {
            rowx[r] = s;
            atomicMax(&s_best, mx);
            if (nc) atomicAdd(&s_cnt, nc);
          }
        }
      }
    }
    cur ^= 1;
    __syncthreads();
    {
      const uint32_t tot = ga_rows_scan(rowx, nrows, warp_sum, &s_carry);
      if (tid == 0) {
        P.tot[blockIdx.x] = tot;
        if (t + 1 < P.n_gens) { atomicMax(&P.best[t + 1], s_best); atomicAdd(&P.count[t + 1], s_cnt); }
        s_best = 0; s_cnt = 0;
      }
    }
    grid.sync();
    if (prof) P.prof[2] += ga_clock() - tp0;
  }
  if (stg && t > 0) {  // the final population was staged: publish it
    unsigned long long *fin = cur ? P.pop1 : P.pop0;
    for (int l = tid; l < (int)len; l += nt) fin[c0 + l] = sg[l];
  }
  if (blockIdx.x == 0 && tid == 0) {
    *P.done = (unsigned long long)t;
    *P.final_buf = cur;
  }
}

}  // namespace tvb

namespace tvb {

// ---------------------------------------------------------------------------
// Replica GA: R independent runs (SPEC:415-432 sweeps, Figs. 9-10 at N = 512),
// one CTA per replica with its population, CDF and statistics in shared
// memory, so a generation needs only block barriers -- no grid barrier.
// Replica r uses seed seeds[r] and is bit-identical to k_ga_run (and to
// oracle/tv_ga_oracle.c) with that seed: same draws (ga_draws), same
// selection (first j with cdf[j] > r), same stop rule (stats of generation t
// are taken before reproduction; a met stop condition ends the run there).
struct GaRepParams {
  GaParams G;            // n, L, mode, target, adapt_count, stop_when, g0, n_gens, T (per-replica seed below)
  int32_t R;
  const uint64_t *seeds;                 // R
  const unsigned long long *init;        // R x n initial genomes, or nullptr (all zero)
  unsigned long long *final_pop;         // R x n, or nullptr
  int64_t *done;                         // R: generations evaluated
  int64_t *disc;                         // R: first generation with count >= 1, else -1
  int64_t *adapt;                        // R: first generation with count >= adapt_count, else -1
  uint32_t *best;                        // R x n_gens, or nullptr
  unsigned long long *sum;               // R x n_gens, or nullptr
  uint32_t *count;                       // R x n_gens, or nullptr
};

__global__ void __launch_bounds__(1024, 1) k_ga_replicas(const __grid_constant__ GaRepParams Q) {
  extern __shared__ unsigned long long rsm[];
  const GaParams &P = Q.G;
  const int rep = blockIdx.x;
  if (rep >= Q.R) return;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int n = (int)P.n;
  unsigned long long *popA = rsm, *popB = rsm + n;
  uint32_t *cdf = reinterpret_cast<uint32_t *>(rsm + 2 * n);
  __shared__ uint32_t w_sum[32], w_best[32], w_cnt[32];
  __shared__ uint32_t s_total;
  __shared__ int s_stop;
  const uint64_t full = P.L == 64 ? ~0ULL : ((1ULL << P.L) - 1);
  const uint64_t seed = Q.seeds[rep];
  for (int i = tid; i < n; i += nt) popA[i] = Q.init ? (Q.init[(int64_t)rep * n + i] & full) : 0ull;
  int64_t disc = -1, adap = -1, t = 0;  // disc/adap tracked by thread 31 (it sees the stats)
  int cur = 0;
  __syncthreads();
  for (; t < P.n_gens; t++) {
    unsigned long long *pop = cur ? popB : popA, *nxt = cur ? popA : popB;
    // fitness + inclusive CDF over the population (index order), stats
    // each thread owns a contiguous run of individuals; warp scan of the run totals
    const int per = (n + nt - 1) / nt, i0 = min(n, tid * per), i1 = min(n, i0 + per);
    uint32_t acc = 0, best = 0, cnt = 0;
    for (int i = i0; i < i1; i++) {
      const uint32_t f = (uint32_t)__popcll(pop[i]);
      acc += f;
      best = max(best, f);
      cnt += f >= P.target;
    }
    uint32_t x = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
      cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    }
    if (lane == 31) w_sum[wid] = x;
    if (lane == 0) { w_best[wid] = best; w_cnt[wid] = cnt; }
    __syncthreads();
    if (wid == 0) {
      const uint32_t v = lane < nw ? w_sum[lane] : 0u;
      uint32_t s = v, b = lane < nw ? w_best[lane] : 0u, q = lane < nw ? w_cnt[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
        if (lane >= o) s += y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        b = max(b, __shfl_xor_sync(0xFFFFFFFFu, b, o));
        q += __shfl_xor_sync(0xFFFFFFFFu, q, o);
      }
      w_sum[lane] = s - v;  // exclusive warp offsets
      if (lane == 31) {
        s_total = s;
        const int64_t gi = (int64_t)rep * P.n_gens + t;
        if (Q.best) Q.best[gi] = b;
        if (Q.sum) Q.sum[gi] = s;
        if (Q.count) Q.count[gi] = q;
        if (disc < 0 && q >= 1u) disc = t;
        if (adap < 0 && (int64_t)q >= P.adapt_count) adap = t;
        s_stop = (P.stop_when == 1 && q >= 1u) || (P.stop_when == 2 && (int64_t)q >= P.adapt_count);
      }
    }
    __syncthreads();
    {
      uint32_t run = w_sum[wid] + x - acc;
      for (int i = i0; i < i1; i++) {
        run += (uint32_t)__popcll(pop[i]);
        cdf[i] = run;
      }
    }
    const uint32_t total = s_total;
    if (s_stop) { t++; break; }
    __syncthreads();
    const uint64_t gkey = mix64(seed ^ (kGold * ((uint64_t)(P.g0 + t) + 1)));
    auto pick = [&](uint32_t r) -> uint32_t {
      if (total == 0) return r;
      int lo = 0, hi = n - 1;  // first j with cdf[j] > r (cdf[n-1] = total > r)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cdf[mid] > r) hi = mid; else lo = mid + 1;
      }
      return (uint32_t)lo;
    };
    if (P.L <= 32) {  // the same draws with 32-bit masks (ga_draws32)
      for (int i = tid; i < n; i += nt) {
        const ChildDraws32 D = ga_draws32(P, gkey, i, total);
        uint32_t c = (uint32_t)pop[pick(D.ra)];
        if (P.mode != 0) c = (c & D.top) | ((uint32_t)pop[pick(D.rb)] & ~D.top);
        nxt[i] = (c ^ D.flips) & (uint32_t)full;
      }
    } else {
      for (int i = tid; i < n; i += nt) {
        const ChildDraws D = ga_draws(P, gkey, i, total);
        uint64_t c = pop[pick(D.ra)];
        if (P.mode != 0) c = (c & D.top) | (pop[pick(D.rb)] & ~D.top);
        nxt[i] = (c ^ D.flips) & full;
      }
    }
    cur ^= 1;
    __syncthreads();
  }
  if (tid == 31) { Q.done[rep] = t; Q.disc[rep] = disc; Q.adapt[rep] = adap; }
  if (Q.final_pop) {  // a stopped run keeps the population it was evaluated on (as k_ga_run)
    __syncthreads();
    const unsigned long long *fin = cur ? popB : popA;
    for (int i = tid; i < n; i += nt) Q.final_pop[(int64_t)rep * n + i] = fin[i];
  }
}

}  // namespace tvb

namespace tvb {

// ---------------------------------------------------------------------------
// Wide genomes (64 < L <= 4096): W = ceil(L/64) words per genome, stored word-major on
// the device (word w of genome i at pop[w * n + i], so every per-word access of a warp
// is coalesced), little-endian words of genome.to_int() (genome position p = integer bit
// L-1-p).  Semantics: oracle/tv_ga_oracle.c orc_ga_child_w / orc_ga_run_w (the narrow
// operators with the uniform-crossover mask drawn one word at a time).  Per generation
// three stream-ordered launches (fitness + stats, 64-bit inclusive CDF by CUB scan,
// children); a device flag turns the launches of generations after a met stop
// condition into no-ops, so a whole call is enqueued without host round trips.
constexpr int kGaMaxWords = 64;  // L <= 4096

struct GaWideParams {
  int64_t n;
  int32_t L, W, mode;
  uint32_t target;
  int64_t adapt_count;
  int32_t stop_when;
  uint64_t seed;
  int64_t g;                      // generation index of this launch (g0 + t)
  int64_t t;                      // stats row
  const uint64_t *T;              // L Poisson thresholds (device)
  const unsigned long long *pop;  // W x n (word-major)
  unsigned long long *nxt;        // W x n
  unsigned long long *f;          // n fitness (64-bit: the scan input)
  unsigned long long *cdf;        // n inclusive CDF
  uint32_t *best;                 // stats rows
  unsigned long long *sum;
  uint32_t *count;
  int32_t *stopped;               // set once a stop condition is met
  int32_t *final_par;             // parity (t & 1) of the generation the run stopped on, -1 = none
  unsigned long long *done;       // generations evaluated
};

__device__ __forceinline__ uint64_t gw_full(int L, int w) {
  const int hi = L - 64 * w;
  return hi >= 64 ? ~0ULL : ((1ULL << hi) - 1);
}

__global__ void __launch_bounds__(256) k_gaw_fitness(const __grid_constant__ GaWideParams P) {
  if (*((volatile int32_t *)P.stopped)) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t f = 0;
  if (i < P.n) {
    for (int w = 0; w < P.W; w++) f += (uint32_t)__popcll(P.pop[(int64_t)w * P.n + i]);
    P.f[i] = f;
  }
  const bool in = i < P.n;
  const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, in ? f : 0u), mx = __reduce_max_sync(0xFFFFFFFFu, f);
  const uint32_t nc = (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, in && f >= P.target));
  if ((threadIdx.x & 31) == 0) {
    if (s) atomicAdd(&P.sum[P.t], (unsigned long long)s);
    if (mx) atomicMax(&P.best[P.t], mx);
    if (nc) atomicAdd(&P.count[P.t], nc);
  }
  if (i == 0) *P.done = (unsigned long long)(P.t + 1);
}

// first j with cdf[j] > r (cdf[n-1] = total > r), or r itself scaled to n when total == 0
__device__ __forceinline__ int64_t gw_select(const GaWideParams &P, uint64_t &s, uint64_t total) {
  const uint64_t x = ga_draw(s);
  if (total == 0) return (int64_t)__umul64hi(x, (uint64_t)P.n);
  const uint64_t r = __umul64hi(x, total);
  int64_t lo = 0, hi = P.n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (P.cdf[mid] > r) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_gaw_children(const __grid_constant__ GaWideParams P) {
  if (*((volatile int32_t *)P.stopped)) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // stop after recording this generation's stats (evaluated before reproduction)
  const uint32_t c = *((volatile uint32_t *)&P.count[P.t]);
  if ((P.stop_when == 1 && c >= 1u) || (P.stop_when == 2 && (int64_t)c >= P.adapt_count)) {
    __syncthreads();
    if (i == 0) { *P.stopped = 1; *P.final_par = (int32_t)(P.t & 1); }
    return;
  }
  if (i >= P.n) return;
  const int L = P.L, W = P.W;
  const uint64_t total = P.cdf[P.n - 1];
  uint64_t s = stream_state(P.seed, (uint64_t)P.g, (uint64_t)i);
  const int64_t a = gw_select(P, s, total);
  int64_t b = a;
  uint32_t pcut = 0;
  uint64_t smask = 0;
  if (P.mode != 0) {
    b = gw_select(P, s, total);
    if (P.mode == 1) pcut = __umulhi((uint32_t)(ga_draw(s) >> 32), (uint32_t)L);
    else { smask = s; s += (uint64_t)W * kGold; }  // W mask draws, regenerated per word below
  }
  const uint64_t u = ga_draw(s) >> 1;
  int k = 0;
  while (k < L && u >= P.T[k]) k++;
  uint64_t chosen[kGaMaxWords];
  for (int w = 0; w < W; w++) chosen[w] = 0;
  for (int fl = 0; fl < k;) {
    const uint32_t p = __umulhi((uint32_t)(ga_draw(s) >> 32), (uint32_t)L);
    const int bit = L - 1 - (int)p;
    if ((chosen[bit >> 6] >> (bit & 63)) & 1ULL) continue;
    chosen[bit >> 6] |= 1ULL << (bit & 63);
    fl++;
  }
  const int lo = L - (int)pcut;  // single point: integer bits >= lo come from a
  for (int w = 0; w < W; w++) {
    const uint64_t full = gw_full(L, w);
    const uint64_t av = P.pop[(int64_t)w * P.n + a];
    uint64_t cv = av;
    if (P.mode == 1) {
      const uint64_t top = (lo <= 64 * w) ? ~0ULL : (lo >= 64 * w + 64) ? 0ULL : ~((1ULL << (lo - 64 * w)) - 1);
      cv = (av & top) | (P.pop[(int64_t)w * P.n + b] & ~top);
    } else if (P.mode == 2) {
      const uint64_t m = mix64(smask + (uint64_t)(w + 1) * kGold) & full;
      cv = (av & ~m) | (P.pop[(int64_t)w * P.n + b] & m);
    }
    P.nxt[(int64_t)w * P.n + i] = (cv ^ chosen[w]) & full;
  }
}

// placement calibration input (tv_ga_create): a fixed pseudo-random population of L-bit genomes
__global__ void k_ga_fill_random(unsigned long long *pop, int64_t n, int32_t L) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t full = L >= 64 ? ~0ULL : ((1ULL << L) - 1);
  pop[i] = mix64((uint64_t)i * kGold + kMixA) & full;
}

// genome-major (host layout [n, W]) <-> word-major (device layout [W, n])
__global__ void k_gaw_transpose(const unsigned long long *src, unsigned long long *dst, int64_t n, int32_t W,
                                int32_t to_word_major) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n * W) return;
  const int64_t i = j / W, w = j % W;
  if (to_word_major) dst[w * n + i] = src[j];
  else dst[j] = src[w * n + i];
}

// SPEC ACCEPTANCE 8 mutation benchmark (oracle/tv_ga_oracle.c orc_ga_mutate): genome i of a
// word-major population mutated in place with stream (seed, g, i); method 0 = by
// distribution (the GA's operator: only the touched words are read and written), 1 = bit by
// bit (one draw per bit against the 64-bit threshold pthr, every word rewritten).
__global__ void __launch_bounds__(256) k_ga_mutate(unsigned long long *pop, int64_t n, int32_t L,
                                                   const uint64_t *T, uint64_t pthr, int32_t method, uint64_t seed,
                                                   int64_t g, unsigned long long *flips) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t nf = 0;
  if (i < n) {
    uint64_t s = stream_state(seed, (uint64_t)g, (uint64_t)i);
    if (method == 0) {
      const uint64_t u = ga_draw(s) >> 1;
      int k = 0;
      while (k < L && u >= T[k]) k++;
      // distinct positions by rejection; k is small (lambda = muL), so a short list suffices
      // for the membership test, with a bitset fallback for large k
      int pos[16];
      uint64_t chosen[kGaMaxWords];
      const bool small = k <= 16;
      if (!small)
        for (int w = 0; w < (L + 63) / 64; w++) chosen[w] = 0;
      for (int fl = 0; fl < k;) {
        const uint32_t p = __umulhi((uint32_t)(ga_draw(s) >> 32), (uint32_t)L);
        const int bit = L - 1 - (int)p;
        bool dup = false;
        if (small) {
          for (int j = 0; j < fl; j++) dup |= pos[j] == bit;
          if (dup) continue;
          pos[fl] = bit;
        } else {
          if ((chosen[bit >> 6] >> (bit & 63)) & 1ULL) continue;
          chosen[bit >> 6] |= 1ULL << (bit & 63);
        }
        fl++;
      }
      if (small) {
        for (int j = 0; j < k; j++) pop[(int64_t)(pos[j] >> 6) * n + i] ^= 1ULL << (pos[j] & 63);
      } else {
        for (int w = 0; w < (L + 63) / 64; w++)
          if (chosen[w]) pop[(int64_t)w * n + i] ^= chosen[w];
      }
      nf = (uint32_t)k;
    } else {
      const int W = (L + 63) / 64;
      for (int w = W - 1; w >= 0; w--) {  // bit L-1-p lies in word (L-1-p) >> 6: p ascending = words descending
        uint64_t m = 0;
        const int b_hi = min(63, L - 1 - 64 * w);
        for (int b = b_hi; b >= 0; b--) {  // p = L-1-(64w+b) ascending
          const bool fl = ga_draw(s) < pthr;
          m |= (uint64_t)fl << b;
          nf += fl;
        }
        pop[(int64_t)w * n + i] ^= m;
      }
    }
  }
  if (flips) {
    const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, nf);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(flips, (unsigned long long)tot);
  }
}

}  // namespace tvb
