// tv_ga.cuh -- GA generation loop (SPEC.md evolve module).
//
// One cooperative persistent kernel runs many generations; per generation:
//   A. per-thread sums over a contiguous run of the fitness vector (staged in
//      index order when the children were made), block scan, stats;
//   -- grid barrier --
//   B. chunk offsets -> global inclusive CDF (u32) and a guide table for
//      indexed search (Chen & Asau): the r-range [0, total) is cut into
//      B = min(n, total) monotone buckets b(r) = (r * M) >> 32 and guide[b] =
//      the individual owning the first r of bucket b; individual j writes the
//      buckets whose first r lies in its own range [cdf[j-1], cdf[j]), so the
//      table is built in the same pass;
//   -- grid barrier --
//   C. children: all random draws of a child first (selection draws,
//      crossover mask, mutation mask), then selection = guide[b(r)] plus a short
//      forward scan while cdf[j] <= r (exactly the first j with cdf[j] > r),
//      parent loads and the child, two children interleaved per thread; the
//      child's Fujiyama fitness is staged for the next generation's phase A.
// Two grid barriers per generation.
// Data written by other CTAs is read only after a grid barrier (grid.sync()
// orders and publishes all prior writes of the grid; its gpu-scope acquire
// invalidates L1), so ordinary cached loads are used.
// Semantics (draw order, masks, thresholds) are defined by the CPU
// restatement oracle/tv_ga_oracle.c, which the GPU reproduces bit for bit.
#pragma once
#include <cooperative_groups.h>

#include "tv_device.cuh"

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
  uint32_t *cdf;         // n
  uint32_t *fstage;      // n: fitness staged in index order (own chunk per CTA)
  uint32_t *guide;       // n (first B entries used in a generation)
  unsigned long long *tot;  // per CTA chunk totals
  uint32_t *best;        // n_gens
  unsigned long long *sum;  // n_gens
  uint32_t *count;       // n_gens
  unsigned long long *done;  // generations evaluated (written by CTA 0)
  int32_t *final_buf;    // which pop buffer holds the final population
};

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

// roulette: first j with cdf[j] > r, from the guide entry of r's bucket
__device__ __forceinline__ uint32_t ga_pick(const GaParams &P, uint32_t r, uint32_t total, uint64_t mul) {
  if (total == 0) return r;
  uint32_t j = P.guide[(uint32_t)(((uint64_t)r * mul) >> 32)];  // mul <= 2^32: no overflow
  while (P.cdf[j] <= r) j++;
  return j;
}

__global__ void __launch_bounds__(1024, 1) k_ga_run(const __grid_constant__ GaParams P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t warp_sum[32];
  __shared__ uint32_t s_best, s_cnt;
  __shared__ unsigned long long s_off, s_total;
  __shared__ int s_stop;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * P.chunk;
  const int64_t c1 = min(P.n, c0 + P.chunk);
  const int64_t len = max((int64_t)0, c1 - c0);
  const int64_t per = (len + nt - 1) / nt;     // contiguous items per thread
  const int64_t i0 = c0 + tid * per, i1 = min(c1, i0 + per);
  int cur = 0;
  int64_t t = 0;
  // fitness of the initial population, staged in index order
  for (int64_t i = c0 + tid; i < c1; i += nt)
    P.fstage[i] = P.fitness == 0 ? (uint32_t)__popcll(P.pop0[i]) : P.f_ext[i];
  __syncthreads();
  for (; t < P.n_gens; t++) {
    const int64_t g = P.g0 + t;
    const unsigned long long *pop = cur ? P.pop1 : P.pop0;
    unsigned long long *nxt = cur ? P.pop0 : P.pop1;
    if (tid == 0) { s_best = 0; s_cnt = 0; }
    // ---- A: per-thread sums over a contiguous run of staged fitness, block scan, stats
    uint32_t acc = 0, best = 0, cnt = 0;
    for (int64_t i = i0; i < i1; i++) {
      const uint32_t f = P.fstage[i];
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
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t w = lane < (nt >> 5) ? warp_sum[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w += y;
      }
      warp_sum[lane] = w;
    }
    __syncthreads();
    const uint32_t excl = x - acc + (wid ? warp_sum[wid - 1] : 0u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
      cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    }
    if (lane == 0) { atomicMax(&s_best, best); atomicAdd(&s_cnt, cnt); }
    __syncthreads();
    if (tid == 0) {
      P.tot[blockIdx.x] = warp_sum[(nt >> 5) - 1];
      atomicMax(&P.best[t], s_best);
      atomicAdd(&P.count[t], s_cnt);
    }
    grid.sync();
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
        const uint32_t c = *((volatile uint32_t *)&P.count[t]);
        s_stop = (P.stop_when == 1 && c >= 1u) || (P.stop_when == 2 && (int64_t)c >= P.adapt_count);
      }
    }
    __syncthreads();
    const uint32_t total = (uint32_t)s_total;
    // bucket function b(r) = (r * mul) >> 32, monotone, B = min(n, total) buckets
    const uint64_t nb = min((uint64_t)P.n, (uint64_t)total);
    const uint64_t mul = total ? (nb << 32) / total : 0ull;
    if (blockIdx.x == 0 && tid == 0) P.sum[t] = s_total;
    if (s_stop) { t++; break; }
    {
      uint32_t prev = (uint32_t)s_off + excl, run = prev;
      for (int64_t i = i0; i < i1; i++) {
        run += P.fstage[i];
        P.cdf[i] = run;
        if (run != prev) {  // own r in [prev, run): buckets whose first r falls in it
          const int64_t b0 = prev ? (int64_t)(((uint64_t)(prev - 1) * mul) >> 32) + 1 : 0;
          const int64_t b1 = (int64_t)(((uint64_t)(run - 1) * mul) >> 32);
          for (int64_t b = b0; b <= b1; b++) P.guide[b] = (uint32_t)i;
        }
        prev = run;
      }
    }
    grid.sync();
    const uint64_t gkey = mix64(P.seed ^ (kGold * ((uint64_t)g + 1)));  // stream_state prefix (_k:45-48)
    // ---- C: children, two at a time (draws first, then the dependent loads);
    //      the next generation's fitness is staged as the children are made
    for (int64_t i = c0 + tid; i < c1; i += 2 * nt) {
      const int64_t i2 = i + nt;
      const bool two = i2 < c1;
      const ChildDraws D1 = ga_draws(P, gkey, i, total);
      const ChildDraws D2 = two ? ga_draws(P, gkey, i2, total) : D1;
      const uint32_t a1 = ga_pick(P, D1.ra, total, mul), a2 = ga_pick(P, D2.ra, total, mul);
      uint64_t c1v = pop[a1], c2v = pop[a2];
      if (P.mode != 0) {
        const uint32_t b1 = ga_pick(P, D1.rb, total, mul), b2 = ga_pick(P, D2.rb, total, mul);
        const uint64_t p1 = pop[b1], p2 = pop[b2];
        c1v = (c1v & D1.top) | (p1 & ~D1.top);
        c2v = (c2v & D2.top) | (p2 & ~D2.top);
      }
      const uint64_t full = P.L == 64 ? ~0ULL : ((1ULL << P.L) - 1);
      c1v = (c1v ^ D1.flips) & full;
      nxt[i] = c1v;
      if (P.fitness == 0) P.fstage[i] = (uint32_t)__popcll(c1v);
      if (two) {
        c2v = (c2v ^ D2.flips) & full;
        nxt[i2] = c2v;
        if (P.fitness == 0) P.fstage[i2] = (uint32_t)__popcll(c2v);
      }
    }
    cur ^= 1;
    __syncthreads();  // this CTA's staged fitness is read in index order by phase A
  }
  if (blockIdx.x == 0 && tid == 0) {
    *P.done = (unsigned long long)t;
    *P.final_buf = cur;
  }
}

}  // namespace tvb
