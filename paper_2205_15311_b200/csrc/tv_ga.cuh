// tv_ga.cuh -- GA generation loop (SPEC.md evolve module).
//
// One cooperative persistent kernel runs many generations; per generation:
//   A. fitness (Fujiyama popcount, or an externally computed vector), per
//      thread sums over a contiguous run, a block scan, and the stats;
//   B. grid barrier; chunk offsets -> global inclusive CDF (u32) and a coarse
//      table (last CDF value of every s-entry segment, <= 32768 entries);
//   C. grid barrier; every CTA stages the coarse table in shared memory and
//      produces its chunk of children: roulette selection = search of the
//      coarse table in shared memory + a binary search inside one s-entry
//      segment (one cache line for s = 32), crossover, Poisson mutation;
//   D. grid barrier; swap population buffers.
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
  int64_t seg;           // coarse segment length s (power of two)
  int32_t seg_shift;     // log2(seg)
  int64_t n_coarse;      // ceil(n / seg)
  uint64_t T[64];        // Poisson CDF thresholds x 2^63 (k = #{j < L : (draw >> 1) >= T[j]})
  unsigned long long *pop0, *pop1;
  const uint32_t *f_ext;
  uint32_t *cdf;         // n
  uint32_t *coarse;      // n_coarse
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

// roulette selection: first j with cdf[j] > r, r = mulhi(draw, total)
__device__ __forceinline__ int64_t ga_select(uint64_t &s, const GaParams &P, const uint32_t *coarse_s,
                                             uint32_t total) {
  const uint64_t x = ga_draw(s);
  if (total == 0) return (int64_t)__umul64hi(x, (uint64_t)P.n);  // SPEC:447 uniform fallback
  const uint32_t r = (uint32_t)__umul64hi(x, (uint64_t)total);
  int64_t lo = 0, hi = P.n_coarse - 1;  // first segment whose last value exceeds r
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (coarse_s[mid] > r) hi = mid; else lo = mid + 1;
  }
  int64_t a = lo << P.seg_shift, b = min(P.n, a + P.seg) - 1;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (P.cdf[mid] > r) b = mid; else a = mid + 1;  // one 128-B line for seg = 32: L1 after the first probe
  }
  return a;
}

__device__ __forceinline__ uint64_t ga_child(const GaParams &P, const unsigned long long *pop, int64_t g,
                                             int64_t i, const uint32_t *coarse_s, uint32_t total) {
  uint64_t s = stream_state(P.seed, (uint64_t)g, (uint64_t)i);
  const int L = P.L;
  const uint64_t full = L == 64 ? ~0ULL : ((1ULL << L) - 1);
  const uint64_t a = pop[ga_select(s, P, coarse_s, total)];
  uint64_t child = a;
  if (P.mode != 0) {
    const uint64_t b = pop[ga_select(s, P, coarse_s, total)];
    if (P.mode == 1) {  // positions < p from a, >= p from b
      const uint32_t p = ga_below(s, (uint32_t)L);
      const uint64_t top = p == 0 ? 0ULL : (full & ~((1ULL << (L - p)) - 1));
      child = (a & top) | (b & ~top & full);
    } else {            // each bit from b where the mask is set
      const uint64_t m = ga_draw(s) & full;
      child = (a & ~m) | (b & m);
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
  return (child ^ chosen) & full;
}

__global__ void __launch_bounds__(1024, 1) k_ga_run(const __grid_constant__ GaParams P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint32_t coarse_s[];       // n_coarse
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
  for (; t < P.n_gens; t++) {
    const int64_t g = P.g0 + t;
    const unsigned long long *pop = cur ? P.pop1 : P.pop0;
    unsigned long long *nxt = cur ? P.pop0 : P.pop1;
    if (tid == 0) { s_best = 0; s_cnt = 0; }
    // ---- A: fitness sums per thread, block scan -> thread offsets, stats
    uint32_t acc = 0, best = 0, cnt = 0;
    for (int64_t i = i0; i < i1; i++) {
      const uint32_t f = P.fitness == 0 ? (uint32_t)__popcll(pop[i]) : P.f_ext[i];
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
    // ---- B: chunk offsets -> global CDF + coarse table; stop decision
    if (wid == 0) {
      unsigned long long o = 0, tt = 0;
      for (int j = lane; j < (int)gridDim.x; j += 32) {
        const unsigned long long v = __ldcg(&P.tot[j]);
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
    if (blockIdx.x == 0 && tid == 0) P.sum[t] = s_total;
    if (s_stop) { t++; break; }
    {
      uint32_t run = (uint32_t)s_off + excl;
      for (int64_t i = i0; i < i1; i++) {
        run += P.fitness == 0 ? (uint32_t)__popcll(pop[i]) : P.f_ext[i];
        P.cdf[i] = run;
        if (((i + 1) & (P.seg - 1)) == 0 || i == P.n - 1) P.coarse[i >> P.seg_shift] = run;
      }
    }
    grid.sync();
    // ---- C: children
    for (int64_t j = tid; j < P.n_coarse; j += nt) coarse_s[j] = P.coarse[j];
    __syncthreads();
    for (int64_t i = c0 + tid; i < c1; i += nt) nxt[i] = ga_child(P, pop, g, i, coarse_s, total);
    cur ^= 1;
    grid.sync();
  }
  if (blockIdx.x == 0 && tid == 0) {
    *P.done = (unsigned long long)t;
    *P.final_buf = cur;
  }
}

}  // namespace tvb
