// tv_generic.cuh -- thread-per-genome movelist assembly over global scratch.
//
// The general-shape path: any a <= 16 tiles, any label alphabet b <= 256,
// any odd d (3..181).  Used by classify_batch / enumerate_range when the
// shared-memory bitboard kernel (tv_fast.cuh) does not cover the space, and by
// the single-genome entry points (assemble_single / classify_single).
// Step order is the reference's exactly (_k:96-249; Appendix A of SURVEY.md).
#pragma once
#include "tv_params.cuh"

namespace tvb {

struct GView {
  int16_t *grid;
  uint8_t *mark;
  int32_t *stack;
  int32_t *placed;
  int64_t T, t;  // element j of thread t lives at [j*T + t] (coalesced across threads)
  __device__ __forceinline__ int16_t &G(int j) const { return grid[(int64_t)j * T + t]; }
  __device__ __forceinline__ uint8_t &M(int j) const { return mark[(int64_t)j * T + t]; }
  __device__ __forceinline__ int32_t &St(int j) const { return stack[(int64_t)j * T + t]; }
  __device__ __forceinline__ int32_t &Pl(int j) const { return placed[(int64_t)j * T + t]; }
};

struct GRun {
  int outcome, n_placed, sp, minr, minc, maxr, maxc;
};

// One assembly on clean scratch (_k:96-249).
__device__ GRun g_assemble(const uint8_t *edges, int a, int d, int strict, uint64_t seed,
                           uint64_t idx, int run, const GView &V) {
  GRun R;
  uint64_t s = stream_state(seed, idx, (uint64_t)run);
  const int dd = d * d, half = d >> 1, ctr = half * d + half;
  V.G(ctr) = 0;
  V.Pl(0) = ctr;
  R.n_placed = 1;
  R.minr = R.maxr = R.minc = R.maxc = half;
  int nb0 = ctr - d, nb1 = ctr + 1, nb2 = ctr + d, nb3 = ctr - 1;
  int nb[4] = {nb0, nb1, nb2, nb3};
#pragma unroll
  for (int j = 3; j > 0; j--) {
    const int q = (int)rng_below(s, (uint32_t)(j + 1));
    const int t = nb[j];
    nb[j] = nb[q];
    nb[q] = t;
  }
  int sp = 0;
  for (int j = 0; j < 4; j++) {
    V.M(nb[j]) = 1;
    V.St(sp++) = nb[j];
  }
  while (sp > 0) {
    const int cell = V.St(--sp);
    V.M(cell) = 0;
    const int r = cell / d, c = cell - r * d;
    int p[4] = {-1, -1, -1, -1};
    if (r > 0) { const int v = V.G(cell - d); if (v >= 0) p[0] = edges[(v >> 2) * 16 + (v & 3) * 4 + 2]; }
    if (c < d - 1) { const int v = V.G(cell + 1); if (v >= 0) p[1] = edges[(v >> 2) * 16 + (v & 3) * 4 + 3]; }
    if (r < d - 1) { const int v = V.G(cell + d); if (v >= 0) p[2] = edges[(v >> 2) * 16 + (v & 3) * 4 + 0]; }
    if (c > 0) { const int v = V.G(cell - 1); if (v >= 0) p[3] = edges[(v >> 2) * 16 + (v & 3) * 4 + 1]; }
    int64_t found = -1;
    int found_v = -1;
    bool ambiguous = false;
    for (int t = 0; t < a && !ambiguous; t++) {
      for (int rt = 0; rt < 4; rt++) {
        const uint8_t *e = edges + t * 16 + rt * 4;
        bool bond = false, ok = true;
        for (int k = 0; k < 4 && ok; k++) {
          if (p[k] < 0) continue;
          if (bonds(e[k], p[k])) bond = true;
          else if (strict && e[k] != 0 && p[k] != 0) ok = false;
        }
        if (ok && bond) {
          const int64_t code = ((int64_t)e[0] << 24) | ((int64_t)e[1] << 16) | ((int64_t)e[2] << 8) | e[3];
          if (found < 0) { found = code; found_v = t * 4 + rt; }
          else if (code != found) { ambiguous = true; break; }
        }
      }
    }
    if (ambiguous) { R.outcome = RUN_TRIVIAL; R.sp = sp; return R; }
    if (found < 0) continue;
    if (r == 0 || c == 0 || r == d - 1 || c == d - 1) { R.outcome = RUN_UNBOUND; R.sp = sp; return R; }
    V.G(cell) = (int16_t)found_v;
    V.Pl(R.n_placed++) = cell;
    R.minr = min(R.minr, r); R.maxr = max(R.maxr, r);
    R.minc = min(R.minc, c); R.maxc = max(R.maxc, c);
    int m = 0;
    const int nbc[4] = {cell - d, cell + 1, cell + d, cell - 1};
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (V.G(nbc[k]) < 0 && V.M(nbc[k]) == 0) nb[m++] = nbc[k];
    for (int j = m - 1; j > 0; j--) {
      const int q = (int)rng_below(s, (uint32_t)(j + 1));
      const int t = nb[j];
      nb[j] = nb[q];
      nb[q] = t;
    }
    for (int j = 0; j < m; j++) {
      if (sp >= dd) { R.outcome = RUN_OVERFLOW; R.sp = sp; return R; }
      V.M(nb[j]) = 1;
      V.St(sp++) = nb[j];
    }
  }
  R.outcome = RUN_BOUNDED;
  R.sp = 0;
  return R;
}

__device__ __forceinline__ void g_cleanup(const GView &V, const GRun &R) {
  for (int i = 0; i < R.sp; i++) V.M(V.St(i)) = 0;
  for (int i = 0; i < R.n_placed; i++) V.G(V.Pl(i)) = -1;
}

// OAT over the cropped shape (_k:260-277); optionally packs the bitmap
// (_k:280-292) into out[0..W) (streamed, register-only).
__device__ uint32_t g_hash_region(const GView &V, int d, const GRun &R, int &w, int &h, int &n,
                                  unsigned long long *out, int64_t W) {
  w = R.maxc - R.minc + 1;
  h = R.maxr - R.minr + 1;
  n = 0;
  uint32_t st = oat_step(oat_step(0u, (uint32_t)w), (uint32_t)h);
  int64_t cw = 0;
  unsigned long long acc = 0;
  int bit = 0;
  for (int y = 0; y < h; y++) {
    const int row = (R.minr + y) * d + R.minc;
    for (int x = 0; x < w; x++, bit++) {
      if (V.G(row + x) >= 0) {
        st = oat_step(oat_step(st, (uint32_t)x), (uint32_t)y);
        n++;
        if (out && (bit >> 6) < W) {  // bits past the caller's W words are dropped
          const int64_t wi = bit >> 6;
          while (cw < wi) { out[cw++] = acc; acc = 0; }
          acc |= 1ULL << (bit & 63);
        }
      }
    }
  }
  if (out) {
    while (cw < W) { out[cw++] = acc; acc = 0; }
  }
  return oat_final(st);
}

struct GFold {
  int status, trivial_at, first_unbound, first_mismatch;
  uint32_t hash;
  int w, h, cells;
  int attr_run;  // run whose shape is attributed (DET/STERIC at hist_k), else -1
};

// k-run fold (_k:306-381).  shape_now != nullptr reproduces classify_single's
// buffer semantics (run 0 packed as soon as it is bounded, steric re-run
// overwrites).  Otherwise the attributed run is only reported in attr_run and
// the caller packs it by replaying that run (identical substream).
__device__ GFold g_classify(const uint8_t *edges, int a, int d, int kmax, int hist_k, uint64_t seed,
                            uint64_t idx, int strict, const GView &V, uint32_t *run_hash, int64_t rh_stride,
                            unsigned long long *shape_now, int64_t W) {
  GFold F = {0, -1, -1, -1, 0u, 0, 0, 0, -1};
  int w0 = 0, h0 = 0, c0 = 0;
  uint32_t hash0 = 0;
  for (int run = 0; run < kmax; run++) {
    GRun R = g_assemble(edges, a, d, strict, seed, idx, run, V);
    if (R.outcome == RUN_OVERFLOW) {
      g_cleanup(V, R);
      F.status = 1;
      return F;
    }
    if (R.outcome == RUN_TRIVIAL) { g_cleanup(V, R); F.trivial_at = run; break; }
    if (R.outcome == RUN_UNBOUND) {
      if (F.first_unbound < 0) F.first_unbound = run;
      run_hash[(int64_t)run * rh_stride] = 0;
      g_cleanup(V, R);
      continue;
    }
    int w, h, nc;
    const uint32_t hs = g_hash_region(V, d, R, w, h, nc, run == 0 ? shape_now : nullptr, W);
    run_hash[(int64_t)run * rh_stride] = hs;
    if (run == 0) { w0 = w; h0 = h; c0 = nc; hash0 = hs; }
    else if (F.first_mismatch < 0 && F.first_unbound != 0 && hs != hash0) F.first_mismatch = run;
    g_cleanup(V, R);
  }
  const int hc = class_at(hist_k, F.trivial_at, F.first_unbound, F.first_mismatch);
  if (hc == CLS_DET) { F.hash = hash0; F.w = w0; F.h = h0; F.cells = c0; F.attr_run = 0; return F; }
  if (hc != CLS_STERIC) return F;
  uint32_t best = 0;
  int best_n = 0;
  for (int j = 0; j < hist_k; j++) {
    const uint32_t hj = run_hash[(int64_t)j * rh_stride];
    int cnt = 0;
    for (int l = 0; l < hist_k; l++) cnt += run_hash[(int64_t)l * rh_stride] == hj;
    if (cnt > best_n || (cnt == best_n && hj < best)) { best_n = cnt; best = hj; }
  }
  F.hash = best; F.w = w0; F.h = h0; F.cells = c0; F.attr_run = 0;
  if (best == hash0) return F;
  for (int j = 1; j < hist_k; j++) {
    if (run_hash[(int64_t)j * rh_stride] != best) continue;
    F.attr_run = j;
    if (shape_now) {
      GRun R = g_assemble(edges, a, d, strict, seed, idx, j, V);
      g_hash_region(V, d, R, F.w, F.h, F.cells, shape_now, W);
      g_cleanup(V, R);
    }
    return F;
  }
  return F;
}

// Fill the in-situ edge table for index idx (_k:384-401).
__device__ __forceinline__ void g_decode(const LabelDecoder &D, int a, uint64_t idx, uint8_t *edges) {
  uint8_t lab[64];
  for (int te = 0; te < a * 4; te++) lab[te] = (uint8_t)decode_label(D, te, idx);
  for (int t = 0; t < a; t++)
    for (int rt = 0; rt < 4; rt++)
      for (int dr = 0; dr < 4; dr++) edges[t * 16 + rt * 4 + dr] = lab[t * 4 + ((dr - rt) & 3)];
}

}  // namespace tvb
