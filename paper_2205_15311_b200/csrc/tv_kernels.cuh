// tv_kernels.cuh -- generic / single-genome / histogram maintenance kernels.
#pragma once
#include "tv_generic.cuh"

namespace tvb {

// Thread-per-genome classify over global scratch (general spaces).
__global__ void __launch_bounds__(128) k_classify_generic(const __grid_constant__ ClassifyParams P) {
  const int64_t T = P.g_threads;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  GView V{P.g_grid, P.g_mark, P.g_stack, P.g_placed, T, t};
  uint32_t *rh = P.run_hash + t;  // run r at rh[r*T]
  uint8_t edges[16 * 16];
  for (int64_t item = t; item < P.n; item += T) {
    const uint64_t idx = item_index(P.indices, P.start, P.chunk, P.stride, item);
    g_decode(P.dec, P.a, idx, edges);
    GFold F = g_classify(edges, P.a, P.d, P.kmax, P.hist_k, P.seed, idx, P.strict, V, rh, T, nullptr, 0);
    if (P.fit_mode) {  // GA JaTAM-shape fitness (see ClassifyParams)
      uint32_t fit = 0;
      if (F.status == 0 && class_at(P.hist_k, F.trivial_at, F.first_unbound, F.first_mismatch) == CLS_DET) {
        GRun R = g_assemble(edges, P.a, P.d, P.strict, P.seed, idx, 0, V);
        int ov = 0, nc = 0;
        for (int r = R.minr; r <= R.maxr; r++)
          for (int c = R.minc; c <= R.maxc; c++)
            if (V.G(r * P.d + c) >= 0) { nc++; ov += (P.target_rows[r + 1] >> (c + 1)) & 1u; }
        g_cleanup(V, R);
        fit = (uint32_t)(P.d * P.d - (P.target_cells + nc - 2 * ov));
      }
      P.out_fit[item] = fit;
      if (P.memo_mask) memo_put(P, idx, fit);
      continue;
    }
    if (F.status != 0) {
      if (!P.hist_mode) {
        for (int k = 0; k < P.q; k++) P.out_class[item * P.q + k] = (uint8_t)CLS_ERROR;
      } else {
        for (int k = 0; k < P.q; k++) atomicAdd(&P.hist.tallies[k * 5 + 4], 1ULL);
      }
      continue;
    }
    for (int k = 0; k < P.q; k++) {
      const int c = class_at(P.ks[k], F.trivial_at, F.first_unbound, F.first_mismatch);
      if (!P.hist_mode) P.out_class[item * P.q + k] = (uint8_t)c;
      else atomicAdd(&P.hist.tallies[k * 5 + c], 1ULL);
    }
    const int hc = class_at(P.hist_k, F.trivial_at, F.first_unbound, F.first_mismatch);
    if (hc != CLS_DET && hc != CLS_STERIC) {
      if (!P.hist_mode) { P.out_hash[item] = 0; P.out_w[item] = 0; P.out_h[item] = 0; P.out_cells[item] = 0; }
      continue;
    }
    unsigned long long *dst = P.out_shape + item * P.W;
    int64_t W = P.W, g = -1;
    if (P.hist_mode) {  // count; the claiming genome provides the payload (fixed at export, tv_hist.cuh)
      bool gnew = false;
      g = hist_claim(P.hist, F.hash, gnew);
      if (g < 0) continue;
      const bool det = hc == CLS_DET;
      atomicAdd(det ? &P.hist.det[g] : &P.hist.steric[g], 1ULL);
      if (det) hist_min(&P.hist.rep_det[g], idx);
      hist_min(&P.hist.rep_any[g], idx);
      if (!gnew) continue;
      dst = P.hist.shape + g * P.hist.W;
      W = P.hist.W;
    }
    // replay the attributed run (identical substream) to emit its bitmap
    GRun R = g_assemble(edges, P.a, P.d, P.strict, P.seed, idx, F.attr_run, V);
    int w, h, nc;
    g_hash_region(V, P.d, R, w, h, nc, dst, W);
    g_cleanup(V, R);
    if (!P.hist_mode) {
      P.out_hash[item] = F.hash;
      P.out_w[item] = (uint8_t)w; P.out_h[item] = (uint8_t)h; P.out_cells[item] = (uint16_t)nc;
    } else {
      P.hist.whc[g] = (uint32_t)w | ((uint32_t)h << 8) | ((uint32_t)nc << 16);
      P.hist.pay_idx[g] = idx;
    }
  }
}

// classify_single (_k:471-484) on one device thread; out[0..5] = status, cls, hash, w, h, cells
__global__ void k_classify_single(const uint8_t *edges_in, int a, int d, int k, uint64_t seed, uint64_t gi,
                                  int strict, unsigned long long *shape, int64_t W, int32_t *out,
                                  int16_t *grid, uint8_t *mark, int32_t *stack, int32_t *placed, uint32_t *rh) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint8_t edges[16 * 16];
  for (int i = 0; i < a * 16; i++) edges[i] = edges_in[i];
  GView V{grid, mark, stack, placed, 1, 0};
  GFold F = g_classify(edges, a, d, k, k, seed, gi, strict, V, rh, 1, shape, W);
  out[0] = F.status;
  out[1] = class_at(k, F.trivial_at, F.first_unbound, F.first_mismatch);
  out[2] = (int32_t)F.hash;
  out[3] = F.w; out[4] = F.h; out[5] = F.cells;
}

// assemble_single (_k:455-468); out[0..5] = outcome, minr, minc, maxr, maxc, n_placed
__global__ void k_assemble_single(const uint8_t *edges_in, int a, int d, uint64_t seed, uint64_t gi, int run,
                                  int strict, int16_t *grid, uint8_t *mark, int32_t *stack, int32_t *placed,
                                  int32_t *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint8_t edges[16 * 16];
  for (int i = 0; i < a * 16; i++) edges[i] = edges_in[i];
  GView V{grid, mark, stack, placed, 1, 0};
  GRun R = g_assemble(edges, a, d, strict, seed, gi, run, V);
  out[0] = R.outcome; out[1] = R.minr; out[2] = R.minc; out[3] = R.maxr; out[4] = R.maxc; out[5] = R.n_placed;
}

__global__ void k_fill_i16(int16_t *p, int64_t n, int16_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_oat(const uint8_t *p, int64_t n, uint32_t *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t h = 0;
  for (int64_t i = 0; i < n; i++) h = oat_step(h, p[i]);
  *out = oat_final(h);
}

// ---- histogram maintenance
__global__ void k_hist_reset(HistDev H) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < H.cap; s += (int64_t)gridDim.x * blockDim.x) {
    H.keys[s] = 0ULL; H.det[s] = 0ULL; H.steric[s] = 0ULL;
    H.rep_det[s] = ~0ULL; H.rep_any[s] = ~0ULL; H.whc[s] = 0u; H.pay_idx[s] = ~0ULL;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < H.q * 5; i += blockDim.x) H.tallies[i] = 0ULL;
    if (threadIdx.x == 0) { *H.n_keys = 0u; *H.overflow = 0u; }
  }
}

__global__ void k_hist_compact(HistDev H, uint32_t *keys_out, uint32_t *slot_out, unsigned int *cnt) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < H.cap; s += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = H.keys[s];
    if (k) {
      const unsigned int p = atomicAdd(cnt, 1u);
      keys_out[p] = (uint32_t)k;
      slot_out[p] = (uint32_t)s;
    }
  }
}

// slots whose payload does not belong to their representative (rep_any)
__global__ void k_hist_stale(HistDev H, uint32_t *slot_out, unsigned long long *idx_out, uint32_t *key_out,
                             unsigned int *cnt) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < H.cap; s += (int64_t)gridDim.x * blockDim.x) {
    if (H.keys[s] && H.pay_idx[s] != H.rep_any[s]) {
      const unsigned int p = atomicAdd(cnt, 1u);
      slot_out[p] = (uint32_t)s;
      idx_out[p] = H.rep_any[s];
      key_out[p] = (uint32_t)H.keys[s];
    }
  }
}

// payload rows of the re-classified representatives -> their slots; a row
// whose hash does not reproduce the slot key flags an error
// rows i*R .. i*R+R-1 belong to stale record i (R = runs replayed per record); the
// first row reproducing the key is the representative's payload
__global__ void k_hist_payload(HistDev H, const uint32_t *slots, const unsigned long long *idx, int64_t n, int R,
                               const uint32_t *hash, const uint8_t *w, const uint8_t *h, const uint16_t *cells,
                               const unsigned long long *shape, unsigned int *err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = slots[i];
    const uint32_t key = (uint32_t)H.keys[s];
    int64_t q = -1;
    for (int j = 0; j < R && q < 0; j++)
      if (hash[i * R + j] == key) q = i * R + j;
    if (q < 0) { atomicOr(err, 1u); continue; }
    H.whc[s] = (uint32_t)w[q] | ((uint32_t)h[q] << 8) | ((uint32_t)cells[q] << 16);
    for (int j = 0; j < H.W; j++) H.shape[s * H.W + j] = shape[q * H.W + j];
    H.pay_idx[s] = idx[i];
  }
}

// Packed raw records for the multi-GPU exchange: row = {key, det, steric, rep_det,
// rep_any, pay_idx, whc, shape[W]} (7 + W u64), payload still the claimer's.
__global__ void k_hist_pack(HistDev H, const uint32_t *slots, int64_t n, unsigned long long *rows) {
  const int64_t R = 7 + H.W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = slots[i];
    unsigned long long *r = rows + i * R;
    r[0] = H.keys[s]; r[1] = H.det[s]; r[2] = H.steric[s]; r[3] = H.rep_det[s]; r[4] = H.rep_any[s];
    r[5] = H.pay_idx[s]; r[6] = H.whc[s];
    for (int j = 0; j < H.W; j++) r[7 + j] = H.shape[s * H.W + j];
  }
}

// Merge packed rows (several rows may share a key: one per rank).  Pass 1 adds the
// counts, lowers the representatives and the per-slot minimum incoming payload owner
// (pmin); pass 2 lets the row holding that owner write the payload if it beats the
// slot's own.  Payload owners are genome indices, distinct across ranks.
__global__ void k_hist_merge_rows1(HistDev H, int64_t n, const unsigned long long *rows, unsigned long long *pmin,
                                   int64_t *slot_of) {
  const int64_t R = 7 + H.W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long *r = rows + i * R;
    if (r[0] == 0ULL) { slot_of[i] = -1; continue; }  // padding row (keys carry a 1 << 32 tag)
    bool gnew = false;
    const int64_t g = hist_claim(H, (uint32_t)r[0], gnew);
    slot_of[i] = g;
    if (g < 0) continue;
    if (r[1]) atomicAdd(&H.det[g], r[1]);
    if (r[2]) atomicAdd(&H.steric[g], r[2]);
    if (r[3] != ~0ULL) hist_min(&H.rep_det[g], r[3]);
    if (r[4] != ~0ULL) hist_min(&H.rep_any[g], r[4]);
    if (r[5] != ~0ULL) atomicMin(&pmin[g], r[5]);
  }
}
__global__ void k_hist_merge_rows2(HistDev H, int64_t n, const unsigned long long *rows,
                                   const unsigned long long *pmin, const int64_t *slot_of) {
  const int64_t R = 7 + H.W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = slot_of[i];
    if (g < 0) continue;
    const unsigned long long *r = rows + i * R;
    if (r[5] == ~0ULL || r[5] != pmin[g] || r[5] >= H.pay_idx[g]) continue;
    H.whc[g] = (uint32_t)r[6];
    for (int j = 0; j < H.W; j++) H.shape[g * H.W + j] = r[7 + j];
    H.pay_idx[g] = r[5];
  }
}

struct HistRecords {  // SoA record arrays (device)
  uint32_t *keys;
  unsigned long long *det, *steric, *rep_det, *rep_any;
  uint8_t *w, *h;
  uint16_t *cells;
  unsigned long long *shape;  // n * W
};

__global__ void k_hist_gather(HistDev H, const uint32_t *slots, int64_t n, HistRecords R) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = slots[i];
    R.det[i] = H.det[s]; R.steric[i] = H.steric[s];
    R.rep_det[i] = H.rep_det[s]; R.rep_any[i] = H.rep_any[s];
    const uint32_t whc = H.whc[s];
    R.w[i] = (uint8_t)(whc & 255u); R.h[i] = (uint8_t)((whc >> 8) & 255u); R.cells[i] = (uint16_t)(whc >> 16);
    for (int j = 0; j < H.W; j++) R.shape[i * H.W + j] = H.shape[s * H.W + j];
  }
}

__global__ void k_hist_merge(HistDev H, int64_t n, HistRecords R, const long long *tallies) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool gnew = false;
    const int64_t g = hist_claim(H, R.keys[i], gnew);
    if (g < 0) continue;
    if (R.det[i]) atomicAdd(&H.det[g], R.det[i]);
    if (R.steric[i]) atomicAdd(&H.steric[g], R.steric[i]);
    if (R.rep_det[i] != ~0ULL) hist_min(&H.rep_det[g], R.rep_det[i]);
    if (R.rep_any[i] != ~0ULL) hist_min(&H.rep_any[g], R.rep_any[i]);
    // an incoming record carries its representative's payload: keep the lowest one
    // (keys are unique within one merge call, so no other thread touches slot g here)
    if (R.rep_any[i] != ~0ULL && R.rep_any[i] < H.pay_idx[g]) {
      H.whc[g] = (uint32_t)R.w[i] | ((uint32_t)R.h[i] << 8) | ((uint32_t)R.cells[i] << 16);
      for (int j = 0; j < H.W; j++) H.shape[g * H.W + j] = R.shape[i * H.W + j];
      H.pay_idx[g] = R.rep_any[i];
    }
    (void)gnew;
  }
  if (tallies && blockIdx.x == 0)
    for (int i = threadIdx.x; i < H.q * 5; i += blockDim.x)
      if (tallies[i]) atomicAdd(&H.tallies[i], (unsigned long long)tallies[i]);
}

}  // namespace tvb
