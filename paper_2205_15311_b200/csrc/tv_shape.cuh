// tv_shape.cuh -- canonical phenotype labels of cropped shapes (extra columns).
//
// The reference phenotype key is the translation-invariant OAT hash of the
// cropped shape (_k:260-277).  Two canonical labels are derived
// from the packed bitmap (_k:280-292: bit y*w+x, LSB-first per u64 word):
//   rot4 : SPEC.md:270-278 rotation-invariant hash -- the four clockwise
//          rotations' shape hashes, sorted ascending, OAT over their 16
//          little-endian bytes (no reflections);
//   d4   : minimum shape hash over the 8 rotations and reflections (dihedral
//          group D4), the north star's canonical min-hash label.
// Neither replaces the histogram key (parity with the reference requires the
// plain hash); they are computed per histogram record or per genome row.
//
// Layout: 8 consecutive lanes per shape, lane t = transform (t & 3 clockwise
// quarter turns of the shape, mirrored left-right first when t >= 4).  Each
// lane walks its transformed frame row-major and hashes (x', y') of occupied
// cells; the group reduces with shuffles.  Shapes are tiny (<= 17x17 cells
// at d = 19) and there are 10^3..10^5 records, so this is latency, not
// bandwidth: one launch, 8 lanes per record, bitmap words read through L1.
#pragma once
#include "tv_device.cuh"

namespace tvb {

// occupancy of source cell (x, y) of a w-wide packed bitmap
__device__ __forceinline__ uint32_t shape_bit(const unsigned long long *words, int w, int x, int y) {
  const int b = y * w + x;
  return (uint32_t)(words[b >> 6] >> (b & 63)) & 1u;
}

// shape hash of transform t of the (w, h) shape: OAT(w', h', then x', y' of
// occupied cells row-major in the transformed frame), _k:264-277
__device__ uint32_t transformed_hash(const unsigned long long *words, int w, int h, int t) {
  const int r = t & 3;
  const bool mir = t >= 4;
  const int wt = (r & 1) ? h : w, ht = (r & 1) ? w : h;
  uint32_t s = oat_step(oat_step(0u, (uint32_t)wt), (uint32_t)ht);
  for (int yp = 0; yp < ht; yp++) {
    for (int xp = 0; xp < wt; xp++) {
      // inverse of the clockwise rotation: frame (xp, yp) -> (xm, ym) of the (mirrored) source
      int xm, ym;
      if (r == 0) { xm = xp; ym = yp; }
      else if (r == 1) { xm = yp; ym = h - 1 - xp; }
      else if (r == 2) { xm = w - 1 - xp; ym = h - 1 - yp; }
      else { xm = w - 1 - yp; ym = xp; }
      const int x = mir ? w - 1 - xm : xm;
      if (shape_bit(words, w, x, ym)) s = oat_step(oat_step(s, (uint32_t)xp), (uint32_t)yp);
    }
  }
  return oat_final(s);
}

// One group of 8 lanes per record; blockDim.x must be a multiple of 32.
__global__ void k_shape_labels(const unsigned long long *shape, const uint8_t *w, const uint8_t *h, int64_t n,
                               int64_t W, uint32_t *out_rot4, uint32_t *out_d4) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = threadIdx.x & 7;
  const int64_t rec = tid >> 3;
  const bool valid = rec < n;
  uint32_t hv = 0xFFFFFFFFu;
  int ww = 0, hh = 0;
  if (valid) {
    ww = w[rec]; hh = h[rec];
    if (ww > 0 && hh > 0 && (int64_t)ww * hh <= W * 64) hv = transformed_hash(shape + rec * W, ww, hh, t);
  }
  const unsigned full = 0xFFFFFFFFu;  // every lane of the block reaches the shuffles
  // d4: min over the 8 lanes
  uint32_t mn = hv;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) mn = min(mn, __shfl_xor_sync(full, mn, o, 8));
  // rot4: lanes 0..3 hold the four rotations; sort ascending and re-hash 16 LE bytes
  uint32_t r0 = __shfl_sync(full, hv, 0, 8), r1 = __shfl_sync(full, hv, 1, 8);
  uint32_t r2 = __shfl_sync(full, hv, 2, 8), r3 = __shfl_sync(full, hv, 3, 8);
  if (valid && t == 0) {
    uint32_t a0 = min(r0, r1), a1 = max(r0, r1), a2 = min(r2, r3), a3 = max(r2, r3);
    const uint32_t b0 = min(a0, a2), b3 = max(a1, a3);
    const uint32_t m1 = max(a0, a2), m2 = min(a1, a3);
    const uint32_t s[4] = {b0, min(m1, m2), max(m1, m2), b3};
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int byte = 0; byte < 4; byte++) x = oat_step(x, (s[i] >> (8 * byte)) & 0xFFu);
    const bool ok = ww > 0 && hh > 0 && (int64_t)ww * hh <= W * 64;
    if (out_rot4) out_rot4[rec] = ok ? oat_final(x) : 0u;
    if (out_d4) out_d4[rec] = ok ? mn : 0u;
  }
}

}  // namespace tvb
