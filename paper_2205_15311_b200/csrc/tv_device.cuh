// tv_device.cuh -- device-side primitives shared by the tilevolve-b200 kernels.
//
// Semantics follow the reference numba kernels
// (/root/reference/pkg/src/tilevolve/_kernels.py, cited "_k:LINE").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvb {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ULL;  // _k:31
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ULL;  // _k:32
constexpr uint64_t kMixB = 0x94D049BB133111EBULL;  // _k:33

enum RunOutcome : int { RUN_BOUNDED = 0, RUN_TRIVIAL = 1, RUN_UNBOUND = 2, RUN_OVERFLOW = 3 };
enum ClassCode : int { CLS_DET = 0, CLS_TRIV = 1, CLS_STERIC = 2, CLS_UNB = 3, CLS_ERROR = 255 };

// splitmix64 finaliser (_k:38-42)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return z ^ (z >> 31);
}

// substream keyed by (seed, enumeration index, run) (_k:45-48)
__host__ __device__ __forceinline__ uint64_t stream_state(uint64_t seed, uint64_t idx, uint64_t run) {
  const uint64_t z = mix64(seed ^ (kGold * (idx + 1)));
  return mix64(z ^ (kMixA * (run + 1)));
}

// counter-based draw: advance then mix; bounded draw uses the high word (_k:51-60).
// Only the high 32 bits of the mixed value are consumed, so the last xor-shift
// is evaluated on the high word alone.
__device__ __forceinline__ uint32_t rng_hi(uint64_t z) {  // high word of mix64(z)
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return (uint32_t)(z >> 32) ^ (uint32_t)(z >> 63);
}
__device__ __forceinline__ uint32_t rng_below(uint64_t &s, uint32_t n) {
  s += kGold;
  return __umulhi(rng_hi(s), n);
}

// one-at-a-time hash steps (_k:65-76)
__host__ __device__ __forceinline__ uint32_t oat_step(uint32_t h, uint32_t k) {
  h += k;
  h += h << 10;
  return h ^ (h >> 6);
}
__host__ __device__ __forceinline__ uint32_t oat_final(uint32_t h) {
  h += h << 3;
  h ^= h >> 11;
  return h + (h << 15);
}

// prefix class at k' with precedence TRIV > UNB > STERIC > DET (_k:295-303)
__host__ __device__ __forceinline__ int class_at(int kp, int trivial_at, int first_unbound, int first_mismatch) {
  if (trivial_at >= 0 && trivial_at < kp) return CLS_TRIV;
  if (first_unbound >= 0 && first_unbound < kp) return CLS_UNB;
  if (first_mismatch >= 0 && first_mismatch < kp) return CLS_STERIC;
  return CLS_DET;
}

// label pairing 1-2, 3-4, ... (_k:90-93)
__host__ __device__ __forceinline__ bool bonds(int i, int j) { return i != 0 && j == (((i - 1) ^ 1) + 1); }

// Enumeration index -> label decoder (_k:384-397, semantics gen:158-165,
// 199-202, 246-255).  The host simulates the reference's bit writes (mask
// first, then free bit j -> free_pos[j], last write wins) and reduces every
// label field te (tile-major, N,E,S,W, MSB-first) to either
//   fast form:    label = fix | (((idx >> lo) & ((1<<nf)-1)) << sh)
// which covers every SearchSpace (a label's free bits are consecutive index
// bits because free_positions() is descending), or, for arbitrary raw arrays,
//   general form: label bit k <- index bit src[te*8+k] (0xFF = constant).
struct LabelDecoder {
  int32_t nlab;     // a*4
  int32_t bpl;
  int32_t general;  // 0: fast form for every label
  int32_t pad_;
  uint8_t lo[64], nf[64], sh[64], fix[64];
  uint32_t pk[64];  // fast form packed: lo | ((1 << nf) - 1) << 8 | sh << 16 | fix << 24
  uint8_t src[64 * 8];
};

__device__ __forceinline__ uint32_t decode_label(const LabelDecoder &D, int te, uint64_t idx) {
  if (!D.general) {  // one constant load, no branch
    const uint32_t w = D.pk[te];
    return (w >> 24) | (((uint32_t)(idx >> (w & 63u)) & ((w >> 8) & 0xFFu)) << ((w >> 16) & 0xFFu));
  }
  uint32_t v = D.fix[te];
  {
    for (int k = 0; k < D.bpl; k++) {
      const uint32_t s = D.src[te * 8 + k];
      if (s != 0xFF) v |= (uint32_t)((idx >> s) & 1ULL) << k;
    }
  }
  return v;
}

// enumeration index of work item i (explicit list, plain range, or strided chunks)
__device__ __forceinline__ uint64_t item_index(const uint64_t *indices, uint64_t start, uint64_t chunk,
                                               uint64_t stride, int64_t item) {
  if (indices) return indices[item];
  if (chunk == 0) return start + (uint64_t)item;
  const uint64_t c = (uint64_t)item / chunk;
  return start + c * stride + ((uint64_t)item - c * chunk);
}

}  // namespace tvb
