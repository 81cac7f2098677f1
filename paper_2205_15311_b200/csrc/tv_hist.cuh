// tv_hist.cuh -- device phenotype histogram (SPEC classify:235-240, 297-306, 322).
//
// Open-addressed global table keyed by the 32-bit shape hash.  Per key:
// det/steric genome counts, the lowest DET index and the lowest DET-or-STERIC
// index ("representative = lowest enumeration index"), and the
// payload (w, h, cells, cropped bitmap) of the representative rep_any: the
// genome that claims a key writes its payload (pay_idx = its index) during
// the enumeration; tv_hist_export then re-derives the payload of every slot
// whose pay_idx is not its rep_any from that one genome, so
// colliding shapes under one 32-bit hash resolve to the lowest index exactly
// as the per-genome aggregation does (with ~5e5 keys in S32, distinct shapes
// sharing a 32-bit hash are expected).
// Global class tallies per prefix k (DET, TRIV, STERIC, UNB, ERROR).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvb {

struct HistDev {
  unsigned long long *keys;      // cap; 0 = empty, else (1<<32) | hash
  unsigned long long *det;       // cap
  unsigned long long *steric;    // cap
  unsigned long long *rep_det;   // cap; ~0 = none
  unsigned long long *rep_any;   // cap
  uint32_t *whc;                 // cap; w | h<<8 | cells<<16
  unsigned long long *pay_idx;   // cap; genome whose payload whc/shape hold (~0 = none)
  unsigned long long *shape;     // cap * W
  unsigned long long *tallies;   // q * 5
  unsigned int *n_keys;          // claimed slots
  unsigned int *overflow;        // table full
  int64_t cap;                   // power of two
  int32_t W;
  int32_t q;
};

__device__ __forceinline__ uint64_t hist_home(uint32_t hash, int64_t cap) {
  uint64_t z = (uint64_t)hash * 0x9E3779B97F4A7C15ULL;
  return (z >> 32) & (uint64_t)(cap - 1);
}

// find-or-claim; returns slot or -1 when the table is full
__device__ __forceinline__ int64_t hist_claim(const HistDev &H, uint32_t hash, bool &is_new) {
  const unsigned long long key = (1ULL << 32) | hash;
  uint64_t s = hist_home(hash, H.cap);
  is_new = false;
  for (int64_t p = 0; p < H.cap; p++) {
    unsigned long long k = *((volatile unsigned long long *)&H.keys[s]);
    if (k == key) return (int64_t)s;
    if (k == 0ULL) {
      const unsigned long long old = atomicCAS(&H.keys[s], 0ULL, key);
      if (old == 0ULL) {
        is_new = true;
        atomicAdd(H.n_keys, 1u);
        return (int64_t)s;
      }
      if (old == key) return (int64_t)s;
    }
    s = (s + 1) & (uint64_t)(H.cap - 1);
  }
  atomicOr(H.overflow, 1u);
  return -1;
}

__device__ __forceinline__ void hist_min(unsigned long long *p, unsigned long long v) {
  if (*((volatile unsigned long long *)p) > v) atomicMin(p, v);
}

}  // namespace tvb
