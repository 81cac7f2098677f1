// tv_params.cuh -- launch parameter blocks shared by host (tv_capi.cu) and kernels.
#pragma once
#include <cstdint>
#include "tv_device.cuh"
#include "tv_hist.cuh"

namespace tvb {

constexpr int kMaxKs = 64;

struct ClassifyParams {
  LabelDecoder dec;
  const uint64_t *indices;  // classify mode: enumeration indices; nullptr in range mode
  uint64_t start;           // range mode: item i -> index start + (i / chunk) * stride + (i % chunk)
  uint64_t chunk, stride;   // chunk == 0: plain range start + i
  int64_t n;                // work items
  int64_t item0;            // histogram-mode slice: work item i of this launch is item item0 + i
  int32_t a, d, strict, q, kmax, hist_k;
  int32_t ks[kMaxKs];       // ascending prefix redundancies (_k:410-413)
  uint64_t seed;
  // classify_batch outputs (_k:404-452), all device pointers
  uint8_t *out_class;
  uint32_t *out_hash;
  uint8_t *out_w, *out_h;
  uint16_t *out_cells;
  unsigned long long *out_shape;
  int64_t W;
  // histogram mode (enumerate_range): no per-genome outputs
  int32_t hist_mode;
  HistDev hist;
  // payload mode (histogram export, fast kernel), R = 2^pay_shift runs per record:
  // item i replays run i % R of record i / R (all runs in parallel lanes); if it ends
  // BOUNDED with hash pay_key[i / R] it writes its hash/w/h/cells/shape row i, else
  // out_hash[i] = ~pay_key[i / R].  The caller takes each record's first matching run.
  int32_t pay_mode;
  int32_t pay_shift;
  const uint32_t *pay_key;
  // GA fitness mode (JaTAM-shape fitness): out_fit[i] =
  // d^2 - shapediff(target, run-0 grid) for genomes DET at hist_k, else 0.
  // target_rows[R] bit C = target occupancy of padded cell (R, C) (d <= 29).
  int32_t fit_mode;
  int32_t target_cells;
  uint32_t *out_fit;
  const uint32_t *fit_known;  // per item: fitness known from the GA generation (~0 = unknown), or nullptr
  // GA fitness memo (fit mode): open-addressed genome -> fitness table the GA handle keeps across
  // generations while the fitness parameters stay the same; key = genome index + 1 (0 = empty).
  // The pre-pass skips genomes found in it, the classify kernels insert what they compute.
  unsigned long long *memo_keys;
  uint32_t *memo_vals;
  uint64_t memo_mask;       // capacity - 1 (a power of two), 0 = no memo
  uint32_t target_rows[32];
  // scratch
  uint32_t *run_hash;       // per lane, kmax entries
  uint16_t *spill;          // fast kernel: per lane stack entries beyond the shared-memory part
  int32_t S;                // fast kernel: shared-memory stack capacity (entries, multiple of 2)
  int32_t spill_cap;        // d*d - S
  int32_t GW;               // fast kernel: grid words per lane
  int32_t cta_slots;        // fast kernel: per-CTA shared histogram slots (power of 2; 0 = off)
  int32_t service_thresh;   // fast kernel: parked lanes that trigger a warp service pass (0 = default)
  int32_t forced_check;     // fast kernel: skip runs 1.. of genomes whose run-0 assembly is locally forced
                            // (1: check every genome, 2: only provably trivial-free ones)
  const uint32_t *tf_flags; // fast kernel: per-item trivial-freedom bits (early unbound cut-off), or nullptr
  const uint32_t *order;    // fast kernel, histogram mode: work-item permutation (k_prepass sort), or nullptr
  const unsigned long long *n_skip;  // fast kernel: the last *n_skip order entries (1-mers) are done, or nullptr
  unsigned long long *work; // dynamic work counter
  unsigned long long *prof_t;  // optional (TV_TAIL_PROF): globaltimer at first CTA start, work queue
                               // found empty, last CTA end (fast kernel)
  // generic kernel scratch (per thread, interleaved)
  int16_t *g_grid;
  uint8_t *g_mark;
  int32_t *g_stack;
  int32_t *g_placed;
  int64_t g_threads;
};

// GA fitness memo (ClassifyParams::memo_*): linear probing from a mixed slot, at most
// kMemoProbes slots; a full neighbourhood only loses the memo entry, never exactness.
constexpr int kMemoProbes = 16;
__device__ __forceinline__ uint64_t memo_slot(uint64_t idx, uint64_t mask) {
  return mix64(idx ^ 0xD1B54A32D192ED03ULL) & mask;
}
__device__ __forceinline__ uint32_t memo_get(const ClassifyParams &P, uint64_t idx) {
  const unsigned long long key = idx + 1;
  uint64_t s = memo_slot(idx, P.memo_mask);
  for (int p = 0; p < kMemoProbes; p++) {
    const unsigned long long k = P.memo_keys[s];
    if (k == key) return P.memo_vals[s];
    if (k == 0ULL) break;
    s = (s + 1) & P.memo_mask;
  }
  return 0xFFFFFFFFu;
}
// values are read only by later launches (the next generation's pre-pass); two inserts of
// one genome in a launch store the same value
__device__ __forceinline__ void memo_put(const ClassifyParams &P, uint64_t idx, uint32_t fit) {
  const unsigned long long key = idx + 1;
  uint64_t s = memo_slot(idx, P.memo_mask);
  for (int p = 0; p < kMemoProbes; p++) {
    const unsigned long long prev = atomicCAS(&P.memo_keys[s], 0ULL, key);
    if (prev == 0ULL || prev == key) {
      P.memo_vals[s] = fit;
      return;
    }
    s = (s + 1) & P.memo_mask;
  }
}

}  // namespace tvb
