// tv_capi.cu -- extern "C" boundary of libtilevolve_b200.so (include/tilevolve_b200.h).
#include <nvtx3/nvToolsExt.h>  // header-only NVTX ranges (no-ops unless a profiler is attached)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tilevolve_b200.h"
#include "tv_fast.cuh"
#include "tv_ga.cuh"
#include "tv_kernels.cuh"
#include "tv_shape.cuh"

using namespace tvb;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launch[5] = {0, 0, 0, 0, 0};

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(expr)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) return fail(TV_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                       \
  } while (0)

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

std::once_flag g_pool_once[64];
void setup_pool(int dev) {
  if (dev < 0 || dev >= 64) return;
  std::call_once(g_pool_once[dev], [dev]() {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

// Stream-ordered scratch owned by one call.
struct Scratch {
  cudaStream_t s;
  std::vector<void *> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <typename T> cudaError_t get(T **p, size_t count) {
    void *v = nullptr;
    cudaError_t e = cudaMallocAsync(&v, std::max<size_t>(count * sizeof(T), 16), s);
    if (e == cudaSuccess) ptrs.push_back(v);
    *p = static_cast<T *>(v);
    return e;
  }
  ~Scratch() {
    for (void *v : ptrs) cudaFreeAsync(v, s);
  }
};

// A handle's buffers live on the device it was created on: calls with another device current
// would launch there on foreign memory, so they fail loudly instead.
int on_device(int want) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return fail(TV_ERR_CUDA, "no CUDA device");
  if (cur != want) return fail(TV_ERR_ARG, "handle belongs to device %d, the current device is %d", want, cur);
  return 0;
}

int current_device(int *dev) {
  cudaError_t e = cudaGetDevice(dev);
  if (e != cudaSuccess) return fail(TV_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(TV_ERR_CUDA, "no CUDA device");
  setup_pool(*dev);
  return 0;
}

// Reduce the reference's bit writes (_k:387-397) to per-label decoders.
int build_decoder(int a, int bpl, const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                  const int64_t *free_pos, int64_t nfree, LabelDecoder &D) {
  if (a < 1 || a > 16) return fail(TV_ERR_ARG, "tile count a=%d outside [1, 16]", a);
  if (bpl < 1 || bpl > 8) return fail(TV_ERR_ARG, "bits per label %d outside [1, 8]", bpl);
  if (nfree > 64) return fail(TV_ERR_ARG, "%lld free bits exceed the 64-bit enumeration index", (long long)nfree);
  const int L = a * 4 * bpl;
  std::vector<int> src(L, -1), cval(L, 0);
  for (int64_t j = 0; j < m; j++) {
    if (mask_pos[j] < 0 || mask_pos[j] >= L) return fail(TV_ERR_ARG, "mask position %lld outside [0, %d)", (long long)mask_pos[j], L);
    if (mask_val[j] > 1) return fail(TV_ERR_ARG, "mask value %d is not a bit", (int)mask_val[j]);
    src[mask_pos[j]] = -1;
    cval[mask_pos[j]] = mask_val[j];
  }
  for (int64_t j = 0; j < nfree; j++) {
    if (free_pos[j] < 0 || free_pos[j] >= L) return fail(TV_ERR_ARG, "free position %lld outside [0, %d)", (long long)free_pos[j], L);
    src[free_pos[j]] = (int)j;
  }
  memset(&D, 0, sizeof D);
  D.nlab = a * 4;
  D.bpl = bpl;
  bool general = false;
  for (int te = 0; te < a * 4; te++) {
    int fix = 0, nf = 0, lo = -1, sh = -1;
    bool contiguous = true;
    for (int k = 0; k < bpl; k++) {  // label bit k (LSB = 0) <- genome position te*bpl + bpl-1-k
      const int p = te * bpl + (bpl - 1 - k);
      D.src[te * 8 + k] = src[p] < 0 ? 0xFF : (uint8_t)src[p];
      if (src[p] < 0) {
        fix |= cval[p] << k;
      } else {
        if (nf == 0) { lo = src[p]; sh = k; }
        else if (src[p] != lo + nf || k != sh + nf) contiguous = false;
        nf++;
      }
    }
    D.fix[te] = (uint8_t)fix;
    D.nf[te] = (uint8_t)nf;
    D.lo[te] = (uint8_t)(lo < 0 ? 0 : lo);
    D.sh[te] = (uint8_t)(sh < 0 ? 0 : sh);
    D.pk[te] = (uint32_t)D.lo[te] | (((1u << nf) - 1u) << 8) | ((uint32_t)D.sh[te] << 16) | ((uint32_t)fix << 24);
    if (!contiguous) general = true;
  }
  D.general = general ? 1 : 0;
  return 0;
}

struct Common {
  ClassifyParams P;
  bool fast;
};

int fill_common(int32_t a, int32_t bpl, const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                const int64_t *free_pos, int64_t nfree, int32_t d, const int64_t *ks, int64_t q, int32_t hist_k,
                uint64_t seed, int32_t strict, Common &C) {
  memset(&C.P, 0, sizeof C.P);
  if (int rc = build_decoder(a, bpl, mask_pos, mask_val, m, free_pos, nfree, C.P.dec)) return rc;
  if (d < 3 || d > 181) return fail(TV_ERR_ARG, "grid dimension d=%d outside [3, 181]", d);
  if (q < 1 || q > kMaxKs) return fail(TV_ERR_ARG, "len(ks)=%lld outside [1, %d]", (long long)q, kMaxKs);
  for (int64_t i = 0; i < q; i++) {
    if (ks[i] < 1 || ks[i] > 4096) return fail(TV_ERR_ARG, "ks[%lld]=%lld outside [1, 4096]", (long long)i, (long long)ks[i]);
    if (i && ks[i] < ks[i - 1]) return fail(TV_ERR_ARG, "ks must be ascending");
    C.P.ks[i] = (int32_t)ks[i];
  }
  const int kmax = (int)ks[q - 1];
  if (hist_k < 1 || hist_k > kmax) return fail(TV_ERR_ARG, "hist_k=%d outside [1, ks[-1]=%d]", hist_k, kmax);
  C.P.a = a; C.P.d = d; C.P.strict = strict ? 1 : 0; C.P.q = (int32_t)q; C.P.kmax = kmax; C.P.hist_k = hist_k;
  C.P.seed = seed;
  C.fast = a <= 3 && bpl <= 3 && d <= 118;  // row stride < 128 (byte cell offsets, tv_fast.cuh)
  return 0;
}

// k_classify_fast<A, STRICT, MODE> for runtime (a, strict, mode)
template <int A, bool S> const void *fast_kernel_fn_m(int mode) {
  switch (mode) {
    case FM_HIST: return (const void *)k_classify_fast<A, S, FM_HIST>;
    case FM_FIT: return (const void *)k_classify_fast<A, S, FM_FIT>;
    case FM_PAY: return (const void *)k_classify_fast<A, S, FM_PAY>;
    default: return (const void *)k_classify_fast<A, S, FM_ROWS>;
  }
}
const void *fast_kernel_fn(int a, bool strict, int mode, int d) {
  // d = 19 (the reference's grid, _k:8) with compile-time board geometry for the throughput modes
  if (d == 19 && a >= 2 && (mode == FM_HIST || mode == FM_FIT)) {
    if (mode == FM_HIST)
      return strict ? (a == 2 ? (const void *)k_classify_fast<2, true, FM_HIST, 19> : (const void *)k_classify_fast<3, true, FM_HIST, 19>)
                    : (a == 2 ? (const void *)k_classify_fast<2, false, FM_HIST, 19> : (const void *)k_classify_fast<3, false, FM_HIST, 19>);
    return strict ? (a == 2 ? (const void *)k_classify_fast<2, true, FM_FIT, 19> : (const void *)k_classify_fast<3, true, FM_FIT, 19>)
                  : (a == 2 ? (const void *)k_classify_fast<2, false, FM_FIT, 19> : (const void *)k_classify_fast<3, false, FM_FIT, 19>);
  }
  if (strict) return a == 1 ? fast_kernel_fn_m<1, true>(mode) : a == 2 ? fast_kernel_fn_m<2, true>(mode)
                                                                     : fast_kernel_fn_m<3, true>(mode);
  return a == 1 ? fast_kernel_fn_m<1, false>(mode) : a == 2 ? fast_kernel_fn_m<2, false>(mode)
                                                             : fast_kernel_fn_m<3, false>(mode);
}

// Launch the chosen kernel for P (n items, indices or range already set).
int launch_classify(Common &C, Scratch &S, cudaStream_t st) {
  ClassifyParams &P = C.P;
  int dev;
  if (int rc = current_device(&dev)) return rc;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  g_launch[4] = 0;
  if (P.n <= 0) return 0;
  unsigned long long *work;
  CK(S.get(&work, 1));
  CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
  P.work = work;
  const int d = P.d, dd = d * d;
  if (C.fast) {
    P.GW = fast_board_words(P.a, d);
    // tunables (env overrides exist for A/B measurements only)
    const char *es = getenv("TV_STACK_S"), *ec = getenv("TV_CTA_SLOTS"), *et = getenv("TV_SERVICE_THRESH");
    const char *eth = getenv("TV_FAST_THREADS");
    // parked lanes that trigger a service pass (measured: a = 2 best at 14 after the round-2 work
    // elimination, 18.62 vs 18.82 ms at 12; a = 3 at 16-20)
    P.service_thresh = et ? atoi(et) : (P.a == 3 ? 20 : 14);
    // locally-forced run-0 assemblies end the genome DET after one run (TV_FORCED=0 disables).
    // a = 3 checks only provably trivial-free genomes (2): the 64-bit check costs about what it
    // saves on the others (S32 2^24 block 24.27 -> 24.03 ms); a <= 2 checks all (S28 18.5 vs 19.5 ms)
    const char *efz = getenv("TV_FORCED");
    P.forced_check = efz ? std::max(0, std::min(2, atoi(efz))) : (P.a == 3 ? 2 : 1);
    // per-CTA phenotype cache: 256 slots (with the behaviour-sorted order a CTA sees many
    // phenotypes of alike genomes: S28 32.3 -> 31.6 ms vs 128 slots; 512 halves occupancy)
    P.cta_slots = P.hist_mode ? (ec ? atoi(ec) : 256) : 0;
    const int maxt = P.a == 3 ? fast_threads<3>() : fast_threads<2>();
    int threads = eth ? std::min(atoi(eth), maxt) & ~31 : maxt;
    if (es) {
      P.S = std::max(4, atoi(es)) & ~1;
    } else {  // largest shared movelist part (<= 64 entries) that keeps two CTAs per SM
      P.S = 64;
      while (P.S > 8 && 2 * (fast_smem_bytes(threads, P.GW, P.S, P.cta_slots, P.q) + 1024) > 228 * 1024) P.S -= 2;
    }
    P.S = std::max(4, std::min(P.S, (dd + 1) & ~1));
    if (P.a <= 2 || TV_A3_ROWS || TV_A3_RING) {  // the movelist ring (FastLane<true>): power-of-two slots
      int r = 4;
      while (2 * r <= P.S) r *= 2;
      P.S = r;
    }
    P.spill_cap = dd;  // spilled entries live at their own stack index
    size_t smem = fast_smem_bytes(threads, P.GW, P.S, P.cta_slots, P.q);
    int maxsmem = 0;
    CK(cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    while (smem > (size_t)maxsmem && threads > 32) {  // whole warps only (the kernel's ballots)
      threads -= 32;
      smem = fast_smem_bytes(threads, P.GW, P.S, P.cta_slots, P.q);
    }
    if (smem <= (size_t)maxsmem) {
      const int mode = P.hist_mode ? FM_HIST : P.pay_mode ? FM_PAY : P.fit_mode ? FM_FIT : FM_ROWS;
      const char *ed = getenv("TV_GENERIC_D");  // A/B: 1 = run-time d even for d = 19
      const void *fn = fast_kernel_fn(P.a, P.strict != 0, mode, (ed && atoi(ed)) ? 0 : d);
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
      if (per_sm < 1) per_sm = 1;
      int64_t blocks = (int64_t)nsm * per_sm;
      const int64_t need = (P.n + threads - 1) / threads;
      if (blocks > need) blocks = std::max<int64_t>(1, need);
      const int64_t warps = blocks * (threads / 32);
      CK(S.get(&P.spill, (size_t)std::max(1, P.spill_cap) * 32 * warps));
      CK(S.get(&P.run_hash, (size_t)P.kmax * 32 * warps));
      // early unbound cut-off: per-genome trivial-freedom bits from a full-SIMT pre-pass
      // (fixpoint proof, CandSwar::trivial_free).  Full S_{2,8} 25.0 -> 18.8 ms, S32 2^24
      // block 28.7 -> 24.4 ms (pre-pass 1.4 / 2.9 ms included).  TV_EARLY_UNBOUND=0/1 forces it.
      const char *eu = getenv("TV_EARLY_UNBOUND");
      const char *eo = getenv("TV_ORDER");
      // (payload and fitness modes stop at the first UNBOUND run anyway)
      const bool want_flags = !P.pay_mode && !P.fit_mode && (eu ? atoi(eu) != 0 : true);
      // behaviour-sorted processing order for every mode (outputs stay addressed by item):
      // see k_prepass.  Classify-type calls above 2^30 items keep item order (sort scratch).
      // TV_ORDER=0 disables it.
      const bool want_order = (P.hist_mode || P.n <= ((int64_t)1 << 30)) && P.n >= 4096 && !P.pay_mode &&
                              (eo ? atoi(eo) != 0 : true);  // (payload-mode items are (record, run) pairs)
      // 1-mers (seed faces bond nothing) classified by the pre-pass and sorted past the end of
      // the fast kernel's work (k_prepass).  TV_ONEMER=0 disables it.
      const char *e1 = getenv("TV_ONEMER");
      const bool want_onemer = want_order && (e1 ? atoi(e1) != 0 : true);
      // histogram mode runs in slices of <= 2^26 items (sort and flag scratch stay bounded;
      // the histogram accumulates across slices)
      const char *esl = getenv("TV_SLICE_LOG2");  // A/B: histogram-mode slice size (items <= 2^31)
      const int slog = esl ? std::max(16, std::min(30, atoi(esl))) : 26;
      const int64_t n_all = P.n, slice = P.hist_mode ? ((int64_t)1 << slog) : n_all;
      const int64_t smax = std::min(n_all, slice);
      uint32_t *flags = nullptr, *order = nullptr, *iota = nullptr, *tile_hist = nullptr, *bintot = nullptr;
      uint16_t *key = nullptr;
      unsigned long long *n_skip = nullptr;
      if (want_onemer) CK(S.get(&n_skip, 1));
      const int64_t nwmax = (smax + 31) / 32, ntmax = (smax + 1023) / 1024;  // key_tile_for() >= 1024
      if (want_flags) CK(S.get(&flags, (size_t)nwmax));
      if (want_order) {  // counting sort by key (k_prepass tile histograms + k_key_*), no library sort
        CK(S.get(&order, (size_t)smax)); CK(S.get(&iota, (size_t)smax)); CK(S.get(&key, (size_t)smax));
        CK(S.get(&tile_hist, (size_t)kNumKeys * ntmax)); CK(S.get(&bintot, (size_t)kNumKeys));
      }
      const void *ff = P.strict
          ? (P.a == 1 ? (const void *)k_prepass<1, true>
             : P.a == 2 ? (const void *)k_prepass<2, true> : (const void *)k_prepass<3, true>)
          : (P.a == 1 ? (const void *)k_prepass<1, false>
             : P.a == 2 ? (const void *)k_prepass<2, false> : (const void *)k_prepass<3, false>);
      for (int64_t off = 0; off < n_all; off += slice) {
        P.item0 = off;
        P.n = std::min(slice, n_all - off);
        P.tf_flags = nullptr;
        P.order = nullptr;
        P.n_skip = nullptr;
        if (off > 0) CK(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
        if (n_skip) CK(cudaMemsetAsync(n_skip, 0, sizeof(unsigned long long), st));
        if (want_flags || want_order) {
          int64_t tile = key_tile_for(P.n, nsm);
          int64_t ntiles = (P.n + tile - 1) / tile;
          uint16_t *kk = want_order ? key : nullptr;
          uint32_t *ff_flags = want_flags ? flags : nullptr;
          uint32_t *th = want_order ? tile_hist : nullptr;
          void *fargs[] = {&P, &ff_flags, &kk, &iota, &n_skip, &th, &ntiles, &tile};
          CK(cudaLaunchKernel(ff, dim3((unsigned)ntiles), dim3(256), fargs, 0, st));
          if (want_order) {  // counting sort of the items by their behaviour key
            k_key_binscan<<<kNumKeys, 1024, 0, st>>>(tile_hist, ntiles, bintot);
            k_key_basescan<<<1, 1024, 0, st>>>(bintot);
            k_key_scatter<<<(unsigned)ntiles, 1024, 0, st>>>(key, iota, tile_hist, ntiles, bintot, P.n, tile, order);
            CK(cudaGetLastError());
          }
          P.tf_flags = ff_flags;
          P.order = want_order ? order : nullptr;
          P.n_skip = n_skip;
        }
        unsigned long long *pt = nullptr;
        const bool tail_prof = getenv("TV_TAIL_PROF") != nullptr;  // development aid
        if (tail_prof) {
          const unsigned long long init[3] = {~0ULL, ~0ULL, 0ULL};
          CK(S.get(&pt, 3));
          CK(cudaMemcpyAsync(pt, init, 24, cudaMemcpyHostToDevice, st));
          CK(cudaStreamSynchronize(st));
        }
        P.prof_t = pt;
        void *args[] = {&P};
        CK(cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(threads), args, smem, st));
        if (tail_prof) {
          unsigned long long t[3];
          CK(cudaMemcpyAsync(t, pt, 24, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          fprintf(stderr, "k_classify_fast %lld items: %.3f ms, work queue empty after %.3f ms, drain %.3f ms\n",
                  (long long)P.n, (t[2] - t[0]) / 1e6, (t[1] - t[0]) / 1e6, (t[2] - t[1]) / 1e6);
        }
        P.prof_t = nullptr;
      }
      P.n = n_all;
      P.item0 = 0;
      g_launch[0] = 1; g_launch[1] = blocks; g_launch[2] = threads; g_launch[3] = (int64_t)smem;
      g_launch[4] = (n_all + slice - 1) / slice;
      return 0;
    }
  }
  // generic thread-per-genome kernel
  const int threads = 128;
  int64_t T = (int64_t)nsm * 8 * threads;
  const size_t per_thread = (size_t)dd * (2 + 1 + 4 + 4) + (size_t)P.kmax * 4;
  const size_t budget = (size_t)2 << 30;
  while (T > threads && (size_t)T * per_thread > budget) T /= 2;
  if (T > P.n) T = std::max<int64_t>(1, P.n);
  P.g_threads = T;
  CK(S.get(&P.g_grid, (size_t)dd * T));
  CK(S.get(&P.g_mark, (size_t)dd * T));
  CK(S.get(&P.g_stack, (size_t)dd * T));
  CK(S.get(&P.g_placed, (size_t)dd * T));
  CK(S.get(&P.run_hash, (size_t)P.kmax * T));
  k_fill_i16<<<512, 256, 0, st>>>(P.g_grid, (int64_t)dd * T, (int16_t)-1);
  CK(cudaMemsetAsync(P.g_mark, 0, (size_t)dd * T, st));
  const int64_t blocks = (T + threads - 1) / threads;
  k_classify_generic<<<(unsigned)blocks, threads, 0, st>>>(P);
  CK(cudaGetLastError());
  g_launch[0] = 2; g_launch[1] = blocks; g_launch[2] = threads; g_launch[3] = 0; g_launch[4] = 2;
  return 0;
}

// Device view of a [h|d] array: either the pointer itself or a staged copy.
template <typename T>
int stage_in(const T *p, size_t count, bool copy_in, Scratch &S, T **dptr, bool &was_host) {
  was_host = !is_device_ptr(p);
  if (!was_host) { *dptr = const_cast<T *>(p); return 0; }
  CK(S.get(dptr, count));
  if (copy_in && count) CK(cudaMemcpyAsync(*dptr, p, count * sizeof(T), cudaMemcpyHostToDevice, S.s));
  return 0;
}


// Integer-ALU peak probe (roofline denominator): 8 independent IADD3/LOP3
// chains per thread, 2 int32 ops per chain step.
__global__ void __launch_bounds__(256) k_int_peak(int64_t iters, uint32_t seed, uint32_t *sink) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = seed + threadIdx.x * 8 + i; b[i] = seed ^ (blockIdx.x + i); }
  for (int64_t t = 0; t < iters; t++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(b[i]) : "r"(a[i]));
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) x ^= a[i] + b[i];
  if (x == 0x12345678u) sink[0] = x;
}

}  // namespace

struct tv_hist {
  void *block = nullptr;  // the single device allocation holding every table of H
  HistDev H;
  int device;
  bool has_params = false;  // enumeration parameters of the genomes counted since the last clear
  Common params;            // (needed to re-classify representatives for their payloads)
};

namespace {
// same space / k / seed / contact rule: histogram contents stay consistent
bool same_enumeration(const ClassifyParams &a, const ClassifyParams &b) {
  if (memcmp(&a.dec, &b.dec, sizeof a.dec) != 0) return false;
  if (a.a != b.a || a.d != b.d || a.strict != b.strict || a.q != b.q || a.kmax != b.kmax || a.hist_k != b.hist_k ||
      a.seed != b.seed)
    return false;
  for (int i = 0; i < a.q; i++)
    if (a.ks[i] != b.ks[i]) return false;
  return true;
}

// Fill the payload of every slot whose payload is not its representative's
// (tv_hist.cuh): replay those representatives' runs until one reproduces the key.
int fix_payloads(tv_hist *h, cudaStream_t st, int64_t nkeys) {  // nkeys: tv_hist_count's, just read
  const HistDev &H = h->H;
  Scratch S(st);
  unsigned int *cnt;
  uint32_t *slots;
  unsigned long long *idx;
  if (nkeys == 0) return 0;
  uint32_t *keys;
  CK(S.get(&cnt, 2)); CK(S.get(&slots, nkeys)); CK(S.get(&idx, nkeys)); CK(S.get(&keys, nkeys));
  CK(cudaMemsetAsync(cnt, 0, 8, st));
  k_hist_stale<<<256, 256, 0, st>>>(H, slots, idx, keys, cnt);
  CK(cudaGetLastError());
  unsigned int ns = 0;
  CK(cudaMemcpyAsync(&ns, cnt, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ns == 0) return 0;
  if (!h->has_params)
    return fail(TV_ERR_ARG, "%u histogram records lack their representative's payload and no enumeration "
                            "parameters are known (merge complete records or enumerate into this histogram)", ns);
  // Fast spaces: payload mode, every run < hist_k of every representative replayed in its own
  // lane (the attributed run of a DET / STERIC genome lies below hist_k, _k:357-381) and the
  // first run reproducing the key taken -- the latency of one run instead of a chain of runs.
  // Others: full classification of the representative, whose attributed row is the payload.
  Common C = h->params;
  ClassifyParams &P = C.P;
  int shift = 0;
  while (C.fast && (1 << shift) < P.hist_k) shift++;
  const int R = 1 << shift;  // runs >= hist_k only ever follow a matching run
  const int64_t rows = (int64_t)ns * R;
  P.hist_mode = 0; P.fit_mode = 0; P.indices = reinterpret_cast<const uint64_t *>(idx); P.n = rows;
  P.start = 0; P.chunk = 0; P.stride = 0;
  P.pay_mode = C.fast ? 1 : 0;
  P.pay_shift = shift;
  P.pay_key = keys;
  uint8_t *cls, *w, *hh; uint32_t *hash; uint16_t *cells; unsigned long long *shape;
  CK(S.get(&cls, (size_t)rows * P.q)); CK(S.get(&hash, rows)); CK(S.get(&w, rows)); CK(S.get(&hh, rows));
  CK(S.get(&cells, rows)); CK(S.get(&shape, (size_t)rows * H.W));
  P.out_class = cls; P.out_hash = hash; P.out_w = w; P.out_h = hh; P.out_cells = cells; P.out_shape = shape;
  P.W = H.W;
  if (int rc = launch_classify(C, S, st)) return rc;
  const int blocks = (int)std::min<int64_t>(256, ((int64_t)ns + 255) / 256);
  k_hist_payload<<<blocks, 256, 0, st>>>(H, slots, idx, ns, R, hash, w, hh, cells, shape, cnt + 1);
  CK(cudaGetLastError());
  unsigned int err = 0;
  CK(cudaMemcpyAsync(&err, cnt + 1, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (err) return fail(TV_ERR_ARG, "a representative did not reproduce its hash: the histogram mixes "
                                   "enumeration parameters");
  return 0;
}
}  // namespace


// NVTX range around every batch-level C-ABI call (SURVEY section 5 tracing): visible in
// Nsight Systems / ncu --nvtx timelines, free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name, long long n = -1) {
    char buf[96];
    if (n >= 0) snprintf(buf, sizeof buf, "%s n=%lld", name, n);
    nvtxRangePushA(n >= 0 ? buf : name);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

extern "C" {

int tv_version(void) { return 10000; }

const char *tv_last_error(void) { return g_err.c_str(); }

int tv_last_launch_info(int64_t *info5) {
  for (int i = 0; i < 5; i++) info5[i] = g_launch[i];
  return 0;
}

int tv_classify_batch(const uint64_t *indices, int64_t n, int32_t a, int32_t bpl, const int64_t *mask_pos,
                      const uint8_t *mask_val, int64_t m, const int64_t *free_pos, int64_t nfree, int32_t d,
                      const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict,
                      uint8_t *out_class, uint32_t *out_hash, uint8_t *out_w, uint8_t *out_h, uint16_t *out_cells,
                      uint64_t *out_shape, int64_t W, void *stream) {
  NvtxRange nvtx_("tv_classify_batch", (long long)n);
  Common C;
  if (n < 0) return fail(TV_ERR_ARG, "negative n");
  if (int rc = fill_common(a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, ks, q, hist_k, seed, strict, C)) return rc;
  // The reference writes shape words unchecked (_k:283-291); shapes wider
  // than W words are truncated here instead of overrunning the row.
  if (W < 1) return fail(TV_ERR_ARG, "out_shape needs at least one word per row");
  int dev;
  if (int rc = current_device(&dev)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  bool any_host = false;
  {
    Scratch S(st);
    uint64_t *d_idx; uint8_t *d_cls, *d_w, *d_h; uint32_t *d_hash; uint16_t *d_cells; uint64_t *d_shape;
    bool h0, h1, h2, h3, h4, h5, h6;
    // outputs are copied in too: rows the reference leaves untouched must survive (_k:434-452)
    if (int rc = stage_in(indices, (size_t)n, true, S, &d_idx, h0)) return rc;
    if (int rc = stage_in(out_class, (size_t)n * q, true, S, &d_cls, h1)) return rc;
    if (int rc = stage_in(out_hash, (size_t)n, true, S, &d_hash, h2)) return rc;
    if (int rc = stage_in(out_w, (size_t)n, true, S, &d_w, h3)) return rc;
    if (int rc = stage_in(out_h, (size_t)n, true, S, &d_h, h4)) return rc;
    if (int rc = stage_in(out_cells, (size_t)n, true, S, &d_cells, h5)) return rc;
    if (int rc = stage_in(out_shape, (size_t)n * W, true, S, &d_shape, h6)) return rc;
    any_host = h0 || h1 || h2 || h3 || h4 || h5 || h6;
    C.P.indices = d_idx; C.P.n = n;
    C.P.out_class = d_cls; C.P.out_hash = d_hash; C.P.out_w = d_w; C.P.out_h = d_h; C.P.out_cells = d_cells;
    C.P.out_shape = reinterpret_cast<unsigned long long *>(d_shape); C.P.W = W;
    if (int rc = launch_classify(C, S, st)) return rc;
    if (h1) CK(cudaMemcpyAsync(out_class, d_cls, (size_t)n * q, cudaMemcpyDeviceToHost, st));
    if (h2) CK(cudaMemcpyAsync(out_hash, d_hash, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    if (h3) CK(cudaMemcpyAsync(out_w, d_w, (size_t)n, cudaMemcpyDeviceToHost, st));
    if (h4) CK(cudaMemcpyAsync(out_h, d_h, (size_t)n, cudaMemcpyDeviceToHost, st));
    if (h5) CK(cudaMemcpyAsync(out_cells, d_cells, (size_t)n * 2, cudaMemcpyDeviceToHost, st));
    if (h6) CK(cudaMemcpyAsync(out_shape, d_shape, (size_t)n * W * 8, cudaMemcpyDeviceToHost, st));
  }
  if (any_host) CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  return 0;
}

static int single_scratch(int d, Scratch &S, int16_t **grid, uint8_t **mark, int32_t **stack, int32_t **placed) {
  const size_t dd = (size_t)d * d;
  CK(S.get(grid, dd));
  CK(S.get(mark, dd));
  CK(S.get(stack, dd));
  CK(S.get(placed, dd));
  k_fill_i16<<<1, 256, 0, S.s>>>(*grid, (int64_t)dd, (int16_t)-1);
  CK(cudaMemsetAsync(*mark, 0, dd, S.s));
  return 0;
}

int tv_classify_single(const uint8_t *edges, int32_t a, int32_t d, int32_t k, uint64_t seed, uint64_t genome_index,
                       int32_t strict, uint64_t *shape_words, int64_t W, int32_t *out6) {
  if (a < 1 || a > 16) return fail(TV_ERR_ARG, "tile count a=%d outside [1, 16]", a);
  if (d < 3 || d > 181) return fail(TV_ERR_ARG, "grid dimension d=%d outside [3, 181]", d);
  if (k < 1 || k > 4096) return fail(TV_ERR_ARG, "k=%d outside [1, 4096]", k);
  if (W < 1) return fail(TV_ERR_ARG, "shape buffer needs at least one word");
  int dev;
  if (int rc = current_device(&dev)) return rc;
  cudaStream_t st = nullptr;
  {
    Scratch S(st);
    int16_t *grid; uint8_t *mark; int32_t *stack, *placed; uint32_t *rh; uint8_t *de; int32_t *dout;
    unsigned long long *dsh;
    if (int rc = single_scratch(d, S, &grid, &mark, &stack, &placed)) return rc;
    CK(S.get(&rh, (size_t)k));
    CK(S.get(&de, (size_t)a * 16));
    CK(S.get(&dout, 6));
    CK(S.get(&dsh, (size_t)W));
    CK(cudaMemcpyAsync(de, edges, (size_t)a * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dsh, shape_words, (size_t)W * 8, cudaMemcpyHostToDevice, st));
    k_classify_single<<<1, 32, 0, st>>>(de, a, d, k, seed, genome_index, strict, dsh, W, dout, grid, mark, stack,
                                         placed, rh);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out6, dout, 6 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(shape_words, dsh, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

int tv_assemble_single(const uint8_t *edges, int32_t a, int32_t d, uint64_t seed, uint64_t genome_index,
                       int32_t run_index, int32_t strict, int16_t *out_grid, int32_t *out6) {
  if (a < 1 || a > 16) return fail(TV_ERR_ARG, "tile count a=%d outside [1, 16]", a);
  if (d < 3 || d > 181) return fail(TV_ERR_ARG, "grid dimension d=%d outside [3, 181]", d);
  int dev;
  if (int rc = current_device(&dev)) return rc;
  cudaStream_t st = nullptr;
  {
    Scratch S(st);
    int16_t *grid; uint8_t *mark; int32_t *stack, *placed; uint8_t *de; int32_t *dout;
    if (int rc = single_scratch(d, S, &grid, &mark, &stack, &placed)) return rc;
    CK(S.get(&de, (size_t)a * 16));
    CK(S.get(&dout, 6));
    CK(cudaMemcpyAsync(de, edges, (size_t)a * 16, cudaMemcpyHostToDevice, st));
    k_assemble_single<<<1, 32, 0, st>>>(de, a, d, seed, genome_index, run_index, strict, grid, mark, stack, placed,
                                         dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out6, dout, 6 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_grid, grid, (size_t)d * d * 2, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

int tv_oat_hash_bytes(const uint8_t *data, int64_t n, uint32_t *out) {
  if (n < 0) return fail(TV_ERR_ARG, "negative length");
  int dev;
  if (int rc = current_device(&dev)) return rc;
  cudaStream_t st = nullptr;
  {
    Scratch S(st);
    uint8_t *dd; bool host; uint32_t *dout;
    if (int rc = stage_in(data, (size_t)n, true, S, &dd, host)) return rc;
    CK(S.get(&dout, 1));
    k_oat<<<1, 32, 0, st>>>(dd, n, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout, 4, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

// ---------------------------------------------------------------- canonical shape labels
int tv_shape_labels(const uint64_t *shape, const uint8_t *w, const uint8_t *h, int64_t n, int64_t W,
                    uint32_t *out_rot4, uint32_t *out_d4, void *stream) {
  if (n < 0) return fail(TV_ERR_ARG, "negative n");
  if (W < 1) return fail(TV_ERR_ARG, "W must be >= 1");
  if (!out_rot4 && !out_d4) return 0;
  int dev;
  if (int rc = current_device(&dev)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  bool any_host = false;
  {
    Scratch S(st);
    uint64_t *d_shape; uint8_t *d_w, *d_h; uint32_t *d_r = nullptr, *d_d = nullptr;
    bool h0, h1, h2, h3 = false, h4 = false;
    if (int rc = stage_in(shape, (size_t)n * W, true, S, &d_shape, h0)) return rc;
    if (int rc = stage_in(w, (size_t)n, true, S, &d_w, h1)) return rc;
    if (int rc = stage_in(h, (size_t)n, true, S, &d_h, h2)) return rc;
    if (out_rot4) if (int rc = stage_in(out_rot4, (size_t)n, false, S, &d_r, h3)) return rc;
    if (out_d4) if (int rc = stage_in(out_d4, (size_t)n, false, S, &d_d, h4)) return rc;
    any_host = h0 || h1 || h2 || h3 || h4;
    if (n > 0) {
      const int threads = 256;
      const int64_t blocks = (n * 8 + threads - 1) / threads;
      k_shape_labels<<<(unsigned)blocks, threads, 0, st>>>(reinterpret_cast<const unsigned long long *>(d_shape),
                                                           d_w, d_h, n, W, d_r, d_d);
      CK(cudaGetLastError());
    }
    if (h3) CK(cudaMemcpyAsync(out_rot4, d_r, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    if (h4) CK(cudaMemcpyAsync(out_d4, d_d, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  }
  if (any_host) CK(cudaStreamSynchronize(st));
  return 0;
}

// ---------------------------------------------------------------- histogram
int tv_hist_create(int64_t capacity, int32_t q, int32_t W, tv_hist **out) {
  if (capacity < 1 || capacity > ((int64_t)1 << 30)) return fail(TV_ERR_ARG, "capacity outside [1, 2^30]");
  if (q < 1 || q > kMaxKs) return fail(TV_ERR_ARG, "q outside [1, %d]", kMaxKs);
  if (W < 1 || W > 1024) return fail(TV_ERR_ARG, "W outside [1, 1024]");
  int dev;
  if (int rc = current_device(&dev)) return rc;
  int64_t cap = 1;
  while (cap < capacity) cap <<= 1;
  tv_hist *h = new tv_hist();
  h->device = dev;
  HistDev &H = h->H;
  H.cap = cap; H.W = W; H.q = q;
  // one allocation carved into the tables (one cudaMalloc / cudaFree per histogram)
  const size_t sizes[11] = {(size_t)cap * 8, (size_t)cap * 8, (size_t)cap * 8, (size_t)cap * 8, (size_t)cap * 8,
                            (size_t)cap * 4, (size_t)cap * 8, (size_t)cap * 8 * W, (size_t)q * 5 * 8, 4, 4};
  size_t total = 0;
  for (size_t sz : sizes) total += (sz + 255) & ~(size_t)255;
  cudaError_t e = cudaMalloc(&h->block, total);
  if (e == cudaSuccess) {
    char *p = static_cast<char *>(h->block);
    void **dst[11] = {(void **)&H.keys, (void **)&H.det, (void **)&H.steric, (void **)&H.rep_det,
                      (void **)&H.rep_any, (void **)&H.whc, (void **)&H.pay_idx, (void **)&H.shape,
                      (void **)&H.tallies, (void **)&H.n_keys, (void **)&H.overflow};
    for (int i = 0; i < 11; i++) {
      *dst[i] = p;
      p += (sizes[i] + 255) & ~(size_t)255;
    }
  }
  if (e != cudaSuccess) {
    tv_hist_destroy(h);
    return fail(TV_ERR_CUDA, "histogram allocation: %s", cudaGetErrorString(e));
  }
  if (int rc = tv_hist_clear(h, nullptr)) { tv_hist_destroy(h); return rc; }
  CK(cudaStreamSynchronize(nullptr));
  *out = h;
  return 0;
}

int tv_hist_destroy(tv_hist *h) {
  if (!h) return 0;
  HistDev &H = h->H;
  (void)H;
  if (h->block) cudaFree(h->block);
  delete h;
  return 0;
}

namespace {
// Page-locked staging for histogram exports, one per process (grown on demand, never freed:
// a page-locked allocation costs milliseconds, so it is paid once, not per histogram).
std::mutex g_pinned_mu;
void *g_pinned = nullptr;
size_t g_pinned_bytes = 0;
}  // namespace

int tv_hist_clear(tv_hist *h, void *stream) {
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  h->has_params = false;
  k_hist_reset<<<256, 256, 0, (cudaStream_t)stream>>>(h->H);
  CK(cudaGetLastError());
  return 0;
}

int tv_hist_count(tv_hist *h, int64_t *n_keys, int32_t *overflow, void *stream) {
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  unsigned int v[2];
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(&v[0], h->H.n_keys, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&v[1], h->H.overflow, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (n_keys) *n_keys = v[0];
  if (overflow) *overflow = (int32_t)v[1];
  return 0;
}

int tv_hist_export(tv_hist *h, int64_t max_records, uint32_t *keys, uint64_t *det, uint64_t *steric,
                   uint64_t *rep_det, uint64_t *rep_any, uint8_t *w, uint8_t *hh, uint16_t *cells, uint64_t *shape,
                   int64_t *tallies, int64_t *n_out, void *stream) {
  NvtxRange nvtx_("tv_hist_export");
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t n = 0;
  int32_t ovf = 0;
  if (int rc = tv_hist_count(h, &n, &ovf, stream)) return rc;
  if (ovf) return fail(TV_ERR_HIST_FULL, "histogram overflowed its %lld slots", (long long)h->H.cap);
  if (int rc = fix_payloads(h, st, n)) return rc;
  if (n > max_records) return fail(TV_ERR_ARG, "%lld records do not fit max_records=%lld", (long long)n, (long long)max_records);
  const HistDev &H = h->H;
  // host outputs (the documented case): every column is gathered into one device block and
  // comes back in ONE copy through page-locked staging (ten pageable copies cost ~0.3 ms)
  const void *outs[10] = {keys, det, steric, rep_det, rep_any, w, hh, cells, shape, tallies};
  bool all_host = true;
  for (const void *o : outs) all_host = all_host && (!o || !is_device_ptr(o));
  if (all_host) {
    const size_t sz[10] = {(size_t)n * 4, (size_t)n * 8, (size_t)n * 8, (size_t)n * 8, (size_t)n * 8, (size_t)n,
                           (size_t)n, (size_t)n * 2, (size_t)n * H.W * 8, (size_t)H.q * 5 * 8};
    size_t off[10], total = 0;
    for (int i = 0; i < 10; i++) { off[i] = total; total += (sz[i] + 15) / 16 * 16; }
    std::lock_guard<std::mutex> lock(g_pinned_mu);
    if (g_pinned_bytes < total) {
      if (g_pinned) cudaFreeHost(g_pinned);
      g_pinned = nullptr;
      g_pinned_bytes = 0;
      CK(cudaHostAlloc(&g_pinned, std::max<size_t>(total, 1 << 20), cudaHostAllocDefault));
      g_pinned_bytes = std::max<size_t>(total, 1 << 20);
    }
    {
      Scratch S(st);
      char *blk;
      uint32_t *k0, *s0, *s1;
      unsigned int *cnt;
      CK(S.get(&blk, total)); CK(S.get(&k0, std::max<int64_t>(n, 1))); CK(S.get(&s0, std::max<int64_t>(n, 1)));
      CK(S.get(&s1, std::max<int64_t>(n, 1))); CK(S.get(&cnt, 1));
      HistRecords R;
      R.keys = reinterpret_cast<uint32_t *>(blk + off[0]);
      R.det = reinterpret_cast<unsigned long long *>(blk + off[1]);
      R.steric = reinterpret_cast<unsigned long long *>(blk + off[2]);
      R.rep_det = reinterpret_cast<unsigned long long *>(blk + off[3]);
      R.rep_any = reinterpret_cast<unsigned long long *>(blk + off[4]);
      R.w = reinterpret_cast<uint8_t *>(blk + off[5]);
      R.h = reinterpret_cast<uint8_t *>(blk + off[6]);
      R.cells = reinterpret_cast<uint16_t *>(blk + off[7]);
      R.shape = reinterpret_cast<unsigned long long *>(blk + off[8]);
      CK(cudaMemsetAsync(cnt, 0, 4, st));
      CK(cudaMemsetAsync(blk, 0, total, st));  // (the alignment padding travels with the one copy)
      k_hist_compact<<<256, 256, 0, st>>>(H, k0, s0, cnt);
      CK(cudaGetLastError());
      if (n > 0) {
        size_t tmp_bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, R.keys, s0, s1, (int)n, 0, 32, st));
        uint8_t *tmp;
        CK(S.get(&tmp, tmp_bytes));
        CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, R.keys, s0, s1, (int)n, 0, 32, st));
        k_hist_gather<<<64, 256, 0, st>>>(H, s1, n, R);
        CK(cudaGetLastError());
      }
      CK(cudaMemcpyAsync(blk + off[9], H.tallies, sz[9], cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(g_pinned, blk, total, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    void *dst[10] = {keys, det, steric, rep_det, rep_any, w, hh, cells, shape, tallies};
    for (int i = 0; i < 10; i++)
      if (dst[i] && sz[i]) memcpy(dst[i], static_cast<char *>(g_pinned) + off[i], sz[i]);
    if (n_out) *n_out = n;
    return 0;
  }
  {
    Scratch S(st);
    uint32_t *k0, *s0, *k1, *s1;
    unsigned int *cnt;
    CK(S.get(&k0, n)); CK(S.get(&s0, n)); CK(S.get(&k1, n)); CK(S.get(&s1, n)); CK(S.get(&cnt, 1));
    CK(cudaMemsetAsync(cnt, 0, 4, st));
    k_hist_compact<<<256, 256, 0, st>>>(H, k0, s0, cnt);
    CK(cudaGetLastError());
    if (n > 0) {
      size_t tmp_bytes = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, s0, s1, (int)n, 0, 32, st));
      uint8_t *tmp;
      CK(S.get(&tmp, tmp_bytes));
      CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, s0, s1, (int)n, 0, 32, st));
      HistRecords R;
      R.keys = k1;
      CK(S.get(&R.det, n)); CK(S.get(&R.steric, n)); CK(S.get(&R.rep_det, n)); CK(S.get(&R.rep_any, n));
      CK(S.get(&R.w, n)); CK(S.get(&R.h, n)); CK(S.get(&R.cells, n)); CK(S.get(&R.shape, (size_t)n * H.W));
      k_hist_gather<<<64, 256, 0, st>>>(H, s1, n, R);
      CK(cudaGetLastError());
      if (keys) CK(cudaMemcpyAsync(keys, k1, n * 4, cudaMemcpyDefault, st));
      if (det) CK(cudaMemcpyAsync(det, R.det, n * 8, cudaMemcpyDefault, st));
      if (steric) CK(cudaMemcpyAsync(steric, R.steric, n * 8, cudaMemcpyDefault, st));
      if (rep_det) CK(cudaMemcpyAsync(rep_det, R.rep_det, n * 8, cudaMemcpyDefault, st));
      if (rep_any) CK(cudaMemcpyAsync(rep_any, R.rep_any, n * 8, cudaMemcpyDefault, st));
      if (w) CK(cudaMemcpyAsync(w, R.w, n, cudaMemcpyDefault, st));
      if (hh) CK(cudaMemcpyAsync(hh, R.h, n, cudaMemcpyDefault, st));
      if (cells) CK(cudaMemcpyAsync(cells, R.cells, n * 2, cudaMemcpyDefault, st));
      if (shape) CK(cudaMemcpyAsync(shape, R.shape, (size_t)n * H.W * 8, cudaMemcpyDefault, st));
    }
    if (tallies) CK(cudaMemcpyAsync(tallies, H.tallies, (size_t)H.q * 5 * 8, cudaMemcpyDefault, st));
  }
  CK(cudaStreamSynchronize(st));
  if (n_out) *n_out = n;
  return 0;
}

int tv_hist_pack(tv_hist *h, int64_t max_records, uint64_t *rows, int64_t *tallies, int64_t *n_out,
                 void *stream) {
  NvtxRange nvtx_("tv_hist_pack");
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t n = 0;
  int32_t ovf = 0;
  if (int rc = tv_hist_count(h, &n, &ovf, stream)) return rc;
  if (ovf) return fail(TV_ERR_HIST_FULL, "histogram overflowed its %lld slots", (long long)h->H.cap);
  if (n > max_records) return fail(TV_ERR_ARG, "%lld records do not fit max_records=%lld", (long long)n, (long long)max_records);
  const HistDev &H = h->H;
  bool any_host = false;
  {
    Scratch S(st);
    uint32_t *keys, *slots;
    unsigned int *cnt;
    CK(S.get(&keys, std::max<int64_t>(n, 1))); CK(S.get(&slots, std::max<int64_t>(n, 1))); CK(S.get(&cnt, 1));
    CK(cudaMemsetAsync(cnt, 0, 4, st));
    k_hist_compact<<<256, 256, 0, st>>>(H, keys, slots, cnt);
    CK(cudaGetLastError());
    unsigned long long *d_rows;
    bool hr;
    if (int rc = stage_in(reinterpret_cast<unsigned long long *>(rows), (size_t)n * (7 + H.W), false, S, &d_rows,
                          hr)) return rc;
    any_host = hr;
    if (n > 0) {
      k_hist_pack<<<(unsigned)std::min<int64_t>(256, (n + 255) / 256), 256, 0, st>>>(H, slots, n, d_rows);
      CK(cudaGetLastError());
      if (hr) CK(cudaMemcpyAsync(rows, d_rows, (size_t)n * (7 + H.W) * 8, cudaMemcpyDeviceToHost, st));
    }
    if (tallies) {
      CK(cudaMemcpyAsync(tallies, H.tallies, (size_t)H.q * 5 * 8, cudaMemcpyDefault, st));
      any_host = any_host || !is_device_ptr(tallies);
    }
  }
  if (any_host) CK(cudaStreamSynchronize(st));
  if (n_out) *n_out = n;
  return 0;
}

int tv_hist_replace_rows(tv_hist *h, int64_t n, const uint64_t *rows, const int64_t *tallies, void *stream) {
  NvtxRange nvtx_("tv_hist_replace_rows", (long long)n);
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  if (n < 0) return fail(TV_ERR_ARG, "negative n");
  cudaStream_t st = (cudaStream_t)stream;
  HistDev &H = h->H;
  bool any_host = false;
  {
    Scratch S(st);
    const bool keep = h->has_params;  // the enumeration parameters survive (payload fix-up at export)
    if (int rc = tv_hist_clear(h, stream)) return rc;
    h->has_params = keep;
    if (tallies) {
      long long *dt;
      CK(S.get(&dt, (size_t)H.q * 5));
      CK(cudaMemcpyAsync(dt, tallies, (size_t)H.q * 5 * 8, cudaMemcpyDefault, st));
      k_hist_merge<<<1, 256, 0, st>>>(H, 0, HistRecords{}, dt);
      CK(cudaGetLastError());
      any_host = !is_device_ptr(tallies);
    }
    if (n > 0) {
      unsigned long long *d_rows, *pmin;
      int64_t *slot_of;
      bool hr;
      if (int rc = stage_in(reinterpret_cast<const unsigned long long *>(rows), (size_t)n * (7 + H.W), true, S,
                            &d_rows, hr)) return rc;
      any_host = any_host || hr;
      CK(S.get(&pmin, (size_t)H.cap));
      CK(S.get(&slot_of, (size_t)n));
      CK(cudaMemsetAsync(pmin, 0xFF, (size_t)H.cap * 8, st));
      const unsigned blocks = (unsigned)std::min<int64_t>(1024, (n + 255) / 256);
      k_hist_merge_rows1<<<blocks, 256, 0, st>>>(H, n, d_rows, pmin, slot_of);
      k_hist_merge_rows2<<<blocks, 256, 0, st>>>(H, n, d_rows, pmin, slot_of);
      CK(cudaGetLastError());
    }
  }
  if (any_host) CK(cudaStreamSynchronize(st));
  return 0;
}

int tv_hist_merge(tv_hist *h, int64_t n, const uint32_t *keys, const uint64_t *det, const uint64_t *steric,
                  const uint64_t *rep_det, const uint64_t *rep_any, const uint8_t *w, const uint8_t *hh,
                  const uint16_t *cells, const uint64_t *shape, const int64_t *tallies, void *stream) {
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  if (n < 0) return fail(TV_ERR_ARG, "negative n");
  cudaStream_t st = (cudaStream_t)stream;
  const HistDev &H = h->H;
  bool any_host = false;
  {
    Scratch S(st);
    HistRecords R;
    bool b[9];
    uint64_t *d0, *d1, *d2, *d3, *d8;
    if (int rc = stage_in(keys, n, true, S, &R.keys, b[0])) return rc;
    if (int rc = stage_in(det, n, true, S, &d0, b[1])) return rc;
    if (int rc = stage_in(steric, n, true, S, &d1, b[2])) return rc;
    if (int rc = stage_in(rep_det, n, true, S, &d2, b[3])) return rc;
    if (int rc = stage_in(rep_any, n, true, S, &d3, b[4])) return rc;
    if (int rc = stage_in(w, n, true, S, &R.w, b[5])) return rc;
    if (int rc = stage_in(hh, n, true, S, &R.h, b[6])) return rc;
    if (int rc = stage_in(cells, n, true, S, &R.cells, b[7])) return rc;
    if (int rc = stage_in(shape, (size_t)n * H.W, true, S, &d8, b[8])) return rc;
    R.det = reinterpret_cast<unsigned long long *>(d0);
    R.steric = reinterpret_cast<unsigned long long *>(d1);
    R.rep_det = reinterpret_cast<unsigned long long *>(d2);
    R.rep_any = reinterpret_cast<unsigned long long *>(d3);
    R.shape = reinterpret_cast<unsigned long long *>(d8);
    for (bool x : b) any_host = any_host || x;
    long long *dt = nullptr;
    if (tallies) {
      CK(S.get(&dt, (size_t)H.q * 5));
      CK(cudaMemcpyAsync(dt, tallies, (size_t)H.q * 5 * 8, cudaMemcpyDefault, st));
      any_host = true;
    }
    const int blocks = (int)std::min<int64_t>(256, std::max<int64_t>(1, (n + 255) / 256));
    k_hist_merge<<<blocks, 256, 0, st>>>(H, n, R, dt);
    CK(cudaGetLastError());
  }
  if (any_host) CK(cudaStreamSynchronize(st));
  return 0;
}

static int enumerate_common(const uint64_t *indices, uint64_t start, uint64_t chunk, uint64_t stride,
                            int64_t count, int32_t a, int32_t bpl,
                            const int64_t *mask_pos, const uint8_t *mask_val, int64_t m, const int64_t *free_pos,
                            int64_t nfree, int32_t d, const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed,
                            int32_t strict, tv_hist *h, void *stream) {
  NvtxRange nvtx_("tv_enumerate", (long long)count);
  if (!h) return fail(TV_ERR_ARG, "null histogram");
  if (int rc = on_device(h->device)) return rc;
  if (count < 0) return fail(TV_ERR_ARG, "negative count");
  Common C;
  if (int rc = fill_common(a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, ks, q, hist_k, seed, strict, C)) return rc;
  if (q != h->H.q) return fail(TV_ERR_ARG, "histogram was created for q=%d, got %lld", h->H.q, (long long)q);
  if ((int64_t)h->H.W * 64 < (int64_t)(d - 2) * (d - 2)) return fail(TV_ERR_ARG, "histogram W too small for d=%d", d);
  if (h->has_params && !same_enumeration(h->params.P, C.P))
    return fail(TV_ERR_ARG, "histogram holds genomes enumerated with other parameters (space, ks, seed, d or "
                            "contact rule); clear it first");
  if (!h->has_params) { h->params = C; h->has_params = true; }
  cudaStream_t st = (cudaStream_t)stream;
  bool host = false;
  {
    Scratch S(st);
    uint64_t *d_idx = nullptr;
    if (indices) {
      if (int rc = stage_in(indices, (size_t)count, true, S, &d_idx, host)) return rc;
    }
    C.P.indices = d_idx;
    C.P.start = start;
    C.P.chunk = chunk;
    C.P.stride = stride;
    C.P.n = count;
    C.P.hist_mode = 1;
    C.P.hist = h->H;
    if (int rc = launch_classify(C, S, st)) return rc;
  }
  if (host) CK(cudaStreamSynchronize(st));
  return 0;
}

// The space has 2^nfree indices; the decoder ignores index bits >= nfree, so an index
// past the end would alias (idx mod 2^nfree) and be counted twice: reject it.
static int check_last_index(uint64_t last, int64_t nfree) {
  if (nfree < 0 || nfree > 64) return fail(TV_ERR_ARG, "nfree=%lld outside [0, 64]", (long long)nfree);
  if (nfree < 64 && last >= ((uint64_t)1 << nfree))
    return fail(TV_ERR_ARG, "index %llu is outside the space (2^%lld indices)", (unsigned long long)last,
                (long long)nfree);
  return 0;
}

int tv_enumerate_range(uint64_t start, uint64_t count, int32_t a, int32_t bpl, const int64_t *mask_pos,
                       const uint8_t *mask_val, int64_t m, const int64_t *free_pos, int64_t nfree, int32_t d,
                       const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict, tv_hist *h,
                       void *stream) {
  if (count > ((uint64_t)1 << 62)) return fail(TV_ERR_ARG, "count too large for one call");
  if (count > 0) {
    if (start + (count - 1) < start) return fail(TV_ERR_ARG, "index range wraps around 2^64");
    if (int rc = check_last_index(start + (count - 1), nfree)) return rc;
  }
  return enumerate_common(nullptr, start, 0, 0, (int64_t)count, a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, ks, q,
                          hist_k, seed, strict, h, stream);
}

int tv_enumerate_chunks(uint64_t start, uint64_t count, uint64_t chunk, uint64_t stride, int32_t a, int32_t bpl,
                        const int64_t *mask_pos, const uint8_t *mask_val, int64_t m, const int64_t *free_pos,
                        int64_t nfree, int32_t d, const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed,
                        int32_t strict, tv_hist *h, void *stream) {
  if (count > ((uint64_t)1 << 62)) return fail(TV_ERR_ARG, "count too large for one call");
  if (chunk == 0 || stride < chunk) return fail(TV_ERR_ARG, "need 0 < chunk <= stride");
  if (count > 0) {
    const uint64_t c = (count - 1) / chunk, r = (count - 1) % chunk;  // the last item's chunk and offset
    if (c > 0 && stride > (~0ULL - start) / c) return fail(TV_ERR_ARG, "chunk layout wraps around 2^64");
    const uint64_t last = start + c * stride;
    if (last + r < last) return fail(TV_ERR_ARG, "chunk layout wraps around 2^64");
    if (int rc = check_last_index(last + r, nfree)) return rc;
  }
  return enumerate_common(nullptr, start, chunk, stride, (int64_t)count, a, bpl, mask_pos, mask_val, m, free_pos,
                          nfree, d, ks, q, hist_k, seed, strict, h, stream);
}

int tv_enumerate_indices(const uint64_t *indices, int64_t n, int32_t a, int32_t bpl, const int64_t *mask_pos,
                         const uint8_t *mask_val, int64_t m, const int64_t *free_pos, int64_t nfree, int32_t d,
                         const int64_t *ks, int64_t q, int32_t hist_k, uint64_t seed, int32_t strict, tv_hist *h,
                         void *stream) {
  if (!indices && n > 0) return fail(TV_ERR_ARG, "null indices");
  return enumerate_common(indices, 0, 0, 0, n, a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, ks, q, hist_k, seed,
                          strict, h, stream);
}

int tv_int_peak_launch(int64_t iters, int32_t blocks, int32_t threads, void *stream, double *ops) {
  int dev;
  if (int rc = current_device(&dev)) return rc;
  static uint32_t *sink = nullptr;
  if (!sink) CK(cudaMalloc(&sink, 4));
  k_int_peak<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, 12345u, sink);
  CK(cudaGetLastError());
  if (ops) *ops = (double)blocks * threads * (double)iters * 16.0;
  return 0;
}

// L2 ceilings for the GA roofline (its working set is L2-resident): streaming read+write of
// a buffer that fits in L2 (16-byte .cg accesses, grid-stride), or independent random 16-byte
// reads (the access pattern of roulette selection).
__global__ void __launch_bounds__(256) k_l2_probe(uint4 *buf, int64_t n16, int32_t reps, int32_t random) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  if (!random) {
    for (int r = 0; r < reps; r++)
      for (int64_t i = tid; i < n16; i += nth) {
        uint4 v = __ldcg(buf + i);
        v.x += 1u;
        __stcg(buf + i, v);
      }
  } else {
    // n16 rounded down to a power of two: the index is a mask of a Weyl sequence through a
    // multiplicative hash (a few integer ops per load, so the probe is bound by L2, not issue)
    uint32_t m = 1u;
    while ((int64_t)m * 2 <= n16) m *= 2;
    uint32_t acc = 0, x = (uint32_t)tid * 0x9E3779B9u;
    const int64_t per = (n16 + nth - 1) / nth;
    for (int r = 0; r < reps; r++)
      for (int64_t k = 0; k < per; k += 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {  // 8 independent loads in flight per thread
          x += 0x6D2B79F5u;
          v[u] = __ldcg(buf + (((x ^ (x >> 15)) * 0x2C1B3C6Du >> 7) & (m - 1u)));
        }
#pragma unroll
        for (int u = 0; u < 8; u++) acc += v[u].x ^ v[u].w;
      }
    if (acc == 0x12345678u) buf[0].y = acc;  // keep the loads
  }
}

// grid-barrier floor: the GA kernel's launch geometry (one 1024-thread CTA per SM), `syncs`
// grid.sync() calls back to back
__global__ void __launch_bounds__(1024, 1) k_gridsync_probe(int32_t syncs) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < syncs; i++) grid.sync();
}

int tv_l2_probe_launch(void *buf, int64_t bytes, int32_t reps, int32_t random, void *stream, double *bytes_moved) {
  int dev;
  if (int rc = current_device(&dev)) return rc;
  if (!buf || bytes < 16) return fail(TV_ERR_ARG, "probe buffer");
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int64_t n16 = bytes / 16;
  k_l2_probe<<<nsm * 8, 256, 0, (cudaStream_t)stream>>>((uint4 *)buf, n16, reps, random);
  CK(cudaGetLastError());
  if (bytes_moved) {
    const int64_t nth = (int64_t)nsm * 8 * 256, per = (n16 + nth - 1) / nth;
    *bytes_moved = random ? (double)nth * (double)((per + 7) / 8 * 8) * 16.0 * reps : 32.0 * (double)n16 * reps;
  }
  return 0;
}

int tv_gridsync_probe_launch(int32_t syncs, void *stream) {
  int dev;
  if (int rc = current_device(&dev)) return rc;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  void *args[] = {&syncs};
  CK(cudaLaunchCooperativeKernel((const void *)k_gridsync_probe, dim3(nsm), dim3(1024), args, 0, (cudaStream_t)stream));
  return 0;
}

int tv_sm_count(int32_t *n) {
  int dev;
  if (int rc = current_device(&dev)) return rc;
  CK(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev));
  return 0;
}

// ---------------------------------------------------------------- GA
struct tv_ga {
  GaParams P;
  int device;
  int cur;  // which population buffer is current
  int nblocks;
  size_t smem;
  // wide genomes (L > 64): word-major populations in P.pop0 / P.pop1 (W x n words)
  int W;                            // words per genome (1 = the narrow cooperative kernel)
  uint64_t *Tw;                     // L thresholds (device)
  unsigned long long *fw, *cdfw;    // n fitness / inclusive CDF (64-bit)
  int32_t *flags;                   // [stopped, final parity]
  unsigned long long *donew;
  void *scan_tmp;
  size_t scan_bytes;
  void *arena;  // narrow GA: one allocation holding P's buffers
  uint32_t *fknown;   // per individual of the current population: its fitness if known (GaParams::f_known)
  bool fknown_valid;  // fknown describes the current population
  // JaTAM fitness memo (ClassifyParams::memo_*), allocated at the first fitness call; valid for
  // the fitness parameters whose signature is memo_sig (cleared when they change)
  unsigned long long *memo_keys;
  uint32_t *memo_vals;
  uint64_t memo_cap;
  uint64_t memo_sig;
  bool memo_clear;             // set_population started a new run: clear before the next use
  // which fitness function fknown's values come from (the JaTAM parameter signature), so a
  // fitness call with other parameters never inherits them
  uint64_t fknown_sig;
  uint64_t fit_sig_last;       // signature and output buffer of the last tv_ga_fitness_jatam call
  const uint32_t *fit_out_last;
};

// FNV-1a over the parameters a JaTAM fitness value depends on (besides the genome)
static uint64_t fit_signature(int32_t a, int32_t bpl, const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                              const int64_t *free_pos, int64_t nfree, int32_t d, int32_t k, uint64_t seed,
                              int32_t strict, const uint8_t *target_occ) {
  uint64_t h = 0xCBF29CE484222325ULL;
  auto mix = [&h](const void *p, size_t nb) {
    const unsigned char *c = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < nb; i++) { h ^= c[i]; h *= 0x100000001B3ULL; }
  };
  mix(&a, 4); mix(&bpl, 4); mix(&m, 8); mix(&nfree, 8); mix(&d, 4); mix(&k, 4); mix(&seed, 8); mix(&strict, 4);
  if (m > 0) { mix(mask_pos, (size_t)m * 8); mix(mask_val, (size_t)m); }
  if (nfree > 0) mix(free_pos, (size_t)nfree * 8);
  mix(target_occ, (size_t)d * d);
  return h;
}

// Bind the handle's fitness memo to P (allocating it on first use, clearing it when the fitness
// parameters changed).  On by default for populations >= 2^21, where the fitness pass is
// throughput-bound (below that it sits on its single-chain floor and the probes only cost:
// DESIGN.md section 6); TV_FITMEMO=1 / 0 forces it on / off.  Capacity: a power of two
// >= 8 n, <= 2^24 slots.
static int memo_bind(tv_ga *h, uint64_t sig, ClassifyParams &P, cudaStream_t st) {
  P.memo_keys = nullptr; P.memo_vals = nullptr; P.memo_mask = 0;
  const char *em = getenv("TV_FITMEMO");
  if (em ? atoi(em) == 0 : h->P.n < ((int64_t)1 << 21)) return 0;
  if (!h->memo_keys) {
    uint64_t cap = 1;
    while (cap < 8 * (uint64_t)h->P.n && cap < ((uint64_t)1 << 24)) cap <<= 1;
    cudaError_t e = cudaMalloc(&h->memo_keys, cap * 8);
    e = e ? e : cudaMalloc(&h->memo_vals, cap * 4);
    if (e != cudaSuccess) {
      cudaFree(h->memo_keys); cudaFree(h->memo_vals);
      h->memo_keys = nullptr; h->memo_vals = nullptr;
      cudaGetLastError();
      return 0;  // no memo: every genome is classified
    }
    h->memo_cap = cap;
    h->memo_sig = ~sig;  // force the clear below
  }
  if (h->memo_sig != sig || h->memo_clear) {
    CK(cudaMemsetAsync(h->memo_keys, 0, h->memo_cap * 8, st));
    h->memo_sig = sig;
    h->memo_clear = false;
  }
  P.memo_keys = h->memo_keys; P.memo_vals = h->memo_vals; P.memo_mask = h->memo_cap - 1;
  return 0;
}

int tv_ga_create(int64_t n, int32_t L, int32_t mode, const uint64_t *T, tv_ga **out) {
  if (n < 2 || n > ((int64_t)1 << 28)) return fail(TV_ERR_ARG, "population %lld outside [2, 2^28]", (long long)n);
  if (L < 1 || L > 64 * kGaMaxWords) return fail(TV_ERR_ARG, "genome length %d outside [1, %d]", L, 64 * kGaMaxWords);
  if (mode < 0 || mode > 2) return fail(TV_ERR_ARG, "reproduction mode %d not in {0,1,2}", mode);
  if (L <= 64 && (uint64_t)L * (uint64_t)n >= ((uint64_t)1 << 32)) return fail(TV_ERR_ARG, "L * population must be < 2^32");
  int dev;
  if (int rc = current_device(&dev)) return rc;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (L > 64) {  // wide genomes: per-generation launches over word-major populations
    tv_ga *h = new tv_ga();
    memset(&h->P, 0, sizeof h->P);
    h->P.n = n; h->P.L = L; h->P.mode = mode;
    h->W = (L + 63) / 64;
    h->device = dev;
    h->cur = 0;
    cudaError_t e = cudaSuccess;
    const size_t words = (size_t)n * h->W;
    e = e ? e : cudaMalloc(&h->P.pop0, words * 8);
    e = e ? e : cudaMalloc(&h->P.pop1, words * 8);
    e = e ? e : cudaMalloc(&h->Tw, (size_t)L * 8);
    e = e ? e : cudaMalloc(&h->fw, (size_t)n * 8);
    e = e ? e : cudaMalloc(&h->cdfw, (size_t)n * 8);
    e = e ? e : cudaMalloc(&h->flags, 8);
    e = e ? e : cudaMalloc(&h->donew, 8);
    e = e ? e : cudaMemset(h->P.pop0, 0, words * 8);
    e = e ? e : cudaMemcpy(h->Tw, T, (size_t)L * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cub::DeviceScan::InclusiveSum(nullptr, h->scan_bytes, h->fw, h->cdfw, (int)n);
    e = e ? e : cudaMalloc(&h->scan_tmp, std::max<size_t>(h->scan_bytes, 16));
    if (e != cudaSuccess) { tv_ga_destroy(h); return fail(TV_ERR_CUDA, "GA allocation: %s", cudaGetErrorString(e)); }
    *out = h;
    return 0;
  }
  tv_ga *h = new tv_ga();
  memset(&h->P, 0, sizeof h->P);
  h->W = 1;
  GaParams &P = h->P;
  P.n = n; P.L = L; P.mode = mode;
  for (int j = 0; j < 64; j++) P.T[j] = j < L ? T[j] : ~0ULL;
  h->nblocks = nsm;
  if (const char *ec = getenv("TV_GA_CTAS")) h->nblocks = std::max(1, std::min(nsm, atoi(ec)));  // A/B only
  P.chunk = ((n + h->nblocks - 1) / h->nblocks + 31) / 32 * 32;  // whole rows of 32 (k_ga_run)
  {  // staged mode: the chunk's genomes, fitness and row offsets in shared memory (k_ga_run)
    const size_t bytes = (size_t)(2 * P.chunk + P.chunk / 32) * 4;
    const char *es = getenv("TV_GA_STG"), *ep = getenv("TV_GA_PAIR");  // A/B only
    P.stg = L <= 32 && bytes <= (size_t)200 * 1024 && (es ? atoi(es) != 0 : true);
    P.pair = ep ? atoi(ep) != 0 : 1;
    h->smem = P.stg ? bytes : 0;
    // once per device, at the cap (handles differ in chunk size)
    static std::atomic<unsigned long long> attr_set{0};
    if (P.stg && dev < 64 && !((attr_set.load() >> dev) & 1ULL)) {
      CK(cudaFuncSetAttribute(k_ga_run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr_set.fetch_or(1ULL << dev);
    } else if (P.stg && dev >= 64) {
      CK(cudaFuncSetAttribute(k_ga_run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
  }
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ga_run, TV_GA_THREADS, h->smem));
  if (per_sm < 1) { delete h; return fail(TV_ERR_CUDA, "GA kernel does not fit one CTA per SM"); }
  h->device = dev;
  h->cur = 0;
  cudaError_t e = cudaSuccess;
  {  // one arena for the generation loop's buffers
    const size_t al = 4096;
    const size_t sz[11] = {(size_t)n * 8, (size_t)n * 8, (size_t)n * 4, (size_t)n * sizeof(ulonglong2), (size_t)n * 4,
                          (size_t)h->nblocks * 8, (size_t)h->nblocks * (size_t)(P.chunk / 32) * 4, 8, 4,
                          (size_t)n * 4, (size_t)h->nblocks * 4};
    size_t off[11], total = 0;
    for (int i = 0; i < 11; i++) { off[i] = total; total += (sz[i] + al - 1) / al * al; }
    auto bind = [&](char *base) {
      h->arena = base;
      P.pop0 = reinterpret_cast<unsigned long long *>(base + off[0]);
      P.pop1 = reinterpret_cast<unsigned long long *>(base + off[1]);
      P.cdf = reinterpret_cast<uint32_t *>(base + off[2]);
      P.guide = reinterpret_cast<ulonglong2 *>(base + off[3]);
      P.fstage = reinterpret_cast<uint32_t *>(base + off[4]);
      P.tot = reinterpret_cast<unsigned long long *>(base + off[5]);
      P.rowx = reinterpret_cast<uint32_t *>(base + off[6]);
      P.done = reinterpret_cast<unsigned long long *>(base + off[7]);
      P.final_buf = reinterpret_cast<int32_t *>(base + off[8]);
      h->fknown = reinterpret_cast<uint32_t *>(base + off[9]);
      P.first_g = reinterpret_cast<uint32_t *>(base + off[10]);
    };
    // Placement calibration (large populations): the same loop runs at ~23, ~27 or ~29 us per
    // generation at 2^20 depending on where its buffers land physically (about 30 % of arenas
    // are fast, tools/ga_bench_order.py), so K arenas (TV_GA_CALIB=K,
    // default 8; 0 or 1 disables) are timed on a short generation loop over a random population
    // and the fastest is kept (~10 ms once per handle; evolve pools handles).  Results do not
    // depend on it.
    const char *ec = getenv("TV_GA_CALIB");
    int K = ec ? atoi(ec) : 8;
    K = std::max(1, std::min(K, 8));
    if (n < ((int64_t)1 << 16) || (size_t)K * total > ((size_t)2 << 30)) K = 1;
    char *arena[8] = {nullptr}, *gap[8] = {nullptr};
    float ms[8] = {0.f};
    const char *eg = getenv("TV_GA_CALIB_GAP");  // development aid: MiB allocated between arenas
    const size_t gap_bytes = eg ? (size_t)atoi(eg) << 20 : 0;
    for (int a = 0; a < K && e == cudaSuccess; a++) {
      if (a && gap_bytes) e = cudaMalloc(&gap[a], gap_bytes);
      e = e ? e : cudaMalloc(&arena[a], total);
      if (e != cudaSuccess && a > 0) {  // out of memory for more candidates: calibrate what there is
        cudaGetLastError();
        e = cudaSuccess;
        if (gap[a]) cudaFree(gap[a]);
        gap[a] = arena[a] = nullptr;
        K = a;
        break;
      }
      if (e != cudaSuccess || K == 1) break;
      bind(arena[a]);
      GaParams Q = P;
      const int gens = 24;
      Q.seed = 1; Q.g0 = 0; Q.n_gens = gens; Q.target = (uint32_t)L; Q.adapt_count = n; Q.stop_when = 0;
      Q.fitness = 0; Q.f_ext = nullptr; Q.f_known = nullptr; Q.prof = nullptr;
      for (int j = 0; j < 64; j++) Q.T[j] = j < L ? T[j] : ~0ULL;
      uint32_t *sb = nullptr;
      unsigned long long *ss = nullptr;
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      e = e ? e : cudaMalloc(&sb, (size_t)gens * 8);
      e = e ? e : cudaMalloc(&ss, (size_t)gens * 8);
      if (e == cudaSuccess) {
        k_ga_fill_random<<<(unsigned)((n + 255) / 256), 256>>>(Q.pop0, n, L);
        e = cudaGetLastError();
      }
      e = e ? e : cudaMemset(sb, 0, (size_t)gens * 8);
      e = e ? e : cudaMemset(ss, 0, (size_t)gens * 8);
      Q.best = sb; Q.count = sb + gens; Q.sum = ss;
      e = e ? e : cudaEventCreate(&e0);
      e = e ? e : cudaEventCreate(&e1);
      void *args[] = {&Q};
      for (int rep = 0; rep < 2 && e == cudaSuccess; rep++) {  // the first launch warms up
        e = cudaEventRecord(e0, 0);
        e = e ? e : cudaLaunchCooperativeKernel((const void *)k_ga_run, dim3(h->nblocks), dim3(TV_GA_THREADS), args,
                                                h->smem, 0);
        e = e ? e : cudaEventRecord(e1, 0);
        e = e ? e : cudaEventSynchronize(e1);
        e = e ? e : cudaEventElapsedTime(&ms[a], e0, e1);
      }
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
      cudaFree(sb); cudaFree(ss);
    }
    if (e == cudaSuccess) {
      int keep = 0;
      for (int a = 1; a < K; a++)
        if (arena[a] && ms[a] < ms[keep]) keep = a;
      if (getenv("TV_GA_CALIB_LOG")) {
        fprintf(stderr, "tv_ga_create calibration (us/gen):");
        for (int a = 0; a < K; a++)
          fprintf(stderr, " %.2f%s[%p]", ms[a] * 1e3 / 24, a == keep ? "*" : "", (void *)arena[a]);
        fprintf(stderr, "\n");
      }
      for (int a = 0; a < K; a++) {
        if (a != keep && arena[a]) cudaFree(arena[a]);
        if (gap[a]) cudaFree(gap[a]);
      }
      bind(arena[keep]);
    } else {
      for (int a = 0; a < K; a++) { cudaFree(arena[a]); cudaFree(gap[a]); }
      h->arena = nullptr;
    }
  }
  e = e ? e : cudaMemset(P.pop0, 0, n * 8);
  if (e != cudaSuccess) { tv_ga_destroy(h); return fail(TV_ERR_CUDA, "GA allocation: %s", cudaGetErrorString(e)); }
  *out = h;
  return 0;
}

int tv_ga_destroy(tv_ga *h) {
  if (!h) return 0;
  GaParams &P = h->P;
  if (h->arena) {
    cudaFree(h->arena);
  } else {
    cudaFree(P.pop0); cudaFree(P.pop1); cudaFree(P.cdf); cudaFree(P.guide); cudaFree(P.fstage); cudaFree(P.tot);
    cudaFree(P.rowx);
    cudaFree(P.done); cudaFree(P.final_buf);
  }
  cudaFree(h->Tw); cudaFree(h->fw); cudaFree(h->cdfw); cudaFree(h->flags); cudaFree(h->donew); cudaFree(h->scan_tmp);
  cudaFree(h->memo_keys); cudaFree(h->memo_vals);
  delete h;
  return 0;
}

int tv_ga_set_population(tv_ga *h, const uint64_t *genomes, void *stream) {
  if (!h) return fail(TV_ERR_ARG, "null GA");
  if (int rc = on_device(h->device)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  h->fknown_valid = false;
  h->memo_clear = true;  // a new run: the fitness memo starts empty (a repeated run is re-classified)
  unsigned long long *dst = h->cur ? h->P.pop1 : h->P.pop0;
  const int64_t words = h->P.n * h->W;
  if (!genomes) {
    CK(cudaMemsetAsync(dst, 0, words * 8, st));
  } else if (h->W == 1) {
    CK(cudaMemcpyAsync(dst, genomes, h->P.n * 8, cudaMemcpyDefault, st));
  } else {  // host / caller layout [n, W] -> device word-major [W, n]
    Scratch S(st);
    unsigned long long *tmp;
    CK(S.get(&tmp, (size_t)words));
    CK(cudaMemcpyAsync(tmp, genomes, words * 8, cudaMemcpyDefault, st));
    k_gaw_transpose<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(tmp, dst, h->P.n, h->W, 1);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

int tv_ga_get_population(tv_ga *h, uint64_t *out, void *stream) {
  if (!h) return fail(TV_ERR_ARG, "null GA");
  if (int rc = on_device(h->device)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned long long *src = h->cur ? h->P.pop1 : h->P.pop0;
  if (h->W == 1) {
    CK(cudaMemcpyAsync(out, src, h->P.n * 8, cudaMemcpyDefault, st));
  } else {  // device word-major [W, n] -> caller layout [n, W]
    const int64_t words = h->P.n * h->W;
    Scratch S(st);
    unsigned long long *tmp;
    CK(S.get(&tmp, (size_t)words));
    k_gaw_transpose<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(src, tmp, h->P.n, h->W, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp, words * 8, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

int tv_ga_population_ptr(tv_ga *h, uint64_t **dev_ptr) {
  if (!h) return fail(TV_ERR_ARG, "null GA");
  *dev_ptr = reinterpret_cast<uint64_t *>(h->cur ? h->P.pop1 : h->P.pop0);
  return 0;
}

int tv_ga_run(tv_ga *h, uint64_t seed, int64_t g0, int64_t n_gens, uint32_t target, int64_t adapt_count,
              int32_t stop_when, const uint32_t *f_ext, uint32_t *best, uint64_t *sum, uint32_t *count,
              int64_t *gens_done, void *stream) {
  NvtxRange nvtx_("tv_ga_run", (long long)n_gens);
  if (!h) return fail(TV_ERR_ARG, "null GA");
  if (int rc = on_device(h->device)) return rc;
  if (n_gens < 1) return fail(TV_ERR_ARG, "n_gens must be >= 1");
  if (f_ext && n_gens != 1) return fail(TV_ERR_ARG, "an external fitness vector covers exactly one generation");
  if (f_ext && !is_device_ptr(f_ext)) return fail(TV_ERR_ARG, "external fitness must be a device pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (h->W > 1) {
    if (f_ext) return fail(TV_ERR_ARG, "external fitness needs L <= 64");
    GaWideParams Q;
    memset(&Q, 0, sizeof Q);
    Q.n = h->P.n; Q.L = h->P.L; Q.W = h->W; Q.mode = h->P.mode; Q.target = target; Q.adapt_count = adapt_count;
    Q.stop_when = stop_when; Q.seed = seed; Q.T = h->Tw; Q.f = h->fw; Q.cdf = h->cdfw;
    Q.stopped = h->flags; Q.final_par = h->flags + 1; Q.done = h->donew;
    Scratch S(st);
    uint32_t *d_best, *d_count; unsigned long long *d_sum;
    CK(S.get(&d_best, n_gens)); CK(S.get(&d_count, n_gens)); CK(S.get(&d_sum, n_gens));
    CK(cudaMemsetAsync(d_best, 0, n_gens * 4, st));
    CK(cudaMemsetAsync(d_count, 0, n_gens * 4, st));
    CK(cudaMemsetAsync(d_sum, 0, n_gens * 8, st));
    const int32_t init_flags[2] = {0, -1};
    CK(cudaMemcpyAsync(h->flags, init_flags, 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(h->donew, 0, 8, st));
    Q.best = d_best; Q.count = d_count; Q.sum = d_sum;
    const unsigned blocks = (unsigned)((Q.n + 255) / 256);
    for (int64_t t = 0; t < n_gens; t++) {
      const int par = (h->cur + (int)(t & 1)) & 1;
      Q.pop = par ? h->P.pop1 : h->P.pop0;
      Q.nxt = par ? h->P.pop0 : h->P.pop1;
      Q.g = g0 + t; Q.t = t;
      k_gaw_fitness<<<blocks, 256, 0, st>>>(Q);
      size_t tb = h->scan_bytes;
      CK(cub::DeviceScan::InclusiveSum(h->scan_tmp, tb, h->fw, h->cdfw, (int)Q.n, st));
      k_gaw_children<<<blocks, 256, 0, st>>>(Q);
    }
    CK(cudaGetLastError());
    g_launch[0] = 4; g_launch[1] = blocks; g_launch[2] = 256; g_launch[3] = 0; g_launch[4] = 3 * n_gens;
    unsigned long long done = 0;
    int32_t fl[2];
    CK(cudaMemcpyAsync(&done, h->donew, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fl, h->flags, 8, cudaMemcpyDeviceToHost, st));
    if (best) CK(cudaMemcpyAsync(best, d_best, n_gens * 4, cudaMemcpyDefault, st));
    if (count) CK(cudaMemcpyAsync(count, d_count, n_gens * 4, cudaMemcpyDefault, st));
    if (sum) CK(cudaMemcpyAsync(sum, d_sum, n_gens * 8, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    // current buffer: the generation the run stopped on, else the one after the last
    const int64_t last = fl[0] ? (int64_t)(done - 1) : n_gens;
    h->cur = (h->cur + (int)(last & 1)) & 1;
    if (gens_done) *gens_done = (int64_t)done;
    return 0;
  }
  GaParams P = h->P;
  if (h->cur) std::swap(P.pop0, P.pop1);
  P.seed = seed; P.g0 = g0; P.n_gens = n_gens; P.target = target; P.adapt_count = adapt_count;
  P.stop_when = stop_when; P.fitness = f_ext ? 1 : 0; P.f_ext = f_ext;
  P.f_known = f_ext ? h->fknown : nullptr;  // children equal to a parent inherit its fitness (one generation)
  int64_t done = 0;
  int32_t fb = 0;
  {
    Scratch S(st);
    uint32_t *d_best, *d_count; unsigned long long *d_sum;
    CK(S.get(&d_best, n_gens)); CK(S.get(&d_count, n_gens)); CK(S.get(&d_sum, n_gens));
    CK(cudaMemsetAsync(d_best, 0, n_gens * 4, st));
    CK(cudaMemsetAsync(d_count, 0, n_gens * 4, st));
    CK(cudaMemsetAsync(d_sum, 0, n_gens * 8, st));
    P.best = d_best; P.count = d_count; P.sum = d_sum;
    P.prof = nullptr;
    const bool prof = getenv("TV_GA_PROF") != nullptr;  // phase timing of CTA 0 (development aid)
    if (prof) { CK(S.get(&P.prof, 3)); CK(cudaMemsetAsync(P.prof, 0, 24, st)); }
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k_ga_run, dim3(h->nblocks), dim3(TV_GA_THREADS), args, h->smem, st));
    g_launch[0] = 3; g_launch[1] = h->nblocks; g_launch[2] = TV_GA_THREADS; g_launch[3] = (int64_t)h->smem; g_launch[4] = 1;
    CK(cudaMemcpyAsync(&done, P.done, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&fb, P.final_buf, 4, cudaMemcpyDeviceToHost, st));
    if (best) CK(cudaMemcpyAsync(best, d_best, n_gens * 4, cudaMemcpyDefault, st));
    if (count) CK(cudaMemcpyAsync(count, d_count, n_gens * 4, cudaMemcpyDefault, st));
    if (sum) CK(cudaMemcpyAsync(sum, d_sum, n_gens * 8, cudaMemcpyDefault, st));
    if (prof) {
      unsigned long long ph[3];
      CK(cudaMemcpyAsync(ph, P.prof, 24, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      const double g = (double)std::max<int64_t>(1, done);
      fprintf(stderr, "tv_ga_run phases (CTA 0, us/gen): A+barrier %.2f  B+barrier %.2f  C %.2f\n",
              ph[0] / g / 1e3, ph[1] / g / 1e3, ph[2] / g / 1e3);
    }
  }
  CK(cudaStreamSynchronize(st));
  h->cur ^= fb;
  h->fknown_valid = f_ext && fb;  // a reproduced generation with external fitness wrote fknown
  // its values are those of the last JaTAM fitness call if f_ext is that call's output
  h->fknown_sig = f_ext == h->fit_out_last ? h->fit_sig_last : 0;
  if (gens_done) *gens_done = done;
  return 0;
}

int tv_ga_replicas(int64_t n, int32_t L, int32_t mode, const uint64_t *T, int32_t R, const uint64_t *seeds,
                   const uint64_t *init, int64_t g0, int64_t n_gens, uint32_t target, int64_t adapt_count,
                   int32_t stop_when, int64_t *done, int64_t *disc, int64_t *adapt, uint32_t *best, uint64_t *sum,
                   uint32_t *count, uint64_t *final_pop, void *stream) {
  NvtxRange nvtx_("tv_ga_replicas", (long long)R);
  if (n < 2 || n > 8192) return fail(TV_ERR_ARG, "replica population %lld outside [2, 8192]", (long long)n);
  if (L < 1 || L > 64) return fail(TV_ERR_ARG, "genome length %d outside [1, 64]", L);
  if (mode < 0 || mode > 2) return fail(TV_ERR_ARG, "reproduction mode %d not in {0,1,2}", mode);
  if (R < 1) return fail(TV_ERR_ARG, "need at least one replica");
  if (n_gens < 1) return fail(TV_ERR_ARG, "n_gens must be >= 1");
  if (stop_when < 0 || stop_when > 2) return fail(TV_ERR_ARG, "stop_when %d not in {0,1,2}", stop_when);
  if (!seeds || !done || !disc || !adapt) return fail(TV_ERR_ARG, "seeds, done, disc and adapt are required");
  int dev;
  if (int rc = current_device(&dev)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  GaRepParams Q;
  memset(&Q, 0, sizeof Q);
  GaParams &P = Q.G;
  P.n = n; P.L = L; P.mode = mode; P.target = target; P.adapt_count = adapt_count; P.stop_when = stop_when;
  P.g0 = g0; P.n_gens = n_gens;
  for (int j = 0; j < 64; j++) P.T[j] = j < L ? T[j] : ~0ULL;
  Q.R = R;
  const size_t gens = (size_t)R * (size_t)n_gens;
  {
    Scratch S(st);
    uint64_t *d_seeds, *d_init = nullptr, *d_fin = nullptr, *d_sum = nullptr;
    int64_t *d_done, *d_disc, *d_adapt;
    uint32_t *d_best = nullptr, *d_count = nullptr;
    bool hs, hi = false;
    if (int rc = stage_in(seeds, (size_t)R, true, S, &d_seeds, hs)) return rc;
    if (init) if (int rc = stage_in(init, (size_t)R * n, true, S, &d_init, hi)) return rc;
    CK(S.get(&d_done, R)); CK(S.get(&d_disc, R)); CK(S.get(&d_adapt, R));
    if (best) CK(S.get(&d_best, gens));
    if (sum) CK(S.get(&d_sum, gens));
    if (count) CK(S.get(&d_count, gens));
    if (final_pop) CK(S.get(&d_fin, (size_t)R * n));
    Q.seeds = d_seeds; Q.init = reinterpret_cast<const unsigned long long *>(d_init);
    Q.final_pop = reinterpret_cast<unsigned long long *>(d_fin);
    Q.done = d_done; Q.disc = d_disc; Q.adapt = d_adapt;
    Q.best = d_best; Q.sum = reinterpret_cast<unsigned long long *>(d_sum); Q.count = d_count;
    const int threads = (int)std::min<int64_t>(1024, (n + 31) / 32 * 32);
    const size_t smem = (size_t)n * (2 * 8 + 4);
    CK(cudaFuncSetAttribute((const void *)k_ga_replicas, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void *args[] = {&Q};
    CK(cudaLaunchKernel((const void *)k_ga_replicas, dim3((unsigned)R), dim3(threads), args, smem, st));
    g_launch[0] = 3; g_launch[1] = R; g_launch[2] = threads; g_launch[3] = (int64_t)smem; g_launch[4] = 1;
    CK(cudaMemcpyAsync(done, d_done, (size_t)R * 8, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(disc, d_disc, (size_t)R * 8, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(adapt, d_adapt, (size_t)R * 8, cudaMemcpyDefault, st));
    if (best) CK(cudaMemcpyAsync(best, d_best, gens * 4, cudaMemcpyDefault, st));
    if (sum) CK(cudaMemcpyAsync(sum, d_sum, gens * 8, cudaMemcpyDefault, st));
    if (count) CK(cudaMemcpyAsync(count, d_count, gens * 4, cudaMemcpyDefault, st));
    if (final_pop) CK(cudaMemcpyAsync(final_pop, d_fin, (size_t)R * n * 8, cudaMemcpyDefault, st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

int tv_ga_mutate(uint64_t *pop, int64_t n, int32_t L, const uint64_t *T, uint64_t pthr, int32_t method,
                 uint64_t seed, int64_t g, uint64_t *flips, void *stream) {
  NvtxRange nvtx_(method ? "tv_ga_mutate bitwise" : "tv_ga_mutate distribution", (long long)n);
  if (!pop || !is_device_ptr(pop)) return fail(TV_ERR_ARG, "population must be a device pointer");
  if (n < 1 || L < 1 || L > 64 * kGaMaxWords) return fail(TV_ERR_ARG, "n / L out of range");
  if (method != 0 && method != 1) return fail(TV_ERR_ARG, "method must be 0 (distribution) or 1 (bit by bit)");
  cudaStream_t st = (cudaStream_t)stream;
  Scratch S(st);
  uint64_t *Td = nullptr;
  if (method == 0) {
    if (is_device_ptr(T)) Td = const_cast<uint64_t *>(T);
    else { CK(S.get(&Td, (size_t)L)); CK(cudaMemcpyAsync(Td, T, (size_t)L * 8, cudaMemcpyHostToDevice, st)); }
  }
  unsigned long long *fd = nullptr;
  if (flips) { CK(S.get(&fd, 1)); CK(cudaMemsetAsync(fd, 0, 8, st)); }
  k_ga_mutate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(reinterpret_cast<unsigned long long *>(pop), n, L, Td,
                                                            pthr, method, seed, g, fd);
  CK(cudaGetLastError());
  if (flips) {
    CK(cudaMemcpyAsync(flips, fd, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return 0;
}

int tv_ga_fitness_jatam(tv_ga *h, int32_t a, int32_t bpl, const int64_t *mask_pos, const uint8_t *mask_val,
                        int64_t m, const int64_t *free_pos, int64_t nfree, int32_t d, int32_t k, uint64_t seed,
                        int32_t strict, const uint8_t *target_occ, uint32_t *f_out, void *stream) {
  NvtxRange nvtx_("tv_ga_fitness_jatam");
  if (!h) return fail(TV_ERR_ARG, "null GA");
  if (int rc = on_device(h->device)) return rc;
  if (h->W > 1) return fail(TV_ERR_ARG, "JaTAM fitness needs L <= 64");
  if (d > 29) return fail(TV_ERR_ARG, "JaTAM fitness supports d <= 29");
  if (nfree != h->P.L) return fail(TV_ERR_ARG, "GA genome length %d != %lld free bits", h->P.L, (long long)nfree);
  if ((uint64_t)d * d * (uint64_t)h->P.n >= ((uint64_t)1 << 32)) return fail(TV_ERR_ARG, "d^2 * population must be < 2^32");
  if (!is_device_ptr(f_out)) return fail(TV_ERR_ARG, "fitness output must be a device pointer");
  Common C;
  const int64_t ks[1] = {k};
  if (int rc = fill_common(a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, ks, 1, k, seed, strict, C)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  ClassifyParams &P = C.P;
  P.fit_mode = 1;
  P.out_fit = f_out;
  int tc = 0;
  for (int r = 0; r < d; r++)
    for (int c = 0; c < d; c++)
      if (target_occ[r * d + c]) { P.target_rows[r + 1] |= 1u << (c + 1); tc++; }
  P.target_cells = tc;
  P.indices = reinterpret_cast<const uint64_t *>(h->cur ? h->P.pop1 : h->P.pop0);
  P.n = h->P.n;
  const char *efc = getenv("TV_FITCACHE");  // 0: classify every genome (A/B)
  const uint64_t sig = fit_signature(a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, k, seed, strict, target_occ);
  P.fit_known = (h->fknown_valid && h->fknown_sig == sig && (efc ? atoi(efc) != 0 : true)) ? h->fknown : nullptr;
  if (int rc = memo_bind(h, sig, P, st)) return rc;
  h->fit_sig_last = sig;
  h->fit_out_last = f_out;
  Scratch S(st);
  return launch_classify(C, S, st);
}

int tv_ga_run_jatam(tv_ga *h, int32_t a, int32_t bpl, const int64_t *mask_pos, const uint8_t *mask_val, int64_t m,
                    const int64_t *free_pos, int64_t nfree, int32_t d, int32_t k, uint64_t fit_seed, int32_t strict,
                    const uint8_t *target_occ, uint64_t seed, int64_t g0, int64_t n_gens, uint32_t target,
                    uint32_t *best, uint64_t *sum, uint32_t *count, void *stream) {
  NvtxRange nvtx_("tv_ga_run_jatam", (long long)n_gens);
  if (!h) return fail(TV_ERR_ARG, "null GA");
  if (int rc = on_device(h->device)) return rc;
  if (h->W > 1) return fail(TV_ERR_ARG, "JaTAM fitness needs L <= 64");
  if (n_gens < 1) return fail(TV_ERR_ARG, "n_gens must be >= 1");
  if (d > 29) return fail(TV_ERR_ARG, "JaTAM fitness supports d <= 29");
  if (nfree != h->P.L) return fail(TV_ERR_ARG, "GA genome length %d != %lld free bits", h->P.L, (long long)nfree);
  if ((uint64_t)d * d * (uint64_t)h->P.n >= ((uint64_t)1 << 32)) return fail(TV_ERR_ARG, "d^2 * population must be < 2^32");
  Common C0;
  const int64_t ks[1] = {k};
  if (int rc = fill_common(a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, ks, 1, k, fit_seed, strict, C0)) return rc;
  C0.P.fit_mode = 1;
  int tc = 0;
  for (int r = 0; r < d; r++)
    for (int c = 0; c < d; c++)
      if (target_occ[r * d + c]) { C0.P.target_rows[r + 1] |= 1u << (c + 1); tc++; }
  C0.P.target_cells = tc;
  C0.P.n = h->P.n;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t sig = fit_signature(a, bpl, mask_pos, mask_val, m, free_pos, nfree, d, k, fit_seed, strict,
                                     target_occ);
  if (int rc = memo_bind(h, sig, C0.P, st)) return rc;
  Scratch S(st);
  uint32_t *f, *d_best, *d_count; unsigned long long *d_sum;
  CK(S.get(&f, (size_t)h->P.n));
  CK(S.get(&d_best, n_gens)); CK(S.get(&d_count, n_gens)); CK(S.get(&d_sum, n_gens));
  CK(cudaMemsetAsync(d_best, 0, n_gens * 4, st));
  CK(cudaMemsetAsync(d_count, 0, n_gens * 4, st));
  CK(cudaMemsetAsync(d_sum, 0, n_gens * 8, st));
  const char *efc = getenv("TV_FITCACHE");
  const bool cache = efc ? atoi(efc) != 0 : true;
  // every generation reproduces (no stop rule), so the current buffer alternates on the host
  // side without reading the device back: the whole call is enqueued in one go
  for (int64_t t = 0; t < n_gens; t++) {
    Common C = C0;
    C.P.out_fit = f;
    C.P.indices = reinterpret_cast<const uint64_t *>(h->cur ? h->P.pop1 : h->P.pop0);
    C.P.fit_known = (h->fknown_valid && h->fknown_sig == sig && cache) ? h->fknown : nullptr;
    {
      Scratch SC(st);
      if (int rc = launch_classify(C, SC, st)) return rc;
    }
    GaParams P = h->P;
    if (h->cur) std::swap(P.pop0, P.pop1);
    P.seed = seed; P.g0 = g0 + t; P.n_gens = 1; P.target = target; P.adapt_count = h->P.n; P.stop_when = 0;
    P.fitness = 1; P.f_ext = f; P.f_known = h->fknown; P.prof = nullptr;
    P.best = d_best + t; P.count = d_count + t; P.sum = d_sum + t;
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k_ga_run, dim3(h->nblocks), dim3(TV_GA_THREADS), args, h->smem, st));
    h->cur ^= 1;
    h->fknown_valid = true;
    h->fknown_sig = sig;
  }
  if (best) CK(cudaMemcpyAsync(best, d_best, n_gens * 4, cudaMemcpyDefault, st));
  if (count) CK(cudaMemcpyAsync(count, d_count, n_gens * 4, cudaMemcpyDefault, st));
  if (sum) CK(cudaMemcpyAsync(sum, d_sum, n_gens * 8, cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

}  // extern "C"
