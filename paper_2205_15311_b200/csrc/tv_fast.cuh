// tv_fast.cuh -- the enumeration hot kernel: lane-per-genome movelist assembly
// on a shared-memory nibble bitboard with SWAR candidate masks.
//
// Covers a <= 3 tile types, b <= 8 labels, odd d with (d+2)^2 < 2^16.
// Bit-exact with the reference step order (_k:96-249).
//
// Layout (per warp, word-interleaved so lane L always hits bank L):
//   grid  : GW words/lane; cell (r,c) of the (d+2)x(d+2) padded board is
//           nibble lin = r*(d+2)+c; 0..4a-1 = placed candidate t*4+orient,
//           0xE = empty + on the movelist, 0xF = empty.
//   stack : S u16 entries/lane (entry = r<<8 | c), spilled to global beyond S.
// Per CTA: a small open-addressed phenotype cache (histogram mode) and the
// class tallies, flushed to the global table once at the end.
//
// Candidate scan (_k:166-209) as SWAR over nibble lanes, one nibble per
// candidate c = t*4 + orient: E[dir] holds the label each candidate shows in
// direction dir, so "bonds the neighbour's label p" is a nibble-equality with
// partner(p) and "strict conflict" is nonzero & !bond.  The first hit is
// ffs(cand); ambiguity is any other hit with a different in-situ 4-label
// code (precomputed class ids, _k:199-205).
#pragma once
#include "tv_params.cuh"

namespace tvb {

template <int A> struct FastMask { typedef uint32_t T; };
template <> struct FastMask<3> { typedef uint64_t T; };

template <typename M> __device__ __forceinline__ M rep_nib(uint32_t v) {
  return (M)v * (M)0x1111111111111111ULL;
}
template <typename M> __device__ __forceinline__ M nz_nib(M x) {  // bit 4i+3 set iff nibble i != 0
  const M l7 = (M)0x7777777777777777ULL, l8 = (M)0x8888888888888888ULL;
  return (((x & l7) + l7) | x) & l8;
}
template <typename M> __device__ __forceinline__ uint32_t get_nib(M x, uint32_t i) {
  return (uint32_t)(x >> (4 * i)) & 15u;
}
__device__ __forceinline__ int ffs_m(uint32_t x) { return __ffs(x) - 1; }
__device__ __forceinline__ int ffs_m(uint64_t x) { return __ffsll((long long)x) - 1; }

struct FastLane {
  uint32_t *gw;          // &grid word 0 of this lane (stride 32 words)
  uint32_t *sw;          // &stack word 0 of this lane (stride 32 words, 2 entries per word)
  uint16_t *spill;       // &spill entry 0 of this lane (stride 32)
  int S;
  __device__ __forceinline__ uint32_t nib(int lin) const {
    return (gw[(lin >> 3) * 32] >> ((lin & 7) * 4)) & 15u;
  }
  __device__ __forceinline__ void set_nib(int lin, uint32_t v) const {
    uint32_t *p = gw + (lin >> 3) * 32;
    const int s = (lin & 7) * 4;
    *p = (*p & ~(15u << s)) | (v << s);
  }
  __device__ __forceinline__ uint32_t st_read(int j) const {
    if (j < S) return reinterpret_cast<const uint16_t *>(sw + (j >> 1) * 32)[j & 1];
    return spill[(int64_t)(j - S) * 32];
  }
  __device__ __forceinline__ void st_write(int j, uint32_t e) const {
    if (j < S) reinterpret_cast<uint16_t *>(sw + (j >> 1) * 32)[j & 1] = (uint16_t)e;
    else spill[(int64_t)(j - S) * 32] = (uint16_t)e;
  }
};

enum { ST_NEED = 0, ST_RUN = 1, ST_DONE = 2 };

template <int A>
__global__ void __launch_bounds__(256, 2) k_classify_fast(const __grid_constant__ ClassifyParams P) {
  typedef typename FastMask<A>::T M;
  constexpr int NC = 4 * A;
  const M VALID = (M)(0x8888888888888888ULL >> (64 - 4 * NC));
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int words_per_warp = (P.GW + P.S / 2) * 32;
  FastLane Ln;
  Ln.gw = smem + warp * words_per_warp + lane;
  Ln.sw = Ln.gw + P.GW * 32;
  Ln.S = P.S;
  const int64_t gwarp = (int64_t)blockIdx.x * nwarps + warp;
  Ln.spill = P.spill + gwarp * (int64_t)P.spill_cap * 32 + lane;
  uint32_t *rh = P.run_hash + gwarp * (int64_t)P.kmax * 32 + lane;  // run r at rh[r*32]

  // per-CTA histogram cache + tallies
  uint32_t *cta = smem + nwarps * words_per_warp;
  const int HS = P.cta_slots;
  unsigned long long *c_key = reinterpret_cast<unsigned long long *>(cta);
  unsigned long long *c_rdet = c_key + HS;
  unsigned long long *c_rany = c_rdet + HS;
  uint32_t *c_det = reinterpret_cast<uint32_t *>(c_rany + HS);
  uint32_t *c_ste = c_det + HS;
  int32_t *c_gs = reinterpret_cast<int32_t *>(c_ste + HS);
  uint32_t *c_tal = reinterpret_cast<uint32_t *>(c_gs + HS);
  if (P.hist_mode) {
    for (int s = threadIdx.x; s < HS; s += blockDim.x) {
      c_key[s] = 0ULL; c_rdet[s] = ~0ULL; c_rany[s] = ~0ULL; c_det[s] = 0; c_ste[s] = 0; c_gs[s] = -1;
    }
    for (int s = threadIdx.x; s < P.q * 5; s += blockDim.x) c_tal[s] = 0;
  }
  for (int w = 0; w < P.GW; w++) Ln.gw[w * 32] = 0xFFFFFFFFu;
  __syncthreads();

  const int d = P.d, PD = d + 2, dd = d * d;
  const uint32_t magic = (uint32_t)(0x100000000ULL / (uint64_t)PD) + 1u;
  const int cE = ((d >> 1) + 1) * 257;  // centre entry (r<<8|c), padded coords
  const M strict_mask = P.strict ? ~(M)0 : (M)0;

  int st = ST_NEED;
  int64_t item = 0;
  uint64_t idx = 0, rs = 0;
  int run = 0, replay = 0, sp = 0;
  int minr = 0, maxr = 0, minc = 0, maxc = 0;
  int trivial_at = -1, first_unbound = -1, first_mismatch = -1;
  uint32_t hash0 = 0, best = 0;
  int64_t pslot = -1;  // histogram slot owning the payload being replayed
  M E0 = 0, E1 = 0, E2 = 0, E3 = 0, N0 = 0, N1 = 0, N2 = 0, N3 = 0, CLS = 0;

  auto start_run = [&]() {
    rs = stream_state(P.seed, idx, (uint64_t)run);
    const int cr = cE >> 8, cl = cr * PD + (cE & 255);
    Ln.set_nib(cl, 0u);                                  // seed tile, orientation 0 (_k:115)
    minr = maxr = minc = maxc = cr;
    uint32_t nbp = 0x03020100u;                          // N,E,S,W then shuffle (_k:122-131)
#pragma unroll
    for (int j = 3; j > 0; j--) {
      const uint32_t q = rng_below(rs, (uint32_t)(j + 1));
      const uint32_t x = ((nbp >> (8 * j)) ^ (nbp >> (8 * q))) & 0xFFu;
      nbp ^= (x << (8 * j)) | (x << (8 * q));
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {                        // push (_k:133-136)
      const uint32_t dir = (nbp >> (8 * j)) & 3u;
      const int de = dir == 0 ? -256 : dir == 1 ? 1 : dir == 2 ? 256 : -1;
      const int dl = dir == 0 ? -PD : dir == 1 ? 1 : dir == 2 ? PD : -1;
      Ln.st_write(j, (uint32_t)(cE + de));
      Ln.set_nib(cl + dl, 0xEu);
    }
    sp = 4;
  };

  auto cleanup = [&]() {  // all marks and tiles lie inside bbox +- 1 (Appendix A.8/9)
    const int lo = ((minr - 1) * PD + (minc - 1)) >> 3;
    const int hi = ((maxr + 1) * PD + (maxc + 1)) >> 3;
    for (int w = lo; w <= hi; w++) Ln.gw[w * 32] = 0xFFFFFFFFu;
  };

  // OAT over w, h, (x, y)... of the cropped shape (_k:260-277); optional pack (_k:280-292)
  auto scan = [&](int &w, int &h, int &n, unsigned long long *out, int64_t W) -> uint32_t {
    w = maxc - minc + 1;
    h = maxr - minr + 1;
    n = 0;
    uint32_t hs = oat_step(oat_step(0u, (uint32_t)w), (uint32_t)h);
    const int lo = (minr * PD + minc) >> 3, hi = (maxr * PD + maxc) >> 3;
    int64_t cw = 0;
    unsigned long long acc = 0;
    for (int wi = lo; wi <= hi; wi++) {
      uint32_t occ = nz_nib<uint32_t>(~Ln.gw[wi * 32]);
      while (occ) {
        const int b = __ffs(occ) - 1;
        occ &= occ - 1;
        const uint32_t L = (uint32_t)(wi * 8 + (b >> 2));
        const uint32_t R = __umulhi(L, magic);
        const int y = (int)R - minr, x = (int)(L - R * PD) - minc;
        hs = oat_step(oat_step(hs, (uint32_t)x), (uint32_t)y);
        n++;
        if (out) {
          const int bit = y * w + x;
          const int64_t wj = bit >> 6;
          while (cw < wj) { out[cw++] = acc; acc = 0; }
          acc |= 1ULL << (bit & 63);
        }
      }
    }
    if (out) { while (cw < W) { out[cw++] = acc; acc = 0; } }
    return oat_final(hs);
  };

  for (;;) {
    // ---- refill lanes that need a genome (warp-aggregated work counter)
    const unsigned need = __ballot_sync(0xFFFFFFFFu, st == ST_NEED);
    if (need) {
      const int leader = __ffs(need) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(P.work, (unsigned long long)__popc(need));
      base = __shfl_sync(0xFFFFFFFFu, base, leader);
      if (st == ST_NEED) {
        item = (int64_t)base + __popc(need & ((1u << lane) - 1u));
        if (item >= P.n) {
          st = ST_DONE;
        } else {
          idx = item_index(P.indices, P.start, P.chunk, P.stride, item);
          // decode labels, in-situ edge planes and equivalence ids (_k:384-401, _k:199)
          uint32_t lab[NC];
#pragma unroll
          for (int te = 0; te < NC; te++) lab[te] = decode_label(P.dec, te, idx);
          E0 = E1 = E2 = E3 = 0;
          uint32_t code[NC];
#pragma unroll
          for (int t = 0; t < A; t++) {
#pragma unroll
            for (int r = 0; r < 4; r++) {
              const int c = t * 4 + r;
              const uint32_t e0 = lab[t * 4 + ((0 - r) & 3)], e1 = lab[t * 4 + ((1 - r) & 3)];
              const uint32_t e2 = lab[t * 4 + ((2 - r) & 3)], e3 = lab[t * 4 + ((3 - r) & 3)];
              E0 |= (M)e0 << (4 * c); E1 |= (M)e1 << (4 * c);
              E2 |= (M)e2 << (4 * c); E3 |= (M)e3 << (4 * c);
              code[c] = e0 | (e1 << 4) | (e2 << 8) | (e3 << 12);
            }
          }
          CLS = 0;
#pragma unroll
          for (int c = 0; c < NC; c++) {
            uint32_t id = (uint32_t)c;
#pragma unroll
            for (int c2 = NC - 1; c2 >= 0; c2--)
              if (c2 < c && code[c2] == code[c]) id = (uint32_t)c2;
            CLS |= (M)id << (4 * c);
          }
          N0 = nz_nib<M>(E0) & VALID; N1 = nz_nib<M>(E1) & VALID;
          N2 = nz_nib<M>(E2) & VALID; N3 = nz_nib<M>(E3) & VALID;
          trivial_at = first_unbound = first_mismatch = -1;
          run = 0;
          replay = 0;
          start_run();
          st = ST_RUN;
        }
      }
    }
    if (!__any_sync(0xFFFFFFFFu, st == ST_RUN)) break;
    if (st != ST_RUN) continue;

    // ---- one movelist pop (_k:138-248)
    int ended = -1;
    if (sp == 0) {
      ended = RUN_BOUNDED;
    } else {
      const uint32_t e = Ln.st_read(--sp);
      const int r = (int)(e >> 8), c = (int)(e & 255u);
      const int lin = r * PD + c;
      const uint32_t vN = Ln.nib(lin - PD), vE = Ln.nib(lin + 1);
      const uint32_t vS = Ln.nib(lin + PD), vW = Ln.nib(lin - 1);
      M bond = 0, conf = 0;
      {
        // label each occupied neighbour shows toward this cell (_k:145-164); absent == inert
        const uint32_t pN = vN < (uint32_t)NC ? get_nib<M>(E2, vN) : 0u;
        const uint32_t pE = vE < (uint32_t)NC ? get_nib<M>(E3, vE) : 0u;
        const uint32_t pS = vS < (uint32_t)NC ? get_nib<M>(E0, vS) : 0u;
        const uint32_t pW = vW < (uint32_t)NC ? get_nib<M>(E1, vW) : 0u;
#define TV_DIR(Ed, Nd, p)                                                        \
  {                                                                              \
    const M on = (p) ? VALID : (M)0;                                             \
    const M bm = ~nz_nib<M>((Ed) ^ rep_nib<M>((((p) - 1u) ^ 1u) + 1u)) & on;     \
    bond |= bm;                                                                  \
    conf |= (Nd) & ~bm & on;                                                     \
  }
        TV_DIR(E0, N0, pN)
        TV_DIR(E1, N1, pE)
        TV_DIR(E2, N2, pS)
        TV_DIR(E3, N3, pW)
#undef TV_DIR
      }
      const M cand = bond & ~(conf & strict_mask);
      if (cand == 0) {
        Ln.set_nib(lin, 0xFu);                           // dropped, re-pushable (_k:210-211)
      } else {
        const uint32_t cf = (uint32_t)ffs_m(cand) >> 2;  // first hit in t-major, orient-minor order
        const M amb = nz_nib<M>(CLS ^ rep_nib<M>(get_nib<M>(CLS, cf))) & cand;
        if (amb) {
          ended = RUN_TRIVIAL;                           // _k:208-209
        } else if (r == 1 || c == 1 || r == d || c == d) {
          ended = RUN_UNBOUND;                           // _k:212-213
        } else {
          Ln.set_nib(lin, cf);                           // place (_k:214-224)
          minr = min(minr, r); maxr = max(maxr, r);
          minc = min(minc, c); maxc = max(maxc, c);
          uint32_t nbp = 0;
          int m = 0;                                     // new frontier N,E,S,W (_k:225-237)
          if (vN == 0xFu) { nbp |= 0u << (8 * m); m++; }
          if (vE == 0xFu) { nbp |= 1u << (8 * m); m++; }
          if (vS == 0xFu) { nbp |= 2u << (8 * m); m++; }
          if (vW == 0xFu) { nbp |= 3u << (8 * m); m++; }
          if (m == 3) {                                  // Fisher-Yates n=m..2 (_k:238-242)
            const uint32_t q = rng_below(rs, 3u);
            const uint32_t x = ((nbp >> 16) ^ (nbp >> (8 * q))) & 0xFFu;
            nbp ^= (x << 16) | (x << (8 * q));
          }
          if (m >= 2) {
            const uint32_t q = rng_below(rs, 2u);
            const uint32_t x = ((nbp >> 8) ^ (nbp >> (8 * q))) & 0xFFu;
            nbp ^= (x << 8) | (x << (8 * q));
          }
          for (int j = 0; j < m; j++) {                  // push (_k:243-248)
            if (sp >= dd) { ended = RUN_OVERFLOW; break; }
            const uint32_t dir = (nbp >> (8 * j)) & 3u;
            const int de = dir == 0 ? -256 : dir == 1 ? 1 : dir == 2 ? 256 : -1;
            const int dl = dir == 0 ? -PD : dir == 1 ? 1 : dir == 2 ? PD : -1;
            Ln.st_write(sp++, e + de);
            Ln.set_nib(lin + dl, 0xEu);
          }
        }
      }
    }
    if (ended < 0) continue;

    // ---- run end
    if (replay) {
      // replay of the attributed run: emit hash/w/h/cells + packed bitmap
      int w, h, n;
      if (!P.hist_mode) {
        unsigned long long *row = P.out_shape + item * P.W;
        scan(w, h, n, row, P.W);
        P.out_hash[item] = best;
        P.out_w[item] = (uint8_t)w;
        P.out_h[item] = (uint8_t)h;
        P.out_cells[item] = (uint16_t)n;
      } else {
        scan(w, h, n, P.hist.shape + pslot * P.hist.W, P.hist.W);
        P.hist.whc[pslot] = (uint32_t)w | ((uint32_t)h << 8) | ((uint32_t)n << 16);
      }
      cleanup();
      st = ST_NEED;
      continue;
    }
    bool genome_done = false, overflow = false;
    if (ended == RUN_BOUNDED) {
      int w, h, n;
      const uint32_t hs = scan(w, h, n, nullptr, 0);
      rh[run * 32] = hs;
      if (run == 0) hash0 = hs;
      else if (first_mismatch < 0 && first_unbound != 0 && hs != hash0) first_mismatch = run;  // _k:347-348
    } else if (ended == RUN_UNBOUND) {
      if (first_unbound < 0) first_unbound = run;
      rh[run * 32] = 0u;
    } else if (ended == RUN_TRIVIAL) {
      trivial_at = run;
      genome_done = true;
    } else {
      overflow = true;
      genome_done = true;
    }
    cleanup();
    run++;
    if (!genome_done && run < P.kmax) { start_run(); continue; }

    // ---- genome fold (_k:351-381, _k:434-452)
    if (overflow) {
      if (!P.hist_mode) {
        for (int k = 0; k < P.q; k++) P.out_class[item * P.q + k] = (uint8_t)CLS_ERROR;
      } else {
        for (int k = 0; k < P.q; k++) atomicAdd(&c_tal[k * 5 + 4], 1u);
      }
      st = ST_NEED;
      continue;
    }
    if (!P.hist_mode) {
      for (int k = 0; k < P.q; k++)
        P.out_class[item * P.q + k] = (uint8_t)class_at(P.ks[k], trivial_at, first_unbound, first_mismatch);
    } else {
      for (int k = 0; k < P.q; k++)
        atomicAdd(&c_tal[k * 5 + class_at(P.ks[k], trivial_at, first_unbound, first_mismatch)], 1u);
    }
    const int hc = class_at(P.hist_k, trivial_at, first_unbound, first_mismatch);
    if (hc != CLS_DET && hc != CLS_STERIC) {
      if (!P.hist_mode) {
        P.out_hash[item] = 0u; P.out_w[item] = 0; P.out_h[item] = 0; P.out_cells[item] = 0;
      }
      st = ST_NEED;
      continue;
    }
    int attr = 0;
    best = hash0;
    if (hc == CLS_STERIC) {  // majority hash over the first hist_k runs, ties -> smaller
      int best_n = 0;
      best = 0u;
      for (int j = 0; j < P.hist_k; j++) {
        const uint32_t hj = rh[j * 32];
        int cnt = 0;
        for (int l = 0; l < P.hist_k; l++) cnt += rh[l * 32] == hj;
        if (cnt > best_n || (cnt == best_n && hj < best)) { best_n = cnt; best = hj; }
      }
      if (best != hash0)
        for (int j = 1; j < P.hist_k; j++)
          if (rh[j * 32] == best) { attr = j; break; }
    }
    bool need_payload = true;
    if (P.hist_mode) {
      const bool det = hc == CLS_DET;
      bool gnew = false;
      int64_t g = -1;
      bool cached = false;
      if (HS > 0) {
        const unsigned long long key = (1ULL << 32) | best;
        uint32_t s = (uint32_t)hist_home(best, HS);
        for (int p = 0; p < 16; p++) {
          unsigned long long k = *((volatile unsigned long long *)&c_key[s]);
          if (k == 0ULL) {
            k = atomicCAS(&c_key[s], 0ULL, key);
            if (k == 0ULL) {
              g = hist_claim(P.hist, best, gnew);
              *((volatile int32_t *)&c_gs[s]) = (int32_t)g;
              k = key;
            }
          }
          if (k == key) {
            atomicAdd(det ? &c_det[s] : &c_ste[s], 1u);
            if (det) atomicMin(&c_rdet[s], (unsigned long long)idx);
            atomicMin(&c_rany[s], (unsigned long long)idx);
            cached = true;
            break;
          }
          s = (s + 1) & (uint32_t)(HS - 1);
        }
      }
      if (!cached) {
        g = hist_claim(P.hist, best, gnew);
        if (g >= 0) {
          atomicAdd(det ? &P.hist.det[g] : &P.hist.steric[g], 1ULL);
          if (det) hist_min(&P.hist.rep_det[g], idx);
          hist_min(&P.hist.rep_any[g], idx);
        }
      }
      need_payload = gnew;
      pslot = g;
    }
    if (need_payload) {
      replay = 1;
      run = attr;
      start_run();
    } else {
      st = ST_NEED;
    }
  }

  if (P.hist_mode) {
    __syncthreads();
    for (int s = threadIdx.x; s < HS; s += blockDim.x) {
      if (c_key[s] == 0ULL) continue;
      const int32_t g = c_gs[s];
      if (g < 0) continue;
      if (c_det[s]) atomicAdd(&P.hist.det[g], (unsigned long long)c_det[s]);
      if (c_ste[s]) atomicAdd(&P.hist.steric[g], (unsigned long long)c_ste[s]);
      if (c_rdet[s] != ~0ULL) hist_min(&P.hist.rep_det[g], c_rdet[s]);
      if (c_rany[s] != ~0ULL) hist_min(&P.hist.rep_any[g], c_rany[s]);
    }
    for (int s = threadIdx.x; s < P.q * 5; s += blockDim.x)
      if (c_tal[s]) atomicAdd(&P.hist.tallies[s], (unsigned long long)c_tal[s]);
  }
}

// shared-memory bytes per CTA for the fast kernel
inline size_t fast_smem_bytes(int threads, int GW, int S, int cta_slots, int q) {
  size_t per_warp = (size_t)(GW + S / 2) * 32 * 4;
  size_t cta = (size_t)cta_slots * (8 * 3 + 4 * 3) + (size_t)q * 5 * 4;
  return per_warp * (threads / 32) + cta;
}

}  // namespace tvb
