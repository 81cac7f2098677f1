// tv_fast.cuh -- the enumeration hot kernel: lane-per-genome movelist assembly
// on a shared-memory nibble board with per-genome candidate tables.
//
// Covers a <= 3 tile types, b <= 8 labels, d <= 118 (row stride < 128).
// Bit-exact with the reference step order (_k:96-249).
//
// Layout (per warp, interleaved by lane so lane L always hits bank L):
//   board : GW words/lane; cell (r,c) of the (d+2)x(d+2) padded board is
//           nibble lin = r*RS+c (RS = 8*ceil((d+2)/8) for a <= 2: whole-word
//           rows, N/S neighbours at a fixed word offset; RS = d+2 for a = 3);
//           0..4a-1 = placed candidate t*4+orient, 0xE = empty + on the
//           movelist, 0xF = empty.
//   stack : S u16 slots/lane (entry = lin; slot k of lane L at halfword k*32+L).
//           a <= 2: a ring holding the top S entries (S a power of two), the
//           ones below spilled to global and refilled ahead of use
//           (FastLane<true>); a = 3: entries 0..S-1 here, deeper ones in
//           global (FastLane<false>).
// Per CTA: a small open-addressed phenotype cache (histogram mode) and the
// class tallies, flushed to the global table once at the end.
//
// Candidate scan (_k:166-209) as SWAR over nibble lanes, one nibble per
// candidate c = t*4 + orient (scan order): E[dir] holds the label each
// candidate shows in direction dir, so "bonds the neighbour's label p" is a
// nibble-equality with partner(p) and "strict conflict" is nonzero & !bond.
// The first hit is ffs(cand); ambiguity is any other hit whose in-situ 4-label
// code differs (precomputed equivalence-class ids, _k:199-205).  (Per-genome
// lookup tables indexed by neighbour value were measured slower: building
// them costs ~900 instructions per genome in the divergent service pass.)
//
// Lane service (run end, k-run fold, histogram insert, refill) is divergent
// and several times longer than a pop, so a lane whose run ended parks and
// the warp services all parked lanes in one pass once enough accumulated.
#pragma once
#include "tv_params.cuh"

namespace tvb {

template <typename M> __device__ __forceinline__ M rep_nib(uint32_t v) {
  return (M)v * (M)0x1111111111111111ULL;
}
template <> __device__ __forceinline__ uint64_t rep_nib<uint64_t>(uint32_t v) {  // v < 16: one multiply
  const uint32_t r = v * 0x11111111u;
  return ((uint64_t)r << 32) | r;
}
template <typename M> __device__ __forceinline__ M nz_nib(M x) {  // bit 4i+3 set iff nibble i != 0
  const M l7 = (M)0x7777777777777777ULL, l8 = (M)0x8888888888888888ULL;
  return (((x & l7) + l7) | x) & l8;
}
template <> __device__ __forceinline__ uint64_t nz_nib<uint64_t>(uint64_t x) {  // no carry crosses a nibble
  const uint32_t lo = nz_nib<uint32_t>((uint32_t)x), hi = nz_nib<uint32_t>((uint32_t)(x >> 32));
  return ((uint64_t)hi << 32) | lo;
}
template <typename M> __device__ __forceinline__ uint32_t get_nib(M x, uint32_t i) {
  return (uint32_t)(x >> (4 * i)) & 15u;
}
__device__ __forceinline__ int ffs_m(uint32_t x) { return __ffs(x) - 1; }
__device__ __forceinline__ int ffs_m(uint64_t x) {  // candidate flags never reach bit 63: halves suffice
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return lo ? __ffs(lo) - 1 : 31 + __ffs(hi);
}

__device__ __forceinline__ unsigned long long fast_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <bool RING> struct FastLane {
  uint32_t *gw;     // &board word 0 of this lane (stride 32 words)
  uint16_t *sw;     // &movelist slot 0 of this lane: slot k at sw[k * 32] (lanes 2k, 2k+1 share a bank word)
  uint16_t *spill;  // &spill entry 0 of this lane (stride 32)
  int mask;         // RING: ring slots - 1 (a power of two); else the shared slots S (linear stack)
  __device__ __forceinline__ uint32_t nib(int lin) const {
    return (gw[(lin >> 3) * 32] >> ((lin & 7) * 4)) & 15u;
  }
  __device__ __forceinline__ void set_nib(int lin, uint32_t v) const {
    uint32_t *p = gw + (lin >> 3) * 32;
    const int s = (lin & 7) * 4;
    *p = (*p & ~(15u << s)) | (v << s);
  }
  // Movelist as a window over a deeper stack: entries lo .. sp-1 (the top, where every push and
  // pop happens) in a shared-memory ring of mask+1 slots, entries 0 .. lo-1 in the global spill.
  // A push that overflows the ring evicts its bottom entry (a store, off the critical path); a pop
  // that leaves fewer than two ring entries above spilled ones refills up to four of them (loads
  // issued a pop ahead of their use).  So pops never wait on the spill, however deep the stack.
  // (a = 3 keeps a linear stack: its dense board leaves ~54 shared slots, deeper stacks are rare)
  __device__ __forceinline__ uint32_t pop(int &sp, int &lo) const {
    if (!RING) {
      --sp;
      return sp < mask ? sw[sp * 32] : spill[(int64_t)sp * 32];
    }
    const uint32_t e = sw[((--sp) & mask) * 32];
    if (sp - lo < 2 && lo > 0) {
      const int n = min(lo, 4);
      for (int i = 0; i < n; i++) {
        --lo;
        sw[(lo & mask) * 32] = spill[(int64_t)lo * 32];
      }
    }
    return e;
  }
  __device__ __forceinline__ void push(int &sp, int &lo, uint32_t e) const {
    if (!RING) {
      if (sp < mask) sw[sp * 32] = (uint16_t)e;
      else spill[(int64_t)sp * 32] = (uint16_t)e;
      ++sp;
      return;
    }
    if (sp - lo > mask) {  // ring full: the bottom entry moves to the spill
      spill[(int64_t)lo * 32] = sw[(lo & mask) * 32];
      ++lo;
    }
    sw[(sp & mask) * 32] = (uint16_t)e;
    ++sp;
  }
};

// ---- candidate tables -------------------------------------------------------
template <int A, bool STRICT> struct Cand;

// SWAR over NC nibble lanes (NC = 4a; a <= 2 fits 32-bit masks, a == 3 64-bit):
// E[dir] holds every candidate's dir-face label, P[dir] its partner
// (partner(0) := 0xF, never a label), so "candidate c bonds the neighbour's
// label p" is the nibble equality P[dir][c] == p (p = 0 never matches);
// CLS holds each candidate's equivalence-class id (in-situ 4-label code).
template <typename M, int NC, bool STRICT> struct CandSwar {
  M E0, E1, E2, E3, P0, P1, P2, P3, N0, N1, N2, N3, CLS;
  static constexpr M VALID = (M)(0x8888888888888888ULL >> (64 - 4 * NC));


  // face labels and partners of every candidate (E, P); build() adds the rest.
  // Candidate (t, r) shows lab[4t + ((k - r) & 3)] on side k, so tile t's 16-bit chunk of
  // E3 is its labels nibble-reversed (rev = L3 L2 L1 L0, nibble 0 first) and E0 / E1 / E2
  // are rev rotated left by 1 / 2 / 3 nibbles.  Partners ((e - 1) ^ 1) + 1, 0 -> 15, in SWAR
  // (labels <= 7 on this path: no borrow or carry crosses a nibble).
  __device__ __forceinline__ void build_faces(const uint32_t *lab) {
    E0 = E1 = E2 = E3 = 0;
#pragma unroll
    for (int t = 0; t < NC / 4; t++) {
      const uint32_t rev = lab[4 * t + 3] | (lab[4 * t + 2] << 4) | (lab[4 * t + 1] << 8) | (lab[4 * t] << 12);
      const uint32_t dup = rev | (rev << 16);
      E0 |= (M)((dup >> 12) & 0xFFFFu) << (16 * t); E1 |= (M)((dup >> 8) & 0xFFFFu) << (16 * t);
      E2 |= (M)((dup >> 4) & 0xFFFFu) << (16 * t); E3 |= (M)rev << (16 * t);
    }
    P0 = partners(E0); P1 = partners(E1); P2 = partners(E2); P3 = partners(E3);
  }
  __device__ __forceinline__ static M partners(M x) {
    constexpr M ONES = VALID >> 3;                   // 0x11..1 over the NC candidate nibbles
    const M z = (~nz_nib<M>(x) & VALID) >> 3;        // 1 in every zero nibble
    const M x1 = x | z;                              // zero nibbles -> 1 (no borrow below)
    return ((((x1 - ONES) ^ ONES) + ONES) | (z * (M)15));
  }

  __device__ __forceinline__ void build(const uint32_t *lab, int ntiles) {
    build_faces(lab);
    // equivalence-class id = lowest candidate with the same in-situ code (_k:199).  Candidate
    // (t, r) has code rotl16(X_t, 4r), X_t = L0 | L1 << 4 | L2 << 8 | L3 << 12, so inside a tile
    // the ids repeat with the tile's rotational period, and tile t2's rotations map onto those
    // of the first earlier tile t1 with X_t2 = rotl16(X_t1, 4s): code(t2, r) = code(t1, r + s).
    constexpr int T = NC / 4;
    uint32_t X[T], id[NC];
#pragma unroll
    for (int t = 0; t < T; t++) {
      X[t] = lab[4 * t] | (lab[4 * t + 1] << 4) | (lab[4 * t + 2] << 8) | (lab[4 * t + 3] << 12);
      const uint32_t dup = X[t] | (X[t] << 16);
      const uint32_t m = t >= ntiles ? 3u  // absent tiles: unique ids, never equal to anything
                         : ((dup >> 12) & 0xFFFFu) == X[t] ? 0u : ((dup >> 8) & 0xFFFFu) == X[t] ? 1u : 3u;
#pragma unroll
      for (int r = 0; r < 4; r++) id[4 * t + r] = (uint32_t)(4 * t) + ((uint32_t)r & m);
    }
#pragma unroll
    for (int t2 = 1; t2 < T; t2++) {
      bool matched = t2 >= ntiles;
#pragma unroll
      for (int t1 = 0; t1 < t2; t1++) {
        const uint32_t dup = X[t1] | (X[t1] << 16);
#pragma unroll
        for (int sft = 0; sft < 4; sft++) {
          const uint32_t rot = sft ? (dup >> (16 - 4 * sft)) & 0xFFFFu : X[t1];
          const bool hit = !matched && rot == X[t2];
#pragma unroll
          for (int r = 0; r < 4; r++) id[4 * t2 + r] = hit ? id[4 * t1 + ((r + sft) & 3)] : id[4 * t2 + r];
          matched = matched || hit;
        }
      }
    }
    CLS = 0;
#pragma unroll
    for (int c = 0; c < NC; c++) CLS |= (M)id[c] << (4 * c);
    N0 = nz_nib<M>(E0) & VALID; N1 = nz_nib<M>(E1) & VALID;
    N2 = nz_nib<M>(E2) & VALID; N3 = nz_nib<M>(E3) & VALID;
  }

  // candidates at a cell whose N,E,S,W neighbours hold board values vN..vW, passed as 4 v
  // (>= NC: empty, shows no label); strict: a nonzero face against a nonzero
  // non-partner label excludes the candidate (_k:176-198)
  __device__ __forceinline__ M cand(uint32_t sN, uint32_t sE, uint32_t sS, uint32_t sW) const {
    // board values are < 16; nibbles >= NC of the zero-extended tables are 0, so an empty
    // neighbour (0xE / 0xF) reads label 0 without a compare
    const uint32_t pN = (uint32_t)(((uint64_t)E2 >> sN) & 15u);
    const uint32_t pE = (uint32_t)(((uint64_t)E3 >> sE) & 15u);
    const uint32_t pS = (uint32_t)(((uint64_t)E0 >> sS) & 15u);
    const uint32_t pW = (uint32_t)(((uint64_t)E1 >> sW) & 15u);
    M bond = 0, conf = 0;
#define TV_DIR(Pd, Nd, p)                                                    \
  {                                                                          \
    const M x = (Pd) ^ rep_nib<M>(p);                                        \
    const M bm = ~nz_nib<M>(x) & VALID; /* nibble == 0 */                    \
    bond |= bm;                                                              \
    if (STRICT) conf |= (p) ? ((Nd) & ~bm) : (M)0;                           \
  }
    TV_DIR(P0, N0, pN)
    TV_DIR(P1, N1, pE)
    TV_DIR(P2, N2, pS)
    TV_DIR(P3, N3, pW)
#undef TV_DIR
    return STRICT ? (bond & ~conf) : bond;
  }
  __device__ __forceinline__ uint32_t first(M cand) const { return (uint32_t)ffs_m(cand) >> 2; }
  __device__ __forceinline__ bool ambiguous(M cand, uint32_t cf) const {
    return (nz_nib<M>(CLS ^ rep_nib<M>(get_nib<M>(CLS, cf))) & cand) != 0;
  }

  // Locally-forced check for one placed tile (candidate v) of a finished BOUNDED assembly:
  // the candidates that bond v's face toward its neighbour cell q (a one-neighbour context,
  // no strict conflict possible) must all have q's in-situ code (q occupied, value qv < NC)
  // or not exist (q empty).  Sides j = N, E, S, W of v; q sees v from side (j + 2) & 3.
  __device__ __forceinline__ bool forced_at(uint32_t v, uint32_t qN, uint32_t qE, uint32_t qS, uint32_t qW) const {
    const M H0 = eqn(P2, get_nib<M>(E0, v)), H1 = eqn(P3, get_nib<M>(E1, v));
    const M H2 = eqn(P0, get_nib<M>(E2, v)), H3 = eqn(P1, get_nib<M>(E3, v));
    const bool o0 = qN < NC ? !ambiguous(H0, qN) : H0 == 0, o1 = qE < NC ? !ambiguous(H1, qE) : H1 == 0;
    const bool o2 = qS < NC ? !ambiguous(H2, qS) : H2 == 0, o3 = qW < NC ? !ambiguous(H3, qW) : H3 == 0;
    return o0 && o1 && o2 && o3;
  }

  // nibble c of X equals v -> bit 4c+3
  __device__ __forceinline__ static M eqn(M X, uint32_t v) { return ~nz_nib<M>(X ^ rep_nib<M>(v)) & VALID; }

  // Static proof that no run of this genome can end TRIVIAL (early unbound
  // cut-off).  Over-approximates what a popped cell can
  // see: S[k] = labels a placed tile can show toward a popped cell from side k,
  // bond[c] = sides through which candidate c bonds a label of S.  A placed tile
  // never shows a label toward a popped cell through a side it bonded at
  // placement (that neighbour was occupied then, and cells never empty again),
  // so candidate c contributes its face f = (k+2)&3 to S[k] only if it can bond
  // through some side other than f; the seed (no bonded side) shows all four
  // faces.  S and bond grow to a joint fixpoint.  A context = at most one label
  // of S[k] per side k (empty sides are always compatible).  A TRIVIAL needs two
  // hits with different in-situ codes in one context (_k:199-209): pair (c1, c2)
  // can co-hit iff one side bonds both (same partner label), or two different
  // sides bond one each while the other candidate tolerates that label (strict:
  // its face there is 0 or bonds it, _k:176-198).  No such pair -> TRIVIAL is
  // impossible.  (Checked against the oracle on all of S_{2,8}: no genome it
  // proves goes TRIVIAL; tools/work_analysis.c.)
  //
  // Byte-SWAR over the four sides (byte k <-> side k): S = labels shown from each side (bit
  // per label), PM[c] = c's partner label per side (one-hot; faces 0 and 7 bond nothing),
  // FM[c] = the label c shows, as a tile at side k of a popped cell, toward that cell (its
  // face (k+2)&3), FC[c] = c's four faces.  ~10 int ops per candidate per
  // fixpoint round; the pair test compares byte-packed faces (equal faces <=> equal
  // in-situ codes, and <=> equal partners since the partner map is injective).
  __device__ __forceinline__ static uint32_t nz_byte(uint32_t x) {  // bit 8k+7 set iff byte k != 0
    return (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
  }
  __device__ __forceinline__ bool trivial_free() const {
    uint32_t PM[NC], FM[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) {
      const uint32_t e0 = get_nib<M>(E0, c), e1 = get_nib<M>(E1, c), e2 = get_nib<M>(E2, c), e3 = get_nib<M>(E3, c);
      FM[c] = (1u << e2) | ((1u << e3) << 8) | ((1u << e0) << 16) | ((1u << e1) << 24);
      PM[c] = ((1u << get_nib<M>(P0, c)) & 0xFEu) | (((1u << get_nib<M>(P1, c)) & 0xFEu) << 8) |
              (((1u << get_nib<M>(P2, c)) & 0xFEu) << 16) | (((1u << get_nib<M>(P3, c)) & 0xFEu) << 24);
    }
    uint32_t S = FM[0];  // the seed (no bonded side) shows all four faces
#pragma unroll 1
    for (int it = 0; it < 32; it++) {  // in-place (Gauss-Seidel) rounds: S only grows, so any order
      const uint32_t S0 = S;           // reaches the same least fixpoint, in fewer rounds
#pragma unroll
      for (int c = 0; c < NC; c++) {
        // T: sides through which c can bond (bit 7 of byte j); c shows its face toward side k' iff
        // it bonds through a side other than the opposite one, (k'+2)&3: OR of T's bytes k'-1,
        // k', k'+1 = T | rotl8(T) | rotr8(T), spread to whole bytes
        const uint32_t T = nz_byte(PM[c] & S);
        const uint32_t A = T | __funnelshift_l(T, T, 8) | __funnelshift_r(T, T, 8);
        S |= FM[c] & ((A >> 7) * 0xFFu);
      }
      if (S == S0) break;
    }
    // pair test, SWAR over c2 for each c1 (nibble flags bit 4c+3): BK[k] = candidates that
    // bond through side k, ZK[k] = zero face at side k, SK = same face as c1 at side k
    M BK[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < NC; c++) {
      const uint32_t b = nz_byte(PM[c] & S);
#pragma unroll
      for (int k = 0; k < 4; k++) BK[k] |= (M)((b >> (8 * k + 7)) & 1u) << (4 * c + 3);
    }
    const M E[4] = {E0, E1, E2, E3};
    M bad = 0;
#pragma unroll
    for (int c1 = 0; c1 < NC; c1++) {
      M SK[4], A = 0, tol2 = 0, bnd2 = 0;
      uint32_t nb1 = 0;  // sides c1 bonds through (bit k)
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t ek = get_nib<M>(E[k], c1);
        SK[k] = eqn(E[k], ek);
        const bool b1k = ((BK[k] >> (4 * c1 + 3)) & 1u) != 0;
        nb1 |= (uint32_t)b1k << k;
        A |= b1k ? SK[k] : (M)0;                               // one side bonds both
        if (STRICT) {
          tol2 |= b1k ? (SK[k] | (~nz_nib<M>(E[k]) & VALID)) : (M)0;  // c2 tolerates c1's bond side
          bnd2 |= BK[k] & (ek == 0u ? VALID : SK[k]);         // c2 bonds where c1 tolerates
        }
      }
      if (!STRICT) {  // c1 bonds k1, c2 bonds some k2 != k1 (no tolerance needed)
        const bool single = (nb1 & (nb1 - 1u)) == 0u;
        M other = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) other |= (single && ((nb1 >> k) & 1u)) ? (M)0 : BK[k];
        tol2 = nb1 ? VALID : (M)0;
        bnd2 = other;
      }
      const M differ = ~(SK[0] & SK[1] & SK[2] & SK[3]) & VALID;  // different in-situ code
      bad |= (A | (tol2 & bnd2)) & differ;
    }
    const bool ok = bad == 0;
    return ok;
  }
};
template <bool S> struct Cand<3, S> : CandSwar<uint64_t, 12, S> {};
template <bool S> struct Cand<2, S> : CandSwar<uint32_t, 8, S> {};
template <bool S> struct Cand<1, S> : CandSwar<uint32_t, 8, S> {};

enum { ST_NEED = 0, ST_RUN = 1, ST_DONE = 2 };

// board layout of the fast kernel: row-aligned (a <= 2) or dense (a = 3), see k_classify_fast
#ifndef TV_A3_ROWS
#define TV_A3_ROWS 0  // a = 3 on the row-aligned board with the movelist ring too (A/B)
#endif
#ifndef TV_H2_LAZY
#define TV_H2_LAZY 1  // the second Fisher-Yates draw only for m == 3 (S28 -0.9 %, S32 -1.1 %; 0 = both always)
#endif
#ifndef TV_A3_RING
#define TV_A3_RING 0  // a = 3 dense board with the movelist ring (A/B)
#endif
template <int A> __host__ __device__ constexpr bool fast_rows() { return A <= 2 || TV_A3_ROWS; }
template <int A> __host__ __device__ constexpr bool fast_ring() { return fast_rows<A>() || TV_A3_RING; }
__host__ __device__ inline int fast_board_words(int a, int d) {
  const int PD = d + 2;
  return (a <= 2 || TV_A3_ROWS) ? PD * ((PD + 7) / 8) : (PD * PD + 7) / 8;
}

#define TV_KEY_BITS 11  // width of the k_prepass behaviour key

#ifndef TV_PREPASS_MINB
#define TV_PREPASS_MINB 2  // k_prepass at <= 128 registers (2 CTAs of 256 per SM; the fixpoint proof spills at 80)
#endif
#ifndef TV_FAST_MINB
#define TV_FAST_MINB 2
#endif
#ifndef TV_FAST_MAXT
#define TV_FAST_MAXT 384  // 2 x 384 lanes per SM: 24 warps at <= 80 registers (measured +10% vs 2 x 256)
#endif
#ifndef TV_FAST_MAXT3
#define TV_FAST_MAXT3 352  // a = 3: 2 x 352 lanes at <= 80 registers (round 2: S32 block 22.07 -> 21.44 ms vs 2 x 320 at 96)
#endif
template <int A> constexpr int fast_threads() { return A == 3 ? TV_FAST_MAXT3 : TV_FAST_MAXT; }

// MODE (compile time, so each variant carries only its own service code): 0 histogram,
// 1 classify_batch rows, 2 GA fitness, 3 representative payloads (HIST / fit_mode / pay_mode)
enum { FM_HIST = 0, FM_ROWS = 1, FM_FIT = 2, FM_PAY = 3 };

// D > 0: the grid dimension as a compile-time constant (board geometry folds into immediates);
// D = 0: P.d at run time.
template <int A, bool STRICT, int MODE, int D = 0>
__global__ void __launch_bounds__(fast_threads<A>(), TV_FAST_MINB) k_classify_fast(const __grid_constant__ ClassifyParams P) {
  constexpr int NC = 4 * A;
  const int GW = D ? fast_board_words(A, D) : P.GW;
  constexpr bool HIST = MODE == FM_HIST, FIT = MODE == FM_FIT, PAY = MODE == FM_PAY;
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int words_per_warp = (GW + P.S / 2) * 32;
  FastLane<fast_ring<A>()> Ln;  // a <= 2: movelist ring; a = 3: linear stack (TV_A3_RING: ring)
  Ln.gw = smem + warp * words_per_warp + lane;
  Ln.sw = reinterpret_cast<uint16_t *>(smem + warp * words_per_warp + GW * 32) + lane;
  Ln.mask = fast_ring<A>() ? P.S - 1 : P.S;  // ring: the host sizes it as a power of two
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
  if (HIST) {
    for (int s = threadIdx.x; s < HS; s += blockDim.x) {
      c_key[s] = 0ULL; c_rdet[s] = ~0ULL; c_rany[s] = ~0ULL; c_det[s] = 0; c_ste[s] = 0; c_gs[s] = -1;
    }
    for (int s = threadIdx.x; s < P.q * 5; s += blockDim.x) c_tal[s] = 0;
  }
  for (int w = 0; w < GW; w++) Ln.gw[w * 32] = 0xFFFFFFFFu;
  __syncthreads();

  // board row stride RS nibbles, cell (r, c) = nibble lin = r RS + c.  a <= 2: rows of RW whole
  // words (RS = 8 RW >= d + 2), so the N and S neighbours sit RW words above / below in the same
  // nibble position; a = 3: RS = d + 2 (dense; its service passes scan and clear fewer words)
  constexpr bool ROWS = fast_rows<A>();
  const int d = D ? D : P.d, dd = d * d, RW = (d + 2 + 7) >> 3, RS = ROWS ? 8 * RW : d + 2;
  const uint32_t magic = (uint32_t)(0x100000000ULL / (uint64_t)RS) + 1u;
  const int cr = (d >> 1) + 1, centre = cr * RS + cr;
  const int thresh = P.service_thresh > 0 ? P.service_thresh : 16;

  const int64_t n_run = P.n - (P.n_skip ? (int64_t)*P.n_skip : 0);  // 1-mers classified by k_prepass
  int st = ST_NEED, pend = -1;
  int64_t item = 0;
  uint64_t idx = 0, rs = 0;
  int run = 0, replay = 0, sp = 0, lo = 0;  // movelist: sp entries, the lowest lo of them spilled
  int minr = 0, maxr = 0, minc = 0, maxc = 0;
  int trivial_at = -1, first_unbound = -1, first_mismatch = -1;
  uint32_t hash0 = 0, best = 0, fit0 = 0;
  int64_t pslot = -1;  // histogram slot whose payload the claiming genome's replay writes
  bool tfree = false;  // no run of this genome can go TRIVIAL (k_prepass)
  Cand<A, STRICT> K;

  if (P.prof_t && threadIdx.x == 0) atomicMin(&P.prof_t[0], fast_clock());
  // lanes not DONE (warp-uniform; lanes only finish in the refill below) and the parked-lane
  // count that triggers a service pass: min(thresh, half the live lanes), so never above nlive
  int nlive = 32, trig = min(thresh, 16);
  for (;;) {
    const unsigned parked = __ballot_sync(0xFFFFFFFFu, st == ST_NEED || pend >= 0);
    if (__popc(parked) >= trig) {
      // =================== service pass over parked lanes ===================
      bool start = false;
      if (pend >= 0) {
        const int ended = pend;
        pend = -1;
        // hash (+ pack on replay) the bounded shape before clearing (_k:260-292)
        uint32_t hs = 0;
        int w = 0, h = 0, n = 0, ov = 0;
        const bool fit_scan = FIT && !replay && run == 0;  // overlap with the GA target shape
        // run 0 of a genome: is its assembly locally forced (every run must reproduce it)?
        bool forced = P.forced_check && (P.forced_check == 1 || tfree) && !replay && !PAY && run == 0;
        if (ended == RUN_BOUNDED) {
          unsigned long long *out = nullptr;
          int64_t W = 0;
          if (replay || PAY) {
            out = HIST ? P.hist.shape + pslot * P.hist.W : P.out_shape + item * P.W;
            W = HIST ? P.hist.W : P.W;
          }
          w = maxc - minc + 1;
          h = maxr - minr + 1;
          hs = oat_step(oat_step(0u, (uint32_t)w), (uint32_t)h);
          const int lo = (minr * RS + minc) >> 3, hi = (maxr * RS + maxc) >> 3;
          int64_t cw = 0;
          unsigned long long acc = 0;
          for (int wi = lo; wi <= hi; wi++) {
            uint32_t occ = nz_nib<uint32_t>(~Ln.gw[wi * 32]);
            while (occ) {
              const int b = __ffs(occ) - 1;
              occ &= occ - 1;
              const uint32_t L = (uint32_t)(wi * 8 + (b >> 2));
              const uint32_t R = __umulhi(L, magic);
              const int col = (int)(L - R * RS);
              const int y = (int)R - minr, x = col - minc;
              hs = oat_step(oat_step(hs, (uint32_t)x), (uint32_t)y);
              n++;
              if (forced)
                forced = K.forced_at((Ln.gw[wi * 32] >> (b & ~3)) & 15u, Ln.nib((int)L - RS), Ln.nib((int)L + 1),
                                     Ln.nib((int)L + RS), Ln.nib((int)L - 1));
              if (fit_scan) ov += (P.target_rows[R] >> col) & 1u;
              if (out) {
                const int bit = y * w + x;
                const int64_t wj = bit >> 6;
                if (wj < W) {  // bits past the caller's W words are dropped
                  while (cw < wj) { out[cw++] = acc; acc = 0; }
                  acc |= 1ULL << (bit & 63);
                }
              }
            }
          }
          if (out) { while (cw < W) { out[cw++] = acc; acc = 0; } }
          hs = oat_final(hs);
        }
        {  // clear: every tile and movelist mark lies inside bbox +- 1
          const int lo = ((minr - 1) * RS + (minc - 1)) >> 3;
          const int hi = ((maxr + 1) * RS + (maxc + 1)) >> 3;
          for (int wi = lo; wi <= hi; wi++) Ln.gw[wi * 32] = 0xFFFFFFFFu;
        }
        if (replay) {
          if (!HIST) {
            P.out_hash[item] = best;
            P.out_w[item] = (uint8_t)w; P.out_h[item] = (uint8_t)h; P.out_cells[item] = (uint16_t)n;
          } else {  // the genome that claimed the key provides its payload (fixed at export
                    // if a lower-index genome carries the same key, tv_hist.cuh)
            P.hist.whc[pslot] = (uint32_t)w | ((uint32_t)h << 8) | ((uint32_t)n << 16);
            P.hist.pay_idx[pslot] = idx;
          }
          st = ST_NEED;
        } else if (PAY) {  // representative payload: does this run reproduce the key?
          const uint32_t key = P.pay_key[item >> P.pay_shift];
          if (ended == RUN_BOUNDED && hs == key) {
            P.out_hash[item] = hs;
            P.out_w[item] = (uint8_t)w; P.out_h[item] = (uint8_t)h; P.out_cells[item] = (uint16_t)n;
          } else {
            P.out_hash[item] = ~key;
          }
          st = ST_NEED;
        } else {
          // ---- fold one run (_k:323-349)
          bool done = false;
          if (ended == RUN_BOUNDED) {
            rh[run * 32] = hs;
            if (run == 0) {
              hash0 = hs; fit0 = (uint32_t)n | ((uint32_t)ov << 16);
              // locally forced: every later run assembles the same shape BOUNDED, so the
              // genome is DET at every k with this hash
              if (forced) done = true;
            }
            else if (first_mismatch < 0 && first_unbound != 0 && hs != hash0) first_mismatch = run;
            if (FIT && first_mismatch >= 0) done = true;  // not DET: fitness 0 whatever follows
          } else if (ended == RUN_UNBOUND) {
            rh[run * 32] = 0u;
            if (first_unbound < 0) {
              first_unbound = run;
              // early unbound cut-off: every prefix k' > run is now UNBOUND unless a
              // later run goes TRIVIAL, which the genome's flag proves impossible
              if (tfree) done = true;
            }
            if (FIT) done = true;  // not DET: fitness 0 whatever follows
          } else {
            done = true;
            if (ended == RUN_TRIVIAL) trivial_at = run;
          }
          run++;
          if (!done && run < P.kmax) {
            start = true;
          } else if (FIT) {  // GA JaTAM-shape fitness: d^2 - shapediff for DET, else 0
            const int hc = ended == RUN_OVERFLOW ? CLS_ERROR : class_at(P.hist_k, trivial_at, first_unbound, first_mismatch);
            const int diff = P.target_cells + (int)(fit0 & 0xFFFFu) - 2 * (int)(fit0 >> 16);
            const uint32_t fit = hc == CLS_DET ? (uint32_t)(dd - diff) : 0u;
            P.out_fit[item] = fit;
            if (P.memo_mask) memo_put(P, idx, fit);
            st = ST_NEED;
          } else if (ended == RUN_OVERFLOW) {  // _k:434-437
            if (!HIST) {
              for (int k = 0; k < P.q; k++) P.out_class[item * P.q + k] = (uint8_t)CLS_ERROR;
            } else {
              for (int k = 0; k < P.q; k++) atomicAdd(&c_tal[k * 5 + 4], 1u);
            }
            st = ST_NEED;
          } else {
            // ---- genome fold (_k:351-381, _k:438-452)
            if (!HIST) {
              for (int k = 0; k < P.q; k++)
                P.out_class[item * P.q + k] = (uint8_t)class_at(P.ks[k], trivial_at, first_unbound, first_mismatch);
            } else {
              for (int k = 0; k < P.q; k++)
                atomicAdd(&c_tal[k * 5 + class_at(P.ks[k], trivial_at, first_unbound, first_mismatch)], 1u);
            }
            const int hc = class_at(P.hist_k, trivial_at, first_unbound, first_mismatch);
            st = ST_NEED;
            if (hc == CLS_DET || hc == CLS_STERIC) {
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
              if (HIST) {
                const bool det = hc == CLS_DET;
                bool gnew = false, cached = false;
                int64_t g = -1;
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
                      if (det && c_rdet[s] > idx) atomicMin(&c_rdet[s], (unsigned long long)idx);
                      if (c_rany[s] > idx) atomicMin(&c_rany[s], (unsigned long long)idx);
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
              if (need_payload) {  // replay the attributed run to emit its bitmap
                replay = 1;
                run = attr;
                start = true;
                st = ST_RUN;
              }
            } else if (!HIST) {
              P.out_hash[item] = 0u; P.out_w[item] = 0; P.out_h[item] = 0; P.out_cells[item] = 0;
            }
          }
        }
      }
      // ---- refill lanes that need a genome (warp-aggregated work counter)
      const unsigned need = __ballot_sync(0xFFFFFFFFu, st == ST_NEED);
      if (need) {
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(P.work, (unsigned long long)__popc(need));
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        if (st == ST_NEED) {
          item = (int64_t)base + __popc(need & ((1u << lane) - 1u));
          if (item >= n_run) {
            st = ST_DONE;
            if (P.prof_t) atomicMin(&P.prof_t[1], fast_clock());
          } else {
            // behaviour-sorted processing order (k_prepass); every per-item output and flag below
            // is addressed by the item's own number, so the order is invisible to the caller
            bool tf = false;  // trivial-freedom bit (k_prepass): bit 31 of the order entry or a flag
            if (P.order) {
              const uint32_t o = P.order[item];
              item = (int64_t)(o & 0x7FFFFFFFu);
              tf = (o >> 31) != 0u;
            } else if (P.tf_flags) {
              tf = ((P.tf_flags[item >> 5] >> (item & 31)) & 1u) != 0u;
            }
            const int64_t rec = item >> P.pay_shift;  // payload mode: item = (record, run)
            idx = item_index(P.indices, P.start, P.chunk, P.stride, P.item0 + rec);
            uint32_t lab[12];  // decode labels (_k:384-401)
#pragma unroll
            for (int te = 0; te < 12; te++) lab[te] = te < NC ? decode_label(P.dec, te, idx) : 0u;
            K.build(lab, A);
            tfree = tf;
            trivial_at = first_unbound = first_mismatch = -1;
            run = (int)item & ((1 << P.pay_shift) - 1);
            replay = 0;
            start = true;
            st = ST_RUN;
          }
        }
      }
      if (start) {  // ---- run start: seed + shuffled centre neighbours (_k:110-136)
        rs = stream_state(P.seed, idx, (uint64_t)run);
        Ln.set_nib(centre, 0u);
        minr = maxr = minc = maxc = cr;
        uint32_t nbp = 0x03020100u;
#pragma unroll
        for (int j = 3; j > 0; j--) {
          const uint32_t q = rng_below(rs, (uint32_t)(j + 1));
          const uint32_t x = ((nbp >> (8 * j)) ^ (nbp >> (8 * q))) & 0xFFu;
          nbp ^= (x << (8 * j)) | (x << (8 * q));
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t dir = (nbp >> (8 * j)) & 3u;
          const int dl = (dir & 1u) ? 1 : RS;
          const int nl = ((dir + 1u) & 2u) ? centre + dl : centre - dl;
          Ln.sw[j * 32] = (uint16_t)nl;  // ring slots 0..3 (the ring has >= 4 slots)
          Ln.set_nib(nl, 0xEu);
        }
        sp = 4;
        lo = 0;
      }
      nlive = __popc(__ballot_sync(0xFFFFFFFFu, st != ST_DONE));
      if (nlive == 0) break;
      trig = min(thresh, (nlive + 1) >> 1);
    }
    if (st != ST_RUN || pend >= 0) continue;

    // =================== one movelist pop (_k:138-248) ===================
    const int lin = (int)Ln.pop(sp, lo);
    uint32_t *const pw = Ln.gw + (lin >> 3) * 32;  // the popped cell's word
    const int sh = (lin & 7) * 4;
    // neighbour values times 4 (0x3C = empty), each one rotate of its word: nibble at bit p
    // lands at bits 2..5 after a right rotate by p - 2
    uint32_t vN, vS, vE, vW;
    if (ROWS) {  // W / E from the own word or its neighbour word (a row never ends mid-word)
      const uint32_t wm = pw[-32], w0 = pw[0], wp = pw[32];
      vN = __funnelshift_r(pw[-RW * 32], pw[-RW * 32], (sh - 2) & 31) & 0x3Cu;
      vS = __funnelshift_r(pw[RW * 32], pw[RW * 32], (sh - 2) & 31) & 0x3Cu;
      const uint32_t ww = sh ? w0 : wm, we = sh == 28 ? wp : w0;
      vW = __funnelshift_r(ww, ww, (sh - 6) & 31) & 0x3Cu;
      vE = __funnelshift_r(we, we, (sh + 2) & 31) & 0x3Cu;
    } else {
      vN = 4 * Ln.nib(lin - RS); vS = 4 * Ln.nib(lin + RS);
      vE = 4 * Ln.nib(lin + 1); vW = 4 * Ln.nib(lin - 1);
    }
    const auto cand = K.cand(vN, vE, vS, vW);
    const uint32_t cf = K.first(cand);
    const int r = (int)__umulhi((uint32_t)lin, magic), c = lin - r * RS;
    bool place = false;
    if (cand != 0) {
      if (K.ambiguous(cand, cf)) pend = RUN_TRIVIAL;                           // _k:208-209
      else if (r == 1 || c == 1 || r == d || c == d) pend = RUN_UNBOUND;     // _k:212-213
      else place = true;
    }
    // a popped cell always holds 0xE (on the movelist), so one XOR writes the placed
    // candidate or 0xF (drop, re-pushable, _k:210-211); the word is lane-private
    atomicXor(pw, (0xEu ^ (place ? cf : 0xFu)) << sh);
    if (!place) {
      if (pend < 0 && sp == 0) pend = RUN_BOUNDED;  // movelist exhausted (_k:138, 249)
      continue;
    }
    minr = min(minr, r); maxr = max(maxr, r);                                 // _k:217-224
    minc = min(minc, c); maxc = max(maxc, c);
    // new frontier N,E,S,W (_k:225-237) as cell offsets + 128, one per byte (RS < 128)
    uint32_t nbp = 0;
    int m = 0;
    if (vN == 0x3Cu) { nbp |= (uint32_t)(128 - RS) << (8 * m); m++; }
    if (vE == 0x3Cu) { nbp |= 129u << (8 * m); m++; }
    if (vS == 0x3Cu) { nbp |= (uint32_t)(128 + RS) << (8 * m); m++; }
    if (vW == 0x3Cu) { nbp |= 127u << (8 * m); m++; }
    if (m >= 2) {  // Fisher-Yates (_k:238-242): both draws of m == 3 mixed side by side
      const bool three = m == 3;
#if TV_H2_LAZY
      const uint32_t h1 = rng_hi(rs + kGold), h2 = three ? rng_hi(rs + 2 * kGold) : 0u;
#else
      const uint32_t h1 = rng_hi(rs + kGold), h2 = rng_hi(rs + 2 * kGold);
#endif
      rs += three ? 2 * kGold : kGold;
      const uint32_t q3 = three ? __umulhi(h1, 3u) : 2u;  // m == 2: swap 2 with itself
      uint32_t x = ((nbp >> 16) ^ (nbp >> (8 * q3))) & 0xFFu;
      nbp ^= (x << 16) | (x << (8 * q3));
      const uint32_t q2 = (three ? h2 : h1) >> 31;  // below(2) = high bit
      x = ((nbp >> 8) ^ (nbp >> (8 * q2))) & 0xFFu;
      nbp ^= (x << 8) | (x << (8 * q2));
    }
    const int mm = min(m, dd - sp);  // capacity check before each push (_k:243-245)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      if (j < mm) {
        const int nl = lin + (int)((nbp >> (8 * j)) & 0xFFu) - 128;
        Ln.push(sp, lo, (uint32_t)nl);
        atomicAnd(&Ln.gw[(nl >> 3) * 32], ~(1u << ((nl & 7) * 4)));  // F -> E (one ATOMS, lane-private word)
      }
    }
    if (mm < m) pend = RUN_OVERFLOW;
    else if (sp == 0) pend = RUN_BOUNDED;
  }

  if (P.prof_t) atomicMax(&P.prof_t[2], fast_clock());
  if (HIST) {
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

// Pre-pass over the work items (full SIMT: every lane runs the same straight-line
// code), two optional products:
//  * flags: trivial-freedom bits for the early unbound cut-off, bit (i & 31) of
//    flags[i >> 5] for work item i (CandSwar::trivial_free);
//  * key: an 11-bit behaviour key per genome (the lowest bit: trivial freedom); the
//    items are counting-sorted by it (k_key_* below), so (1) line-prone genomes (a tile bonds a copy of itself
//    through opposite faces: long UNBOUND runs -- in S_{2,8} 33 % of the genomes,
//    45 % of the pops, 98 % of the slowest 0.1 %) run first and the kernel's tail
//    is made of short genomes, and (2) the lanes of a warp hold genomes of the same
//    structure (seed self-bonding, bondable faces of the seed, other tiles
//    self-bonding, their bondable faces), whose runs have similar lengths and
//    outcomes: fewer idle lanes.
//    Results cannot depend on the order (per-genome substreams, commutative
//    histogram updates).
//  * 1-mers (with key): a genome whose seed faces bond no label of the genome gets
//    no hit at any centre neighbour, so every run drops the four and ends BOUNDED
//    with the 1x1 shape (_k:138-249): DET at every k, hash 0x3a9be4cf.  When
//    n_skip is given the pre-pass classifies these itself (histogram: tallies,
//    counts, representatives, payload; classify mode: the output rows), gives
//    them the largest key so they sort to the end of the order, and counts them
//    in *n_skip; k_classify_fast stops at n - *n_skip.
constexpr uint32_t kOneMerHash = 0x3a9be4cfu;  // OAT of (w, h, x, y) = (1, 1, 0, 0), _k:260-277
constexpr uint16_t kOneMerKey = (1u << TV_KEY_BITS) - 1u;

//  * work order (with key): the items are counting-sorted by key (k_key_binscan / _basescan /
//    _scatter below, no library sort): CTA b handles the tile of items [b TILE, (b+1) TILE) and
//    writes the tile's key histogram to tile_hist[key * ntiles + b].
constexpr int kNumKeys = 1 << TV_KEY_BITS;
// items per pre-pass / scatter CTA: a multiple of 32, sized by the host so that even small
// launches get a few CTAs per SM (key_tile_for)
inline int64_t key_tile_for(int64_t n, int nsm) {
  int64_t t = (n + 4 * (int64_t)nsm - 1) / (4 * (int64_t)nsm);
  t = (t + 31) / 32 * 32;
  return t < 1024 ? 1024 : t;
}

template <int A, bool STRICT>
__global__ void __launch_bounds__(256, TV_PREPASS_MINB) k_prepass(const __grid_constant__ ClassifyParams P, uint32_t *flags,
                                                 uint16_t *key_out, uint32_t *iota_out,
                                                 unsigned long long *n_skip, uint32_t *tile_hist, int64_t ntiles,
                                                 int64_t tile) {
  constexpr int NC = 4 * A;
  const int lane = threadIdx.x & 31;
  __shared__ unsigned long long s_om_min;
  __shared__ unsigned int s_om_cnt;
  __shared__ uint32_t s_hist[kNumKeys];
  if (threadIdx.x == 0) { s_om_min = ~0ULL; s_om_cnt = 0u; }
  if (tile_hist)
    for (int b = threadIdx.x; b < kNumKeys; b += blockDim.x) s_hist[b] = 0u;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * tile, t1 = min(P.n, t0 + tile);
  for (int64_t base = t0 + (threadIdx.x & ~31); base < t1; base += blockDim.x) {
    const int64_t item = base + lane;
    bool f = false, om = false;
    const bool valid = item < t1;
    uint64_t idx = 0;
    uint32_t fk = 0xFFFFFFFFu;      // fit mode: the item's known fitness (~0 = unknown)
    uint32_t kk_all = 0xFFFFFFFFu;  // this item's key for the tile histogram (none if invalid)
    if (valid) {
      idx = item_index(P.indices, P.start, P.chunk, P.stride, P.item0 + item);
      uint32_t lab[12];
#pragma unroll
      for (int te = 0; te < 12; te++) lab[te] = te < NC ? decode_label(P.dec, te, idx) : 0u;
      uint32_t kk = 0;
      if (key_out) {
        // behaviour key (bonds, _k:90-93): line-prone (a tile bonds a copy of itself through
        // opposite faces), seed tile bonds itself, bondable faces of the seed, another tile
        // bonds itself, bondable faces of the other tiles; smaller keys run first
        uint32_t present = 0;
#pragma unroll
        for (int te = 0; te < NC; te++) present |= 1u << lab[te];
        bool line = false, self0 = false, selfr = false;
        int nb0 = 0, nbr = 0;
#pragma unroll
        for (int t = 0; t < A; t++)
          line |= bonds((int)lab[4 * t], (int)lab[4 * t + 2]) || bonds((int)lab[4 * t + 1], (int)lab[4 * t + 3]);
#pragma unroll
        for (int te = 0; te < NC; te++) {
          const uint32_t x = lab[te];
          const uint32_t px = x ? (((x - 1u) ^ 1u) + 1u) : 31u;  // partner; label 0 bonds nothing
          const bool can = px < 31u && ((present >> px) & 1u);
          if (te < 4) {
            nb0 += can;
#pragma unroll
            for (int g = 0; g < 4; g++) self0 |= bonds((int)x, (int)lab[g]);
          } else {
            nbr += can;
#pragma unroll
            for (int g = 4; g < NC; g++) selfr |= (g >> 2) == (te >> 2) && bonds((int)x, (int)lab[g]);
          }
        }
        kk = ((line ? 0u : 1u) << 9) | ((self0 ? 0u : 1u) << 8) | ((uint32_t)(4 - nb0) << 5) |
             ((selfr ? 0u : 1u) << 4) | (uint32_t)(8 - nbr);
        // GA fitness mode: a genome whose fitness is already known (a child equal to its parent,
        // GaParams::f_known, or a genome in the fitness memo) is skipped like a 1-mer
        if (P.fit_mode) {
          fk = P.fit_known ? P.fit_known[item] : 0xFFFFFFFFu;
          if (fk == 0xFFFFFFFFu && P.memo_mask && nb0 != 0) fk = memo_get(P, idx);
        }
        om = n_skip != nullptr && (nb0 == 0 || fk != 0xFFFFFFFFu);
      }
      if (flags && !om) {  // (1-mers never reach the fast kernel)
        Cand<A, STRICT> K;
        K.build_faces(lab);  // tiles >= A have all-zero faces: they never bond, so never pair
        f = K.trivial_free();
      }
      if (key_out) {
        kk = (kk << 1) | (f ? 0u : 1u);  // trivial-freedom as the lowest key bit
        kk = om ? kOneMerKey : kk;
        key_out[item] = (uint16_t)kk;
        kk_all = kk;
        iota_out[item] = (uint32_t)item | (f ? 0x80000000u : 0u);  // items < 2^31; bit 31 = flag
        if (om && P.fit_mode) {  // known fitness, or that of a DET 1x1 genome: d^2 - shapediff(target, centre)
          const int cr = (P.d >> 1) + 1;
          const int ov = (int)((P.target_rows[cr] >> cr) & 1u);
          P.out_fit[item] = fk != 0xFFFFFFFFu ? fk : (uint32_t)(P.d * P.d - (P.target_cells + 1 - 2 * ov));
        } else if (om && !P.hist_mode) {  // classify_batch row of a DET 1x1 genome (_k:438-452)
          for (int k = 0; k < P.q; k++) P.out_class[item * P.q + k] = (uint8_t)CLS_DET;
          P.out_hash[item] = kOneMerHash;
          P.out_w[item] = 1; P.out_h[item] = 1; P.out_cells[item] = 1;
          for (int64_t wj = 0; wj < P.W; wj++) P.out_shape[item * P.W + wj] = wj == 0 ? 1ULL : 0ULL;
        }
      }
    }
    if (flags) {
      const uint32_t w = __ballot_sync(0xFFFFFFFFu, f);
      if (lane == 0) flags[base >> 5] = w;
    }
    if (tile_hist) {  // warp-aggregated count per key
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, kk_all);
      if (kk_all != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&s_hist[kk_all], (uint32_t)__popc(peers));
    }
    if (n_skip) {
      const unsigned om_mask = __ballot_sync(0xFFFFFFFFu, om);
      if (om_mask) {
        unsigned long long m = om ? idx : ~0ULL;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long x = __shfl_xor_sync(0xFFFFFFFFu, m, o);
          m = x < m ? x : m;
        }
        if (lane == 0) { atomicAdd(&s_om_cnt, (unsigned)__popc(om_mask)); atomicMin(&s_om_min, m); }
      }
    }
  }
  if (tile_hist) {
    __syncthreads();
    for (int b = threadIdx.x; b < kNumKeys; b += blockDim.x) tile_hist[(int64_t)b * ntiles + blockIdx.x] = s_hist[b];
  }
  if (n_skip) {
    __syncthreads();
    if (threadIdx.x == 0 && s_om_cnt) {
      atomicAdd(n_skip, (unsigned long long)s_om_cnt);
      if (P.hist_mode) {
        for (int k = 0; k < P.q; k++) atomicAdd(&P.hist.tallies[k * 5 + CLS_DET], (unsigned long long)s_om_cnt);
        bool gnew = false;
        const int64_t g = hist_claim(P.hist, kOneMerHash, gnew);
        if (g >= 0) {
          atomicAdd(&P.hist.det[g], (unsigned long long)s_om_cnt);
          hist_min(&P.hist.rep_det[g], s_om_min);
          hist_min(&P.hist.rep_any[g], s_om_min);
          if (gnew) {  // this CTA's lowest 1-mer provides the payload (fixed at export if another is lower)
            P.hist.whc[g] = 1u | (1u << 8) | (1u << 16);
            for (int wj = 0; wj < P.hist.W; wj++) P.hist.shape[g * P.hist.W + wj] = wj == 0 ? 1ULL : 0ULL;
            P.hist.pay_idx[g] = s_om_min;
          }
        }
      }
    }
  }
}

// Counting sort of the work items by key (replaces a library radix sort on the hot step).
// tile_hist is key-major [key][tile]; after k_key_binscan it holds each (key, tile)'s offset
// inside its key's run and bintot[key] the key's total; k_key_basescan turns bintot into the
// key runs' starts; k_key_scatter places every item (warp-aggregated shared cursor per key).
// Within one key the order follows the tiles and, inside a tile, the warps' arrival -- results
// never depend on the order (per-genome substreams, commutative histogram updates).
__global__ void __launch_bounds__(1024) k_key_binscan(uint32_t *tile_hist, int64_t ntiles, uint32_t *bintot) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  uint32_t *row = tile_hist + (int64_t)blockIdx.x * ntiles;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0u;
  __syncthreads();
  for (int64_t t0 = 0; t0 < ntiles; t0 += blockDim.x) {
    const int64_t t = t0 + threadIdx.x;
    const uint32_t v = t < ntiles ? row[t] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const uint32_t w0 = lane < nwp ? ws[lane] : 0u;
      uint32_t w = w0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w - w0;
    }
    __syncthreads();
    const uint32_t c = carry;
    if (t < ntiles) row[t] = c + ws[wid] + x - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c + ws[wid] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) bintot[blockIdx.x] = carry;
}

// exclusive scan of the kNumKeys key totals in place (kNumKeys a multiple of 1024)
__global__ void __launch_bounds__(1024) k_key_basescan(uint32_t *bintot) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0u;
  __syncthreads();
  for (int b0 = 0; b0 < kNumKeys; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const uint32_t v = bintot[b];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const uint32_t w0 = ws[lane];
      uint32_t w = w0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w - w0;
    }
    __syncthreads();
    const uint32_t c = carry;
    bintot[b] = c + ws[wid] + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + ws[wid] + x;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_key_scatter(const uint16_t *key, const uint32_t *iota,
                                                     const uint32_t *tile_hist, int64_t ntiles,
                                                     const uint32_t *binbase, int64_t n, int64_t tile,
                                                     uint32_t *order) {
  __shared__ uint32_t cur[kNumKeys];
  for (int b = threadIdx.x; b < kNumKeys; b += blockDim.x)
    cur[b] = binbase[b] + tile_hist[(int64_t)b * ntiles + blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t t0 = (int64_t)blockIdx.x * tile, t1 = min(n, t0 + tile);
  for (int64_t base = t0 + (threadIdx.x & ~31); base < t1; base += blockDim.x) {
    const int64_t item = base + lane;
    const bool valid = item < t1;
    const uint32_t k = valid ? key[item] : 0u;
    // lanes holding the same key: one ballot per key bit (cheaper than __match_any_sync here)
    unsigned peers = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
    for (int b = 0; b < TV_KEY_BITS; b++) {
      const bool bit = (k >> b) & 1u;
      const unsigned m = __ballot_sync(0xFFFFFFFFu, bit);
      peers &= bit ? m : ~m;
    }
    const int leader = __ffs(peers) - 1;
    uint32_t pos = 0;
    if (valid && lane == leader) pos = atomicAdd(&cur[k], (uint32_t)__popc(peers));
    pos = __shfl_sync(0xFFFFFFFFu, pos, leader) + (uint32_t)__popc(peers & ((1u << lane) - 1u));
    if (valid) order[pos] = iota[item];
  }
}

// shared-memory bytes per CTA for the fast kernel
inline size_t fast_smem_bytes(int threads, int GW, int S, int cta_slots, int q) {
  size_t per_warp = (size_t)(GW + S / 2) * 32 * 4;
  size_t cta = (size_t)cta_slots * (8 * 3 + 4 * 3) + (size_t)q * 5 * 4;
  return per_warp * (threads / 32) + cta;
}

}  // namespace tvb
