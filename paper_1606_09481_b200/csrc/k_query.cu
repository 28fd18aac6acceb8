// k_query.cu -- K5..K8: the range queries of Alg. 1 lines 13-21.
//
// For every vertex v and slab b_j (all slabs for CSR; slabs with c_{j+1} > r_v,
// i.e. "outward", for the undirected list):
//
//  * Outer window (the paper's getMinMaxPhi, Eqs. 6-9):
//    every neighbour w in b_j has |dphi| <= W(r_v, c_j).  Evaluated without
//    cancellation (Z3) and padded outward: a superset.
//  * Inner window (this build's addition):
//    W(r_v, r) decreases in r and every w in b_j has r_w <= c_{j+1}, so every w
//    with |dphi| <= W(r_v, c_{j+1}) is a neighbour.  Evaluated with a lower bound
//    and shrunk by a relative margin 2^-17, and only used when both
//    T - sinh^2((r_v - c)/2) >= 2^-10 T at c = c_j, c_{j+1}: the accepted pairs
//    are >= 2^-27 T inside the threshold, so the exact test from either end would
//    also accept them (CSR stays symmetric).  These candidates are edges without
//    a test: the count pass adds their number, the emit pass copies their ids.
//  * The annulus between the windows holds the candidates that need the exact
//    test, dist <= R, in the cancellation-free form of Eq. 3
//    (Z2):
//       h  = e^{r_v/2} e^{-r_w/2} - e^{-r_v/2} e^{r_w/2} = 2 sinh((r_v - r_w)/2)
//       S4 = h^2 + 4 sinh r_v sinh r_w sin^2(dphi/2)  = 2 (cosh d - 1)
//       edge iff S4 <= T4 = 4 sinh^2(R/2) = 2 (cosh R - 1).
//  * Index ranges come from the slab's bucket directory (the binary search of
//    PAPER.md:214, replaced by a lookup).  Every slab is stored twice in a row
//    (the "doubled" SoA), so an arc that crosses 2 pi (DESIGN.md
//    Z13) is one contiguous index range: per (vertex, slab) the candidates are
//    one range [a, b) with the certain sub-range [h0, h1) cut out of it.
//
// Work decomposition (B200): one warp owns 32 consecutive entries of the
// sector-major query order (same slab and angular sector: their candidate ranges
// overlap, so the point SoA is read from L2, not HBM, about once per pass); lane =
// vertex, slabs in lock step.  Per slab each lane computes its vertex's window and
// walks its own candidates: the count pass tests the annulus and stores one bit per
// test; the emit pass recomputes the window, writes the certain ids and replays
// the set bits.  Rows leave the SM in whole 32-byte sectors (a shared-memory ring
// for sample ids, eight sector registers for sequential ids).  Hub vertices take
// the chunked path at the end of this file.  DESIGN.md §7 lists the layouts that
// were measured against this one.
#include <cstdio>
#include <type_traits>

#include "rhg_internal.cuh"
#include "rhg_predicate.cuh"

namespace rhg {

// Debug builds (-DRHG_BOUNDS, scripts/): the first failed check is recorded in
// DevScalars::dbg_line / dbg[] and printed by the host after the emit pass.
#ifdef RHG_BOUNDS
#define RHG_CHECK(cond)                                                      \
  do {                                                                       \
    if (!(cond)) {                                                           \
      if (atomicCAS(&A.sc->dbg_line, 0u, (unsigned)__LINE__) == 0u) {        \
        A.sc->dbg[0] = blockIdx.x;                                           \
        A.sc->dbg[1] = threadIdx.x;                                          \
      }                                                                      \
    }                                                                        \
  } while (0)
#else
#define RHG_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// RHG_ABL (measurement builds only, wrong output): 1 = no certain-id copy, 2 = no hit
// replay, 4 = no row stores.  Attributes the emit kernel's time and DRAM traffic
// (profiles/r02_emit_ablation.txt).
#ifndef RHG_ABL
#define RHG_ABL 0
#endif
#ifndef RHG_QK_WARPS
#define RHG_QK_WARPS 4
#endif
constexpr int QK_WARPS = RHG_QK_WARPS;
constexpr int QK_THREADS = QK_WARPS * 32;
constexpr uint32_t FULL = 0xffffffffu;

// test range of one owner lane (indexed by its rank among the lanes with tests):
// candidate t (flattened index) -> doubled position aoff + t (+ hlen past thr)
struct __align__(16) QRec {
  uint32_t aoff, thr, hlen, lane;
};
// own-slab exclusion (global doubled positions): p excluded iff (p - e1) < w or (p - e2) < w
struct __align__(16) XRec {
  uint32_t e1, e2, w, pad;
};
// certain pieces of one owner: t -> src0 + t (t < thr) or src1 + t; row slot dst + t
struct __align__(16) CRec {
  uint32_t src0, thr, src1, vid;
  unsigned long long dst;
  unsigned long long pad;
};

struct WarpSm {
  double2 qA[2];   // per group vertex: (theta, 4 sinh r)
  double2 qB[2];   // (e^{r/2}, e^{-r/2})
  QRec rec[32];
  XRec xr[32];
  CRec cr[32];
};

struct BandSm {
  uint32_t start[kMaxBands + 1];
  uint32_t dir_off[kMaxBands];
  uint32_t shift[kMaxBands];
};

__device__ __forceinline__ void load_band_sm(BandSm& bs, const BandLayout* lay, int L) {
  if (threadIdx.x <= (unsigned)L) bs.start[threadIdx.x] = lay->start[threadIdx.x];
  if (threadIdx.x < (unsigned)L) {
    bs.dir_off[threadIdx.x] = lay->dir_off[threadIdx.x];
    bs.shift[threadIdx.x] = lay->shift[threadIdx.x];
  }
}

template <typename T>
__device__ __forceinline__ T warp_incl(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T a = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += a;
  }
  return v;
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));  // ftz: denormal ratios -> 0 (still a superset / subset)
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Candidate set of one query vertex in slab j, in positions relative to the slab's
// doubled segment [0, 2 n_j): test the range [a, b) minus [h0, h1); [cs, ce) are
// certain edges.  (Non-full window: h0 = cs, h1 = ce; full window: the tested
// range is the complement of the certain one, hole empty.)
// I = int32_t when every slab has < 2^30 points (positions in [-n_j, 2 n_j] fit),
// int64_t otherwise.
template <typename I>
struct SlabWin {
  I a, b, h0, h1, cs, ce;
  int32_t dq;  // light kernel: outer half-width in quanta incl. bucket rounding (2^30 if full)
};

// num = T4 - 4 sinh^2((r_v - c_j)/2), num1 = the same at c_{j+1} (num1 of slab j
// is num of slab j+1, carried by the caller); q = q27(theta_v); qinv4s = 1/(4 sinh r_v).
// MUFU square roots: their ~2^-22 relative error is inside the 2^-12 / 2^-17 pads.
template <typename I>
__device__ __forceinline__ void slab_window(int j, const BandConst& bc, const BandSm& B, I q,
                                            double num, double num1, double qinv4s,
                                            const uint32_t* __restrict__ dir, SlabWin<I>& w) {
  const uint32_t bstart = B.start[j];
  const I nj = (I)(B.start[j + 1] - bstart);
  // outer window at c_j: d_o >= 2 tan(dphi/2) K27 (1 + 2^-12) + 2 quanta
  bool full = true;
  I d_o = 0;
  const double invS = bc.invS[j];
  if (invS != 0.0) {
    const double ratio = __fma_rn(num, __dmul_rn(qinv4s, invS), __dmul_rn(qinv4s, bc.padS[j]));
    if (ratio < 0.99) {
      const float rf = fmaxf((float)ratio, 0.0f);
      const float dqf = sqrt_approx(rf) * rsqrt_approx(1.0f - rf) *
                        (2.0f * (float)RHG_Q27_SCALE * 1.000244140625f);
      if (dqf < 67108860.0f) {
        full = false;
        d_o = (I)dqf + 2;
      }
    }
  }
  // certain window at c_{j+1}: d_i <= 2 sqrt(ratio1) K27 (1 - 2^-17) - 1 quantum
  I d_i = -1;
  const double invS1 = bc.invS[j + 1];
  if (invS1 != 0.0 && num >= bc.T4min && num1 >= bc.T4min) {
    const float rf1 = fminf((float)__dmul_rn(num1, __dmul_rn(qinv4s, invS1)), 1.0f);
    d_i = (I)(sqrt_approx(rf1) * (2.0f * (float)RHG_Q27_SCALE * 0.99999237060546875f)) - 1;
  }
  // Bucket-only boundaries (no key probing): outer ends round outward to whole
  // buckets, certain ends round inward; boundary-bucket points land in the tested
  // annulus.  Unwrapped bucket bu -> unwrapped slab position (periodic in nb).
  const uint32_t sh = B.shift[j], off = B.dir_off[j];
  const uint32_t lgnb = kQBits - sh, nbm = (1u << lgnb) - 1u;
  auto P = [&](I bu) -> I {  // bu >> lgnb is -1, 0 or 1
    const I per = bu >> lgnb;
    return (I)(__ldg(dir + off + ((uint32_t)bu & nbm)) - bstart) +
           (per < 0 ? -nj : (per > 0 ? nj : (I)0));
  };
  I ls = 0, re = 0, cs = 0, ce = 0;
  if (!full) {
    ls = P((q - d_o) >> sh);
    re = P(((q + d_o) >> sh) + 1);
    if (re - ls >= nj) full = true;
  }
  bool cert = false;
  if (d_i >= 0) {
    cs = P(((q - d_i) >> sh) + 1);
    ce = P((q + d_i) >> sh);
    cert = ce > cs;
  }
  if (!full) {  // shift the arc so that it starts in the first copy
    const I sft = ls < 0 ? nj : (ls >= nj ? -nj : (I)0);
    w.a = ls + sft;
    w.b = re + sft;
    if (cert) {
      w.h0 = cs + sft;
      w.h1 = ce + sft;
    } else {
      w.h0 = w.h1 = w.b;
    }
    w.cs = w.h0;
    w.ce = w.h1;
  } else if (cert) {
    const I sft = cs < 0 ? nj : (cs >= nj ? -nj : (I)0);
    w.cs = cs + sft;
    w.ce = ce + sft;
    w.a = w.ce;
    w.b = w.cs + nj;
    w.h0 = w.h1 = w.b;
  } else {
    w.a = 0;
    w.b = nj;
    w.h0 = w.h1 = nj;
    w.cs = w.ce = 0;
  }
}

// Per-slab constants of the light kernel, staged in shared memory.
struct SlabC {
  double invS, padS;      // 1/sinh c_j (0 for c_j = 0), T4 2^-48 / sinh c_j
  double A0, B0;          // e^{c_j/2}, e^{-c_j/2}
  double A1, B1, invS1;   // e^{c_{j+1}/2}, e^{-c_{j+1}/2}, 1/sinh c_{j+1}
  uint32_t start, nj, off, sh;
};

// slab_window for slabs of < 2^30 points, written for few instructions: the same
// windows, pads and bucket rounding, with selects instead of branches.
__device__ __forceinline__ void win32(const SlabC& S, int32_t q, double num, double num1,
                                      double qinv4s, double T4min,
                                      const uint32_t* __restrict__ dir, SlabWin<int32_t>& w) {
  const int32_t nj = (int32_t)S.nj;
  // outer window at c_j: d_o >= 2 tan(dphi/2) K27 (1 + 2^-12) + 2 quanta
  const double ratio = __dmul_rn(qinv4s, __fma_rn(num, S.invS, S.padS));
  bool full = !(ratio < 0.99) || S.invS == 0.0;
  const float rf = fminf(fmaxf((float)ratio, 0.0f), 0.99f);
  const float dqf = sqrt_approx(rf) * rsqrt_approx(1.0f - rf) *
                    (2.0f * (float)RHG_Q27_SCALE * 1.000244140625f);
  full = full || !(dqf < 67108860.0f);
  const int32_t d_o = full ? 0 : (int32_t)dqf + 2;
  // certain window at c_{j+1}: d_i <= 2 sqrt(ratio1) K27 (1 - 2^-17) - 1 quantum
  const bool certok = S.invS1 != 0.0 && num >= T4min && num1 >= T4min;
  const float rf1 = fminf((float)__dmul_rn(num1, __dmul_rn(qinv4s, S.invS1)), 1.0f);
  const int32_t d_i =
      certok ? (int32_t)(sqrt_approx(rf1) * (2.0f * (float)RHG_Q27_SCALE * 0.99999237060546875f)) - 1
             : -1;
  const uint32_t sh = S.sh, lgnb = kQBits - sh, nbm = (1u << lgnb) - 1u, off = S.off;
  const int32_t mstart = -(int32_t)S.start;
  auto P = [&](int32_t bu) -> int32_t {  // unwrapped bucket -> unwrapped slab position
    const uint32_t e = off + ((uint32_t)bu & nbm);  // 32-bit index: one wide IMAD address
    return (int32_t)__ldg(dir + e) + (bu >> lgnb) * nj + mstart;
  };
  int32_t ls = P((q - d_o) >> sh), re = P(((q + d_o) >> sh) + 1);
  full = full || (re - ls >= nj);
  int32_t cs = P(((q - d_i) >> sh) + 1), ce = P((q + d_i) >> sh);  // d_i = -1: ce <= cs
  const bool cert = ce > cs;
  const int32_t base = full ? cs : ls;  // shift the arc so that it starts in the first copy
  const int32_t sft = base < 0 ? nj : (base >= nj ? -nj : 0);
  ls += sft; re += sft; cs += sft; ce += sft;
  if (!cert) ce = cs;
  // non-full: test [ls, re) minus [cs, ce); full: test [ce, cs + nj) (or all of it)
  w.dq = full ? (1 << 30) : d_o + (1 << sh);
  w.cs = cert ? cs : 0;
  w.ce = cert ? ce : 0;
  if (full) {
    w.a = cert ? ce : 0;
    w.b = cert ? cs + nj : nj;
    w.h0 = w.h1 = w.b;
  } else {
    w.a = ls;
    w.b = re;
    w.h0 = cert ? cs : re;
    w.h1 = cert ? ce : re;
  }
}

// [x, y) minus the periodic exclusion [e1, e1 + wx) u [e1 + nj, e1 + nj + wx)
// (y - x <= nj, so at most two pieces survive).  CSR: e1 = own position, wx = 1
// (no self-loop); undirected list: e1 = 0, wx = own position + 1 (only partners
// sorted after v, Z9).
template <typename I>
__device__ __forceinline__ void cut_piece(I x, I y, I e1, I wx, I nj, I& lo0, I& len0, I& lo1,
                                          I& len1) {
  // pieces below, between and above the two excluded intervals; the first and
  // the last cannot both be non-empty
  const I l1 = max(min(y, e1) - x, (I)0);
  const I s2 = max(x, e1 + wx), l2 = max(min(y, e1 + nj) - s2, (I)0);
  const I s3 = max(x, e1 + nj + wx), l3 = max(y - s3, (I)0);
  if (l1 > 0) {
    lo0 = x; len0 = l1; lo1 = s2; len1 = l2;
  } else {
    lo0 = s2; len0 = l2; lo1 = s3; len1 = l3;
  }
}

// L2 policy for the id array sid2: it is re-read by every neighbourhood, while the
// output streams 4-8 GB through L2, so keep it resident (evict_last).
__device__ __forceinline__ uint64_t policy_keep() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* ptr, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}

template <int FMT>
__device__ __forceinline__ void write_edge(const QueryArgs& A, unsigned long long o, uint32_t vid,
                                           uint32_t w) {
  RHG_CHECK(o < A.out_cap);
  if (FMT == RHG_CSR) A.col[o] = w;
  else reinterpret_cast<uint2*>(A.pairs)[o] = vid < w ? make_uint2(vid, w) : make_uint2(w, vid);
}

// 32 x 32 bit-matrix transpose across the warp: on entry lane r holds row r (bit c =
// element (r, c)); on exit lane c holds column c (bit r = element (r, c)).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t M[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int sft = 16 >> k;
    const uint32_t m = M[k];
    const uint32_t o = __shfl_xor_sync(FULL, x, sft);
    x = (lane & sft) ? ((x & ~m) | ((o >> sft) & m)) : ((x & m) | ((o << sft) & ~m));
  }
  return x;
}

// lanes [lo, hi) of a 32-bit mask (0 <= lo, hi <= 32)
__device__ __forceinline__ uint32_t lane_range_mask(int lo, int hi) {
  if (hi <= lo) return 0u;
  const uint32_t mh = hi >= 32 ? FULL : ((1u << hi) - 1u);
  return mh & ~((1u << lo) - 1u);
}

// Light vertices: one warp per 32 consecutive entries of the sector-major query
// order, one vertex per lane, slabs in lock step.  Per slab every lane computes
// its window (the paper's per-vertex loop body) and then walks
// its own candidates sequentially: certain pieces are copied, the annulus is
// tested exactly.  A lane writes only its own row, through an 8-word shared-memory
// stage, so rows leave the SM as whole 32-byte sectors (one STG.256 each).
//   QM_COUNT     : deg[v]; test results as bits, word w of lane l of warp g at
//                  bits[(g * kLightBitRows + w) * 32 + l] (warp_over[g] = 1 if
//                  some lane needs more than kLightBitRows words)
//   QM_EMIT      : writes the rows, re-testing
//   QM_EMIT_BITS : writes the rows, replaying the bits (re-tests warps with warp_over)
constexpr int kStageStride = 16;  // 16-word ring per lane, 16-byte groups XOR-swizzled by lane

template <int FMT>
struct RowWriter {
  // CSR: 8 ids per 32-byte sector; pairs: 4 (u, v) pairs per sector.  The stage is
  // a two-sector ring; a sector goes out (one STG.256) when the next one starts.
  // Word w of the ring lives at w ^ sw (sw flips bits 2-3 by lane: 16-byte groups
  // stay whole, so a sector is read back with two LDS.128).
  static constexpr uint32_t EPS = FMT == RHG_CSR ? 8u : 4u;
  uint32_t* stage;                 // this lane's ring (16 words, 64-byte aligned)
  uint32_t sw;                     // swizzle
  unsigned long long pos, start;   // next slot, first slot of the row (elements)
  __device__ __forceinline__ void store_elem(uint32_t slot, uint32_t vid, uint32_t w) {
    if (FMT == RHG_CSR) {
      stage[slot ^ sw] = w;
    } else {
      *reinterpret_cast<uint2*>(stage + ((2 * slot) ^ sw)) =
          vid < w ? make_uint2(vid, w) : make_uint2(w, vid);
    }
  }
  // words [8 h + a, 8 h + a + k) of the ring (k = 1, 2, 4; a a multiple of k) -> dst
  __device__ __forceinline__ void store_words(uint32_t* dst, uint32_t h, uint32_t a, uint32_t k) {
    const uint32_t* src = stage + ((8u * h + a) ^ sw);
    if (k == 4) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    else if (k == 2) *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
    else *dst = *src;
  }
  // elements [lo, hi) of the sector in ring half h (a partial sector: the first or
  // last of the row) with at most five aligned vector stores
  __device__ __forceinline__ void store_range(const QueryArgs& A, unsigned long long s0, uint32_t h,
                                              uint32_t lo, uint32_t hi) {
    uint32_t* base = FMT == RHG_CSR ? A.col + s0 : A.pairs + 2 * s0;
    uint32_t x = lo;
    if (FMT == RHG_CSR) {
      if ((x & 1u) && x < hi) { store_words(base + x, h, x, 1); x += 1; }
      if ((x & 2u) && x + 2u <= hi) { store_words(base + x, h, x, 2); x += 2; }
      if (x + 4u <= hi) { store_words(base + x, h, x, 4); x += 4; }
      if (x + 2u <= hi) { store_words(base + x, h, x, 2); x += 2; }
      if (x < hi) store_words(base + x, h, x, 1);
    } else {  // element = one (u, v) pair, two words
      if ((x & 1u) && x < hi) { store_words(base + 2 * x, h, 2 * x, 2); x += 1; }
      if (x + 2u <= hi) { store_words(base + 2 * x, h, 2 * x, 4); x += 2; }
      if (x < hi) store_words(base + 2 * x, h, 2 * x, 2);
    }
  }
  __device__ __forceinline__ void flush(const QueryArgs& A, unsigned long long sec) {
    const uint32_t h = (uint32_t)(sec & 1);
    const unsigned long long s0 = sec * EPS;
    if (RHG_ABL & 4) return;
    if (s0 >= start) {
      uint32_t* dst = FMT == RHG_CSR ? A.col + s0 : A.pairs + 2 * s0;
      const uint4 a = *reinterpret_cast<const uint4*>(stage + ((8u * h) ^ sw));
      const uint4 b = *reinterpret_cast<const uint4*>(stage + ((8u * h + 4u) ^ sw));
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(a.x),
                   "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                   : "memory");
    } else {  // first sector of the row: the slots before `start` belong to the previous row
      store_range(A, s0, h, (uint32_t)(start - s0), EPS);
    }
  }
  // append w[lo..hi) (hi - lo <= 4 < 2 EPS)
  __device__ __forceinline__ void put4(const QueryArgs& A, uint32_t vid, const uint32_t* w,
                                       uint32_t lo, uint32_t hi) {
    const uint32_t p0 = (uint32_t)pos;  // ring arithmetic on the low bits
#pragma unroll
    for (uint32_t u = 0; u < 4; ++u)
      if (u >= lo && u < hi) store_elem((p0 + u - lo) & (2 * EPS - 1), vid, w[u]);
    const uint32_t p1 = p0 + (hi - lo);
    pos += hi - lo;
    if ((p0 ^ p1) & ~(EPS - 1)) flush(A, (pos - (hi - lo)) / EPS);  // a sector completed
  }
  __device__ __forceinline__ void put(const QueryArgs& A, uint32_t vid, uint32_t w) {
    store_elem((uint32_t)pos & (2 * EPS - 1), vid, w);
    ++pos;
    if ((pos & (EPS - 1)) == 0) flush(A, pos / EPS - 1);
  }
  __device__ __forceinline__ void finish(const QueryArgs& A) {
    const uint32_t x = (uint32_t)pos & (EPS - 1);
    if (x) {
      const unsigned long long sec = pos / EPS, s0 = sec * EPS;
      store_range(A, s0, (uint32_t)(sec & 1), s0 >= start ? 0u : (uint32_t)(start - s0), x);
    }
  }
};

// Row writer for sequential vertex ids (rhg_options.vertex_order = 1: the id of a
// vertex is its position in the (slab, angle) order, so the ids of a certain piece
// are consecutive integers and the id of a tested candidate is its position).
// The lane assembles its current 32-byte output sector in eight registers: a run
// of consecutive ids or a single id is merged in with per-slot selects (no
// shared memory, no loads), and a completed sector leaves as one STG.256.  The
// sectors holding the row's first and last slots are written slot by slot.
// Pairs (u, v) = (the query vertex, the partner): the partner's id is larger.
template <int FMT>
struct SecWriter {
  static constexpr uint32_t EPS = FMT == RHG_CSR ? 8u : 4u;  // elements per sector
  uint32_t r[8];
  uint32_t f;                      // filled elements of the current sector
  unsigned long long sec, start;   // current sector, first element of the row
  __device__ __forceinline__ void init(unsigned long long pos, uint32_t vid) {
    sec = pos / EPS;
    f = (uint32_t)(pos % EPS);
    start = pos;
#pragma unroll
    for (int x = 0; x < 8; ++x) r[x] = vid;  // pairs: even words stay = vid
  }
  __device__ __forceinline__ void store_slots(const QueryArgs& A, uint32_t lo, uint32_t hi) {
#pragma unroll
    for (uint32_t x = 0; x < EPS; ++x) {
      if (x >= lo && x < hi) {
        if (FMT == RHG_CSR) A.col[sec * EPS + x] = r[x];
        else reinterpret_cast<uint2*>(A.pairs)[sec * EPS + x] = make_uint2(r[2 * x], r[2 * x + 1]);
      }
    }
  }
  __device__ __forceinline__ void flush(const QueryArgs& A) {
    const unsigned long long s0 = sec * EPS;
    RHG_CHECK(s0 + EPS <= A.out_cap);
    if (s0 >= start) {
      uint32_t* dst = FMT == RHG_CSR ? A.col + s0 : A.pairs + 2 * s0;
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(r[0]),
                   "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                   : "memory");
    } else {
      store_slots(A, (uint32_t)(start - s0), EPS);
    }
    ++sec;
    f = 0;
  }
  // ids v0, v0 + 1, ..., v0 + len - 1 (all lanes call; len may be 0)
  __device__ __forceinline__ void run(const QueryArgs& A, uint32_t v0, uint32_t len) {
    while (__any_sync(FULL, len != 0)) {
      const uint32_t t = min(len, EPS - f);
      const uint32_t base = v0 - f;
#pragma unroll
      for (uint32_t x = 0; x < EPS; ++x) {
        const bool in = (x - f) < t;
        if (FMT == RHG_CSR) r[x] = in ? base + x : r[x];
        else r[2 * x + 1] = in ? base + x : r[2 * x + 1];
      }
      f += t;
      v0 += t;
      len -= t;
      if (f == EPS) flush(A);
    }
  }
  __device__ __forceinline__ void put(const QueryArgs& A, uint32_t v) {
#pragma unroll
    for (uint32_t x = 0; x < EPS; ++x) {
      if (FMT == RHG_CSR) r[x] = x == f ? v : r[x];
      else r[2 * x + 1] = x == f ? v : r[2 * x + 1];
    }
    if (++f == EPS) flush(A);
  }
  __device__ __forceinline__ void finish(const QueryArgs& A) {
    if (f) {
      const unsigned long long s0 = sec * EPS;
      store_slots(A, s0 >= start ? 0u : (uint32_t)(start - s0), f);
    }
  }
};

// id of doubled position p of a slab starting at s with nj points (sequential ids)
__device__ __forceinline__ uint32_t seq_id(uint32_t p, uint32_t s, uint32_t nj) {
  const uint32_t x = p - 2u * s;
  return s + (x >= nj ? x - nj : x);
}

__device__ __forceinline__ uint4 ld4_keep(const uint32_t* ptr, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}

// 1 / (4 sinh r) to ~1 ulp: float reciprocal + two Newton steps (the window pads
// absorb far larger relative errors)
__device__ __forceinline__ double inv4s_of(double s) {
  const double y = 4.0 * s;
  double x = (double)__frcp_rn((float)y);
  x = __fma_rn(x, __fma_rn(-y, x, 1.0), x);
  x = __fma_rn(x, __fma_rn(-y, x, 1.0), x);
  return x;
}

#ifndef RHG_QK_MINB_COUNT
#define RHG_QK_MINB_COUNT 8  // 64 registers (measured at config 3: 2.43 ms vs 2.49 ms with 56)
#endif
#ifndef RHG_QK_MINB_COUNT_LIST
#define RHG_QK_MINB_COUNT_LIST 8  // count pass of the list output (its own instantiation)
#endif
#ifndef RHG_QK_MINB_EMIT
#define RHG_QK_MINB_EMIT 9
#endif
#ifndef RHG_QK_MINB_SEQ
#define RHG_QK_MINB_SEQ 7  // 72 registers: the eight sector registers of SecWriter
#endif
#ifndef RHG_QK_MINB_LIST
#define RHG_QK_MINB_LIST 10  // list emit (COOP), sample ids: no row stage; 48 registers (config 5
                             // emit 6.24 ms at 8 blocks / 64 registers, 6.13 at 9, 6.07 at 10)
#endif
#ifndef RHG_QK_MINB_LIST_SEQ
#define RHG_QK_MINB_LIST_SEQ 9  // list emit, vertex_order 1: 56 registers (5.72 ms at 8, 5.59 at 9, 5.70 at 10)
#endif
template <int MODE, int FMT, bool WIDE, bool SEQ>
__global__ void __launch_bounds__(QK_THREADS, MODE == QM_COUNT ? (FMT == RHG_EDGES_UNDIRECTED ? RHG_QK_MINB_COUNT_LIST : RHG_QK_MINB_COUNT)
                                              : (FMT == RHG_EDGES_UNDIRECTED ? (SEQ ? RHG_QK_MINB_LIST_SEQ : RHG_QK_MINB_LIST)
                                              : (SEQ ? RHG_QK_MINB_SEQ : RHG_QK_MINB_EMIT)))
    k_query(const QueryArgs A, const __grid_constant__ BandConst bc) {
  using I = typename std::conditional<WIDE, int64_t, int32_t>::type;
  // Undirected list: the 32 rows of a warp are adjacent in the output (offsets by
  // processing position) and the order of the pairs inside that region is free, so
  // the warp fills it iteration by iteration -- every lane with a pair in this
  // iteration writes it at the warp cursor + its rank among those lanes (ballot +
  // popc): coalesced stores, no per-lane ring, no bit transpose, no per-lane loops.
  constexpr bool COOP = MODE != QM_COUNT && FMT == RHG_EDGES_UNDIRECTED;
  // emit launched before the host has seen the edge total: nothing is written
  // unless it fits the caller's capacity (block-uniform exit)
  if (MODE != QM_COUNT && A.total_dev && *A.total_dev > A.cap) return;
  __shared__ BandSm bs;
  __shared__ SlabC scs[kMaxBands];
  __shared__ __align__(16) uint32_t stage_all[(MODE == QM_COUNT || SEQ || COOP) ? 4 : QK_THREADS * kStageStride];
  load_band_sm(bs, A.lay, bc.L);
  if (threadIdx.x < (unsigned)bc.L) {
    const int j = threadIdx.x;
    SlabC c;
    c.invS = bc.invS[j];
    c.padS = bc.padS[j];
    c.A0 = bc.A[j];
    c.B0 = bc.B[j];
    c.A1 = bc.A[j + 1];
    c.B1 = bc.B[j + 1];
    c.invS1 = bc.invS[j + 1];
    c.start = A.lay->start[j];
    c.nj = A.lay->start[j + 1] - c.start;
    c.off = A.lay->dir_off[j];
    c.sh = A.lay->shift[j];
    scs[j] = c;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t g = blockIdx.x * QK_WARPS + (threadIdx.x >> 5);  // light warp (of this shard)
  const uint32_t nlight = A.nquery ? (uint32_t)*A.nquery : A.n - A.lay->heavy_end;
  // shard: a contiguous range of the 32-vertex groups of the sector-major order
  // with an equal share of the estimated work (k_shard.cu)
  const uint32_t ngroups = (nlight + 31u) / 32u;
  uint32_t gbeg = 0, gend = ngroups;
  if (bc.nshards > 1) {
    gbeg = min(A.shard_plan->grp_beg, ngroups);
    gend = min(A.shard_plan->grp_end, ngroups);
  }
  if (gbeg + g >= gend) return;
  const uint32_t idx = (gbeg + g) * 32u + lane;
  const bool valid = idx < nlight;
  const uint32_t k = valid ? __ldg(A.order + idx) : 0u;
  const bool outward = (FMT == RHG_EDGES_UNDIRECTED);
  const uint64_t keep = policy_keep();
  const double T4 = bc.T4;

  uint32_t qkey = 0, qid = 0;
  if (valid) {
    qkey = __ldg(A.skey + k);
    if (MODE != QM_COUNT) qid = SEQ ? k : __ldg(A.sid + k);
  }
  // Emit passes: the slab of sorted position k = the last j with start[j] <= k
  // (start[L] = n > k) is found in shared memory, so that the record load does not wait
  // for the key load (one level less in the group's chain of dependent loads: order ->
  // key, id, record; config 5 emit 6.41 -> 6.24 ms).  The count pass keeps the key's
  // slab bits: the search costs it a register it does not have (config 3 count +0.04 ms).
  uint32_t qband = qkey >> kBandShift;
  if (MODE != QM_COUNT) {
    qband = 0;
#pragma unroll
    for (uint32_t step = kMaxBands / 2; step; step >>= 1) {
      const uint32_t t = qband + step;
      if (t < (uint32_t)bc.L && bs.start[t] <= k) qband = t;
    }
    RHG_CHECK(!valid || qband == (qkey >> kBandShift));
  }
  const I qq = (I)(qkey & kQMask);
  PointRec q;
  q.theta = 0.0; q.s = 1.0; q.a = 1.0; q.b = 1.0;
  if (valid) q = A.pts[k + bs.start[qband]];  // first copy of the doubled slab
  const double qinv4s = inv4s_of(q.s);
  const double q4s = 4.0 * q.s;

  // rows.  Sample ids: slab by slab, certain ids then hits, all through the
  // shared-memory ring.  Sequential ids: [certain ids, slab by slab][hits, slab by
  // slab]; the certain part through the sector registers, hits stored one by one
  // from hcur (the count pass left the certain count in cdeg).
  RowWriter<FMT> rw;
  SecWriter<FMT> sw;
  unsigned long long hcur = 0;
  unsigned long long wc = 0;  // COOP: the warp's output cursor (warp-uniform)
  const uint32_t ltmask = (1u << lane) - 1u;
  if (COOP) {
    // lane 0 is valid in every launched warp; its row starts the warp's region
    if (lane == 0) wc = A.offs[A.lay->heavy_end + gbeg + g];
    wc = __shfl_sync(FULL, wc, 0);
  } else if (MODE != QM_COUNT) {
    // list output: degrees and offsets by processing position (coalesced), else by id
    const uint32_t slot = A.poff ? A.lay->heavy_end + idx : qid;
    const unsigned long long pos0 = valid ? A.offs[slot] : 0ull;
    if (SEQ) hcur = valid ? pos0 + A.cdeg[slot] : 0ull;
    if (SEQ) {
      sw.init(pos0, qid);
    } else {
      rw.stage = stage_all + threadIdx.x * kStageStride;
      rw.sw = ((threadIdx.x >> 1) & 3u) << 2;
      rw.pos = rw.start = pos0;
    }
  }
  uint32_t deg = 0;           // count pass
  uint32_t word = 0;
  // the warp's test bit stream: one ballot word per test iteration, slab after slab
  uint32_t* const wstream = A.bits + (uint64_t)g * (kLightBitRows * 32u);
  uint32_t F = 0;             // words of earlier slabs
  bool retest = MODE == QM_EMIT;
  if (MODE == QM_EMIT_BITS) retest = A.warp_over[g] != 0;
  bool over = false;          // count: some lane ran out of bit words
  uint32_t tested = 0, certain = 0;  // per lane (certain: also the row-tail start)

  int jlo = 0;
  if (outward) jlo = (int)__reduce_min_sync(FULL, valid ? qband : 0xffffu);
  for (int j = jlo; j < bc.L; ++j) {
    const SlabC& S = scs[j];
    const uint32_t nj = S.nj;
    if (nj == 0) continue;
    const uint32_t bstart = S.start, gbase = 2u * bstart;
    const bool on = valid && (!outward || j >= (int)qband);
    SlabWin<I> w;
    w.a = w.b = w.h0 = w.h1 = w.cs = w.ce = 0;
    w.dq = 0;
    if (on) {
      const double h0 = __fma_rn(q.a, S.B0, -__dmul_rn(q.b, S.A0));
      const double h1 = __fma_rn(q.a, S.B1, -__dmul_rn(q.b, S.A1));
      const double num0 = __fma_rn(-h0, h0, T4), num1 = __fma_rn(-h1, h1, T4);
      if (WIDE) {
        slab_window<I>(j, bc, bs, qq, num0, num1, qinv4s, A.dir, w);
      } else {
        SlabWin<int32_t> w32;
        win32(S, (int32_t)qq, num0, num1, qinv4s, bc.T4min, A.dir, w32);
        w.a = w32.a; w.b = w32.b; w.h0 = w32.h0; w.h1 = w32.h1; w.cs = w32.cs; w.ce = w32.ce;
        w.dq = w32.dq;
      }
    }
    const bool own = on && (j == (int)qband);
    const bool anyown = __any_sync(FULL, own);
    I e1 = 0, wx = 0;
    if (own) {
      const I kv = (I)(k - bstart);
      if (outward) { e1 = 0; wx = kv + 1; } else { e1 = kv; wx = 1; }
      // list: only partners sorted after v.  When the tested range lies in the first
      // copy its excluded part is the prefix [a, kv]: start the range at kv + 1
      // (count and emit trim alike, so the bit streams line up)
      if (outward && w.b <= (I)nj && w.a <= kv) {
        w.a = min(kv + 1, w.b);
        w.h0 = max(w.h0, w.a);
        w.h1 = max(w.h1, w.a);
      }
    }
    // certain pieces (own slab: minus v itself / minus the partners sorted before v)
    I clo0 = w.cs, cln0 = w.ce - w.cs, clo1 = 0, cln1 = 0;
    if (own) cut_piece<I>(w.cs, w.ce, e1, wx, (I)nj, clo0, cln0, clo1, cln1);
    const uint32_t ct = (uint32_t)(cln0 + cln1);
    const uint32_t nt = (uint32_t)((w.b - w.a) - (w.h1 - w.h0));
    if (MODE == QM_COUNT) {
      deg += ct;
      certain += ct;
    } else if (COOP) {
      // ---- certain edges, list output: one pair per lane and iteration ----
      const uint32_t c0 = gbase + (uint32_t)clo0, c1 = gbase + (uint32_t)clo1;
      const uint32_t l0 = (uint32_t)cln0;
      const uint32_t mc = (RHG_ABL & 1) ? 0u : __reduce_max_sync(FULL, ct);
      for (uint32_t u = 0; u < mc; ++u) {
        const bool act = u < ct;
        const uint32_t am = __ballot_sync(FULL, act);
        if (act) {
          const uint32_t x = u < l0 ? c0 + u : c1 + (u - l0);
          const uint32_t w = SEQ ? seq_id(x, bstart, nj) : ld_keep(A.sid2 + x, keep);
          write_edge<FMT>(A, wc + __popc(am & ltmask), qid, w);
        }
        wc += __popc(am);
      }
    } else if (SEQ) {
      // ---- certain edges: consecutive ids, two pieces, each wrapping at most once ----
      const uint32_t rel0 = (uint32_t)clo0 >= nj ? (uint32_t)clo0 - nj : (uint32_t)clo0;
      const uint32_t rel1 = (uint32_t)clo1 >= nj ? (uint32_t)clo1 - nj : (uint32_t)clo1;
      const uint32_t a0 = min((uint32_t)cln0, nj - rel0), a1 = min((uint32_t)cln1, nj - rel1);
      sw.run(A, bstart + rel0, a0);
      sw.run(A, bstart, (uint32_t)cln0 - a0);
      sw.run(A, bstart + rel1, a1);
      sw.run(A, bstart, (uint32_t)cln1 - a1);
    } else {
      // ---- certain edges: copy the ids into my row, 4 aligned ids per load ----
      const uint32_t c0 = gbase + (uint32_t)clo0, c1 = gbase + (uint32_t)clo1;
      const uint32_t l0 = (uint32_t)cln0, l1 = (uint32_t)cln1;
      const uint32_t a0 = c0 & ~3u, a1 = c1 & ~3u;
      const uint32_t n0 = l0 ? (c0 + l0 - a0 + 3u) >> 2 : 0u;
      const uint32_t n1 = l1 ? (c1 + l1 - a1 + 3u) >> 2 : 0u;
      const uint32_t nit = n0 + n1;
      const uint32_t mc = (RHG_ABL & 1) ? 0u : __reduce_max_sync(FULL, nit);
      for (uint32_t i = 0; i < mc; ++i) {
        if (i < nit) {
          const bool second = i >= n0;
          const uint32_t c = second ? c1 : c0, l = second ? l1 : l0;
          const uint32_t x = (second ? a1 + 4u * (i - n0) : a0 + 4u * i);
          const uint4 v = ld4_keep(A.sid2 + x, keep);
          const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
          const uint32_t lo = c > x ? c - x : 0u;
          const uint32_t hi = min(c + l - x, 4u);
          rw.put4(A, qid, wv, lo, hi);
        }
      }
    }
    // ---- annulus: exact tests ----
    const uint32_t mt = __reduce_max_sync(FULL, nt);
    if (mt == 0) continue;
    const uint32_t pa = gbase + (uint32_t)w.a, thr = (uint32_t)(w.h0 - w.a);
    const uint32_t hl = (uint32_t)(w.h1 - w.h0);
    // own-slab exclusion in doubled positions: [x1, x1 + wx) and [x1 + nj, ...)
    const uint32_t x1 = gbase + (uint32_t)e1, xw = (uint32_t)wx;
    if (MODE == QM_COUNT) tested += nt;
    if ((RHG_ABL & 2) && MODE == QM_EMIT_BITS) continue;
    if (COOP && MODE == QM_EMIT_BITS && !retest) {
      // replay, list output: word F + i is the ballot of the count pass's i-th test
      // iteration of this slab; its set lanes write their pairs side by side
      for (uint32_t i0 = 0; i0 < mt; i0 += 32u) {
        const uint32_t wv = i0 + (uint32_t)lane < mt ? wstream[F + i0 + (uint32_t)lane] : 0u;
        const uint32_t cnt = min(32u, mt - i0);
        for (uint32_t u = 0; u < cnt; ++u) {
          const uint32_t m = __shfl_sync(FULL, wv, u);
          if (m == 0u) continue;
          if ((m >> lane) & 1u) {
            const uint32_t i = i0 + u;
            const uint32_t p = pa + i + (i >= thr ? hl : 0u);
            const uint32_t w = SEQ ? seq_id(p, bstart, nj) : ld_keep(A.sid2 + p, keep);
            write_edge<FMT>(A, wc + __popc(m & ltmask), qid, w);
          }
          wc += __popc(m);
        }
      }
      F += mt;
      continue;
    }
    if (MODE == QM_EMIT_BITS && !retest) {
      // replay: word F + i of the warp's bit stream is the ballot of the count pass's
      // i-th test iteration of this slab (bit l: lane l's i-th candidate).  Per 32
      // iterations one coalesced load and a 32 x 32 bit transpose give each lane its
      // own hit mask; then only the set bits are walked.
      for (uint32_t i0 = 0; i0 < mt; i0 += 32u) {
        uint32_t m = i0 + (uint32_t)lane < mt ? wstream[F + i0 + (uint32_t)lane] : 0u;
        m = transpose32(m, lane);
        const uint32_t mh = __reduce_max_sync(FULL, (uint32_t)__popc(m));
        for (uint32_t h = 0; h < mh; ++h) {
          if (m) {
            const uint32_t i = i0 + (uint32_t)(__ffs(m) - 1);
            m &= m - 1u;
            const uint32_t p = pa + i + (i >= thr ? hl : 0u);
            if (SEQ) write_edge<FMT>(A, hcur++, qid, seq_id(p, bstart, nj));
            else rw.put(A, qid, ld_keep(A.sid2 + p, keep));
          }
        }
      }
      F += mt;
      continue;
    }
    // count, or emit with re-tests: every candidate is tested
    const bool store = F + mt <= kLightBitRows * 32u;  // warp-uniform
    if (MODE == QM_COUNT && !store) over = true;
    auto test_loop = [&](auto short_poly, auto own_slab) {
      // chunks of 32 iterations: lane u keeps the ballot word of iteration i0 + u and
      // the chunk's words are stored together (count pass)
      for (uint32_t i0 = 0; i0 < mt; i0 += 32u) {
        const uint32_t cnt = min(32u, mt - i0);
        for (uint32_t u = 0; u < cnt; ++u) {
          const uint32_t i = i0 + u;
          const bool act = i < nt;
          const uint32_t p = pa + i + (i >= thr ? hl : 0u);
          bool tst = act;
          if (decltype(own_slab)::value) tst = tst && !((p - x1) < xw || (p - x1 - nj) < xw);
          uint32_t r[8];
          const PointRec* wp = A.pts + (tst ? p : 0u);
          asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                         "=r"(r[6]), "=r"(r[7])
                       : "l"(wp));
          const double2 w0 = make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
          const double2 w1 = make_double2(__hiloint2double(r[5], r[4]), __hiloint2double(r[7], r[6]));
          const bool hit = decltype(short_poly)::value
                               ? certified_edge_short(q.theta, q4s, q.a, q.b, w0, w1, T4, tst)
                               : certified_edge(q.theta, q4s, q.a, q.b, w0, w1, T4, tst);
          if (MODE == QM_COUNT) {
            deg += hit;
            const uint32_t hm = __ballot_sync(FULL, hit);
            word = u == (uint32_t)lane ? hm : word;
          } else if (COOP) {
            const uint32_t hm = __ballot_sync(FULL, hit);
            if (hit)
              write_edge<FMT>(A, wc + __popc(hm & ltmask), qid,
                              SEQ ? seq_id(p, bstart, nj) : ld_keep(A.sid2 + p, keep));
            wc += __popc(hm);
          } else if (hit) {
            if (SEQ) write_edge<FMT>(A, hcur++, qid, seq_id(p, bstart, nj));
            else rw.put(A, qid, ld_keep(A.sid2 + p, keep));
          }
        }
        if (MODE == QM_COUNT && store && (uint32_t)lane < cnt) wstream[F + i0 + (uint32_t)lane] = word;
      }
    };
    // every candidate of the warp within |dphi| < 2^-4 (300000 quanta < 2^27 2^-4 / 2pi)
    // and no window reaching across theta = 0 (so no seam pair): the short-polynomial
    // test applies
    const int32_t q32 = (int32_t)(qkey & kQMask);
    const bool small = __all_sync(
        FULL, !on || (!WIDE && w.dq < 300000 && q32 >= w.dq && q32 + w.dq < (int32_t)(1u << kQBits)));
    // the own-slab exclusion only where some lane queries its own slab
    if (anyown) {
      if (small) test_loop(std::true_type{}, std::true_type{});
      else test_loop(std::false_type{}, std::true_type{});
    } else {
      if (small) test_loop(std::true_type{}, std::false_type{});
      else test_loop(std::false_type{}, std::false_type{});
    }
    F += mt;
  }
  if (MODE == QM_COUNT) {
    if (FMT == RHG_EDGES_UNDIRECTED) {
      // list output: the warp's rows are one region, so one degree entry per warp
      // (after the hub rows): the scan runs over heavy_end + groups entries
      const uint32_t wsum = __reduce_add_sync(FULL, valid ? deg : 0u);
      if (lane == 0) A.deg[A.lay->heavy_end + gbeg + g] = wsum;
    } else if (valid) {
      const uint32_t id = A.poff ? A.lay->heavy_end + idx : (A.labels ? k : __ldg(A.sid + k));
      A.deg[id] = deg;
      if (A.labels) A.cdeg[id] = (uint32_t)certain;
    }
    const bool anyover = __any_sync(FULL, over);
    if (lane == 0) {
      A.warp_over[g] = anyover ? 1u : 0u;
      if (anyover) atomicAdd(&A.sc->bit_overflow, 1u);  // warps whose emit re-tests
    }
    if (A.stats) {  // timing statistics only
      const unsigned long long tw = warp_incl((unsigned long long)tested);
      const unsigned long long cw = warp_incl((unsigned long long)certain);
      if (lane == 31) {
        atomicAdd(&A.sc->candidates, tw);
        atomicAdd(&A.sc->certain, cw);
      }
    }
  } else if (!COOP && valid) {
    if (SEQ) sw.finish(A);
    else rw.finish(A);
  }
}

// ------------------------------------------------------------------ hub path
// Hub vertices (sorted positions [0, heavy_end), chosen by k_band_layout) have
// 10^3..10^6 candidates each.  One warp per hub materialises its non-empty
// (slab, piece) ranges -- up to 4 tested pieces and 2 certain pieces per slab --
// as a compacted list; the vertex's concatenated candidate sequence is cut into
// chunks of CH candidates (a 32-candidate group belongs to the chunk holding its
// first candidate), and the chunks are spread over every warp of the GPU.
// Output placement stays deterministic: the edges of chunk c land at
// offs[v] + (chunk_pos[c] - chunk_pos[first chunk of v]) in group order.
constexpr int HV_THREADS = 256;
constexpr int HV_WARPS = HV_THREADS / 32;

template <int FMT>
__global__ void __launch_bounds__(HV_THREADS)
    k_heavy_ranges(const QueryArgs A, const HeavyArgs H, const __grid_constant__ BandConst bc) {
  __shared__ BandSm bs;
  load_band_sm(bs, A.lay, bc.L);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * HV_WARPS + (threadIdx.x >> 5);
  const uint32_t TW = gridDim.x * HV_WARPS;
  const uint32_t he = A.lay->heavy_end;
  const int L = bc.L;
  const uint32_t LS = kRangesPerSlab * (uint32_t)L;
  const bool outward = (FMT == RHG_EDGES_UNDIRECTED);

  for (uint32_t i = gw; i < he; i += TW) {
    const uint32_t qkey = A.skey[i];
    const uint32_t qband = qkey >> kBandShift;
    const PointRec q = A.pts[i + bs.start[qband]];
    const double qinv4s = 0.25 / q.s;
    const bool owned = (bc.nshards <= 1 || snake(i, bc.nshards) == bc.shard) &&
                       (!A.hub_mask || A.hub_mask[i] != 0u);
    const int j = owned ? lane : 32;  // other shards' hubs: no pieces
    int64_t lo[6] = {0, 0, 0, 0, 0, 0}, ln[6] = {0, 0, 0, 0, 0, 0};
    uint32_t gbase = 0;
    if (j < L) {
      const uint32_t bstart = bs.start[j], nj = bs.start[j + 1] - bstart;
      gbase = 2u * bstart;
      if (nj > 0 && (!outward || j >= (int)qband)) {
        const double hA = __fma_rn(q.a, bc.B[j], -__dmul_rn(q.b, bc.A[j]));
        const double hB = __fma_rn(q.a, bc.B[j + 1], -__dmul_rn(q.b, bc.A[j + 1]));
        SlabWin<int64_t> w;
        slab_window<int64_t>(j, bc, bs, (int64_t)(qkey & kQMask), __fma_rn(-hA, hA, bc.T4),
                             __fma_rn(-hB, hB, bc.T4), qinv4s, A.dir, w);
        if (j == (int)qband) {
          const int64_t kv = (int64_t)(i - bstart);
          const int64_t e1 = outward ? 0 : kv, wx = outward ? kv + 1 : 1;
          cut_piece<int64_t>(w.a, w.h0, e1, wx, (int64_t)nj, lo[0], ln[0], lo[1], ln[1]);
          cut_piece<int64_t>(w.h1, w.b, e1, wx, (int64_t)nj, lo[2], ln[2], lo[3], ln[3]);
          cut_piece<int64_t>(w.cs, w.ce, e1, wx, (int64_t)nj, lo[4], ln[4], lo[5], ln[5]);
        } else {
          lo[0] = w.a; ln[0] = w.h0 - w.a;
          lo[2] = w.h1; ln[2] = w.b - w.h1;
          lo[4] = w.cs; ln[4] = w.ce - w.cs;
        }
      }
    }
    // compact the lane's non-empty pieces (slab order, then piece order)
    uint32_t cnt = 0, cand = 0;
#pragma unroll
    for (int x = 0; x < 6; ++x) {
      cnt += ln[x] > 0;
      cand += (uint32_t)ln[x];
    }
    const uint32_t ci = warp_incl(cnt), ca = warp_incl(cand);
    uint32_t slot = i * LS + (ci - cnt), off = ca - cand;
#pragma unroll
    for (int x = 0; x < 6; ++x) {
      if (ln[x] > 0) {
        const uint32_t len = (uint32_t)ln[x];
        H.pstart[slot] = gbase + (uint32_t)lo[x];
        H.plen[slot] = len | (x < (int)kTestPieces ? 0u : kCertainPiece);
        H.poff[slot] = off;
        ++slot;
        off += len;
      }
    }
    if (lane == 31) {
      H.np[i] = ci;
      H.vtot[i] = ca;
    }
    if (lane == 0) A.deg[(A.labels || A.poff) ? i : A.sid[i]] = 0u;
  }
}

__global__ void k_heavy_chunk_size(const HeavyArgs H) {
  const unsigned long long C = H.meta->cand, nv = H.meta->nvtx;
  const unsigned long long room = H.chunk_cap > nv ? H.chunk_cap - nv : 1ull;
  unsigned long long ch = (C + room - 1) / room;  // sum_v ceil(C_v / ch) <= C / ch + nv
  if (ch < H.chunk_min) ch = H.chunk_min;
  ch = (ch + 31ull) & ~31ull;  // whole 32-candidate groups
  H.meta->chunk = ch;
}

__global__ void k_heavy_chunk_counts(const HeavyArgs H) {
  const unsigned long long nv = H.meta->nvtx, ch = H.meta->chunk;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < nv;
       i += (unsigned long long)gridDim.x * blockDim.x)
    H.cc[i] = (uint32_t)((H.vtot[i] + ch - 1) / ch);
}

// warp per hub vertex; lane handles chunks c0 + lane, c0 + lane + 32, ...: the
// first piece whose candidates reach past the chunk start (binary search).
__global__ void __launch_bounds__(HV_THREADS) k_heavy_chunk_map(const HeavyArgs H, uint32_t LS) {
  const int lane = threadIdx.x & 31;
  const unsigned long long nv = H.meta->nvtx, ch = H.meta->chunk;
  for (unsigned long long i = blockIdx.x * (unsigned long long)HV_WARPS + (threadIdx.x >> 5);
       i < nv; i += (unsigned long long)gridDim.x * HV_WARPS) {
    const unsigned long long c0 = H.choff[i], c1 = H.choff[i + 1];
    const uint32_t np = H.np[i];
    const uint64_t base = i * LS;
    for (unsigned long long c = c0 + lane; c < c1; c += 32) {
      const unsigned long long lo = (c - c0) * ch;
      uint32_t a = 0, b = np;  // first piece with poff + len > lo
      while (a < b) {
        const uint32_t m = (a + b) >> 1;
        const unsigned long long end =
            (unsigned long long)H.poff[base + m] + (H.plen[base + m] & ~kCertainPiece);
        if (end <= lo) a = m + 1; else b = m;
      }
      H.chunk_vtx[c] = (uint32_t)i;
      H.chunk_piece[c] = a;
    }
  }
}

// One warp per chunk: [lo, hi) of hub vertex i's candidate sequence (the
// concatenation of its pieces).  The warp holds up to 32 of the chunk's pieces in
// registers (one per lane) and walks the chunk 32 candidates per batch; the piece
// of candidate t is found like the light kernel's owner (OR of segment-start bits
// + popcount).  Certain pieces count as hits without a test.  Ballot words are
// stored per chunk (CH / 32 + 8 words per chunk) for the emit pass to replay.
template <int MODE, int FMT>
#ifndef RHG_HV_MINB
#define RHG_HV_MINB 4
#endif
#ifndef RHG_HV_BLOCKS
#define RHG_HV_BLOCKS 8  // per SM
#endif
__global__ void __launch_bounds__(HV_THREADS, RHG_HV_MINB)
    k_heavy(const QueryArgs A, const HeavyArgs H, const __grid_constant__ BandConst bc) {
  if (MODE != QM_COUNT && A.total_dev && *A.total_dev > A.cap) return;  // see k_query
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u, le = (2u << lane) - 1u;
  const unsigned long long gw = blockIdx.x * HV_WARPS + (threadIdx.x >> 5);
  const unsigned long long TW = (unsigned long long)gridDim.x * HV_WARPS;
  const unsigned long long nch = H.meta->nchunks, CH = H.meta->chunk;
  const uint32_t LS = kRangesPerSlab * (uint32_t)bc.L;
  const double T4 = bc.T4;
  const unsigned long long WPC = (CH >> 5) + 8;  // bit words per chunk (+ window seams)
  const bool bits = nch * WPC <= H.bits_cap;
  const uint64_t keep = policy_keep();
  unsigned long long cand_total = 0, cert_total = 0;
  for (unsigned long long c = gw; c < nch; c += TW) {
    const uint32_t i = H.chunk_vtx[c];
    const unsigned long long c0 = H.choff[i];
    const uint32_t lo = (uint32_t)((c - c0) * CH);
    const uint32_t vt = H.vtot[i];
    const uint32_t hi = (uint32_t)min((unsigned long long)vt, (unsigned long long)lo + CH);
    const uint32_t np = H.np[i];
    const uint32_t qid = A.labels ? i : A.sid[i];
    unsigned long long base = 0;
    if (MODE != QM_COUNT) base = A.offs[A.poff ? i : qid] + (H.chunk_pos[c] - H.chunk_pos[c0]);
    const uint32_t qband = A.skey[i] >> kBandShift;
    const PointRec q = A.pts[i + A.lay->start[qband]];
    const double q4s = 4.0 * q.s;
    const unsigned long long wbase = c * WPC;
    uint32_t run = 0, bt = 0;  // hits so far, batch index within the chunk
    uint32_t pc = H.chunk_piece[c];
    uint32_t t0 = 0;           // chunk-relative candidate index of the next batch
    const uint32_t span = hi - lo;
    while (t0 < span) {
      // ---- up to 32 pieces, one per lane, clipped to the chunk ----
      const uint32_t mp = pc + lane;
      uint32_t ps = 0, pe = 0, pst = 0, pcert = 0;
      if (mp < np) {
        const uint64_t sl = (uint64_t)i * LS + mp;
        const uint32_t off = H.poff[sl], lf = H.plen[sl];
        const uint32_t len = lf & ~kCertainPiece;
        ps = max(off, lo) - lo;
        pe = min(off + len, hi);
        pe = pe > lo ? pe - lo : 0u;
        pst = H.pstart[sl] + (lo > off ? lo - off : 0u) - ps;  // position = pst + t
        pcert = lf & kCertainPiece;
      }
      // candidates [t0, wend) are covered by this group of pieces (pieces are
      // contiguous and non-empty; pieces past the chunk end clip to empty)
      const uint32_t pe31 = __shfl_sync(FULL, pe, 31);
      const uint32_t wend = pc + 32 >= np ? span : pe31;
      int R0 = -1;
      for (; t0 < wend; t0 += 32) {
        const uint32_t t = t0 + lane;
        const uint32_t sb = ps - t0;
        const uint32_t bit = (mp < np && pe > ps && sb < 32u) ? (1u << sb) : 0u;
        const uint32_t M = __reduce_or_sync(FULL, bit);
        const int r = min(R0 + __popc(M & le), 31);
        R0 += __popc(M);
        const uint32_t o_st = __shfl_sync(FULL, pst, r);
        const uint32_t o_cert = __shfl_sync(FULL, pcert, r);
        const bool act = t < wend;
        const uint32_t p = o_st + t;
        uint32_t m;
        if (MODE == QM_EMIT_BITS && bits) {
          m = H.bits[wbase + bt];
        } else if (!__any_sync(FULL, act && !o_cert)) {
          // a batch of certain candidates only (hub rows are mostly certain): no loads,
          // no tests
          m = __ballot_sync(FULL, act);
          if (MODE == QM_COUNT && bits && lane == 0) H.bits[wbase + bt] = m;
          if (MODE == QM_COUNT && A.stats) cert_total += __popc(m);
        } else {
          const bool test = act && !o_cert;
          const double2* xp = reinterpret_cast<const double2*>(A.pts + (test ? p : 0u));
          const double2 w0 = __ldg(xp), w1 = __ldg(xp + 1);
          const bool e = certified_edge(q.theta, q4s, q.a, q.b, w0, w1, T4, test);
          m = __ballot_sync(FULL, e || (act && o_cert));
          if (MODE == QM_COUNT && bits && lane == 0) H.bits[wbase + bt] = m;
          if (MODE == QM_COUNT && A.stats) {
            const uint32_t na = __popc(__ballot_sync(FULL, act));
            const uint32_t nc = __popc(__ballot_sync(FULL, act && o_cert));
            cand_total += na - nc;
            cert_total += nc;
          }
        }
        if (MODE != QM_COUNT && ((m >> lane) & 1u))
          write_edge<FMT>(A, base + run + __popc(m & lt), qid, ld_keep(A.sid2 + p, keep));
        run += __popc(m);
        ++bt;
      }
      t0 = wend;
      pc += 32;
    }
    if (MODE == QM_COUNT && lane == 0) {
      H.chunk_hits[c] = run;
      if (run) atomicAdd(&A.deg[A.poff ? i : qid], run);
    }
  }
  if (MODE == QM_COUNT && lane == 0) {
    if (cand_total) atomicAdd(&A.sc->candidates, cand_total);
    if (cert_total) atomicAdd(&A.sc->certain, cert_total);
  }
}

// ------------------------------------------------------------------ shard plan
// Work of the query items for the shard partition (k_shard.cu).
// Candidates of vertex q in slab j = the outer window's index range (the count the
// query kernels visit, tested + certain).
__device__ __forceinline__ uint32_t slab_candidates(const SlabC& S, const PointRec& q, uint32_t qkey,
                                                    double qinv4s, const BandConst& bc,
                                                    const uint32_t* __restrict__ dir) {
  if (S.nj == 0) return 0u;
  const double h0 = __fma_rn(q.a, S.B0, -__dmul_rn(q.b, S.A0));
  const double h1 = __fma_rn(q.a, S.B1, -__dmul_rn(q.b, S.A1));
  SlabWin<int32_t> w;
  win32(S, (int32_t)(qkey & kQMask), __fma_rn(-h0, h0, bc.T4), __fma_rn(-h1, h1, bc.T4), qinv4s,
        bc.T4min, dir, w);
  return w.dq == (1 << 30) ? S.nj : (uint32_t)(w.b - w.a);
}

// fp32 expected candidates of a vertex: E(r) = sum_k n_k min(1, W(r, c_k)/pi), k >= k0
__device__ __forceinline__ float expected_candidates(const PointRec& q, const SlabC* scs, int k0,
                                                     int L, float T4) {
  const float a = (float)q.a, b = (float)q.b;
  const float inv4s = 0.25f / fmaxf((float)q.s, 1e-30f);
  float E = 0.0f;
  for (int k = k0; k < L; ++k) {
    float frac = 1.0f;
    if (scs[k].invS != 0.0) {
      const float h = a * (float)scs[k].B0 - b * (float)scs[k].A0;  // 2 sinh((r - c_k)/2)
      const float ratio = (T4 - h * h) * inv4s * (float)scs[k].invS;
      if (ratio < 1.0f) frac = 0.63661977f * asinf(sqrtf(fmaxf(ratio, 0.0f)));
    }
    E += (float)scs[k].nj * frac;
  }
  return E;
}

// item t < heavy_end: hub vertex t, work = its exact candidate count (lane k: slab k);
// item heavy_end + g: light group g, work = sum of E(r) over its 32 vertices, scaled by
// exact / E of its first vertex (which catches the lumpy angular distribution of the
// few inner-slab points that every vertex of an arc sees).
__global__ void __launch_bounds__(256)
    k_shard_work(const QueryArgs A, const __grid_constant__ BandConst bc, int outward,
                 uint32_t* __restrict__ work) {
  __shared__ SlabC scs[kMaxBands];
  __shared__ uint32_t start[kMaxBands + 1];
  const int L = bc.L;
  if (threadIdx.x < (unsigned)L) {
    const int j = threadIdx.x;
    SlabC c;
    c.invS = bc.invS[j];
    c.padS = bc.padS[j];
    c.A0 = bc.A[j];
    c.B0 = bc.B[j];
    c.A1 = bc.A[j + 1];
    c.B1 = bc.B[j + 1];
    c.invS1 = bc.invS[j + 1];
    c.start = A.lay->start[j];
    c.nj = A.lay->start[j + 1] - c.start;
    c.off = A.lay->dir_off[j];
    c.sh = A.lay->shift[j];
    scs[j] = c;
  }
  if (threadIdx.x <= (unsigned)L) start[threadIdx.x] = A.lay->start[threadIdx.x];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t he = A.lay->heavy_end, nlight = A.n - he, ngroups = (nlight + 31u) / 32u;
  const uint32_t items = he + ngroups, warps = gridDim.x * (blockDim.x >> 5);
  const float T4f = (float)bc.T4;
  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += warps) {
    // representative vertex of the item (a hub, or the group's first vertex)
    const uint32_t k0 = it < he ? it : A.order[(it - he) * 32u];
    const uint32_t key0 = A.skey[k0], j0 = key0 >> kBandShift;
    const PointRec q0 = A.pts[k0 + start[j0]];
    const int kmin = outward ? (int)j0 : 0;
    uint32_t c = 0;
    if ((int)lane >= kmin && (int)lane < L)
      c = slab_candidates(scs[lane], q0, key0, 0.25 / q0.s, bc, A.dir);
    const float exact = (float)__reduce_add_sync(0xffffffffu, c);
    float w;
    if (it < he) {
      w = exact;
    } else {
      const uint32_t idx = (it - he) * 32u + lane;
      float e = 0.0f;
      if (idx < nlight) {
        const uint32_t k = A.order[idx];
        const uint32_t key = A.skey[k], j = key >> kBandShift;
        e = expected_candidates(A.pts[k + start[j]], scs, outward ? (int)j : 0, L, T4f);
      }
      const float e0 = __shfl_sync(0xffffffffu, e, 0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
      w = e0 > 0.0f ? e * (exact + 1.0f) / (e0 + 1.0f) : e;
    }
    if (lane == 0) work[it] = (uint32_t)fminf(ceilf(w) + 1.0f, 4.0e9f);
  }
}

cudaError_t launch_shard_work(const QueryArgs& qa, const BandConst& bc, int outward, uint32_t* work,
                              cudaStream_t st) {
  k_shard_work<<<num_sms() * 8, 256, 0, st>>>(qa, bc, outward, work);
  return cudaGetLastError();
}

cudaError_t launch_heavy_plan(rhg_format fmt, const QueryArgs& qa, const HeavyArgs& ha,
                              const BandConst& bc, void* scan_tmp, cudaStream_t st, int* launches) {
  uint32_t blocks = (uint32_t)((bc.heavy_cap + HV_WARPS - 1) / HV_WARPS);
  if (blocks > (uint32_t)num_sms() * 8) blocks = (uint32_t)num_sms() * 8;
  if (blocks < 1) blocks = 1;
  if (fmt == RHG_CSR) k_heavy_ranges<RHG_CSR><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  else k_heavy_ranges<RHG_EDGES_UNDIRECTED><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  cudaError_t e = exclusive_scan_u32_u64_dev(ha.vcap, &ha.meta->nvtx, ha.vtot, ha.vtot_off,
                                             scan_tmp, &ha.meta->cand, st, launches);
  if (e != cudaSuccess) return e;
  k_heavy_chunk_size<<<1, 1, 0, st>>>(ha);
  k_heavy_chunk_counts<<<num_sms() * 4, 256, 0, st>>>(ha);
  e = exclusive_scan_u32_u64_dev(ha.vcap, &ha.meta->nvtx, ha.cc, ha.choff, scan_tmp,
                                 &ha.meta->nchunks, st, launches);
  if (e != cudaSuccess) return e;
  k_heavy_chunk_map<<<blocks, HV_THREADS, 0, st>>>(ha, kRangesPerSlab * (uint32_t)bc.L);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

cudaError_t launch_heavy(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const HeavyArgs& ha,
                         const BandConst& bc, cudaStream_t st) {
  const uint32_t blocks = (uint32_t)num_sms() * RHG_HV_BLOCKS;
  if (mode == QM_COUNT) {
    if (fmt == RHG_CSR) k_heavy<QM_COUNT, RHG_CSR><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
    else k_heavy<QM_COUNT, RHG_EDGES_UNDIRECTED><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  } else if (mode == QM_EMIT) {
    if (fmt == RHG_CSR) k_heavy<QM_EMIT, RHG_CSR><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
    else k_heavy<QM_EMIT, RHG_EDGES_UNDIRECTED><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  } else {
    if (fmt == RHG_CSR) k_heavy<QM_EMIT_BITS, RHG_CSR><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
    else k_heavy<QM_EMIT_BITS, RHG_EDGES_UNDIRECTED><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  }
  return cudaGetLastError();
}

cudaError_t launch_query(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const BandConst& bc,
                         cudaStream_t st) {
  // one warp per light group (upper bound: hubs are excluded and a shard's range is
  // known on the device only)
  const uint32_t groups = ((qa.nquery_max ? qa.nquery_max : qa.n) + 31) / 32 + 1;
  const uint32_t blocks = (groups + QK_WARPS - 1) / QK_WARPS;
  if (blocks == 0) return cudaSuccess;
  // a slab may hold >= 2^30 points: 64-bit positions (or forced, rhg_options.wide_positions)
  const bool wide = qa.n >= (1u << 30) || qa.force_wide;
#define RHG_LQ(M, F, S)                                                                \
  do {                                                                                 \
    if (wide) k_query<M, F, true, S><<<blocks, QK_THREADS, 0, st>>>(qa, bc);           \
    else k_query<M, F, false, S><<<blocks, QK_THREADS, 0, st>>>(qa, bc);               \
  } while (0)
  const bool seq = qa.labels != 0;
  if (mode == QM_COUNT) {  // the count pass does not write ids
    if (fmt == RHG_CSR) RHG_LQ(QM_COUNT, RHG_CSR, false);
    else RHG_LQ(QM_COUNT, RHG_EDGES_UNDIRECTED, false);
  } else if (mode == QM_EMIT) {
    if (fmt == RHG_CSR) {
      if (seq) RHG_LQ(QM_EMIT, RHG_CSR, true); else RHG_LQ(QM_EMIT, RHG_CSR, false);
    } else {
      if (seq) RHG_LQ(QM_EMIT, RHG_EDGES_UNDIRECTED, true);
      else RHG_LQ(QM_EMIT, RHG_EDGES_UNDIRECTED, false);
    }
  } else {
    if (fmt == RHG_CSR) {
      if (seq) RHG_LQ(QM_EMIT_BITS, RHG_CSR, true); else RHG_LQ(QM_EMIT_BITS, RHG_CSR, false);
    } else {
      if (seq) RHG_LQ(QM_EMIT_BITS, RHG_EDGES_UNDIRECTED, true);
      else RHG_LQ(QM_EMIT_BITS, RHG_EDGES_UNDIRECTED, false);
    }
  }
#undef RHG_LQ
  return cudaGetLastError();
}

}  // namespace rhg
