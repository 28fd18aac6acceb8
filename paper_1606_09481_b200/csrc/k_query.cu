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
//  * The two annuli between the windows hold the candidates that need the exact
//    test, dist <= R, in the cancellation-free form of Eq. 3
//    (Z2):
//       h  = e^{r_v/2} e^{-r_w/2} - e^{-r_v/2} e^{r_w/2} = 2 sinh((r_v - r_w)/2)
//       S4 = h^2 + 4 sinh r_v sinh r_w sin^2(dphi/2)  = 2 (cosh d - 1)
//       edge iff S4 <= T4 = 4 sinh^2(R/2) = 2 (cosh R - 1).
//  * Index ranges come from the slab's bucket directory + a short binary search
//    (the binary search of PAPER.md:214); arcs that cross 2 pi split in two
//    (Z13).
//
// Work decomposition (B200): one warp owns 32 query vertices.  Per slab each lane
// computes its vertex's ranges; the ranges to test go to a shared-memory ring and
// the warp consumes the flattened candidate sequence 32 at a time (every lane
// tests a candidate in every batch regardless of range lengths).  Hub vertices
// take the chunked path at the end of this file.
#include "rhg_internal.cuh"

namespace rhg {

constexpr int QK_WARPS = 4;
constexpr int QK_THREADS = QK_WARPS * 32;
constexpr uint32_t RING = 256;   // >= 31 pending + 4 test ranges x 32 lanes appended per slab
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t NO_BLOCK = 0xffffffffu;
constexpr int kTest = 4;         // test ranges per (vertex, slab)
constexpr int kCert = 3;         // certain ranges per (vertex, slab)

struct WarpSm {
  double2 qA[32];                 // (theta, 4 sinh r)
  double2 qB[32];                 // (e^{r/2}, e^{-r/2})
  unsigned long long e_pref[RING];
  uint32_t e_start[RING];
  uint8_t e_lane[RING];
  unsigned long long cur[32];
  uint32_t degc[32];
  uint32_t qid[32];
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

// sin(d/2) = d * Q(u), u = d^2, Q(u) = sum_k (-1)^k u^k / (2 4^k (2k+1)!)
// short: |d| < 2^-4 (truncation < 3e-18 relative); long: |d| <= pi (+tiny), 12 terms.
__device__ __forceinline__ double poly_short(double u) {
  double p = -0x1.a01a01a01a01ap-20;
  p = __fma_rn(p, u, 0x1.1111111111111p-12);
  p = __fma_rn(p, u, -0x1.5555555555555p-6);
  p = __fma_rn(p, u, 0x1.0000000000000p-1);
  return p;
}
__device__ __forceinline__ double poly_long(double u) {
  double p = -0x1.761b41316381ap-98;
  p = __fma_rn(p, u, 0x1.71b8ef6dcf572p-87);
  p = __fma_rn(p, u, -0x1.2f49b46814157p-76);
  p = __fma_rn(p, u, 0x1.952c77030ad4ap-66);
  p = __fma_rn(p, u, -0x1.ae7f3e733b81fp-56);
  p = __fma_rn(p, u, 0x1.6124613a86d09p-46);
  p = __fma_rn(p, u, -0x1.ae64567f544e4p-37);
  p = __fma_rn(p, u, 0x1.71de3a556c734p-28);
  p = __fma_rn(p, u, -0x1.a01a01a01a01ap-20);
  p = __fma_rn(p, u, 0x1.1111111111111p-12);
  p = __fma_rn(p, u, -0x1.5555555555555p-6);
  p = __fma_rn(p, u, 0x1.0000000000000p-1);
  return p;
}

// first index p in band (given by its directory) with q(p) >= q; q in [0, 2^27]
// (q = 2^27 returns the band end).
__device__ __forceinline__ uint32_t dir_lower(const uint32_t* __restrict__ skey,
                                              const uint32_t* __restrict__ dir, uint32_t off,
                                              uint32_t sh, uint32_t q, uint32_t bend) {
  if (q > kQMax) return bend;
  const uint32_t b = q >> sh;
  uint32_t lo = __ldg(dir + off + b), hi = __ldg(dir + off + b + 1);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(skey + mid) & kQMask) < q) lo = mid + 1; else hi = mid;
  }
  return lo;
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

// The certified test of one (query, candidate) pair, evaluated identically (bit
// for bit) from either endpoint: S4 = h^2 + 4 s_v s_w sin^2(dphi/2) <= T4.
// All lanes of the warp must call it (warp-uniform choice of the sin polynomial).
// q4s = 4 sinh r_v; w0 = (theta_w, sinh r_w), w1 = (e^{r_w/2}, e^{-r_w/2}).
__device__ __forceinline__ bool certified_edge(double qth, double q4s, double qa, double qb,
                                               double2 w0, double2 w1, double T4, bool act) {
  double d = __dsub_rn(qth, w0.x);
  const uint32_t dhi = (uint32_t)__double2hiint(d) & 0x7fffffffu;
  const bool big = act && dhi >= 0x3FB00000u;  // |d| >= 2^-4: long polynomial
  double Qv;
  if (__any_sync(FULL, big)) {
    if (dhi >= 0x400921FBu) {  // |d| >~ pi: the short way round crosses the seam
      const double mx = fmax(qth, w0.x), mn = fmin(qth, w0.x);
      d = __dadd_rn(__dadd_rn(__dsub_rn(RHG_TWO_PI_HI, mx), mn), RHG_TWO_PI_LO);
    }
    const double u = __dmul_rn(d, d);
    Qv = big ? poly_long(u) : poly_short(u);
  } else {
    Qv = poly_short(__dmul_rn(d, d));
  }
  const double sn = __dmul_rn(d, Qv);              // sin(dphi/2)
  const double Bv = __dmul_rn(sn, sn);
  const double p1 = __dmul_rn(qa, w1.y);           // e^{r_v/2} e^{-r_w/2}
  const double p2 = __dmul_rn(qb, w1.x);           // e^{-r_v/2} e^{r_w/2}
  const double h = __dsub_rn(p1, p2);              // 2 sinh((r_v - r_w)/2)
  const double A4 = __dmul_rn(q4s, w0.y);          // 4 sinh r_v sinh r_w
  const double C = __dmul_rn(A4, Bv);
  const double S4 = __fma_rn(h, h, C);
  return act && (S4 <= T4);
}

// Unwrapped index interval [s, e) of a slab with nj points (s in [-nj, 2nj),
// 0 <= e - s <= nj, relative to the slab start) -> <= 2 real ranges in slots x, x+1.
__device__ __forceinline__ void put_interval(int64_t s, int64_t e, uint32_t bstart, uint32_t nj,
                                             uint32_t* lo, uint32_t* hi, int x) {
  if (e <= s) return;
  const int64_t len = e - s;
  if (s < 0) s += nj;
  else if (s >= (int64_t)nj) s -= nj;
  if (s + len <= (int64_t)nj) {
    lo[x] = bstart + (uint32_t)s;
    hi[x] = bstart + (uint32_t)(s + len);
  } else {
    lo[x] = bstart + (uint32_t)s;
    hi[x] = bstart + nj;
    lo[x + 1] = bstart;
    hi[x + 1] = bstart + (uint32_t)(s + len - nj);
  }
}

struct SlabRanges {
  uint32_t tlo[kTest], thi[kTest];  // to test
  uint32_t clo[kCert], chi[kCert];  // certain edges
};

// Own slab: the undirected list keeps only partners sorted after v (DESIGN.md
// Z9); CSR cuts v itself out of whichever range holds it.
__device__ __forceinline__ void own_slab_cut(bool outward, uint32_t k, SlabRanges& rg) {
    if (outward) {
#pragma unroll
      for (int x = 0; x < kTest; ++x) rg.tlo[x] = max(rg.tlo[x], min(k + 1, rg.thi[x]));
#pragma unroll
      for (int x = 0; x < kCert; ++x) rg.clo[x] = max(rg.clo[x], min(k + 1, rg.chi[x]));
    } else {
#pragma unroll
      for (int x = 0; x < 2; ++x)
        if (rg.clo[x] <= k && k < rg.chi[x]) {
          rg.clo[2] = k + 1;
          rg.chi[2] = rg.chi[x];
          rg.chi[x] = k;
        }
      // test ranges: at most 3 of the 4 slots are in use (only one arc can wrap)
#pragma unroll
      for (int x = 0; x < kTest; ++x) {
        if (rg.tlo[x] <= k && k < rg.thi[x]) {
          const uint32_t tail_hi = rg.thi[x];
          rg.thi[x] = k;
          bool placed = false;
#pragma unroll
          for (int y = 0; y < kTest; ++y) {
            if (!placed && y != x && !(rg.thi[y] > rg.tlo[y])) {
              rg.tlo[y] = k + 1;
              rg.thi[y] = tail_hi;
              placed = true;
            }
          }
        }
      }
    }
}

// Ranges of one query vertex (sorted position k, key q) in slab j (general
// 64-bit version: hub vertices and slabs of >= 2^27 points).
__device__ __forceinline__ void slab_ranges(int j, const BandConst& bc, const BandSm& B, uint32_t q,
                                            double qa, double qb, double qinv4s, uint32_t k,
                                            uint32_t qband, bool outward,
                                            const uint32_t* __restrict__ skey,
                                            const uint32_t* __restrict__ dir, SlabRanges& rg) {
  const uint32_t bstart = B.start[j], bend = B.start[j + 1], nj = bend - bstart;
#pragma unroll
  for (int x = 0; x < kTest; ++x) rg.tlo[x] = rg.thi[x] = bend;
#pragma unroll
  for (int x = 0; x < kCert; ++x) rg.clo[x] = rg.chi[x] = bend;
  const double T4 = bc.T4;
  // ---- outer window at c_j (superset) ----
  const double h = __fma_rn(qa, bc.B[j], -__dmul_rn(qb, bc.A[j]));
  const double num = __fma_rn(-h, h, T4);  // T4 - 4 sinh^2((r_v - c_j)/2)
  bool full = false;
  int64_t d_o = 0;
  const double invS = bc.invS[j];
  if (invS == 0.0) {
    full = true;  // c_j = 0: the innermost slab reaches every angle
  } else {
    const double scale = __dmul_rn(qinv4s, invS);
    const double ratio = __fma_rn(num, scale, __dmul_rn(T4 * 0x1.0p-48, scale));
    if (!(ratio < 0.99)) {
      full = true;
    } else {
      // dphi <= 2 tan(dphi/2) = 2 sqrt(ratio / (1 - ratio)); pad 2^-12, +2 quanta
      const float rf = fmaxf((float)ratio, 0.0f);
      const float t = __fsqrt_rn(rf) * rsqrtf(1.0f - rf);
      const float dqf = t * (2.0f * (float)RHG_Q27_SCALE * 1.000244140625f);
      if (dqf >= 67108860.0f) full = true;
      else d_o = (int64_t)dqf + 2;
    }
  }
  // ---- inner window at c_{j+1} (certain subset) ----
  int64_t d_i = -1;
  {
    const double h1 = __fma_rn(qa, bc.B[j + 1], -__dmul_rn(qb, bc.A[j + 1]));
    const double num1 = __fma_rn(-h1, h1, T4);
    const double invS1 = bc.invS[j + 1];
    if (invS1 != 0.0 && num >= T4 * 0x1.0p-10 && num1 >= T4 * 0x1.0p-10) {
      // dphi_in >= 2 asin(sqrt(ratio1)) >= 2 sqrt(ratio1); shrink 2^-17, -1 quantum
      const double ratio1 = __dmul_rn(__dmul_rn(num1, __dmul_rn(qinv4s, invS1)), 1.0 - 0x1.0p-30);
      const float rf1 = fminf((float)ratio1, 1.0f);
      const float dif = __fsqrt_rn(rf1) * (2.0f * (float)RHG_Q27_SCALE * 0.99999237060546875f);
      d_i = (int64_t)dif - 1;
    }
  }
  // Bucket-only boundaries (no key probing): outer ends round outward to whole
  // buckets, certain ends round inward; boundary-bucket points land in the tested
  // annuli, so {left test, certain, right test} still partition the outer window.
  // Unwrapped bucket b maps to the unwrapped slab position P(b) (periodic in nb).
  const uint32_t sh = B.shift[j], off = B.dir_off[j];
  const uint32_t lgnb = kQBits - sh, nbm = (1u << lgnb) - 1u;
  auto P = [&](int64_t bu) -> int64_t {
    const uint32_t bi = (uint32_t)bu & nbm;
    return (int64_t)(__ldg(dir + off + bi) - bstart) + (bu >> lgnb) * (int64_t)nj;
  };
  const int64_t qq = (int64_t)q;
  int64_t ls = 0, re = 0, cs = 0, ce = 0;
  if (!full) {
    ls = P((qq - d_o) >> sh);
    re = P(((qq + d_o) >> sh) + 1);
    if (re - ls >= (int64_t)nj) full = true;
  }
  bool cert = false;
  if (d_i >= 0) {
    cs = P(((qq - d_i) >> sh) + 1);
    ce = P((qq + d_i) >> sh);
    cert = ce > cs;
  }
  if (cert) {
    put_interval(cs, ce, bstart, nj, rg.clo, rg.chi, 0);
    if (full) {
      put_interval(ce, cs + nj, bstart, nj, rg.tlo, rg.thi, 0);
    } else {
      put_interval(ls, cs, bstart, nj, rg.tlo, rg.thi, 0);
      put_interval(ce, re, bstart, nj, rg.tlo, rg.thi, 2);
    }
  } else if (full) {
    rg.tlo[0] = bstart;
    rg.thi[0] = bend;
  } else {
    put_interval(ls, re, bstart, nj, rg.tlo, rg.thi, 0);
  }
  if (j == (int)qband) own_slab_cut(outward, k, rg);
}



__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// [a, b) in [0, 2 nj) relative positions -> <= 2 slab ranges (split at the seam nj)
__device__ __forceinline__ void split_at_seam(int32_t a, int32_t b, int32_t nj, uint32_t bstart,
                                              uint32_t& lo0, uint32_t& hi0, uint32_t& lo1,
                                              uint32_t& hi1) {
  if (b <= nj) {
    lo0 = bstart + a; hi0 = bstart + b;
  } else if (a >= nj) {
    lo0 = bstart + (a - nj); hi0 = bstart + (b - nj);
  } else {
    lo0 = bstart + a; hi0 = bstart + nj;
    lo1 = bstart; hi1 = bstart + (b - nj);
  }
}

// Same ranges as slab_ranges (below), 32-bit positions (slabs < 2^27 points), MUFU
// square roots (their ~2^-22 relative error is inside the 2^-12 / 2^-17 pads) and
// the window numerators supplied by the caller: num = T4 - h(c_j)^2,
// num1 = T4 - h(c_{j+1})^2 (num1 of slab j is num of slab j+1).
__device__ __forceinline__ void slab_ranges_fast(int j, const BandConst& bc, const BandSm& B,
                                                 int32_t q, double num, double num1,
                                                 double qinv4s, uint32_t k, uint32_t qband,
                                                 bool outward, const uint32_t* __restrict__ dir,
                                                 SlabRanges& rg) {
  const uint32_t bstart = B.start[j], bend = B.start[j + 1];
  const int32_t nj = (int32_t)(bend - bstart);
#pragma unroll
  for (int x = 0; x < kTest; ++x) rg.tlo[x] = rg.thi[x] = bstart;
#pragma unroll
  for (int x = 0; x < kCert; ++x) rg.clo[x] = rg.chi[x] = bstart;
  // outer window at c_j: d_o >= 2 tan(dphi/2) K27 (1 + 2^-12) + 2
  bool full = true;
  int32_t d_o = 0;
  const double invS = bc.invS[j];
  if (invS != 0.0) {
    const double ratio = __fma_rn(num, __dmul_rn(qinv4s, invS), __dmul_rn(qinv4s, bc.padS[j]));
    if (ratio < 0.99) {
      const float rf = fmaxf((float)ratio, 0.0f);
      const float dqf = sqrt_approx(rf) * rsqrt_approx(1.0f - rf) *
                        (2.0f * (float)RHG_Q27_SCALE * 1.000244140625f);
      if (dqf < 67108860.0f) {
        full = false;
        d_o = (int32_t)dqf + 2;
      }
    }
  }
  // certain window at c_{j+1}: d_i <= 2 sqrt(ratio1) K27 (1 - 2^-17) - 1
  int32_t d_i = -1;
  const double invS1 = bc.invS[j + 1];
  if (invS1 != 0.0 && num >= bc.T4min && num1 >= bc.T4min) {
    const float rf1 = fminf((float)__dmul_rn(num1, __dmul_rn(qinv4s, invS1)), 1.0f);
    d_i = (int32_t)(sqrt_approx(rf1) * (2.0f * (float)RHG_Q27_SCALE * 0.99999237060546875f)) - 1;
  }
  const uint32_t sh = B.shift[j], off = B.dir_off[j];
  const uint32_t lgnb = kQBits - sh, nbm = (1u << lgnb) - 1u;
  auto P = [&](int32_t bu) -> int32_t {  // unwrapped bucket -> unwrapped slab position
    const int32_t per = bu >> lgnb;       // -1, 0 or 1
    return (int32_t)(__ldg(dir + off + ((uint32_t)bu & nbm)) - bstart) + per * nj;
  };
  int32_t ls = 0, re = 0, cs = 0, ce = 0;
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
  if (!cert) {
    if (full) {
      rg.thi[0] = bend;
    } else {
      const int32_t sft = ls < 0 ? nj : (ls >= nj ? -nj : 0);
      split_at_seam(ls + sft, re + sft, nj, bstart, rg.tlo[0], rg.thi[0], rg.tlo[1], rg.thi[1]);
    }
  } else {
    const int32_t sft = cs < 0 ? nj : (cs >= nj ? -nj : 0);
    cs += sft; ce += sft;
    split_at_seam(cs, ce, nj, bstart, rg.clo[0], rg.chi[0], rg.clo[1], rg.chi[1]);
    if (full) {
      split_at_seam(ce, cs + nj, nj, bstart, rg.tlo[0], rg.thi[0], rg.tlo[1], rg.thi[1]);
    } else {
      ls += sft; re += sft;
      // [ls, cs) may dip below 0 and [ce, re) may pass 2 nj: shift them into range
      if (ls < 0) split_at_seam(ls + nj, cs + nj, nj, bstart, rg.tlo[0], rg.thi[0], rg.tlo[1], rg.thi[1]);
      else split_at_seam(ls, cs, nj, bstart, rg.tlo[0], rg.thi[0], rg.tlo[1], rg.thi[1]);
      if (re > 2 * nj) split_at_seam(ce - nj, re - nj, nj, bstart, rg.tlo[2], rg.thi[2], rg.tlo[3], rg.thi[3]);
      else split_at_seam(ce, re, nj, bstart, rg.tlo[2], rg.thi[2], rg.tlo[3], rg.thi[3]);
    }
  }
  if (j == (int)qband) own_slab_cut(outward, k, rg);
}

__device__ __forceinline__ void write_edge(const QueryArgs& A, unsigned long long o, uint32_t vid,
                                           uint32_t w, int fmt) {
  if (fmt == RHG_CSR) A.col[o] = w;
  else reinterpret_cast<uint2*>(A.pairs)[o] = vid < w ? make_uint2(vid, w) : make_uint2(w, vid);
}

// Light vertices: one warp per 32 consecutive sorted positions >= heavy_end.
//   QM_COUNT     : certain ranges counted, annulus candidates tested; deg[v];
//                  ballot words -> chained bit blocks
//   QM_EMIT      : same sequence, re-tests (fallback when the bit pool ran dry)
//   QM_EMIT_BITS : same sequence, replays the bits
template <int MODE, int FMT, bool WIDE>
__global__ void __launch_bounds__(QK_THREADS)
    k_query(const QueryArgs A, const __grid_constant__ BandConst bc) {
  __shared__ WarpSm sm_all[QK_WARPS];
  __shared__ BandSm bs;
  load_band_sm(bs, A.lay, bc.L);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSm& sm = sm_all[wid];
  const uint32_t g = blockIdx.x * QK_WARPS + wid;  // light warp id
  const uint32_t first = A.lay->heavy_end + g * 32u;
  if (first >= A.n) return;
  const uint32_t k = first + lane;
  const bool valid = k < A.n;
  const bool outward = (FMT == RHG_EDGES_UNDIRECTED);
  const uint32_t lt = (1u << lane) - 1u;

  PointRec q;
  q.theta = 0.0; q.s = 1.0; q.a = 1.0; q.b = 1.0;
  uint32_t qkey = 0, qid = 0;
  if (valid) {
    q = A.pts[k];
    qkey = A.skey[k];
    qid = A.sid[k];
  }
  const uint32_t qband = qkey >> kBandShift, qq = qkey & kQMask;
  const double qinv4s = 0.25 / q.s;
  sm.qA[lane] = make_double2(q.theta, 4.0 * q.s);
  sm.qB[lane] = make_double2(q.a, q.b);
  sm.qid[lane] = qid;
  if (MODE == QM_COUNT) sm.degc[lane] = 0;
  else sm.cur[lane] = valid ? A.offs[qid] : 0ull;
  __syncwarp();
  uint32_t deg_certain = 0;

  // candidate-bit chain (count writes, emit replays)
  uint32_t blk = NO_BLOCK, t32 = 0, myword = 0;
  bool bits_ok = (MODE == QM_COUNT) && (A.bits != nullptr);
  if (MODE == QM_EMIT_BITS) {
    blk = A.warp_first[g];
    if (blk != NO_BLOCK) myword = A.bits[(uint64_t)blk * 32u + lane];
  }

  unsigned long long total = 0, consumed = 0;
  uint32_t head = 0xffffffffu, tail = 0;  // ring entry "-1": nothing consumed yet
  int jlo = 0;
  if (outward) jlo = (int)__reduce_min_sync(FULL, valid ? qband : 0xffffu);
  const double T4 = bc.T4;

  auto flush_bits = [&]() {
    uint32_t nb = NO_BLOCK;
    if (lane == 0) {
      const uint32_t sub = g & (kBitSubPools - 1);
      const uint32_t idx = atomicAdd(&A.pool_cursor[sub], 1u);
      if (idx < A.pool_sub_blocks) nb = sub * A.pool_sub_blocks + idx;
    }
    nb = __shfl_sync(FULL, nb, 0);
    if (nb == NO_BLOCK) {
      bits_ok = false;
      if (lane == 0) atomicOr(&A.sc->bit_overflow, 1u);
      return;
    }
    if (lane == 0) {
      A.bit_next[nb] = NO_BLOCK;  // chain terminator (the emit pass reads one link ahead)
      if (blk == NO_BLOCK) A.warp_first[g] = nb;
      else A.bit_next[blk] = nb;
    }
    A.bits[(uint64_t)nb * 32u + lane] = myword;
    blk = nb;
  };

  // one batch: candidates [consumed, consumed + cnt) of the flattened test-range
  // sequence, cnt = min(32, total - consumed); lane l takes candidate consumed + l.
  auto batch = [&]() {
    const uint32_t cnt = (uint32_t)min(32ull, total - consumed);
    const bool act = (uint32_t)lane < cnt;
    // `head` holds candidate consumed - 1 (or is exhausted); ranges head+1 ..
    // head+32 that start at consumed .. consumed + 31 mark bit (start - consumed).
    const uint32_t e = head + 1u + lane;
    uint32_t bit = 0;
    if (e < tail) {
      if (WIDE) {
        const unsigned long long rel = sm.e_pref[e % RING] - consumed;
        if (rel < 32ull) bit = 1u << (uint32_t)rel;
      } else {  // ranges < 2^27: the 32 entries ahead start < 2^32 after `consumed`
        const uint32_t rel = (uint32_t)sm.e_pref[e % RING] - (uint32_t)consumed;
        if (rel < 32u) bit = 1u << rel;
      }
    }
    const uint32_t M = __reduce_or_sync(FULL, bit);
    const uint32_t my_e = (head + __popc(M & ((2u << lane) - 1u))) % RING;
    const uint32_t ql = sm.e_lane[my_e];
    const uint32_t cand =
        act ? sm.e_start[my_e] + (uint32_t)lane + ((uint32_t)consumed - (uint32_t)sm.e_pref[my_e])
            : 0u;
    uint32_t hm;
    if (MODE == QM_EMIT_BITS) {
      hm = __shfl_sync(FULL, myword, t32);
    } else {
      const double2* pp = reinterpret_cast<const double2*>(A.pts + cand);
      const double2 w0 = __ldg(pp), w1 = __ldg(pp + 1);  // (theta, s), (a, b)
      const double2 qa_ = sm.qA[ql], qb_ = sm.qB[ql];
      hm = __ballot_sync(FULL, certified_edge(qa_.x, qa_.y, qb_.x, qb_.y, w0, w1, T4, act));
    }
    const bool hit = (hm >> lane) & 1u;
    if (MODE == QM_COUNT) {
      if (hit) atomicAdd(&sm.degc[ql], 1u);
      if (bits_ok) {
        if (lane == (int)t32) myword = hm;
        if (t32 == 31) flush_bits();
      }
    } else {
      const uint32_t peers = __match_any_sync(FULL, act ? ql : (32u + lane));
      const unsigned long long base = act ? sm.cur[ql] : 0ull;
      if (hit) write_edge(A, base + __popc(hm & peers & lt), sm.qid[ql], __ldg(A.sid + cand), FMT);
      __syncwarp();
      if (act && (__ffs(peers) - 1) == lane) sm.cur[ql] = base + __popc(hm & peers);
      if (MODE == QM_EMIT_BITS && t32 == 31) {
        blk = (blk != NO_BLOCK) ? A.bit_next[blk] : NO_BLOCK;
        if (blk != NO_BLOCK) myword = A.bits[(uint64_t)blk * 32u + lane];
      }
    }
    t32 = (t32 + 1) & 31u;
    consumed += cnt;
    head += __popc(M);
    __syncwarp();
  };

  // window numerator T4 - 4 sinh^2((r_v - c)/2) at c = c_j, carried from slab to slab
  double num_j = 0.0;
  if (!WIDE) {
    const double h0 = __fma_rn(q.a, bc.B[jlo], -__dmul_rn(q.b, bc.A[jlo]));
    num_j = __fma_rn(-h0, h0, T4);
  }
  for (int j = jlo; j < bc.L; ++j) {
    double num_j1 = 0.0;
    if (!WIDE) {
      const double h1 = __fma_rn(q.a, bc.B[j + 1], -__dmul_rn(q.b, bc.A[j + 1]));
      num_j1 = __fma_rn(-h1, h1, T4);
    }
    const double num_here = num_j;
    num_j = num_j1;
    if (bs.start[j] == bs.start[j + 1]) continue;
    SlabRanges rg;
#pragma unroll
    for (int x = 0; x < kTest; ++x) rg.tlo[x] = rg.thi[x] = 0;
#pragma unroll
    for (int x = 0; x < kCert; ++x) rg.clo[x] = rg.chi[x] = 0;
    if (valid && (!outward || j >= (int)qband)) {
      if (WIDE)
        slab_ranges(j, bc, bs, qq, q.a, q.b, qinv4s, k, qband, outward, A.skey, A.dir, rg);
      else
        slab_ranges_fast(j, bc, bs, (int32_t)qq, num_here, num_j1, qinv4s, k, qband, outward,
                         A.dir, rg);
    }
    uint32_t cc[kCert];
    uint32_t ccs = 0;
#pragma unroll
    for (int x = 0; x < kCert; ++x) {
      cc[x] = rg.chi[x] > rg.clo[x] ? rg.chi[x] - rg.clo[x] : 0u;
      ccs += cc[x];
    }
    if (MODE == QM_COUNT) {
      deg_certain += ccs;
    } else {
      // ---- certain edges: flattened, coalesced id copy into each vertex's row ----
      // (per-warp certain totals are < 2^32: every lane's ranges lie in one slab)
      const uint32_t cinc = warp_incl(ccs);
      const uint32_t ctot = __shfl_sync(FULL, cinc, 31);
      if (ctot) {
        const uint32_t cex = cinc - ccs;
        const unsigned long long cbase = sm.cur[lane];
        const uint32_t cb_lo = (uint32_t)cbase, cb_hi = (uint32_t)(cbase >> 32);
        for (uint32_t t0 = 0; t0 < ctot; t0 += 32) {
          const uint32_t t = t0 + lane;
          // owner lane: the last lane whose exclusive prefix is <= t (register search)
          uint32_t own = 0;
#pragma unroll
          for (uint32_t stp = 16; stp > 0; stp >>= 1) {
            const uint32_t p = __shfl_sync(FULL, cex, own + stp);
            own = (p <= t) ? own + stp : own;
          }
          const uint32_t oex = __shfl_sync(FULL, cex, own);
          const uint32_t n0 = __shfl_sync(FULL, cc[0], own), n1 = __shfl_sync(FULL, cc[1], own);
          const uint32_t l0 = __shfl_sync(FULL, rg.clo[0], own);
          const uint32_t l1 = __shfl_sync(FULL, rg.clo[1], own);
          const uint32_t l2 = __shfl_sync(FULL, rg.clo[2], own);
          const uint32_t blo = __shfl_sync(FULL, cb_lo, own), bhi = __shfl_sync(FULL, cb_hi, own);
          const uint32_t ovid = __shfl_sync(FULL, qid, own);
          if (t < ctot) {
            const uint32_t r = t - oex;
            const uint32_t src = r < n0 ? l0 + r : (r < n0 + n1 ? l1 + (r - n0) : l2 + (r - n0 - n1));
            const unsigned long long ob = ((unsigned long long)bhi << 32) | blo;
            write_edge(A, ob + r, ovid, __ldg(A.sid + src), FMT);
          }
        }
        sm.cur[lane] = cbase + ccs;
        __syncwarp();
      }
    }
    // ---- annulus candidates: append the test ranges to the ring ----
    uint32_t ct[kTest];
    unsigned long long ne = 0, cs = 0;
#pragma unroll
    for (int x = 0; x < kTest; ++x) {
      ct[x] = rg.thi[x] > rg.tlo[x] ? rg.thi[x] - rg.tlo[x] : 0u;
      ne += (ct[x] > 0);
      cs += ct[x];
    }
    const unsigned long long packed = (ne << 56) | cs;  // one scan for slots and candidates
    const unsigned long long inc = warp_incl(packed);
    const unsigned long long tot = __shfl_sync(FULL, inc, 31);
    const unsigned long long cs_tot = tot & ((1ull << 56) - 1);
    if (cs_tot == 0) continue;
    {
      const unsigned long long ex = inc - packed;
      uint32_t slot = tail + (uint32_t)(ex >> 56);
      unsigned long long pref = total + (ex & ((1ull << 56) - 1));
#pragma unroll
      for (int x = 0; x < kTest; ++x) {
        if (ct[x]) {
          sm.e_start[slot % RING] = rg.tlo[x];
          sm.e_pref[slot % RING] = pref;
          sm.e_lane[slot % RING] = (uint8_t)lane;
          ++slot;
          pref += ct[x];
        }
      }
    }
    tail += (uint32_t)(tot >> 56);
    total += cs_tot;
    __syncwarp();
    while (total - consumed >= 32ull) batch();
  }
  while (total > consumed) batch();
  if (MODE == QM_COUNT) {
    if (bits_ok && t32 != 0) flush_bits();
    __syncwarp();
    if (valid) A.deg[qid] = sm.degc[lane] + deg_certain;
    const unsigned long long dc = warp_incl((unsigned long long)deg_certain);
    if (lane == 31) {
      atomicAdd(&A.sc->candidates, total);
      atomicAdd(&A.sc->certain, dc);
    }
  }
}

// ------------------------------------------------------------------ hub path
// Hub vertices (sorted positions [0, heavy_end), chosen by k_band_layout) have
// 10^3..10^6 candidates each.  Their ranges are materialised per (vertex, slab,
// piece) slot -- pieces 0..3 to test, 4..6 certain -- cut into chunks of >=
// chunk_min candidates, and the chunks are spread over every warp of the GPU.
// Output placement stays deterministic: the hits of chunk c land at
// offs[v] + (chunk_pos[c] - chunk_pos[first chunk of v]).
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
  const bool outward = (FMT == RHG_EDGES_UNDIRECTED);
  for (uint32_t i = gw; i < he; i += TW) {
    const PointRec q = A.pts[i];
    const uint32_t qkey = A.skey[i];
    const uint32_t qband = qkey >> kBandShift, qq = qkey & kQMask;
    const double qinv4s = 0.25 / q.s;
    if (lane == 0) A.deg[A.sid[i]] = 0u;
    if (lane < L) {
      const int j = lane;
      SlabRanges rg;
#pragma unroll
      for (int x = 0; x < kTest; ++x) rg.tlo[x] = rg.thi[x] = 0;
#pragma unroll
      for (int x = 0; x < kCert; ++x) rg.clo[x] = rg.chi[x] = 0;
      if (bs.start[j] < bs.start[j + 1] && (!outward || j >= (int)qband))
        slab_ranges(j, bc, bs, qq, q.a, q.b, qinv4s, i, qband, outward, A.skey, A.dir, rg);
      const uint64_t s0 = ((uint64_t)i * (uint64_t)L + (uint64_t)j) * kRangesPerSlab;
#pragma unroll
      for (int x = 0; x < (int)kRangesPerSlab; ++x) {
        const uint32_t lo = x < kTest ? rg.tlo[x] : rg.clo[x - kTest];
        const uint32_t hi = x < kTest ? rg.thi[x] : rg.chi[x - kTest];
        const uint32_t len = hi > lo ? hi - lo : 0u;
        H.start[s0 + x] = lo;
        H.len[s0 + x] = len;
        H.lenw[s0 + x] = x < kTest ? (len + 31u) >> 5 : 0u;  // bits only for tested pieces
      }
    }
  }
}

__global__ void k_heavy_chunk_size(const HeavyArgs H) {
  const unsigned long long C = H.meta->cand;
  const unsigned long long extra = H.chunk_cap - H.nslots_cap;
  unsigned long long ch = (C + extra - 1) / extra;
  if (ch < H.chunk_min) ch = H.chunk_min;
  ch = (ch + 63ull) & ~63ull;  // whole bit words per 32-candidate batch
  H.meta->chunk = ch;
  H.meta->bits_overflow = (H.meta->words > H.bits_cap) ? 1u : 0u;
}

__global__ void k_heavy_chunk_counts(const HeavyArgs H) {
  const unsigned long long ns = H.meta->nslots, ch = H.meta->chunk;
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < ns;
       s += (unsigned long long)gridDim.x * blockDim.x)
    H.cc[s] = (uint32_t)((H.len[s] + ch - 1) / ch);
}

__global__ void k_heavy_chunk_map(const HeavyArgs H) {
  const unsigned long long ns = H.meta->nslots;
  for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < ns;
       s += (unsigned long long)gridDim.x * blockDim.x)
    for (unsigned long long c = H.choff[s]; c < H.choff[s + 1]; ++c) H.chunk_slot[c] = (uint32_t)s;
}

template <int MODE, int FMT>
__global__ void __launch_bounds__(HV_THREADS)
    k_heavy(const QueryArgs A, const HeavyArgs H, const __grid_constant__ BandConst bc) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const unsigned long long gw = blockIdx.x * HV_WARPS + (threadIdx.x >> 5);
  const unsigned long long TW = (unsigned long long)gridDim.x * HV_WARPS;
  const unsigned long long nch = H.meta->nchunks, CH = H.meta->chunk;
  const unsigned long long LS = (unsigned long long)kRangesPerSlab * (unsigned long long)bc.L;
  const double T4 = bc.T4;
  const bool bits = !H.meta->bits_overflow;
  unsigned long long cand_total = 0, cert_total = 0;
  for (unsigned long long c = gw; c < nch; c += TW) {
    const uint32_t s = H.chunk_slot[c];
    const uint32_t i = (uint32_t)(s / LS);
    const bool certain = (s % kRangesPerSlab) >= (uint32_t)kTest;
    const unsigned long long k = c - H.choff[s];
    const uint32_t b0 = H.start[s] + (uint32_t)(k * CH);
    const uint32_t e0 = (uint32_t)min((unsigned long long)H.start[s] + H.len[s],
                                      (unsigned long long)b0 + CH);
    const uint32_t qid = A.sid[i];
    unsigned long long base = 0;
    if (MODE != QM_COUNT)
      base = A.offs[qid] + (H.chunk_pos[c] - H.chunk_pos[H.choff[(unsigned long long)i * LS]]);
    if (certain) {  // every candidate is an edge
      if (MODE == QM_COUNT) {
        if (lane == 0) {
          H.chunk_hits[c] = e0 - b0;
          atomicAdd(&A.deg[qid], e0 - b0);
        }
        cert_total += e0 - b0;
      } else {
        for (uint32_t p = b0 + lane; p < e0; p += 32)
          write_edge(A, base + (p - b0), qid, __ldg(A.sid + p), FMT);
      }
      continue;
    }
    const PointRec q = A.pts[i];
    const double q4s = 4.0 * q.s;
    const unsigned long long wbase = H.soffw[s] + (k * CH) / 32ull;  // word-aligned bits
    uint32_t run = 0;
    for (uint32_t p0 = b0; p0 < e0; p0 += 64) {  // two batches in flight per warp
      const uint32_t pa = p0 + lane, pb = p0 + 32 + lane;
      const bool aa = pa < e0, ab = pb < e0;
      const unsigned long long wi = wbase + (p0 - b0) / 32u;
      uint32_t ma, mb;
      if (MODE == QM_EMIT_BITS && bits) {
        ma = H.bits[wi];
        mb = (p0 + 32 < e0) ? H.bits[wi + 1] : 0u;
      } else {
        const double2* xa = reinterpret_cast<const double2*>(A.pts + (aa ? pa : b0));
        const double2* xb = reinterpret_cast<const double2*>(A.pts + (ab ? pb : b0));
        const double2 w0a = __ldg(xa), w1a = __ldg(xa + 1);
        const double2 w0b = __ldg(xb), w1b = __ldg(xb + 1);
        ma = __ballot_sync(FULL, certified_edge(q.theta, q4s, q.a, q.b, w0a, w1a, T4, aa));
        mb = __ballot_sync(FULL, certified_edge(q.theta, q4s, q.a, q.b, w0b, w1b, T4, ab));
        if (MODE == QM_COUNT && bits && lane == 0) {
          H.bits[wi] = ma;
          if (p0 + 32 < e0) H.bits[wi + 1] = mb;
        }
      }
      if (MODE != QM_COUNT) {
        if ((ma >> lane) & 1u) write_edge(A, base + run + __popc(ma & lt), qid, __ldg(A.sid + pa), FMT);
        run += __popc(ma);
        if ((mb >> lane) & 1u) write_edge(A, base + run + __popc(mb & lt), qid, __ldg(A.sid + pb), FMT);
        run += __popc(mb);
      } else {
        run += __popc(ma) + __popc(mb);
      }
    }
    if (MODE == QM_COUNT && lane == 0) {
      H.chunk_hits[c] = run;
      if (run) atomicAdd(&A.deg[qid], run);
    }
    cand_total += e0 - b0;
  }
  if (MODE == QM_COUNT && lane == 0) {
    if (cand_total) atomicAdd(&A.sc->candidates, cand_total);
    if (cert_total) atomicAdd(&A.sc->certain, cert_total);
  }
}

cudaError_t launch_heavy_plan(rhg_format fmt, const QueryArgs& qa, const HeavyArgs& ha,
                              const BandConst& bc, void* scan_tmp, cudaStream_t st, int* launches) {
  uint32_t blocks = (uint32_t)((bc.heavy_cap + HV_WARPS - 1) / HV_WARPS);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  if (fmt == RHG_CSR) k_heavy_ranges<RHG_CSR><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  else k_heavy_ranges<RHG_EDGES_UNDIRECTED><<<blocks, HV_THREADS, 0, st>>>(qa, ha, bc);
  cudaError_t e = exclusive_scan_u32_u64_dev(ha.nslots_cap, &ha.meta->nslots, ha.len, ha.soff,
                                             scan_tmp, &ha.meta->cand, st, launches);
  if (e != cudaSuccess) return e;
  e = exclusive_scan_u32_u64_dev(ha.nslots_cap, &ha.meta->nslots, ha.lenw, ha.soffw, scan_tmp,
                                 &ha.meta->words, st, launches);
  if (e != cudaSuccess) return e;
  k_heavy_chunk_size<<<1, 1, 0, st>>>(ha);
  k_heavy_chunk_counts<<<148 * 4, 256, 0, st>>>(ha);
  e = exclusive_scan_u32_u64_dev(ha.nslots_cap, &ha.meta->nslots, ha.cc, ha.choff, scan_tmp,
                                 &ha.meta->nchunks, st, launches);
  if (e != cudaSuccess) return e;
  k_heavy_chunk_map<<<148 * 4, 256, 0, st>>>(ha);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

cudaError_t launch_heavy(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const HeavyArgs& ha,
                         const BandConst& bc, cudaStream_t st) {
  const uint32_t blocks = 148 * 8;
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
  const uint32_t groups = (qa.n + 31) / 32;
  const uint32_t blocks = (groups + QK_WARPS - 1) / QK_WARPS;
  if (blocks == 0) return cudaSuccess;
  const bool wide = qa.n >= (1u << 27);  // slabs may exceed 2^27 points: 64-bit positions
#define RHG_LQ(M, F)                                                                   \
  do {                                                                                 \
    if (wide) k_query<M, F, true><<<blocks, QK_THREADS, 0, st>>>(qa, bc);              \
    else k_query<M, F, false><<<blocks, QK_THREADS, 0, st>>>(qa, bc);                  \
  } while (0)
  if (mode == QM_COUNT) {
    if (fmt == RHG_CSR) RHG_LQ(QM_COUNT, RHG_CSR);
    else RHG_LQ(QM_COUNT, RHG_EDGES_UNDIRECTED);
  } else if (mode == QM_EMIT) {
    if (fmt == RHG_CSR) RHG_LQ(QM_EMIT, RHG_CSR);
    else RHG_LQ(QM_EMIT, RHG_EDGES_UNDIRECTED);
  } else {
    if (fmt == RHG_CSR) RHG_LQ(QM_EMIT_BITS, RHG_CSR);
    else RHG_LQ(QM_EMIT_BITS, RHG_EDGES_UNDIRECTED);
  }
#undef RHG_LQ
  return cudaGetLastError();
}

}  // namespace rhg
