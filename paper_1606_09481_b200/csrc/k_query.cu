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
// Work decomposition (B200): one warp owns 32 consecutive query vertices (same
// slab, neighbouring angles: their candidate ranges overlap, so the point SoA is
// read from L2, not HBM, once per neighbourhood).  Per slab each lane computes
// its vertex's ranges; the warp then walks the concatenation of the 32 lanes'
// ranges 32 candidates at a time, so every lane tests a candidate in every batch
// whatever the range lengths.  The owner of a candidate is found with one
// warp-wide OR of segment-start bits and a popcount (no search).  Hub vertices
// take the chunked path at the end of this file.
#include <type_traits>

#include "rhg_internal.cuh"

namespace rhg {

constexpr int QK_WARPS = 4;
constexpr int QK_THREADS = QK_WARPS * 32;
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t NO_BLOCK = 0xffffffffu;

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
  double2 qA[32];  // (theta, 4 sinh r)
  double2 qB[32];  // (e^{r/2}, e^{-r/2})
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

// Candidate set of one query vertex in slab j, in positions relative to the slab's
// doubled segment [0, 2 n_j): test the range [a, b) minus [h0, h1); [cs, ce) are
// certain edges.  (Non-full window: h0 = cs, h1 = ce; full window: the tested
// range is the complement of the certain one, hole empty.)
// I = int32_t when every slab has < 2^30 points (positions in [-n_j, 2 n_j] fit),
// int64_t otherwise.
template <typename I>
struct SlabWin {
  I a, b, h0, h1, cs, ce;
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
    return (I)(__ldg(dir + off + ((uint32_t)bu & nbm)) - bstart) + (per < 0 ? -nj : (per > 0 ? nj : (I)0));
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

template <int FMT>
__device__ __forceinline__ void write_edge(const QueryArgs& A, unsigned long long o, uint32_t vid,
                                           uint32_t w) {
  if (FMT == RHG_CSR) A.col[o] = w;
  else reinterpret_cast<uint2*>(A.pairs)[o] = vid < w ? make_uint2(vid, w) : make_uint2(w, vid);
}

// lanes [lo, hi) of a 32-bit mask (0 <= lo, hi <= 32)
__device__ __forceinline__ uint32_t lane_range_mask(int lo, int hi) {
  if (hi <= lo) return 0u;
  const uint32_t mh = hi >= 32 ? FULL : ((1u << hi) - 1u);
  return mh & ~((1u << lo) - 1u);
}

// Light vertices: one warp per 32 consecutive entries of the sector-major query
// order (sorted positions >= heavy_end).
//   QM_COUNT     : certain pieces counted, annulus candidates tested; deg[v];
//                  ballot words -> chained bit blocks
//   QM_EMIT      : same sequence, re-tests (fallback when the bit pool ran dry)
//   QM_EMIT_BITS : same sequence, replays the bits
template <int MODE, int FMT, bool WIDE>
__global__ void __launch_bounds__(QK_THREADS)
    k_query(const QueryArgs A, const __grid_constant__ BandConst bc) {
  using I = typename std::conditional<WIDE, int64_t, int32_t>::type;
  __shared__ WarpSm sm_all[QK_WARPS];
  __shared__ BandSm bs;
  load_band_sm(bs, A.lay, bc.L);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSm& sm = sm_all[wid];
  const uint32_t g = blockIdx.x * QK_WARPS + wid;  // light warp id
  const uint32_t nlight = A.n - A.lay->heavy_end;
  const uint32_t idx = g * 32u + lane;
  if (g * 32u >= nlight) return;
  const bool valid = idx < nlight;
  const uint32_t k = valid ? __ldg(A.order + idx) : 0u;
  const bool outward = (FMT == RHG_EDGES_UNDIRECTED);
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t le = (2u << lane) - 1u;  // lanes <= lane (lane 31: 2u << 31 == 0 -> all)

  uint32_t qkey = 0, qid = 0;
  if (valid) {
    qkey = A.skey[k];
    qid = A.sid[k];
  }
  const uint32_t qband = qkey >> kBandShift;
  const I qq = (I)(qkey & kQMask);
  PointRec q;
  q.theta = 0.0; q.s = 1.0; q.a = 1.0; q.b = 1.0;
  if (valid) q = A.pts[k + bs.start[qband]];  // first copy of the doubled slab
  const double qinv4s = 0.25 / q.s;
  sm.qA[lane] = make_double2(q.theta, 4.0 * q.s);
  sm.qB[lane] = make_double2(q.a, q.b);
  unsigned long long cur = 0;  // count: degree; emit: next row slot
  if (MODE != QM_COUNT && valid) cur = A.offs[qid];
  __syncwarp();

  // candidate-bit chain (count writes, emit replays)
  uint32_t blk = NO_BLOCK, t32 = 0, myword = 0;
  bool bits_ok = (MODE == QM_COUNT) && (A.bits != nullptr);
  if (MODE == QM_EMIT_BITS) {
    blk = A.warp_first[g];
    if (blk != NO_BLOCK) myword = A.bits[(uint64_t)blk * 32u + lane];
  }
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

  unsigned long long tested = 0, certain = 0;  // count-pass statistics (warp-uniform)
  int jlo = 0;
  if (outward) jlo = (int)__reduce_min_sync(FULL, valid ? qband : 0xffffu);
  const double T4 = bc.T4;

  // window numerator T4 - 4 sinh^2((r_v - c)/2) at c = c_j, carried from slab to slab
  double num_j;
  {
    const double h0 = __fma_rn(q.a, bc.B[jlo], -__dmul_rn(q.b, bc.A[jlo]));
    num_j = __fma_rn(-h0, h0, T4);
  }
  for (int j = jlo; j < bc.L; ++j) {
    const double h1 = __fma_rn(q.a, bc.B[j + 1], -__dmul_rn(q.b, bc.A[j + 1]));
    const double num_j1 = __fma_rn(-h1, h1, T4);
    const double num_here = num_j;
    num_j = num_j1;
    const uint32_t bstart = bs.start[j];
    const uint32_t nj = bs.start[j + 1] - bstart;
    if (nj == 0) continue;
    const uint32_t gbase = 2u * bstart;  // doubled segment of slab j
    const bool on = valid && (!outward || j >= (int)qband);
    SlabWin<I> w;
    w.a = w.b = w.h0 = w.h1 = w.cs = w.ce = 0;
    if (on) slab_window<I>(j, bc, bs, qq, num_here, num_j1, qinv4s, A.dir, w);
    const bool own = on && (j == (int)qband);
    const bool anyown = __any_sync(FULL, own);  // warp-uniform: only near slab boundaries / own slab
    I e1 = 0, wx = 0;
    if (own) {
      const I kv = (I)(k - bstart);
      if (outward) { e1 = 0; wx = kv + 1; } else { e1 = kv; wx = 1; }
    }
    // certain pieces
    I clo[2] = {w.cs, 0}, cln[2] = {w.ce - w.cs, 0};
    if (own) cut_piece<I>(w.cs, w.ce, e1, wx, (I)nj, clo[0], cln[0], clo[1], cln[1]);
    const uint32_t ct = (uint32_t)(cln[0] + cln[1]);
    const uint32_t nt = (uint32_t)((w.b - w.a) - (w.h1 - w.h0));

    if (MODE == QM_COUNT) {
      cur += ct;
      certain += ct;
    } else {
      // ---- certain edges: flattened copy of the 32 lanes' pieces ----
      const uint32_t cinc = warp_incl(ct);
      const uint32_t ctot = __shfl_sync(FULL, cinc, 31);
      if (ctot) {
        const uint32_t cex = cinc - ct;
        const uint32_t NEc = __ballot_sync(FULL, ct > 0);
        if (ct > 0) {
          CRec c;
          c.src0 = gbase + (uint32_t)clo[0] - cex;
          c.thr = cex + (uint32_t)cln[0];
          c.src1 = gbase + (uint32_t)clo[1] - cex - (uint32_t)cln[0];
          c.vid = qid;
          c.dst = cur - cex;
          c.pad = 0;
          sm.cr[__popc(NEc & lt)] = c;
        }
        __syncwarp();
        int R0 = -1;
        for (uint32_t t0 = 0; t0 < ctot; t0 += 32) {
          const uint32_t t = t0 + lane;
          const uint32_t s = cex - t0;
          const uint32_t bit = (ct > 0 && s < 32u) ? (1u << s) : 0u;
          const uint32_t M = __reduce_or_sync(FULL, bit);
          const int r = R0 + __popc(M & le);
          if (t < ctot) {
            const CRec c = sm.cr[r];
            const uint32_t src = (t < c.thr ? c.src0 : c.src1) + t;
            write_edge<FMT>(A, c.dst + t, c.vid, __ldg(A.sid2 + src));
          }
          R0 += __popc(M);
        }
        cur += ct;
        __syncwarp();
      }
    }

    // ---- annulus candidates: flattened exact tests ----
    const uint32_t tinc = warp_incl(nt);
    const uint32_t tot = __shfl_sync(FULL, tinc, 31);
    if (tot == 0) continue;
    const uint32_t tex = tinc - nt;
    {
      const uint32_t NE = __ballot_sync(FULL, nt > 0);
      if (nt > 0) {
        QRec rc;
        rc.aoff = gbase + (uint32_t)w.a - tex;
        rc.thr = tex + (uint32_t)(w.h0 - w.a);
        rc.hlen = (uint32_t)(w.h1 - w.h0);
        rc.lane = (uint32_t)lane;
        const int rk = __popc(NE & lt);
        sm.rec[rk] = rc;
        if (anyown) {
          XRec x;
          x.e1 = gbase + (uint32_t)e1;
          x.e2 = gbase + (uint32_t)e1 + nj;
          x.w = (uint32_t)wx;
          x.pad = 0;
          sm.xr[rk] = x;
        }
      }
    }
    __syncwarp();
    if (MODE == QM_COUNT) tested += tot;
    int R0 = -1;
    for (uint32_t t0 = 0; t0 < tot; t0 += 32) {
      const uint32_t t = t0 + lane;
      bool act = t < tot;
      const uint32_t s = tex - t0;
      const uint32_t bit = (nt > 0 && s < 32u) ? (1u << s) : 0u;
      const uint32_t M = __reduce_or_sync(FULL, bit);
      const int r = R0 + __popc(M & le);
      R0 += __popc(M);
      const QRec rc = sm.rec[r];
      const uint32_t p = rc.aoff + t + (t >= rc.thr ? rc.hlen : 0u);
      uint32_t hm;
      if (MODE == QM_EMIT_BITS) {
        hm = __shfl_sync(FULL, myword, t32);
      } else {
        if (anyown) {
          const XRec x = sm.xr[r];
          act = act && !((p - x.e1) < x.w || (p - x.e2) < x.w);
        }
        const double2* pp = reinterpret_cast<const double2*>(A.pts + (act ? p : 0u));
        const double2 w0 = __ldg(pp), w1 = __ldg(pp + 1);  // (theta, s), (a, b)
        const double2 qa_ = sm.qA[rc.lane], qb_ = sm.qB[rc.lane];
        hm = __ballot_sync(FULL, certified_edge(qa_.x, qa_.y, qb_.x, qb_.y, w0, w1, T4, act));
      }
      // my own candidates in this batch: lanes [tex - t0, tex + nt - t0) of the batch
      const int lo = max((int)tex - (int)t0, 0), hi = min((int)(tex + nt) - (int)t0, 32);
      const uint32_t mine = __popc(hm & lane_range_mask(lo, hi));
      if (MODE == QM_COUNT) {
        cur += mine;
        if (bits_ok) {
          if (lane == (int)t32) myword = hm;
          if (t32 == 31) flush_bits();
        }
      } else {
        const int o = (int)rc.lane;
        const uint32_t olo = (uint32_t)__shfl_sync(FULL, lo, o);
        const unsigned long long ocur = __shfl_sync(FULL, cur, o);
        uint32_t ovid = 0;
        if (FMT != RHG_CSR) ovid = __shfl_sync(FULL, qid, o);
        if ((hm >> lane) & 1u)
          write_edge<FMT>(A, ocur + __popc(hm & lt & ~((1u << olo) - 1u)), ovid,
                          __ldg(A.sid2 + p));
        cur += mine;
        if (MODE == QM_EMIT_BITS && t32 == 31) {
          blk = (blk != NO_BLOCK) ? A.bit_next[blk] : NO_BLOCK;
          if (blk != NO_BLOCK) myword = A.bits[(uint64_t)blk * 32u + lane];
        }
      }
      t32 = (t32 + 1) & 31u;
    }
    __syncwarp();
  }
  if (MODE == QM_COUNT) {
    if (bits_ok && t32 != 0) flush_bits();
    if (valid) A.deg[qid] = (uint32_t)cur;
    certain = warp_incl(certain);
    if (lane == 31) {
      atomicAdd(&A.sc->candidates, tested);
      atomicAdd(&A.sc->certain, certain);
    }
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
    const int j = lane;
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
    uint32_t cnt = 0, cand = 0, words = 0;
#pragma unroll
    for (int x = 0; x < 6; ++x) {
      cnt += ln[x] > 0;
      cand += (uint32_t)ln[x];
      if (x < (int)kTestPieces) words += ((uint32_t)ln[x] + 31u) >> 5;
    }
    const uint32_t ci = warp_incl(cnt), ca = warp_incl(cand), cw = warp_incl(words);
    uint32_t slot = i * LS + (ci - cnt), off = ca - cand, woff = cw - words;
#pragma unroll
    for (int x = 0; x < 6; ++x) {
      if (ln[x] > 0) {
        const uint32_t len = (uint32_t)ln[x];
        H.pstart[slot] = gbase + (uint32_t)lo[x];
        H.plen[slot] = len | (x < (int)kTestPieces ? 0u : kCertainPiece);
        H.poff[slot] = off;
        H.pword[slot] = woff;
        ++slot;
        off += len;
        if (x < (int)kTestPieces) woff += (len + 31u) >> 5;
      }
    }
    if (lane == 31) {
      H.np[i] = ci;
      H.vtot[i] = ca;
      H.vwords[i] = cw;
    }
    if (lane == 0) A.deg[A.sid[i]] = 0u;
  }
}

__global__ void k_heavy_chunk_size(const HeavyArgs H) {
  const unsigned long long C = H.meta->cand, nv = H.meta->nvtx;
  const unsigned long long room = H.chunk_cap > nv ? H.chunk_cap - nv : 1ull;
  unsigned long long ch = (C + room - 1) / room;  // sum_v ceil(C_v / ch) <= C / ch + nv
  if (ch < H.chunk_min) ch = H.chunk_min;
  ch = (ch + 31ull) & ~31ull;  // whole 32-candidate groups
  H.meta->chunk = ch;
  H.meta->bits_overflow = (H.meta->words > H.bits_cap) ? 1u : 0u;
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

template <int MODE, int FMT>
__global__ void __launch_bounds__(HV_THREADS)
    k_heavy(const QueryArgs A, const HeavyArgs H, const __grid_constant__ BandConst bc) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const unsigned long long gw = blockIdx.x * HV_WARPS + (threadIdx.x >> 5);
  const unsigned long long TW = (unsigned long long)gridDim.x * HV_WARPS;
  const unsigned long long nch = H.meta->nchunks, CH = H.meta->chunk;
  const uint32_t LS = kRangesPerSlab * (uint32_t)bc.L;
  const double T4 = bc.T4;
  const bool bits = !H.meta->bits_overflow;
  unsigned long long cand_total = 0, cert_total = 0;
  for (unsigned long long c = gw; c < nch; c += TW) {
    const uint32_t i = H.chunk_vtx[c];
    const unsigned long long c0 = H.choff[i];
    const unsigned long long lo = (c - c0) * CH, hi = lo + CH;
    const uint32_t np = H.np[i];
    const uint32_t qid = A.sid[i];
    unsigned long long base = 0;
    if (MODE != QM_COUNT) base = A.offs[qid] + (H.chunk_pos[c] - H.chunk_pos[c0]);
    const uint32_t qband = A.skey[i] >> kBandShift;
    const PointRec q = A.pts[i + A.lay->start[qband]];
    const double q4s = 4.0 * q.s;
    const unsigned long long wb = H.vwbase[i];
    uint32_t run = 0;
    for (uint32_t pc = H.chunk_piece[c]; pc < np; ++pc) {
      const uint64_t s = (uint64_t)i * LS + pc;
      const unsigned long long off = H.poff[s];
      if (off >= hi) break;
      const uint32_t lf = H.plen[s];
      const uint32_t len = lf & ~kCertainPiece;
      const uint32_t st = H.pstart[s];
      // groups k whose first candidate off + 32 k lies in [lo, hi)
      const uint32_t k0 = off >= lo ? 0u : (uint32_t)((lo - off + 31) >> 5);
      const uint32_t k1 = (uint32_t)min((unsigned long long)((len + 31u) >> 5), (hi - off + 31) >> 5);
      if (lf & kCertainPiece) {  // every candidate is an edge
        if (MODE == QM_COUNT) {
          const uint32_t m = min(32u * k1, len) - min(32u * k0, len);
          run += m;
          cert_total += m;
        } else {
          for (uint32_t k = k0; k < k1; k += 4) {  // 4 groups of loads in flight
            uint32_t w[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const uint32_t u = 32u * (k + g) + lane;
              w[g] = (k + g < k1 && u < len) ? __ldg(A.sid2 + st + u) : 0u;
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const uint32_t u = 32u * (k + g) + lane;
              if (k + g < k1 && u < len) write_edge<FMT>(A, base + run + lane, qid, w[g]);
              if (k + g < k1) run += min(32u, len - 32u * (k + g));
            }
          }
        }
        continue;
      }
      const unsigned long long wq = wb + H.pword[s];
      for (uint32_t k = k0; k < k1; k += 4) {  // 4 groups of loads in flight
        uint32_t m[4];
        uint32_t pp[4];
        if (MODE == QM_EMIT_BITS && bits) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            pp[g] = st + 32u * (k + g) + lane;
            m[g] = (k + g < k1) ? H.bits[wq + k + g] : 0u;
          }
        } else {
          double2 w0[4], w1[4];
          bool act[4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t u = 32u * (k + g) + lane;
            act[g] = (k + g < k1) && u < len;
            pp[g] = st + (act[g] ? u : 0u);
            const double2* xp = reinterpret_cast<const double2*>(A.pts + pp[g]);
            w0[g] = __ldg(xp);
            w1[g] = __ldg(xp + 1);
          }
#pragma unroll
          for (int g = 0; g < 4; ++g)
            m[g] = __ballot_sync(FULL, certified_edge(q.theta, q4s, q.a, q.b, w0[g], w1[g], T4, act[g]));
          if (MODE == QM_COUNT && bits && lane < 4 && k + lane < k1) {
            const uint32_t mine = lane == 0 ? m[0] : (lane == 1 ? m[1] : (lane == 2 ? m[2] : m[3]));
            H.bits[wq + k + lane] = mine;
          }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (MODE != QM_COUNT && ((m[g] >> lane) & 1u))
            write_edge<FMT>(A, base + run + __popc(m[g] & lt), qid, __ldg(A.sid2 + pp[g]));
          run += __popc(m[g]);
          if (MODE == QM_COUNT && k + g < k1) cand_total += min(32u, len - 32u * (k + g));
        }
      }
    }
    if (MODE == QM_COUNT && lane == 0) {
      H.chunk_hits[c] = run;
      if (run) atomicAdd(&A.deg[qid], run);
    }
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
  cudaError_t e = exclusive_scan_u32_u64_dev(ha.vcap, &ha.meta->nvtx, ha.vtot, ha.vtot_off,
                                             scan_tmp, &ha.meta->cand, st, launches);
  if (e != cudaSuccess) return e;
  e = exclusive_scan_u32_u64_dev(ha.vcap, &ha.meta->nvtx, ha.vwords, ha.vwbase, scan_tmp,
                                 &ha.meta->words, st, launches);
  if (e != cudaSuccess) return e;
  k_heavy_chunk_size<<<1, 1, 0, st>>>(ha);
  k_heavy_chunk_counts<<<148 * 4, 256, 0, st>>>(ha);
  e = exclusive_scan_u32_u64_dev(ha.vcap, &ha.meta->nvtx, ha.cc, ha.choff, scan_tmp,
                                 &ha.meta->nchunks, st, launches);
  if (e != cudaSuccess) return e;
  k_heavy_chunk_map<<<blocks, HV_THREADS, 0, st>>>(ha, kRangesPerSlab * (uint32_t)bc.L);
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
  const bool wide = qa.n >= (1u << 30);  // a slab may hold >= 2^30 points: 64-bit positions
#define RHG_LQ(M, F)                                                      \
  do {                                                                    \
    if (wide) k_query<M, F, true><<<blocks, QK_THREADS, 0, st>>>(qa, bc); \
    else k_query<M, F, false><<<blocks, QK_THREADS, 0, st>>>(qa, bc);     \
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
