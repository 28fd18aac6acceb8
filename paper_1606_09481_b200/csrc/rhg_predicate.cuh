// rhg_predicate.cuh -- the point record and the certified edge test of the B200
// path (device code shared by the index build, the query kernels and the dynamic
// update).  Nothing here is shared with oracle/ (DESIGN.md).
#pragma once
#include "rhg_internal.cuh"

namespace rhg {

// Point record: theta, sinh r, e^{r/2}, e^{-r/2}.
// (cosh d - 1 = 2 sinh^2((r_p - r_q)/2) + 2 sinh r_p sinh r_q sin^2(dphi/2), and
//  2 sinh((r_p - r_q)/2) = e^{r_p/2} e^{-r_q/2} - e^{-r_p/2} e^{r_q/2}.)
// The query record of one point: e^{r/2} from exp, e^{-r/2} as its correctly
// rounded reciprocal, and sinh r = (e^{r/2} - e^{-r/2})(e^{r/2} + e^{-r/2}) / 2 for
// r >= 1 (no cancellation there: the first factor is >= 2 sinh(1/2)), sinh() below.
// A few ulp from libm's values at most -- far inside the near-tie window the edge
// predicate is checked against; both endpoints of a pair read the same record.
__device__ __forceinline__ PointRec point_rec(double th, double rr) {
  PointRec p;
  p.theta = th;
  p.a = exp(0.5 * rr);
  p.b = __drcp_rn(p.a);
  p.s = rr >= 1.0 ? 0.5 * ((p.a - p.b) * (p.a + p.b)) : sinh(rr);
  return p;
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
  if (__any_sync(0xffffffffu, big)) {
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

// Same test when every candidate of the warp is known to have |dphi| < 2^-4 (and no
// seam crossing): the short polynomial, which certified_edge also picks for such
// pairs, so the decision is the same bit for bit from either endpoint.
__device__ __forceinline__ bool certified_edge_short(double qth, double q4s, double qa, double qb,
                                                     double2 w0, double2 w1, double T4, bool act) {
  const double d = __dsub_rn(qth, w0.x);
  const double sn = __dmul_rn(d, poly_short(__dmul_rn(d, d)));
  const double Bv = __dmul_rn(sn, sn);
  const double h = __dsub_rn(__dmul_rn(qa, w1.y), __dmul_rn(qb, w1.x));
  const double C = __dmul_rn(__dmul_rn(q4s, w0.y), Bv);
  return act && (__fma_rn(h, h, C) <= T4);
}


}  // namespace rhg
