// k_dynamic.cu -- the dynamic model of Sec. 3.3, SURVEY §8(f) row
// f1: per-vertex step values and one movement step (rotation + Algorithm 2 radial
// move with reflection), applied in place to device point arrays.  The graph of
// the moved points is then rebuilt by the static path (rhg_generate_from_points),
// which gives exactly the threshold edge set of the new positions.
#include "rhg_internal.cuh"

namespace rhg {

// Step values: Philox(key = seed, ctr = (i_lo, i_hi, 1, 0)) -- counter
// word 2 = 1 keeps them independent of the point sample (word 2 = 0), D1.
__global__ void k_movement_init(uint64_t n, uint64_t seed, double phi_lo, double phi_span,
                                double r_lo, double r_span, double* __restrict__ tau_phi,
                                double* __restrict__ tau_r) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 1u, 0u),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const uint64_t a = ((uint64_t)w.y << 32) | w.x, b = ((uint64_t)w.w << 32) | w.z;
    const double u1 = __dmul_rn((double)(a >> 11), 0x1.0p-53);
    const double u2 = __dmul_rn((double)(b >> 11), 0x1.0p-53);
    tau_phi[i] = __dadd_rn(phi_lo, __dmul_rn(phi_span, u1));
    tau_r[i] = __dadd_rn(r_lo, __dmul_rn(r_span, u2));
  }
}

// One movement step (PAPER.md:239 rotation; Alg. 2, radial move;
// PAPER.md:254 reflection, read as folding in the transformed coordinate y at 0 and
// sinh(alpha R), flipping tau_r once per fold, D2).
__global__ void k_move(uint64_t n, double* __restrict__ theta, double* __restrict__ r,
                       const double* __restrict__ tau_phi, double* __restrict__ tau_r, double R,
                       double alpha, double S) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double s = __dadd_rn(theta[i], tau_phi[i]);
    if (s >= RHG_TWO_PI_HI) s = __dsub_rn(s, RHG_TWO_PI_HI);
    else if (s < 0.0) s = __dadd_rn(s, RHG_TWO_PI_HI);
    if (s >= RHG_TWO_PI_HI || s < 0.0) s = 0.0;  // rounding at the seam
    theta[i] = s;
    double t = tau_r[i];
    double y = __dadd_rn(sinh(__dmul_rn(r[i], alpha)), t);
    for (int it = 0; it < 64 && (y < 0.0 || y > S); ++it) {
      y = y < 0.0 ? -y : __dsub_rn(__dmul_rn(2.0, S), y);
      t = -t;
    }
    y = fmin(fmax(y, 0.0), S);
    const double z = __ddiv_rn(asinh(y), alpha);
    r[i] = z > R ? R : z;
    tau_r[i] = t;
  }
}

static int grid_for(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  return (int)(b > (uint32_t)num_sms() * 16u ? (uint32_t)num_sms() * 16u : b);
}

cudaError_t launch_movement_init(uint64_t n, uint64_t seed, double phi_lo, double phi_hi,
                                 double r_lo, double r_hi, double* tau_phi, double* tau_r,
                                 cudaStream_t st) {
  k_movement_init<<<grid_for(n), 256, 0, st>>>(n, seed, phi_lo, phi_hi - phi_lo, r_lo, r_hi - r_lo,
                                               tau_phi, tau_r);
  return cudaGetLastError();
}

cudaError_t launch_move(uint64_t n, double* theta, double* r, const double* tau_phi, double* tau_r,
                        double R, double alpha, cudaStream_t st) {
  k_move<<<grid_for(n), 256, 0, st>>>(n, theta, r, tau_phi, tau_r, R, alpha, sinh(alpha * R));
  return cudaGetLastError();
}

}  // namespace rhg
