// k_sample.cu -- K1 (Philox point sampler) and K2 (band assignment, sort keys,
// band histogram), plus the band-layout kernel.
//
// Paper: Alg. 1 lines 6-10: draw phi ~ U[0, 2pi) and r with
// density f(r) = alpha sinh(alpha r)/(cosh(alpha R) - 1) (Eq. 1),
// insert into the slab b_i with c_i <= r < c_{i+1}.
#include <cmath>

#include "rhg_internal.cuh"

namespace rhg {

// Band j with c_j <= r < c_{j+1}; the last band is closed at R (Reading Z8).
__device__ __forceinline__ uint32_t band_of(double r, const BandConst& bc) {
  int j = bc.L - 1;
  while (j > 0 && r < bc.c[j]) --j;
  return (uint32_t)j;
}

// 27-bit fixed-point angle, monotone non-decreasing in theta.
__device__ __forceinline__ uint32_t q27_of(double theta) {
  uint32_t q = __double2uint_rz(__dmul_rn(theta, RHG_Q27_SCALE));
  return q > kQMax ? kQMax : q;
}

__global__ void k_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t* out) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < count;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint4 w = vertex_words(seed, i0 + t);
    reinterpret_cast<uint4*>(out)[t] = w;
  }
}

// Band of a point from its radial variate u2 (words_to_point): r(u2) is increasing,
// so c_j <= r < c_{j+1} iff ucut[j] <= u2 < ucut[j+1] -- decided here without the
// asinh / sqrt, except within a relative 2^-30 of a threshold (never, in practice),
// where r is evaluated and band_of decides (r's own rounding error is ~1e-16
// relative, far inside that margin).  Same band as band_of(r) for every point.
__device__ __forceinline__ uint32_t band_of_u(double u2, const PhiloxPoints& g, int L, bool& amb) {
  int j = L - 1;
  while (j > 0 && u2 < g.ucut[j]) --j;
  amb = (j > 0 && u2 < g.ucut[j] * (1.0 + 0x1.0p-30)) ||
        (j + 1 < L && u2 > g.ucut[j + 1] * (1.0 - 0x1.0p-30));
  return (uint32_t)j;
}

__global__ void __launch_bounds__(256)
    k_sample(uint64_t n, const __grid_constant__ PhiloxPoints gen,
             const __grid_constant__ BandConst bc, double* __restrict__ theta,
             double* __restrict__ r, uint32_t* __restrict__ keys, uint32_t* __restrict__ idx,
             uint32_t* __restrict__ band_hist) {
  __shared__ uint32_t hist[kMaxBands];
  if (threadIdx.x < kMaxBands) hist[threadIdx.x] = 0;
  __syncthreads();
  // keys only (the generate path): the band from u2, no radius
  const bool cuts = !r && !theta && (bc.L == 1 || gen.ucut[1] > 0.0);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double th, rr = 0.0;
    uint32_t j = 0;
    bool amb = true;
    const uint4 w = vertex_words(gen.seed, i);
    if (cuts) {
      const uint64_t a = ((uint64_t)w.y << 32) | w.x, b = ((uint64_t)w.w << 32) | w.z;
      th = __dmul_rn(RHG_TWO_PI_HI, __dmul_rn((double)(a >> 11), 0x1.0p-53));
      j = band_of_u(__dmul_rn((double)(b >> 11), 0x1.0p-53), gen, bc.L, amb);
    }
    if (amb) {
      words_to_point(w, gen.two_over_alpha, gen.half_span, bc.R, th, rr);
      if (theta) theta[i] = th;
      if (r) r[i] = rr;
      if (keys) j = band_of(rr, bc);
    }
    if (keys) {
      keys[i] = (j << kBandShift) | q27_of(th);
      idx[i] = (uint32_t)i;
      // one shared-memory add per band present in the warp
      const uint32_t peers = __match_any_sync(__activemask(), j);
      if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&hist[j], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  if (keys && threadIdx.x < kMaxBands && hist[threadIdx.x])
    atomicAdd(&band_hist[threadIdx.x], hist[threadIdx.x]);
}

__global__ void __launch_bounds__(256)
    k_keys_from_points(uint64_t n, const double* __restrict__ theta, const double* __restrict__ r,
                       const __grid_constant__ BandConst bc, uint32_t* __restrict__ keys,
                       uint32_t* __restrict__ idx, uint32_t* __restrict__ band_hist,
                       DevScalars* sc) {
  __shared__ uint32_t hist[kMaxBands];
  __shared__ uint32_t bad;
  if (threadIdx.x < kMaxBands) hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double th = theta[i], rr = r[i];
    // domain: theta in [0, 2pi), r in [0, R]; NaN fails both
    bool ok = (th >= 0.0) && (th < RHG_TWO_PI_HI) && (rr >= 0.0) && (rr <= bc.R);
    if (!ok) {
      bad = 1;
      th = 0.0;
      rr = 0.0;
    }
    uint32_t j = band_of(rr, bc);
    keys[i] = (j << kBandShift) | q27_of(th);
    idx[i] = (uint32_t)i;
    atomicAdd(&hist[j], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kMaxBands && hist[threadIdx.x]) atomicAdd(&band_hist[threadIdx.x], hist[threadIdx.x]);
  if (threadIdx.x == 0 && bad) atomicOr(&sc->domain_error, 1u);
}

// One warp: band offsets, bucket-directory geometry.  Buckets per band: the
// power of two >= 4 n_j (1/8 .. 1/4 point per bucket), capped at 2^27.
// Hub split: E_j = sum_k n_k min(1, dphi(c_j, c_k)/pi) bounds the expected
// candidate count of a vertex in band j (its radius is >= c_j and windows shrink
// with radius); bands with E_j above the
// threshold form the hub prefix [0, heavy_end) of the sorted order.
__global__ void k_band_layout(const __grid_constant__ BandConst bc,
                              const uint32_t* __restrict__ band_hist, BandLayout* lay,
                              HeavyMeta* meta) {
  const int L = bc.L;
  int j = threadIdx.x;
  uint32_t cnt = (j < L) ? band_hist[j] : 0u;
  uint32_t nb = 1, sh = kQBits;
  if (j < L) {
    // >= 4 buckets per point: range ends are whole buckets (no key probing in the
    // queries), so fine buckets keep the boundary-bucket overhead small
    uint32_t want = cnt > (1u << 25) ? (1u << 27) : RHG_DIR_PER_PT * cnt;
    while (nb < want && sh > 0) {
      nb <<= 1;
      --sh;
    }
  }
  uint32_t dsz = (j < L) ? nb + 1 : 0u;
  // inclusive warp scans
  uint32_t s_cnt = cnt, s_dir = dsz;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t a = __shfl_up_sync(0xffffffffu, s_cnt, o);
    uint32_t b = __shfl_up_sync(0xffffffffu, s_dir, o);
    if (j >= o) {
      s_cnt += a;
      s_dir += b;
    }
  }
  // expected candidates of a vertex sitting on band j's inner boundary
  double E = 0.0;
  if (j < L) {
    for (int k = 0; k < L; ++k) {
      double nk = (double)band_hist[k];
      if (nk == 0.0) continue;
      double frac = 1.0;
      if (bc.invS[j] != 0.0 && bc.invS[k] != 0.0) {
        double h = bc.A[j] * bc.B[k] - bc.B[j] * bc.A[k];
        double ratio = (bc.T4 - h * h) * (0.25 * bc.invS[j]) * bc.invS[k];
        if (ratio < 1.0) frac = 2.0 * asin(sqrt(fmax(ratio, 0.0))) / 3.141592653589793;
      }
      E += nk * frac;
    }
  }
  bool heavy = (j < L) && (E > bc.heavy_threshold);
  uint32_t hmask = __ballot_sync(0xffffffffu, heavy);
  // bands are ordered inner -> outer and E_j is non-increasing: hubs = prefix
  int J = __ffs(~hmask) - 1;  // first light band
  if (J < 0 || J > L) J = L;
  uint32_t startJ = __shfl_sync(0xffffffffu, s_cnt - cnt, J < 32 ? J : 31);
  uint32_t total = __shfl_sync(0xffffffffu, s_cnt, 31);
  if (J >= L) startJ = total;
  if (j < L) {
    lay->count[j] = cnt;
    lay->start[j] = s_cnt - cnt;
    lay->dir_off[j] = s_dir - dsz;
    lay->shift[j] = sh;
    lay->nb[j] = nb;
    lay->expected[j] = (float)E;
  }
  if (j == L - 1) {
    lay->start[L] = s_cnt;
    lay->dir_off[L] = s_dir;
  }
  if (j == 0) {
    uint32_t he = startJ < bc.heavy_cap ? startJ : bc.heavy_cap;
    lay->heavy_end = he;
    meta->nvtx = he;
    meta->list_len = he + (total - he + 31u) / 32u;
  }
}

static int grid_for(uint64_t n, int threads, int max_blocks) {
  uint64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b > (uint64_t)max_blocks ? max_blocks : b);
}

cudaError_t launch_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t* out,
                                cudaStream_t st) {
  k_philox_words<<<grid_for(count, 256, num_sms() * 16), 256, 0, st>>>(seed, i0, count, out);
  return cudaGetLastError();
}

cudaError_t launch_sample(uint64_t n, const PhiloxPoints& gen, const BandConst& bc, double* theta,
                          double* r, uint32_t* keys, uint32_t* idx, uint32_t* band_hist,
                          cudaStream_t st) {
  k_sample<<<grid_for(n, 256, num_sms() * 32), 256, 0, st>>>(n, gen, bc, theta, r, keys, idx,
                                                       band_hist);
  return cudaGetLastError();
}

cudaError_t launch_keys_from_points(uint64_t n, const double* theta, const double* r,
                                    const BandConst& bc, uint32_t* keys, uint32_t* idx,
                                    uint32_t* band_hist, DevScalars* sc, cudaStream_t st) {
  k_keys_from_points<<<grid_for(n, 256, num_sms() * 32), 256, 0, st>>>(n, theta, r, bc, keys, idx,
                                                                 band_hist, sc);
  return cudaGetLastError();
}

void set_band_cuts(PhiloxPoints& gen, double alpha, const BandConst& bc) {
  for (int j = 0; j <= kMaxBands; ++j) gen.ucut[j] = 0.0;
  for (int j = 1; j < bc.L; ++j) {
    const double s = std::sinh(0.5 * alpha * bc.c[j]);
    gen.ucut[j] = s * s / gen.half_span;
  }
}

cudaError_t launch_band_layout(const BandConst& bc, const uint32_t* band_hist, BandLayout* lay,
                               HeavyMeta* meta, cudaStream_t st) {
  k_band_layout<<<1, 32, 0, st>>>(bc, band_hist, lay, meta);
  return cudaGetLastError();
}

}  // namespace rhg
