// k_stats.cu -- on-device validation statistics of a generated graph (SURVEY §8(f)
// row f4): degree histogram, mean / max degree, the discrete
// maximum-likelihood tail exponent over degrees >= k_min (compared with gamma,
// PAPER.md:78), and the number of emitted edges inside the north star's near-tie
// window |cosh d - cosh R| <= 1e-12 cosh R.  Everything stays on the device; only
// the small result struct is copied back.
#include "rhg_internal.cuh"

namespace rhg {

constexpr int ST_THREADS = 256;

struct StatsAcc {
  unsigned long long edges_dir, tail_n, max_deg, near_ties;
  double tail_log;
  unsigned long long hist[RHG_STATS_BINS];
};

__device__ __forceinline__ uint32_t deg_bin(uint64_t d) {
  // bin 0: degree 0; bin b >= 1: degrees in [2^(b-1), 2^b)
  return d == 0 ? 0u : min(64u - (uint32_t)__clzll((long long)d), (uint32_t)RHG_STATS_BINS - 1u);
}

// pairs format: degree of every vertex by counting endpoints
__global__ void k_stats_pair_degrees(uint64_t m, const uint32_t* __restrict__ pairs,
                                     uint32_t* __restrict__ deg) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    atomicAdd(&deg[pairs[2 * e]], 1u);
    atomicAdd(&deg[pairs[2 * e + 1]], 1u);
  }
}

__global__ void __launch_bounds__(ST_THREADS)
    k_stats_degrees(uint32_t n, const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ deg,
                    double kmin, StatsAcc* acc) {
  __shared__ unsigned long long hist[RHG_STATS_BINS];
  if (threadIdx.x < RHG_STATS_BINS) hist[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long tail_n = 0, mx = 0, tot = 0;
  double tail_log = 0.0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint64_t d = row_ptr ? row_ptr[v + 1] - row_ptr[v] : deg[v];
    tot += d;
    mx = d > mx ? d : mx;
    if ((double)d >= kmin) {
      ++tail_n;
      tail_log += log((double)d / (kmin - 0.5));
    }
    atomicAdd(&hist[deg_bin(d)], 1ull);
  }
  for (int o = 16; o > 0; o >>= 1) {
    tail_n += __shfl_xor_sync(0xffffffffu, tail_n, o);
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
    tail_log += __shfl_xor_sync(0xffffffffu, tail_log, o);
    const unsigned long long om = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = om > mx ? om : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc->tail_n, tail_n);
    atomicAdd(&acc->edges_dir, tot);
    atomicAdd(&acc->tail_log, tail_log);
    atomicMax(&acc->max_deg, mx);
  }
  __syncthreads();
  if (threadIdx.x < RHG_STATS_BINS && hist[threadIdx.x]) atomicAdd(&acc->hist[threadIdx.x], hist[threadIdx.x]);
}

// |cosh d - cosh R| <= 1e-12 cosh R  <=>  |S4 - T4| <= 2e-12 cosh R with the
// cancellation-free S4 = 4 sinh^2((r_u - r_v)/2) + 4 sinh r_u sinh r_v sin^2(dphi/2)
__device__ __forceinline__ bool near_tie(double tu, double ru, double tv, double rv, double T4,
                                         double tol) {
  double d = fabs(tu - tv);
  if (d > 3.141592653589793) d = (RHG_TWO_PI_HI - fmax(tu, tv) + fmin(tu, tv)) + RHG_TWO_PI_LO;
  const double h = 2.0 * sinh(0.5 * (ru - rv));
  const double s = sin(0.5 * d);
  const double S4 = h * h + 4.0 * sinh(ru) * sinh(rv) * s * s;
  return fabs(S4 - T4) <= tol;
}

__global__ void __launch_bounds__(ST_THREADS)
    k_stats_ties_csr(uint32_t n, const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                     const double* __restrict__ theta, const double* __restrict__ r, double T4,
                     double tol, StatsAcc* acc) {
  unsigned long long c = 0;
  // warp per row: lanes over the row's entries with u < v
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (gridDim.x * blockDim.x) >> 5) {
    const double tu = theta[u], ru = r[u];
    for (uint64_t e = row_ptr[u] + lane; e < row_ptr[u + 1]; e += 32) {
      const uint32_t v = col[e];
      if (v > u && near_tie(tu, ru, theta[v], r[v], T4, tol)) ++c;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0 && c) atomicAdd(&acc->near_ties, c);
}

__global__ void __launch_bounds__(ST_THREADS)
    k_stats_ties_pairs(uint64_t m, const uint32_t* __restrict__ pairs, const double* __restrict__ theta,
                       const double* __restrict__ r, double T4, double tol, StatsAcc* acc) {
  unsigned long long c = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = pairs[2 * e], v = pairs[2 * e + 1];
    if (near_tie(theta[u], r[u], theta[v], r[v], T4, tol)) ++c;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&acc->near_ties, c);
}

size_t stats_workspace_bytes(uint64_t n) { return sizeof(StatsAcc) + 4 * (n + 64) + 256; }

cudaError_t launch_graph_stats(uint32_t n, int fmt, const uint64_t* row_ptr, const uint32_t* col,
                               const uint32_t* pairs, uint64_t m, const double* theta,
                               const double* r, double R, double kmin, void* ws,
                               rhg_stats* host_out, cudaStream_t st) {
  StatsAcc* acc = (StatsAcc*)ws;
  uint32_t* deg = (uint32_t*)((char*)ws + ((sizeof(StatsAcc) + 255) & ~(size_t)255));
  cudaError_t e = cudaMemsetAsync(acc, 0, sizeof(StatsAcc), st);
  if (e != cudaSuccess) return e;
  const int blocks = num_sms() * 8;
  if (fmt != RHG_CSR) {
    if ((e = cudaMemsetAsync(deg, 0, 4ull * n, st)) != cudaSuccess) return e;
    k_stats_pair_degrees<<<blocks, ST_THREADS, 0, st>>>(m, pairs, deg);
    k_stats_degrees<<<blocks, ST_THREADS, 0, st>>>(n, nullptr, deg, kmin, acc);
  } else {
    k_stats_degrees<<<blocks, ST_THREADS, 0, st>>>(n, row_ptr, nullptr, kmin, acc);
  }
  if (theta && r) {
    const double h = std::sinh(R / 2.0), T4 = 4.0 * h * h;
    const double tol = 2e-12 * std::cosh(R);
    if (fmt == RHG_CSR) k_stats_ties_csr<<<blocks, ST_THREADS, 0, st>>>(n, row_ptr, col, theta, r, T4, tol, acc);
    else k_stats_ties_pairs<<<blocks, ST_THREADS, 0, st>>>(m, pairs, theta, r, T4, tol, acc);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  StatsAcc h;
  if ((e = cudaMemcpyAsync(&h, acc, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  host_out->num_edges = fmt == RHG_CSR ? h.edges_dir / 2 : h.edges_dir / 2;
  host_out->max_degree = h.max_deg;
  host_out->mean_degree = n ? (double)h.edges_dir / n : 0.0;
  host_out->tail_count = h.tail_n;
  host_out->tail_exponent = h.tail_log > 0.0 ? 1.0 + (double)h.tail_n / h.tail_log : 0.0;
  host_out->near_ties = (theta && r) ? h.near_ties : ~0ull;
  for (int b = 0; b < RHG_STATS_BINS; ++b) host_out->degree_hist[b] = h.hist[b];
  return cudaSuccess;
}

}  // namespace rhg
