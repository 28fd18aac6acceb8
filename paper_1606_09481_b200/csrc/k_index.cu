// k_index.cu -- K4: gather the query SoA in (band, angle) order and build the
// per-band bucket directory that replaces most of the binary search of
// PAPER.md:214 ("find the leftmost and rightmost neighbor candidate in each slab
// using binary search").
#include "rhg_internal.cuh"

namespace rhg {

// Point record for sorted position k: theta, sinh r, e^{r/2}, e^{-r/2}.
// (cosh d - 1 = 2 sinh^2((r_p - r_q)/2) + 2 sinh r_p sinh r_q sin^2(dphi/2), and
//  2 sinh((r_p - r_q)/2) = e^{r_p/2} e^{-r_q/2} - e^{-r_p/2} e^{r_q/2}.)
__global__ void __launch_bounds__(256)
    k_gather(uint32_t n, const double* __restrict__ theta, const double* __restrict__ r,
             const uint32_t* __restrict__ sidx, PointRec* __restrict__ pts) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    uint32_t i = sidx[k];
    double rr = r[i];
    PointRec p;
    p.theta = theta[i];
    p.s = sinh(rr);
    p.a = exp(0.5 * rr);
    p.b = exp(-0.5 * rr);
    pts[k] = p;
  }
}

// Generate path: the points are re-derived from Philox(seed, i) (bit-identical to
// K1, same device code) instead of gathering theta[i], r[i] at random addresses.
__global__ void __launch_bounds__(256)
    k_gather_philox(uint32_t n, uint64_t seed, double two_over_alpha, double half_span, double R,
                    const uint32_t* __restrict__ sidx, PointRec* __restrict__ pts) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t i = sidx[k];
    double th, rr;
    words_to_point(vertex_words(seed, i), two_over_alpha, half_span, R, th, rr);
    PointRec p;
    p.theta = th;
    p.s = sinh(rr);
    p.a = exp(0.5 * rr);
    p.b = exp(-0.5 * rr);
    pts[k] = p;
  }
}

// dir[dir_off[j] + b] = first sorted index of band j whose bucket >= b, for
// b = 0 .. nb_j (entry nb_j = band end).  Thread k fills the entries in
// (bucket(k-1), bucket(k)]; the last point of a band also fills the tail.
__global__ void __launch_bounds__(256)
    k_directory(uint32_t n, const uint32_t* __restrict__ skey, const BandLayout* __restrict__ lay,
                int L, uint32_t* __restrict__ dir) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    uint32_t key = skey[k];
    uint32_t j = key >> kBandShift;
    uint32_t sh = lay->shift[j], off = lay->dir_off[j];
    uint32_t b = (key & kQMask) >> sh;
    int64_t prev = -1;
    if (k > lay->start[j]) prev = (int64_t)((skey[k - 1] & kQMask) >> sh);
    for (int64_t bb = prev + 1; bb <= (int64_t)b; ++bb) dir[off + bb] = k;
    if (k + 1 == lay->start[j + 1]) {
      uint32_t nb = lay->nb[j];
      for (uint32_t bb = b + 1; bb <= nb; ++bb) dir[off + bb] = k + 1;
    }
  }
  // empty bands: both entries = band start
  if (blockIdx.x == 0 && threadIdx.x < (unsigned)L) {
    int j = threadIdx.x;
    if (lay->count[j] == 0) {
      uint32_t off = lay->dir_off[j], nb = lay->nb[j];
      for (uint32_t bb = 0; bb <= nb; ++bb) dir[off + bb] = lay->start[j];
    }
  }
}

cudaError_t launch_build_index(uint32_t n, const double* theta, const double* r,
                               const uint32_t* skey, const uint32_t* sidx, const BandLayout* lay,
                               int L, PointRec* pts, uint32_t* dir, const PhiloxPoints* gen,
                               cudaStream_t st, int* launches) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  if (gen)
    k_gather_philox<<<blocks, 256, 0, st>>>(n, gen->seed, gen->two_over_alpha, gen->half_span,
                                            gen->R, sidx, pts);
  else
    k_gather<<<blocks, 256, 0, st>>>(n, theta, r, sidx, pts);
  k_directory<<<blocks, 256, 0, st>>>(n, skey, lay, L, dir);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

}  // namespace rhg
