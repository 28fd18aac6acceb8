// rhg_internal.cuh -- shared definitions of the B200 product path (kernels + host
// orchestration).  Nothing here is shared with oracle/ (see DESIGN.md).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rhg.h"

namespace rhg {

constexpr int kMaxBands = 32;          // L <= 32: n < 2^32 => ceil(log2 n) <= 32
constexpr int kBandShift = 27;         // sort key = band << 27 | q27(theta)
constexpr uint32_t kQBits = 27;
constexpr uint32_t kQMax = (1u << kQBits) - 1u;
constexpr uint32_t kQMask = kQMax;

// fl(2*pi) and the remainder 2*pi - fl(2*pi): seam differences (Z13)
#define RHG_TWO_PI_HI 0x1.921fb54442d18p+2
#define RHG_TWO_PI_LO 0x1.1a62633145c07p-52
// 2^27 / fl(2*pi): angle -> 27-bit fixed-point key (monotone in theta)
#define RHG_Q27_SCALE 0x1.45f306dc9c883p+24

// Host-computed, per-call constants passed to kernels by value.
struct BandConst {
  int L;
  double R;
  double T4;                 // 4 sinh^2(R/2) = 2 (cosh R - 1)       (Eq. 3 threshold, rewritten)
  double c[kMaxBands + 1];   // slab boundaries c_0 .. c_L
  double A[kMaxBands];       // e^{c_j/2}
  double B[kMaxBands];       // e^{-c_j/2}
  double invS[kMaxBands];    // 1/sinh(c_j)   (0 for c_j = 0 -> full circle)
};

// Device-computed band layout after the band histogram.
struct BandLayout {
  uint32_t count[kMaxBands];       // n_j
  uint32_t start[kMaxBands + 1];   // first sorted index of band j
  uint32_t dir_off[kMaxBands + 1]; // offset of band j's bucket directory
  uint32_t shift[kMaxBands];       // bucket(q) = q >> shift[j]
  uint32_t nb[kMaxBands];          // buckets in band j (power of two)
};

// Scalars the host reads back once per call.
struct DevScalars {
  unsigned long long total;        // edges (directed for CSR, undirected for pairs)
  unsigned long long candidates;   // tests performed by the count pass
  unsigned long long bit_words;    // candidate-bit words allocated by the count pass
  unsigned int domain_error;       // a point outside the disk
  unsigned int bit_overflow;       // bit buffer too small -> emit re-tests
};

// One point in the query SoA, 32 B: theta, sinh r, e^{r/2}, e^{-r/2}.
struct __align__(16) PointRec {
  double theta, s, a, b;
};

struct QueryArgs {
  uint32_t n;
  const PointRec* __restrict__ pts;   // sorted by (band, theta)
  const uint32_t* __restrict__ skey;  // sorted keys
  const uint32_t* __restrict__ sid;   // sorted position -> vertex id
  const uint32_t* __restrict__ dir;   // bucket directory
  const BandLayout* __restrict__ lay;
  const uint32_t* __restrict__ order; // query order (sorted positions), or nullptr = identity
  uint32_t* deg;                      // count pass: degree per vertex id
  const uint64_t* __restrict__ offs;  // emit pass: output offset per vertex id
  uint32_t* col;                      // CSR output
  uint32_t* pairs;                    // undirected output
  uint32_t* bits;                     // candidate-bit buffer
  uint64_t bits_cap;                  // words
  uint64_t* warp_bits;                // per-warp bit base (count writes, emit reads)
  DevScalars* sc;
};

// ---- launch wrappers (each returns cudaError_t of the launch) ----
cudaError_t launch_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t* out,
                                cudaStream_t st);
cudaError_t launch_sample(uint64_t n, uint64_t seed, double alpha, double R, const BandConst& bc,
                          double* theta, double* r, uint32_t* keys, uint32_t* idx,
                          uint32_t* band_hist, cudaStream_t st);
cudaError_t launch_keys_from_points(uint64_t n, const double* theta, const double* r,
                                    const BandConst& bc, uint32_t* keys, uint32_t* idx,
                                    uint32_t* band_hist, DevScalars* sc, cudaStream_t st);
cudaError_t launch_band_layout(const BandConst& bc, const uint32_t* band_hist, BandLayout* lay,
                               cudaStream_t st);
// LSD radix sort of (key, val) pairs, 32-bit keys, stable.  Result lands in
// (keys_a, vals_a).  tmp must hold radix_sort_tmp_bytes(n).
size_t radix_sort_tmp_bytes(uint64_t n);
cudaError_t radix_sort(uint32_t n, uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b,
                       uint32_t* vals_b, void* tmp, int begin_bit, int end_bit, cudaStream_t st,
                       int* launches);
cudaError_t launch_build_index(uint32_t n, const double* theta, const double* r,
                               const uint32_t* skey, const uint32_t* sidx, const BandLayout* lay,
                               int L, PointRec* pts, uint32_t* dir, cudaStream_t st,
                               int* launches);
// Exclusive scan of n uint32 counts into n+1 uint64 offsets (out[n] = total);
// also writes the total into *total_out.  tmp: scan_tmp_bytes(n).
size_t scan_tmp_bytes(uint64_t n);
cudaError_t exclusive_scan_u32_u64(uint32_t n, const uint32_t* in, uint64_t* out, void* tmp,
                                   unsigned long long* total_out, cudaStream_t st, int* launches);

enum QueryMode { QM_COUNT = 0, QM_EMIT = 1, QM_EMIT_BITS = 2 };
cudaError_t launch_query(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const BandConst& bc,
                         cudaStream_t st);

}  // namespace rhg
