// k_index.cu -- K4: gather the query SoA in (band, angle) order and build the
// per-band bucket directory that replaces most of the binary search of
// PAPER.md:214 ("find the leftmost and rightmost neighbor candidate in each slab
// using binary search").
#include "rhg_internal.cuh"
#include "rhg_predicate.cuh"

namespace rhg {

__device__ __forceinline__ uint32_t warp_incl_u32(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += a;
  }
  return v;
}

// Doubled SoA: the record of sorted position k in slab j (start s_j, n_j points)
// is written at k + s_j and k + s_j + n_j, so slab j occupies [2 s_j, 2 s_j + 2 n_j)
// as two back-to-back copies and every arc across 2 pi is one index range.
__device__ __forceinline__ void put_doubled(uint32_t k, uint32_t key, const BandLayout* lay,
                                            const PointRec& p, uint32_t id,
                                            PointRec* __restrict__ pts, uint32_t* __restrict__ sid2) {
  const uint32_t j = key >> kBandShift;
  const uint32_t s = lay->start[j], nj = lay->start[j + 1] - s;
  pts[k + s] = p;
  pts[k + s + nj] = p;
  sid2[k + s] = id;
  sid2[k + s + nj] = id;
}

// ---- bucket directory ----
// dir[dir_off[j] + b] = first sorted position of band j whose bucket >= b, for
// b = 0 .. nb_j (entry nb_j = band end).  Point k owns the entries in
// (bucket(k-1), bucket(k)] (value k); the last point of a band also owns
// (bucket(k), nb_j] (value k + 1, written by its lane).  Warp-cooperative: the
// entries owned by 32 consecutive points are one contiguous stretch of the
// directory (per band), written 32 consecutive entries per store instruction.
// Runs inside the gather kernels (same warp -> 32 positions mapping, the key is
// already in a register; the directory's integer work overlaps the gather's
// memory traffic).  (The sampled path gets its directory from bucket_sort.)
struct DirSmem {
  uint8_t tbl[8][32];
  uint2 own[8][32];
  uint32_t start[kMaxBands + 1], off[kMaxBands], sh[kMaxBands], nb[kMaxBands];
};

__device__ __forceinline__ void dir_smem_init(DirSmem& S, const BandLayout* lay, int L) {
  if (threadIdx.x <= (unsigned)L) S.start[threadIdx.x] = lay->start[threadIdx.x];
  if (threadIdx.x < (unsigned)L) {
    S.off[threadIdx.x] = lay->dir_off[threadIdx.x];
    S.sh[threadIdx.x] = lay->shift[threadIdx.x];
    S.nb[threadIdx.x] = lay->nb[threadIdx.x];
  }
}

// the directory entries owned by positions [32 w, 32 w + 32); key = skey[k] (0 if k >= n)
__device__ __forceinline__ void dir_warp(uint32_t w, uint32_t n, const uint32_t* __restrict__ skey,
                                         uint32_t key, DirSmem& S, uint32_t* __restrict__ dir) {
  const int lane = threadIdx.x & 31, wi = (threadIdx.x >> 5) & 7;
  const uint32_t k = w * 32 + (uint32_t)lane;
  uint32_t len = 0, base = 0;
  uint32_t pkey = __shfl_up_sync(0xffffffffu, key, 1);  // the previous point's key
  if (lane == 0 && k > 0 && k < n) pkey = __ldg(skey + k - 1);
  if (k < n) {
    const uint32_t j = key >> kBandShift;
    const uint32_t sh = S.sh[j], off = S.off[j];
    const uint32_t b = (key & kQMask) >> sh;
    uint32_t first = 0;  // first entry I own
    if (k > S.start[j]) first = ((pkey & kQMask) >> sh) + 1;
    len = b + 1 - first;  // 0 if the previous point shares my bucket
    base = off + first;
    if (k + 1 == S.start[j + 1]) {  // band tail: (b, nb] -> k + 1
      const uint32_t nb = S.nb[j];
      for (uint32_t bb = b + 1; bb <= nb; ++bb) dir[off + bb] = k + 1;
    }
  }
  const uint32_t incl = warp_incl_u32(len), T = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t pre = incl - len;
  const uint32_t NE = __ballot_sync(0xffffffffu, len > 0);
  if (len > 0) {
    S.tbl[wi][__popc(NE & ((1u << lane) - 1u))] = (uint8_t)lane;
    S.own[wi][lane] = make_uint2(base - pre, k);  // entry t -> dir[base - pre + t] = k
  }
  __syncwarp();
  uint32_t R0 = 0;
  for (uint32_t B = 0; B < T; B += 32) {
    const uint32_t sb = pre - B;
    const uint32_t M = __reduce_or_sync(0xffffffffu, (len > 0 && sb < 32u) ? (1u << sb) : 0u);
    const uint32_t rank = R0 + __popc(M & (0xffffffffu >> (31 - lane)));
    R0 += __popc(M);
    const uint32_t t = B + (uint32_t)lane;
    if (t < T) {
      const uint2 o = S.own[wi][S.tbl[wi][(rank - 1u) & 31u]];
      dir[o.x + t] = o.y;
    }
  }
  __syncwarp();
}

// empty bands: both entries = band start
__device__ __forceinline__ void dir_empty_bands(const BandLayout* lay, int L, uint32_t* dir) {
  if (blockIdx.x == 0 && threadIdx.x < (unsigned)L) {
    const int jj = threadIdx.x;
    if (lay->count[jj] == 0) {
      const uint32_t off = lay->dir_off[jj], nb = lay->nb[jj];
      for (uint32_t bb = 0; bb <= nb; ++bb) dir[off + bb] = lay->start[jj];
    }
  }
}

// Gather of the query records in sorted order (+ the directory when dir != null).
// Warp-uniform loop: warp-chunk w covers sorted positions [32 w, 32 w + 32).
// PHILOX: the points are re-derived from Philox(seed, i) (bit-identical to K1,
// same device code) instead of gathering theta[i], r[i] at random addresses.
template <bool PHILOX>
__global__ void __launch_bounds__(256)
    k_gather(uint32_t n, const double* __restrict__ theta, const double* __restrict__ r,
             PhiloxPoints gen, const uint32_t* __restrict__ skey,
             const uint32_t* __restrict__ sidx, const BandLayout* __restrict__ lay, int L,
             PointRec* __restrict__ pts, uint32_t* __restrict__ sid2, uint32_t* __restrict__ dir,
             int seq_ids) {
  __shared__ DirSmem S;
  if (dir) {
    dir_smem_init(S, lay, L);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); (uint64_t)w * 32 < n;
       w += nwarps) {
    const uint32_t k = w * 32 + (uint32_t)lane;
    uint32_t key = 0;
    if (k < n) {
      key = __ldg(skey + k);
      const uint32_t i = __ldg(sidx + k);
      double th, rr;
      if (PHILOX) {
        words_to_point(vertex_words(gen.seed, i), gen.two_over_alpha, gen.half_span, gen.R, th, rr);
      } else {
        th = theta[i];
        rr = r[i];
      }
      put_doubled(k, key, lay, point_rec(th, rr), seq_ids ? k : i, pts, sid2);
    }
    if (dir) dir_warp(w, n, skey, key, S, dir);
  }
  if (dir) dir_empty_bands(lay, L, dir);
}

// ---- query order (sector-major) ----
// The light queries are processed sector by sector: all slabs' vertices with
// angle in sector s (kQuerySectors equal arcs), slab by slab, before sector s+1.
// The warps in flight then all read the candidates of one arc of every slab, so
// each slab's points come from HBM about once per pass (slab-major order re-reads
// every slab once per query slab, SURVEY E-9).  Cell c = s * L + j holds the
// sorted positions of slab j in sector s (hub positions < heavy_end excluded).
__global__ void k_query_cells(const uint32_t* __restrict__ skey, const BandLayout* __restrict__ lay,
                              int L, uint32_t* __restrict__ cell_lo, uint32_t* __restrict__ cell_cnt) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (uint32_t)(kQuerySectors * L)) return;
  const uint32_t sct = c / (uint32_t)L, j = c % (uint32_t)L;
  const uint32_t b0 = lay->start[j], b1 = lay->start[j + 1];
  auto lower = [&](uint32_t q) {  // first position of slab j with q27 >= q
    uint32_t a = b0, b = b1;
    while (a < b) {
      const uint32_t m = (a + b) >> 1;
      if ((skey[m] & kQMask) < q) a = m + 1; else b = m;
    }
    return a;
  };
  const uint32_t sh = kQBits - kQuerySectorBits;
  uint32_t lo = lower(sct << sh);
  const uint32_t hi = (sct + 1 == (uint32_t)kQuerySectors) ? b1 : lower((sct + 1) << sh);
  const uint32_t he = lay->heavy_end;
  if (lo < he) lo = he;
  cell_lo[c] = lo;
  cell_cnt[c] = hi > lo ? hi - lo : 0u;
}

__global__ void __launch_bounds__(256)
    k_query_fill(const uint32_t* __restrict__ cell_lo, const uint32_t* __restrict__ cell_cnt,
                 const uint64_t* __restrict__ cell_off, uint32_t* __restrict__ order) {
  const uint32_t c = blockIdx.x;
  const uint32_t lo = cell_lo[c], cnt = cell_cnt[c];
  const uint64_t o = cell_off[c];
  for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) order[o + t] = lo + t;
}

cudaError_t launch_build_index(uint32_t n, const double* theta, const double* r,
                               const uint32_t* skey, const uint32_t* sidx, const BandLayout* lay,
                               int L, PointRec* pts, uint32_t* sid2, uint32_t* dir,
                               const PhiloxPoints* gen, int seq_ids, cudaStream_t st,
                               int* launches) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > (uint32_t)num_sms() * 32) blocks = (uint32_t)num_sms() * 32;
  if (blocks < 1) blocks = 1;
  if (gen)
    k_gather<true><<<blocks, 256, 0, st>>>(n, theta, r, *gen, skey, sidx, lay, L, pts, sid2, dir,
                                           seq_ids);
  else
    k_gather<false><<<blocks, 256, 0, st>>>(n, theta, r, PhiloxPoints{}, skey, sidx, lay, L, pts,
                                            sid2, dir, seq_ids);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_query_order(const uint32_t* skey, const BandLayout* lay, int L,
                               uint32_t* cell_lo, uint32_t* cell_cnt, uint64_t* cell_off,
                               uint32_t* order, void* scan_tmp, cudaStream_t st, int* launches) {
  const uint32_t cells = (uint32_t)(kQuerySectors * L);
  k_query_cells<<<(cells + 255) / 256, 256, 0, st>>>(skey, lay, L, cell_lo, cell_cnt);
  cudaError_t e = exclusive_scan_u32_u64(cells, cell_cnt, cell_off, scan_tmp, nullptr, st, launches);
  if (e != cudaSuccess) return e;
  k_query_fill<<<cells, 256, 0, st>>>(cell_lo, cell_cnt, cell_off, order);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

}  // namespace rhg
