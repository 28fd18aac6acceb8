// k_update.cu -- SURVEY.md §8(f) f1: incremental edge update of the dynamic model.
//
// PAPER.md:387-389 (§4): "Our implementation allows updating a graph without
// rebuilding it from scratch.  Moving up to 12 % of nodes and updating an existing
// graph is still faster than a new static generation."  The movement itself
// (rotation + Alg. 2 radial step with reflection) is k_dynamic.cu.
//
// Given the new positions of all points, the ids of the vertices that moved and
// their old positions, and the graph of the old positions (CSR over vertex ids),
// the host code (rhg_abi.cu, run_update) indexes the new points, runs the range
// queries of Alg. 1 for the moved vertices only -- their new
// rows -- and these kernels turn old and new rows into the edge delta:
//   removed = { {v, w} : w in old_row(v), dist_new(v, w) > R },
//   added   = { {v, w} : w in new_row(v), dist_old(v, w) > R },
// v over the moved vertices, each pair once (a pair of two moved vertices is
// reported from its smaller id).  dist is decided by the same certified test of
// Eq. 3 (rhg_predicate.cuh) on the same point records as the
// generator, so the old graph's edge set is exactly the set this test accepts and
// (old graph - removed) + added is exactly the graph of the new positions.
#include "rhg_internal.cuh"
#include "rhg_predicate.cuh"

namespace rhg {

constexpr uint32_t kNotMoved = 0xffffffffu;

__global__ void k_update_midx(uint64_t m, const uint32_t* __restrict__ moved,
                              uint32_t* __restrict__ midx) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x)
    midx[moved[k]] = (uint32_t)k;
}

// query item t of the full processing order: hub position t < heavy_end, then the
// sector-major light order; flag = the item's vertex moved
__global__ void k_update_flags(uint32_t n, const BandLayout* __restrict__ lay,
                               const uint32_t* __restrict__ order, const uint32_t* __restrict__ sid,
                               const uint32_t* __restrict__ midx, uint32_t* __restrict__ flag) {
  const uint32_t he = lay->heavy_end;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint32_t p = t < he ? t : order[t - he];
    flag[t] = midx[sid[p]] != kNotMoved ? 1u : 0u;
  }
}

// stable compaction: the moved light vertices' sorted positions in processing order
// (moved hubs take the hub path, selected by flag[0 .. heavy_end))
__global__ void k_update_compact(uint32_t n, const BandLayout* __restrict__ lay,
                                 const uint32_t* __restrict__ order, const uint32_t* __restrict__ flag,
                                 const uint64_t* __restrict__ fpos, uint32_t* __restrict__ qorder,
                                 unsigned long long* __restrict__ nlight_moved) {
  const uint32_t he = lay->heavy_end;
  const uint64_t f0 = fpos[he];
  for (uint32_t t = he + blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    if (flag[t]) qorder[fpos[t] - f0] = order[t - he];
  if (blockIdx.x == 0 && threadIdx.x == 0) *nlight_moved = fpos[n] - f0;
}

__device__ __forceinline__ PointRec rec_of(const double* theta, const double* r, uint32_t i) {
  return point_rec(theta[i], r[i]);
}

// One warp per moved vertex k (grid-stride).  WRITE = false: count the pairs to
// remove / add; WRITE = true: write them at the scanned offsets, in row order.
template <bool WRITE>
__global__ void __launch_bounds__(256)
    k_delta(uint64_t m, const uint32_t* __restrict__ moved, const uint32_t* __restrict__ midx,
            const double* __restrict__ theta, const double* __restrict__ r,
            const double* __restrict__ theta_old, const double* __restrict__ r_old,
            const uint64_t* __restrict__ old_rp, const uint32_t* __restrict__ old_col,
            const uint64_t* __restrict__ new_rp, const uint32_t* __restrict__ new_col, double T4,
            uint32_t* __restrict__ n_rem, uint32_t* __restrict__ n_add,
            const uint64_t* __restrict__ off_rem, const uint64_t* __restrict__ off_add,
            uint32_t* __restrict__ removed, uint32_t* __restrict__ added) {
  const uint32_t lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t k = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < m;
       k += warps) {
    const uint32_t v = moved[k];
    // removed: old row entries that the NEW positions no longer connect
    {
      const PointRec q = rec_of(theta, r, v);
      const uint64_t a = old_rp[v], b = old_rp[v + 1];
      uint64_t base = WRITE ? off_rem[k] : 0;
      uint32_t cnt = 0;
      for (uint64_t i0 = a; i0 < b; i0 += 32) {
        const bool act = i0 + lane < b;
        const uint32_t w = act ? old_col[i0 + lane] : v;
        const bool own = act && !(midx[w] != kNotMoved && w < v);  // pair of two moved: once
        const PointRec p = rec_of(theta, r, own ? w : v);
        const bool e = certified_edge(q.theta, 4.0 * q.s, q.a, q.b, make_double2(p.theta, p.s),
                                      make_double2(p.a, p.b), T4, own);
        const uint32_t bm = __ballot_sync(0xffffffffu, own && !e);
        if (WRITE && own && !e) {
          const uint64_t o = base + __popc(bm & lt);
          removed[2 * o] = min(v, w);
          removed[2 * o + 1] = max(v, w);
        }
        base += __popc(bm);
        cnt += __popc(bm);
      }
      if (!WRITE && lane == 0) n_rem[k] = cnt;
    }
    // added: new row entries that the OLD positions did not connect
    {
      const uint32_t kv = k;
      const PointRec q = point_rec(theta_old[kv], r_old[kv]);
      const uint64_t a = new_rp[v], b = new_rp[v + 1];
      uint64_t base = WRITE ? off_add[k] : 0;
      uint32_t cnt = 0;
      for (uint64_t i0 = a; i0 < b; i0 += 32) {
        const bool act = i0 + lane < b;
        const uint32_t w = act ? new_col[i0 + lane] : v;
        const uint32_t mw = act ? midx[w] : kNotMoved;
        const bool own = act && !(mw != kNotMoved && w < v);
        const PointRec p = !own ? q
                           : (mw != kNotMoved ? point_rec(theta_old[mw], r_old[mw]) : rec_of(theta, r, w));
        const bool e = certified_edge(q.theta, 4.0 * q.s, q.a, q.b, make_double2(p.theta, p.s),
                                      make_double2(p.a, p.b), T4, own);
        const uint32_t bm = __ballot_sync(0xffffffffu, own && !e);
        if (WRITE && own && !e) {
          const uint64_t o = base + __popc(bm & lt);
          added[2 * o] = min(v, w);
          added[2 * o + 1] = max(v, w);
        }
        base += __popc(bm);
        cnt += __popc(bm);
      }
      if (!WRITE && lane == 0) n_add[k] = cnt;
    }
  }
}

cudaError_t launch_update_select(uint32_t n, uint64_t m, const uint32_t* moved, const BandLayout* lay,
                                 const uint32_t* order, const uint32_t* sid, uint32_t* midx,
                                 uint32_t* flag, uint64_t* fpos, uint32_t* qorder,
                                 unsigned long long* nlight_moved, void* scan_tmp, cudaStream_t st,
                                 int* launches) {
  cudaError_t e = cudaMemsetAsync(midx, 0xff, 4ull * n, st);
  if (e != cudaSuccess) return e;
  const int blocks = num_sms() * 8;
  if (m) k_update_midx<<<blocks, 256, 0, st>>>(m, moved, midx);
  k_update_flags<<<blocks, 256, 0, st>>>(n, lay, order, sid, midx, flag);
  e = exclusive_scan_u32_u64(n, flag, fpos, scan_tmp, nullptr, st, launches);
  if (e != cudaSuccess) return e;
  k_update_compact<<<blocks, 256, 0, st>>>(n, lay, order, flag, fpos, qorder, nlight_moved);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_delta(bool write, uint64_t m, const uint32_t* moved, const uint32_t* midx,
                         const double* theta, const double* r, const double* theta_old,
                         const double* r_old, const uint64_t* old_rp, const uint32_t* old_col,
                         const uint64_t* new_rp, const uint32_t* new_col, double T4, uint32_t* n_rem,
                         uint32_t* n_add, const uint64_t* off_rem, const uint64_t* off_add,
                         uint32_t* removed, uint32_t* added, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const uint64_t want = (m + 7) / 8;
  const int blocks = (int)(want < (uint64_t)num_sms() * 16 ? want : (uint64_t)num_sms() * 16);
  if (write)
    k_delta<true><<<blocks, 256, 0, st>>>(m, moved, midx, theta, r, theta_old, r_old, old_rp,
                                          old_col, new_rp, new_col, T4, n_rem, n_add, off_rem,
                                          off_add, removed, added);
  else
    k_delta<false><<<blocks, 256, 0, st>>>(m, moved, midx, theta, r, theta_old, r_old, old_rp,
                                           old_col, new_rp, new_col, T4, n_rem, n_add, off_rem,
                                           off_add, removed, added);
  return cudaGetLastError();
}

}  // namespace rhg
