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
// rows -- and these kernels turn old and new rows into the edge delta (decide ->
// scan -> write):
//   removed = { {v, w} : w in old_row(v) \ new_row(v) },
//   added   = { {v, w} : w in new_row(v) \ old_row(v) },
// v over the moved vertices, each pair once (a pair of two moved vertices is
// reported from its smaller id).  Rows of up to kDeltaHash / 2 (kBlockHash / 2) entries
// are compared through a per-warp (per-block) hash set in shared memory (no point
// records needed); longer new rows (hubs) decide membership with the same certified test of
// Eq. 3 (rhg_predicate.cuh) on the same point records as the
// generator: the old graph's edge set is exactly the set this test accepts, so
// (old graph - removed) + added is exactly the graph of the new positions.
#include "rhg_internal.cuh"
#include "rhg_predicate.cuh"

namespace rhg {

constexpr uint32_t kNotMoved = 0xffffffffu;
constexpr int kDeltaHash = 1024;  // hash slots per warp (new rows up to 512 entries)
constexpr int kDeltaWarps = 8;
constexpr uint32_t kEmpty = 0xffffffffu, kMark = 0x80000000u;  // ids < 2^31

// pm[id] = (sorted position of id in the new index, index of id in `moved` or
// kNotMoved): one 8-byte record per vertex (80 MB at n = 1e7, L2-resident), so that a
// row entry w costs one scattered read plus reads of the sorted SoA, which are local
// for angularly close queries.
__global__ void k_update_pos(uint32_t n, const uint32_t* __restrict__ sid, uint2* __restrict__ pm) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    pm[sid[p]].x = p;
}

__global__ void k_update_midx(uint64_t m, const uint32_t* __restrict__ moved, uint2* __restrict__ pm) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x)
    pm[moved[k]].y = (uint32_t)k;
}

// query item t of the full processing order: hub position t < heavy_end, then the
// sector-major light order; flag = the item's vertex moved
__global__ void k_update_flags(uint32_t n, const BandLayout* __restrict__ lay,
                               const uint32_t* __restrict__ order, const uint32_t* __restrict__ sid,
                               const uint2* __restrict__ pm, uint32_t* __restrict__ flag) {
  const uint32_t he = lay->heavy_end;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint32_t p = t < he ? t : order[t - he];
    flag[t] = pm[sid[p]].y != kNotMoved ? 1u : 0u;
  }
}

// stable compactions: morder = the moved vertices (ids) in processing order (the
// delta kernels walk them in this order, so consecutive warps read nearby parts of
// the sorted SoA); qorder = the moved light vertices' sorted positions (the light
// query kernels; moved hubs take the hub path, selected by flag[0 .. heavy_end))
__global__ void k_update_compact(uint32_t n, const BandLayout* __restrict__ lay,
                                 const uint32_t* __restrict__ order, const uint32_t* __restrict__ sid,
                                 const uint32_t* __restrict__ flag, const uint64_t* __restrict__ fpos,
                                 uint32_t* __restrict__ qorder, uint32_t* __restrict__ morder,
                                 unsigned long long* __restrict__ nlight_moved) {
  const uint32_t he = lay->heavy_end;
  const uint64_t f0 = fpos[he];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (!flag[t]) continue;
    const uint32_t p = t < he ? t : order[t - he];
    morder[fpos[t]] = sid[p];
    if (t >= he) qorder[fpos[t] - f0] = p;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *nlight_moved = fpos[n] - f0;
}

// new-position record of vertex w from the sorted, doubled SoA
__device__ __forceinline__ PointRec new_rec(const PointRec* __restrict__ pts,
                                            const uint32_t* __restrict__ skey,
                                            const uint32_t* start, uint32_t p) {
  return pts[p + start[skey[p] >> kBandShift]];
}

__device__ __forceinline__ uint32_t slot_of(uint32_t w) { return (w * 0x9E3779B1u) >> 22; }  // 10 bits

// Work units of the delta (balanced: no warp walks a hub-sized row alone).  Moved
// vertex j (processing order) is one unit if its new row fits a hash set -- a warp's
// (<= kDeltaHash / 2 entries, k_delta) or a block's (<= kBlockHash / 2,
// k_delta_block) -- and the two rows are compared through it; a longer one is cut
// into kDeltaChunk-entry chunks of its old row (removed, by the certified test at the
// new positions) and of its new row (added, by the test at the old positions).
constexpr uint32_t kDeltaChunk = 512;
constexpr int kBlockHash = 8192;

__device__ __forceinline__ bool is_big(uint64_t new_len) { return new_len > (uint64_t)(kDeltaHash / 2); }
__device__ __forceinline__ bool is_huge(uint64_t new_len) { return new_len > (uint64_t)(kBlockHash / 2); }

__global__ void k_delta_units(uint64_t m, const uint32_t* __restrict__ morder,
                              const uint64_t* __restrict__ old_rp, const uint64_t* __restrict__ new_rp,
                              uint32_t* __restrict__ units) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = morder[j];
    const uint64_t nl = new_rp[v + 1] - new_rp[v], ol = old_rp[v + 1] - old_rp[v];
    units[j] = is_huge(nl) ? (uint32_t)((ol + kDeltaChunk - 1) / kDeltaChunk +
                                        (nl + kDeltaChunk - 1) / kDeltaChunk)
                           : 1u;
  }
}

// unit -> moved vertex; the medium units (block hash) also go to a list (any order:
// outputs are placed by the per-unit scan)
__global__ void k_delta_unit_map(uint64_t m, const uint32_t* __restrict__ morder,
                                 const uint64_t* __restrict__ new_rp, const uint64_t* __restrict__ uoff,
                                 uint32_t* __restrict__ unit_j, uint32_t* __restrict__ mlist,
                                 unsigned int* __restrict__ mcount) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m;
       j += (uint64_t)gridDim.x * blockDim.x) {
    for (uint64_t t = uoff[j]; t < uoff[j + 1]; ++t) unit_j[t] = (uint32_t)j;
    const uint32_t v = morder[j];
    const uint64_t nl = new_rp[v + 1] - new_rp[v];
    if (is_big(nl) && !is_huge(nl)) mlist[atomicAdd(mcount, 1u)] = (uint32_t)uoff[j];
  }
}

// Decisions are recorded as bits over the rows' entries -- rbits over old_col
// (removed), abits over new_col (added), bit i = entry i -- by the decide kernels
// (one pass: per-unit counts + bits); the scans give each unit its output offsets and
// k_delta_write replays the bits in row order (deterministic output, nothing decided
// twice).  A 32-entry batch starting at entry i0 covers bits [i0, i0 + 32): at most two
// words, merged with atomicOr.
__device__ __forceinline__ void put_bits(uint32_t* bits, uint64_t i0, uint32_t bm) {
  if (!bm) return;
  const uint64_t w = i0 >> 5;
  const uint32_t s = (uint32_t)(i0 & 31u);
  atomicOr(bits + w, bm << s);
  if (s && (bm >> (32u - s))) atomicOr(bits + w + 1, bm >> (32u - s));
}
__device__ __forceinline__ uint32_t get_bits(const uint32_t* bits, uint64_t i0) {
  const uint64_t w = i0 >> 5;
  const uint32_t s = (uint32_t)(i0 & 31u);
  return s ? (bits[w] >> s) | (bits[w + 1] << (32u - s)) : bits[w];
}

// One warp per unit (grid-stride): decide which entries leave / join.
__global__ void __launch_bounds__(kDeltaWarps * 32)
    k_delta(const uint64_t* __restrict__ uoff, uint64_t m, const uint32_t* __restrict__ unit_j,
            const uint32_t* __restrict__ morder, const uint2* __restrict__ pm,
            const uint32_t* __restrict__ mbits, const PointRec* __restrict__ pts,
            const uint32_t* __restrict__ skey, const BandLayout* __restrict__ lay, int L,
            const double* __restrict__ theta_old, const double* __restrict__ r_old,
            const uint64_t* __restrict__ old_rp, const uint32_t* __restrict__ old_col,
            const uint64_t* __restrict__ new_rp, const uint32_t* __restrict__ new_col, double T4,
            uint32_t* __restrict__ n_rem, uint32_t* __restrict__ n_add, uint32_t* __restrict__ rbits,
            uint32_t* __restrict__ abits) {
  __shared__ uint32_t tab_all[kDeltaWarps][kDeltaHash];
  __shared__ uint32_t start[kMaxBands + 1];
  if (threadIdx.x <= (unsigned)L) start[threadIdx.x] = lay->start[threadIdx.x];
  __syncthreads();
  uint32_t* tab = tab_all[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t U = uoff[m], warps = (uint64_t)gridDim.x * kDeltaWarps;
  auto moved = [&](uint32_t w) { return (mbits[w >> 5] >> (w & 31u)) & 1u; };
  for (uint64_t u = blockIdx.x * (uint64_t)kDeltaWarps + (threadIdx.x >> 5); u < U; u += warps) {
    const uint32_t j = unit_j[u];
    const uint32_t v = morder[j];
    const uint64_t na = new_rp[v], nb = new_rp[v + 1], oa = old_rp[v], ob = old_rp[v + 1];
    if (is_big(nb - na) && !is_huge(nb - na)) continue;  // k_delta_block
    uint32_t crem = 0, cadd = 0;
    if (!is_big(nb - na)) {
      // ---- hash set of the new row; old entries not in it are removed, new entries
      // whose slot no old entry marked are added ----
      for (int s = lane; s < kDeltaHash; s += 32) tab[s] = kEmpty;
      __syncwarp();
      for (uint64_t i = na + lane; i < nb; i += 32) {
        const uint32_t w = new_col[i];
        uint32_t h = slot_of(w);
        while (true) {
          const uint32_t o = atomicCAS(&tab[h], kEmpty, w);
          if (o == kEmpty || o == w) break;
          h = (h + 1u) & (kDeltaHash - 1u);
        }
      }
      __syncwarp();
      for (uint64_t i0 = oa; i0 < ob; i0 += 32) {
        const bool act = i0 + lane < ob;
        const uint32_t w = act ? old_col[i0 + lane] : 0u;
        const bool dup = act && w < v && moved(w);  // pair of two moved: from the smaller id
        bool found = false;
        if (act) {
          uint32_t h = slot_of(w);
          while (true) {
            const uint32_t t = tab[h];
            if (t == kEmpty) break;
            if ((t & ~kMark) == w) {
              found = true;
              atomicOr(&tab[h], kMark);
              break;
            }
            h = (h + 1u) & (kDeltaHash - 1u);
          }
        }
        const uint32_t bm = __ballot_sync(0xffffffffu, act && !found && !dup);
        if (lane == 0) put_bits(rbits, i0, bm);
        crem += __popc(bm);
      }
      __syncwarp();
      for (uint64_t i0 = na; i0 < nb; i0 += 32) {
        const bool act = i0 + lane < nb;
        const uint32_t w = act ? new_col[i0 + lane] : 0u;
        const bool dup = act && w < v && moved(w);
        bool in_old = false;
        if (act) {
          uint32_t h = slot_of(w);
          while ((tab[h] & ~kMark) != w) h = (h + 1u) & (kDeltaHash - 1u);
          in_old = (tab[h] & kMark) != 0u;
        }
        const uint32_t bm = __ballot_sync(0xffffffffu, act && !in_old && !dup);
        if (lane == 0) put_bits(abits, i0, bm);
        cadd += __popc(bm);
      }
      __syncwarp();
    } else {
      // ---- one chunk of a long row, decided by the certified test ----
      const uint64_t c = u - uoff[j];
      const uint64_t ncr = (ob - oa + kDeltaChunk - 1) / kDeltaChunk;
      const uint2 pv = pm[v];
      if (c < ncr) {  // removed: old row entries the NEW positions do not connect
        const PointRec q = new_rec(pts, skey, start, pv.x);
        const uint64_t a = oa + c * kDeltaChunk, b = min(ob, a + kDeltaChunk);
        for (uint64_t i0 = a; i0 < b; i0 += 32) {
          const bool act = i0 + lane < b;
          const uint32_t w = act ? old_col[i0 + lane] : v;
          const uint2 pw = act ? pm[w] : pv;
          const bool own = act && !(pw.y != kNotMoved && w < v);
          const PointRec p = new_rec(pts, skey, start, own ? pw.x : pv.x);
          const bool e = certified_edge(q.theta, 4.0 * q.s, q.a, q.b, make_double2(p.theta, p.s),
                                        make_double2(p.a, p.b), T4, own);
          const uint32_t bm = __ballot_sync(0xffffffffu, own && !e);
          if (lane == 0) put_bits(rbits, i0, bm);
          crem += __popc(bm);
        }
      } else {  // added: new row entries the OLD positions did not connect
        const PointRec q = point_rec(theta_old[pv.y], r_old[pv.y]);
        const uint64_t a = na + (c - ncr) * kDeltaChunk, b = min(nb, a + kDeltaChunk);
        for (uint64_t i0 = a; i0 < b; i0 += 32) {
          const bool act = i0 + lane < b;
          const uint32_t w = act ? new_col[i0 + lane] : v;
          const uint2 pw = act ? pm[w] : make_uint2(pv.x, kNotMoved);
          const bool own = act && !(pw.y != kNotMoved && w < v);
          const PointRec p = pw.y != kNotMoved ? point_rec(theta_old[pw.y], r_old[pw.y])
                                               : new_rec(pts, skey, start, pw.x);  // static: same
          const bool e = certified_edge(q.theta, 4.0 * q.s, q.a, q.b, make_double2(p.theta, p.s),
                                        make_double2(p.a, p.b), T4, own);
          const uint32_t bm = __ballot_sync(0xffffffffu, own && !e);
          if (lane == 0) put_bits(abits, i0, bm);
          cadd += __popc(bm);
        }
      }
    }
    if (lane == 0) {
      n_rem[u] = crem;
      n_add[u] = cadd;
    }
  }
}

// One block per medium unit (new row of kDeltaHash / 2 .. kBlockHash / 2 entries):
// the same comparison with a block-wide hash set.
__global__ void __launch_bounds__(256)
    k_delta_block(const uint32_t* __restrict__ mlist, const unsigned int* __restrict__ mcount,
                  const uint32_t* __restrict__ unit_j, const uint32_t* __restrict__ morder,
                  const uint32_t* __restrict__ mbits, const uint64_t* __restrict__ old_rp,
                  const uint32_t* __restrict__ old_col, const uint64_t* __restrict__ new_rp,
                  const uint32_t* __restrict__ new_col, uint32_t* __restrict__ n_rem,
                  uint32_t* __restrict__ n_add, uint32_t* __restrict__ rbits,
                  uint32_t* __restrict__ abits) {
  __shared__ uint32_t tab[kBlockHash];
  __shared__ uint32_t wsum[2][8];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t MC = *mcount;
  auto moved = [&](uint32_t w) { return (mbits[w >> 5] >> (w & 31u)) & 1u; };
  constexpr uint32_t msk = kBlockHash - 1u;
  for (uint32_t x = blockIdx.x; x < MC; x += gridDim.x) {
    const uint32_t u = mlist[x];
    const uint32_t v = morder[unit_j[u]];
    const uint64_t na = new_rp[v], nb = new_rp[v + 1], oa = old_rp[v], ob = old_rp[v + 1];
    for (uint32_t s = tid; s < (uint32_t)kBlockHash; s += 256) tab[s] = kEmpty;
    __syncthreads();
    for (uint64_t i = na + tid; i < nb; i += 256) {
      const uint32_t w = new_col[i];
      uint32_t h = (w * 0x9E3779B1u) >> 19;  // 13 bits
      while (true) {
        const uint32_t o = atomicCAS(&tab[h], kEmpty, w);
        if (o == kEmpty || o == w) break;
        h = (h + 1u) & msk;
      }
    }
    __syncthreads();
    uint32_t crem = 0, cadd = 0;  // per warp
    for (uint64_t i0 = oa + 32 * warp; i0 < ob; i0 += 256) {
      const bool act = i0 + lane < ob;
      const uint32_t w = act ? old_col[i0 + lane] : 0u;
      const bool dup = act && w < v && moved(w);
      bool found = false;
      if (act) {
        uint32_t h = (w * 0x9E3779B1u) >> 19;
        while (true) {
          const uint32_t t = tab[h];
          if (t == kEmpty) break;
          if ((t & ~kMark) == w) {
            found = true;
            atomicOr(&tab[h], kMark);
            break;
          }
          h = (h + 1u) & msk;
        }
      }
      const uint32_t bm = __ballot_sync(0xffffffffu, act && !found && !dup);
      if (lane == 0) put_bits(rbits, i0, bm);
      crem += __popc(bm);
    }
    __syncthreads();
    for (uint64_t i0 = na + 32 * warp; i0 < nb; i0 += 256) {
      const bool act = i0 + lane < nb;
      const uint32_t w = act ? new_col[i0 + lane] : 0u;
      const bool dup = act && w < v && moved(w);
      bool in_old = false;
      if (act) {
        uint32_t h = (w * 0x9E3779B1u) >> 19;
        while ((tab[h] & ~kMark) != w) h = (h + 1u) & msk;
        in_old = (tab[h] & kMark) != 0u;
      }
      const uint32_t bm = __ballot_sync(0xffffffffu, act && !in_old && !dup);
      if (lane == 0) put_bits(abits, i0, bm);
      cadd += __popc(bm);
    }
    if (lane == 0) {
      wsum[0][warp] = crem;
      wsum[1][warp] = cadd;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t a = 0, b = 0;
      for (int k = 0; k < 8; ++k) {
        a += wsum[0][k];
        b += wsum[1][k];
      }
      n_rem[u] = a;
      n_add[u] = b;
    }
    __syncthreads();
  }
}

// One warp per unit: write the decided pairs at the unit's offsets, in row order.
__global__ void __launch_bounds__(kDeltaWarps * 32)
    k_delta_write(const uint64_t* __restrict__ uoff, uint64_t m, const uint32_t* __restrict__ unit_j,
                  const uint32_t* __restrict__ morder, const uint64_t* __restrict__ old_rp,
                  const uint32_t* __restrict__ old_col, const uint64_t* __restrict__ new_rp,
                  const uint32_t* __restrict__ new_col, const uint32_t* __restrict__ rbits,
                  const uint32_t* __restrict__ abits, const uint64_t* __restrict__ off_rem,
                  const uint64_t* __restrict__ off_add, uint32_t* __restrict__ removed,
                  uint32_t* __restrict__ added) {
  const uint32_t lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
  const uint64_t U = uoff[m], warps = (uint64_t)gridDim.x * kDeltaWarps;
  auto replay = [&](uint64_t a, uint64_t b, const uint32_t* col, const uint32_t* bits, uint32_t v,
                    uint64_t base, uint32_t* out) {
    for (uint64_t i0 = a; i0 < b; i0 += 32) {
      uint32_t bm = get_bits(bits, i0);
      if (b - i0 < 32) bm &= (1u << (uint32_t)(b - i0)) - 1u;
      if ((bm >> lane) & 1u) {
        const uint32_t w = col[i0 + lane];
        const uint64_t o = base + __popc(bm & lt);
        out[2 * o] = min(v, w);
        out[2 * o + 1] = max(v, w);
      }
      base += __popc(bm);
    }
  };
  for (uint64_t u = blockIdx.x * (uint64_t)kDeltaWarps + (threadIdx.x >> 5); u < U; u += warps) {
    const uint32_t j = unit_j[u];
    const uint32_t v = morder[j];
    const uint64_t na = new_rp[v], nb = new_rp[v + 1], oa = old_rp[v], ob = old_rp[v + 1];
    if (!is_huge(nb - na)) {  // one unit: both rows
      replay(oa, ob, old_col, rbits, v, off_rem[u], removed);
      replay(na, nb, new_col, abits, v, off_add[u], added);
    } else {
      const uint64_t c = u - uoff[j];
      const uint64_t ncr = (ob - oa + kDeltaChunk - 1) / kDeltaChunk;
      if (c < ncr) {
        const uint64_t a = oa + c * kDeltaChunk;
        replay(a, min(ob, a + kDeltaChunk), old_col, rbits, v, off_rem[u], removed);
      } else {
        const uint64_t a = na + (c - ncr) * kDeltaChunk;
        replay(a, min(nb, a + kDeltaChunk), new_col, abits, v, off_add[u], added);
      }
    }
  }
}

__global__ void k_update_bits(uint64_t m, const uint32_t* __restrict__ moved, uint32_t* __restrict__ mbits) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
       k += (uint64_t)gridDim.x * blockDim.x)
    atomicOr(mbits + (moved[k] >> 5), 1u << (moved[k] & 31u));
}

cudaError_t launch_update_select(uint32_t n, uint64_t m, const uint32_t* moved, const BandLayout* lay,
                                 const uint32_t* order, const uint32_t* sid, uint2* pm,
                                 uint32_t* mbits, uint32_t* flag, uint64_t* fpos, uint32_t* qorder,
                                 uint32_t* morder, unsigned long long* nlight_moved, void* scan_tmp,
                                 cudaStream_t st, int* launches) {
  cudaError_t e = cudaMemsetAsync(pm, 0xff, 8ull * n, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(mbits, 0, 4ull * ((n + 31) / 32), st);
  if (e != cudaSuccess) return e;
  const int blocks = num_sms() * 8;
  k_update_pos<<<blocks, 256, 0, st>>>(n, sid, pm);
  if (m) k_update_midx<<<blocks, 256, 0, st>>>(m, moved, pm);
  if (m) k_update_bits<<<blocks, 256, 0, st>>>(m, moved, mbits);
  k_update_flags<<<blocks, 256, 0, st>>>(n, lay, order, sid, pm, flag);
  e = exclusive_scan_u32_u64(n, flag, fpos, scan_tmp, nullptr, st, launches);
  if (e != cudaSuccess) return e;
  k_update_compact<<<blocks, 256, 0, st>>>(n, lay, order, sid, flag, fpos, qorder, morder,
                                           nlight_moved);
  if (launches) *launches += 5;
  return cudaGetLastError();
}

cudaError_t launch_delta_plan(uint64_t m, const uint32_t* morder, const uint64_t* old_rp,
                              const uint64_t* new_rp, uint32_t* units, uint64_t* uoff,
                              uint32_t* unit_j, uint32_t* mlist, unsigned int* mcount,
                              void* scan_tmp, cudaStream_t st, int* launches) {
  cudaError_t e = cudaMemsetAsync(mcount, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess || m == 0) return e;
  const int blocks = num_sms() * 8;
  k_delta_units<<<blocks, 256, 0, st>>>(m, morder, old_rp, new_rp, units);
  e = exclusive_scan_u32_u64((uint32_t)m, units, uoff, scan_tmp, nullptr, st, launches);
  if (e != cudaSuccess) return e;
  k_delta_unit_map<<<blocks, 256, 0, st>>>(m, morder, new_rp, uoff, unit_j, mlist, mcount);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_delta_decide(uint64_t m, uint64_t unit_cap, const uint64_t* uoff,
                                const uint32_t* unit_j, const uint32_t* mlist,
                                const unsigned int* mcount, const uint32_t* morder, const uint2* pm,
                                const uint32_t* mbits, const PointRec* pts, const uint32_t* skey,
                                const BandLayout* lay, int L, const double* theta_old,
                                const double* r_old, const uint64_t* old_rp, const uint32_t* old_col,
                                const uint64_t* new_rp, const uint32_t* new_col, double T4,
                                uint32_t* n_rem, uint32_t* n_add, uint32_t* rbits, uint32_t* abits,
                                cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const uint64_t want = (unit_cap + kDeltaWarps - 1) / kDeltaWarps;
  const int blocks = (int)(want < (uint64_t)num_sms() * 16 ? want : (uint64_t)num_sms() * 16);
  k_delta_block<<<num_sms() * 4, 256, 0, st>>>(mlist, mcount, unit_j, morder, mbits, old_rp, old_col,
                                               new_rp, new_col, n_rem, n_add, rbits, abits);
  k_delta<<<blocks, kDeltaWarps * 32, 0, st>>>(uoff, m, unit_j, morder, pm, mbits, pts, skey, lay, L,
                                               theta_old, r_old, old_rp, old_col, new_rp, new_col,
                                               T4, n_rem, n_add, rbits, abits);
  return cudaGetLastError();
}

cudaError_t launch_delta_write(uint64_t m, uint64_t unit_cap, const uint64_t* uoff,
                               const uint32_t* unit_j, const uint32_t* morder,
                               const uint64_t* old_rp, const uint32_t* old_col,
                               const uint64_t* new_rp, const uint32_t* new_col,
                               const uint32_t* rbits, const uint32_t* abits,
                               const uint64_t* off_rem, const uint64_t* off_add, uint32_t* removed,
                               uint32_t* added, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const uint64_t want = (unit_cap + kDeltaWarps - 1) / kDeltaWarps;
  const int blocks = (int)(want < (uint64_t)num_sms() * 16 ? want : (uint64_t)num_sms() * 16);
  k_delta_write<<<blocks, kDeltaWarps * 32, 0, st>>>(uoff, m, unit_j, morder, old_rp, old_col,
                                                     new_rp, new_col, rbits, abits, off_rem,
                                                     off_add, removed, added);
  return cudaGetLastError();
}

}  // namespace rhg
