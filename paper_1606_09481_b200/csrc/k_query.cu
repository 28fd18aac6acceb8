// k_query.cu -- K5..K8: the range queries of Alg. 1 lines 13-21.
//
// For every vertex v and slab b_j (all slabs for CSR; slabs with c_{j+1} > r_v,
// i.e. "outward", for the undirected list):
//   * getMinMaxPhi (Eqs. 6-9), written without
//     cancellation (Z3) and padded to a superset;
//   * the candidate index range(s) in b_j's angle-sorted segment (binary search
//     of PAPER.md:214, here: bucket directory + short binary search; wrap at 2pi
//     splits into <= 2 ranges, Z13);
//   * every candidate tested exactly: dist <= R via the
//     cancellation-free form of Eq. 3 (Z2):
//       h  = e^{r_v/2} e^{-r_w/2} - e^{-r_v/2} e^{r_w/2} = 2 sinh((r_v - r_w)/2)
//       S4 = h^2 + 4 sinh r_v sinh r_w sin^2(dphi/2)  = 2 (cosh d - 1)
//       edge iff S4 <= T4 = 4 sinh^2(R/2) = 2 (cosh R - 1).
//
// Work decomposition (B200): one warp owns 32 query vertices.  Per slab each lane
// computes its vertex's ranges; the warp appends them to a ring of ranges in
// shared memory and consumes the flattened candidate sequence 32 at a time, so
// every lane tests a candidate in every batch regardless of range lengths.
// The count pass (QM_COUNT) and the emit pass (QM_EMIT) run the same code; the
// emit pass writes hit ids at offset[v] + running rank (ballot + match_any).
#include "rhg_internal.cuh"

namespace rhg {

constexpr int QK_WARPS = 4;
constexpr int QK_THREADS = QK_WARPS * 32;
constexpr uint32_t RING = 128;
constexpr uint32_t FULL = 0xffffffffu;

struct WarpSm {
  double qth[32], q4s[32], qa[32], qb[32];
  unsigned long long e_pref[RING];
  uint32_t e_start[RING];
  uint32_t e_lane[RING];
  unsigned long long cur[32];
  uint32_t degc[32];
  uint32_t qk[32];
  uint32_t qid[32];
};

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

// first index p in [dir[b], dir[b+1]) with q(p) >= q  (all keys of the band)
__device__ __forceinline__ uint32_t dir_lower(const uint32_t* __restrict__ skey,
                                              const uint32_t* __restrict__ dir, uint32_t off,
                                              uint32_t sh, uint32_t q) {
  uint32_t b = q >> sh;
  uint32_t lo = __ldg(dir + off + b), hi = __ldg(dir + off + b + 1);
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(skey + mid) & kQMask) < q) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// first index p with q(p) > q
__device__ __forceinline__ uint32_t dir_upper(const uint32_t* __restrict__ skey,
                                              const uint32_t* __restrict__ dir, uint32_t off,
                                              uint32_t sh, uint32_t q) {
  uint32_t b = q >> sh;
  uint32_t lo = __ldg(dir + off + b), hi = __ldg(dir + off + b + 1);
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(skey + mid) & kQMask) <= q) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <typename T>
__device__ __forceinline__ T warp_incl(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T a = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += a;
  }
  return v;
}

// Candidate index ranges of one query vertex in slab j (<= 2, nonempty ones first).
__device__ __forceinline__ int lane_ranges(int j, const BandConst& bc, uint32_t qq, double qa,
                                           double qb, double qinv4s, const uint32_t* skey,
                                           const uint32_t* dir, uint32_t bstart, uint32_t bend,
                                           uint32_t sh, uint32_t off, uint32_t lo[2],
                                           uint32_t hi[2]) {
  bool full = false;
  uint32_t dq = 0;
  const double invS = bc.invS[j];
  if (invS == 0.0) {
    full = true;  // c_j = 0: the innermost slab reaches every angle
  } else {
    // sin^2(dphi/2) <= (T - sinh^2((r_v - c_j)/2)) / (sinh r_v sinh c_j)
    //               = (T4 - h_c^2) / (4 sinh r_v sinh c_j),  h_c = 2 sinh((r_v - c_j)/2)
    // The window at the slab's inner boundary bounds the whole slab (DESIGN.md,
    // "Window monotonicity").  Upward pad: + T4 2^-48 / (4 s_v S_j).
    double h = __fma_rn(qa, bc.B[j], -__dmul_rn(qb, bc.A[j]));
    double num = __fma_rn(-h, h, bc.T4);
    double scale = __dmul_rn(qinv4s, invS);
    double ratio = __fma_rn(num, scale, __dmul_rn(bc.T4 * 0x1.0p-48, scale));
    if (!(ratio < 1.0)) {
      full = true;
    } else {
      float x = sqrtf(fmaxf((float)ratio, 0.0f));
      float dl = 2.0f * asinf(x);
      // angle -> q27 units, relative pad 2^-12 (fp32 error is < 1e-6), +2 quanta
      float dqf = dl * (float)RHG_Q27_SCALE * 1.000244140625f;
      if (dqf >= 67108860.0f) full = true;
      else dq = (uint32_t)dqf + 2u;
    }
  }
  if (full) {
    lo[0] = bstart; hi[0] = bend;
    lo[1] = bend; hi[1] = bend;
    return 1;
  }
  int64_t ql = (int64_t)qq - (int64_t)dq, qh = (int64_t)qq + (int64_t)dq;
  if (ql < 0) {
    lo[0] = bstart;
    hi[0] = dir_upper(skey, dir, off, sh, (uint32_t)qh);
    lo[1] = dir_lower(skey, dir, off, sh, (uint32_t)(ql + (1ll << kQBits)));
    hi[1] = bend;
    return 2;
  }
  if (qh > (int64_t)kQMax) {
    lo[0] = dir_lower(skey, dir, off, sh, (uint32_t)ql);
    hi[0] = bend;
    lo[1] = bstart;
    hi[1] = dir_upper(skey, dir, off, sh, (uint32_t)(qh - (1ll << kQBits)));
    return 2;
  }
  lo[0] = dir_lower(skey, dir, off, sh, (uint32_t)ql);
  hi[0] = dir_upper(skey, dir, off, sh, (uint32_t)qh);
  lo[1] = bend; hi[1] = bend;
  return 1;
}

template <int MODE, int FMT>
__global__ void __launch_bounds__(QK_THREADS)
    k_query(const QueryArgs A, const __grid_constant__ BandConst bc) {
  __shared__ WarpSm sm_all[QK_WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSm& sm = sm_all[wid];
  const uint32_t first = (blockIdx.x * QK_WARPS + wid) * 32u;
  if (first >= A.n) return;
  const uint32_t pos = first + lane;
  const bool valid = pos < A.n;
  const uint32_t k = valid ? (A.order ? A.order[pos] : pos) : 0u;

  PointRec q;
  q.theta = 0.0; q.s = 1.0; q.a = 1.0; q.b = 1.0;
  uint32_t qkey = 0, qid = 0;
  if (valid) {
    q = A.pts[k];
    qkey = A.skey[k];
    qid = A.sid[k];
  }
  const uint32_t qband = qkey >> kBandShift, qq = qkey & kQMask;
  const double qinv4s = 0.25 / q.s;
  sm.qth[lane] = q.theta;
  sm.q4s[lane] = 4.0 * q.s;
  sm.qa[lane] = q.a;
  sm.qb[lane] = q.b;
  sm.qk[lane] = valid ? k : 0xffffffffu;
  sm.qid[lane] = qid;
  if (MODE == QM_COUNT) sm.degc[lane] = 0;
  else sm.cur[lane] = valid ? A.offs[qid] : 0ull;
  __syncwarp();

  unsigned long long total = 0, consumed = 0;
  uint32_t head = 0, tail = 0;
  const bool outward = (FMT == RHG_EDGES_UNDIRECTED);
  int jlo = 0;
  if (outward) jlo = (int)__reduce_min_sync(FULL, valid ? qband : 0xffffu);
  const double T4 = bc.T4;

  // one batch: candidates [consumed, consumed + min(32, total - consumed)) of the
  // flattened range sequence; lane l tests candidate consumed + l.
  auto batch = [&]() {
      // -------------------------------------------------------------- batch
    const uint32_t cnt = (uint32_t)min(32ull, total - consumed);
    const bool act = (uint32_t)lane < cnt;
    const uint32_t e = head + lane;
    const bool ex = e < tail;
    const unsigned long long pl = ex ? sm.e_pref[e % RING] : ~0ull;
    const uint32_t bit =
        (lane > 0 && ex && pl < consumed + cnt) ? (1u << (uint32_t)(pl - consumed)) : 0u;
    const uint32_t M = __reduce_or_sync(FULL, bit);
    const uint32_t my_e = head + __popc(M & ((2u << lane) - 1u));
    const uint32_t es = sm.e_start[my_e % RING];
    const unsigned long long ep = sm.e_pref[my_e % RING];
    const uint32_t ql = sm.e_lane[my_e % RING] & 31u;
    const uint32_t cand = act ? es + (uint32_t)(consumed + lane - ep) : 0u;

    const double2* pp = reinterpret_cast<const double2*>(A.pts + cand);
    const double2 w0 = __ldg(pp), w1 = __ldg(pp + 1);  // (theta, s), (a, b)
    const double qth = sm.qth[ql];
    double d = __dsub_rn(qth, w0.x);
    const uint32_t dhi = (uint32_t)__double2hiint(d) & 0x7fffffffu;
    const bool big = act && dhi >= 0x3FB00000u;  // |d| >= 2^-4
    double Qv;
    if (__any_sync(FULL, big)) {
      if (dhi >= 0x400921FBu) {  // |d| >~ pi: go across the seam
        const double mx = fmax(qth, w0.x), mn = fmin(qth, w0.x);
        d = __dadd_rn(__dadd_rn(__dsub_rn(RHG_TWO_PI_HI, mx), mn), RHG_TWO_PI_LO);
      }
      const double u = __dmul_rn(d, d);
      Qv = big ? poly_long(u) : poly_short(u);
    } else {
      Qv = poly_short(__dmul_rn(d, d));
    }
    const double sn = __dmul_rn(d, Qv);
    const double Bv = __dmul_rn(sn, sn);
    const double p1 = __dmul_rn(sm.qa[ql], w1.y);
    const double p2 = __dmul_rn(sm.qb[ql], w1.x);
    const double h = __dsub_rn(p1, p2);
    const double A4 = __dmul_rn(sm.q4s[ql], w0.y);
    const double C = __dmul_rn(A4, Bv);
    const double S4 = __fma_rn(h, h, C);
    bool hit = act && (S4 <= T4);
    if (!outward) hit = hit && (cand != sm.qk[ql]);  // no self-loops

    const uint32_t hm = __ballot_sync(FULL, hit);
    const uint32_t peers = __match_any_sync(FULL, act ? ql : (32u + lane));
    const bool leader = act && (__ffs(peers) - 1) == lane;
    if (MODE == QM_COUNT) {
      if (leader) {
        const uint32_t c = __popc(hm & peers);
        if (c) sm.degc[ql] += c;
      }
    } else {
      const unsigned long long base = act ? sm.cur[ql] : 0ull;
      if (hit) {
        const unsigned long long o = base + __popc(hm & peers & ((1u << lane) - 1u));
        const uint32_t wid_ = __ldg(A.sid + cand);
        if (FMT == RHG_CSR) {
          A.col[o] = wid_;
        } else {
          const uint32_t vid = sm.qid[ql];
          uint2 pr = vid < wid_ ? make_uint2(vid, wid_) : make_uint2(wid_, vid);
          reinterpret_cast<uint2*>(A.pairs)[o] = pr;
        }
      }
      __syncwarp();
      if (leader) sm.cur[ql] = base + __popc(hm & peers);
    }
    // advance the ring head to the range holding candidate consumed + cnt
    const uint32_t e_last = __shfl_sync(FULL, my_e, cnt - 1);
    const unsigned long long end_last =
        (e_last + 1 < tail) ? sm.e_pref[(e_last + 1) % RING] : total;
    consumed += cnt;
    head = (end_last == consumed) ? e_last + 1 : e_last;
    __syncwarp();
  };

  for (int j = jlo; j < bc.L; ++j) {
    const uint32_t bstart = A.lay->start[j], bend = A.lay->start[j + 1];
    if (bstart == bend) continue;
    uint32_t lo[2] = {0, 0}, hi[2] = {0, 0};
    if (valid && (!outward || j >= (int)qband)) {
      lane_ranges(j, bc, qq, q.a, q.b, qinv4s, A.skey, A.dir, bstart, bend, A.lay->shift[j],
                  A.lay->dir_off[j], lo, hi);
      if (outward && j == (int)qband) {  // same slab: only partners sorted after v (Z9)
        if (lo[0] < k + 1) lo[0] = k + 1;
        if (lo[1] < k + 1) lo[1] = k + 1;
      }
    }
    const uint32_t c0 = hi[0] > lo[0] ? hi[0] - lo[0] : 0u;
    const uint32_t c1 = hi[1] > lo[1] ? hi[1] - lo[1] : 0u;
    const uint32_t ne = (c0 > 0) + (c1 > 0);
    const unsigned long long cs = (unsigned long long)c0 + c1;
    const uint32_t ne_inc = warp_incl(ne);
    const unsigned long long cs_inc = warp_incl(cs);
    const uint32_t ne_tot = __shfl_sync(FULL, ne_inc, 31);
    const unsigned long long cs_tot = __shfl_sync(FULL, cs_inc, 31);
    if (cs_tot == 0) continue;
    {
      uint32_t slot = tail + ne_inc - ne;
      unsigned long long pref = total + cs_inc - cs;
      if (c0) {
        sm.e_start[slot % RING] = lo[0];
        sm.e_pref[slot % RING] = pref;
        sm.e_lane[slot % RING] = (uint32_t)lane;
        ++slot;
        pref += c0;
      }
      if (c1) {
        sm.e_start[slot % RING] = lo[1];
        sm.e_pref[slot % RING] = pref;
        sm.e_lane[slot % RING] = (uint32_t)lane;
      }
    }
    tail += ne_tot;
    total += cs_tot;
    __syncwarp();

    while (total - consumed >= 32ull) batch();
  }
  while (total > consumed) batch();
  if (MODE == QM_COUNT) {
    if (valid) A.deg[qid] = sm.degc[lane];
    if (lane == 0) atomicAdd(&A.sc->candidates, total);
  }
}

cudaError_t launch_query(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const BandConst& bc,
                         cudaStream_t st) {
  uint32_t groups = (qa.n + 31) / 32;
  uint32_t blocks = (groups + QK_WARPS - 1) / QK_WARPS;
  if (blocks == 0) return cudaSuccess;
  if (mode == QM_COUNT) {
    if (fmt == RHG_CSR) k_query<QM_COUNT, RHG_CSR><<<blocks, QK_THREADS, 0, st>>>(qa, bc);
    else k_query<QM_COUNT, RHG_EDGES_UNDIRECTED><<<blocks, QK_THREADS, 0, st>>>(qa, bc);
  } else {
    if (fmt == RHG_CSR) k_query<QM_EMIT, RHG_CSR><<<blocks, QK_THREADS, 0, st>>>(qa, bc);
    else k_query<QM_EMIT, RHG_EDGES_UNDIRECTED><<<blocks, QK_THREADS, 0, st>>>(qa, bc);
  }
  return cudaGetLastError();
}

}  // namespace rhg
