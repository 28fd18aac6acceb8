// rhg_abi.cu -- the C-ABI (include/rhg.h): argument validation, host-side model
// parameters (L0), workspace layout and the launch sequence of Algorithm 1.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>

#include <vector>

#include "rhg_internal.cuh"

using namespace rhg;

#define RHG_VERSION "rhg-b200 r01"

namespace {

// ------------------------------------------------------------------ L0 math
// Expected average degree, Krioukov Eq. (22) as printed in PAPER.md:178-182 with
// zeta = 1:
//   kbar(R) = 2/pi xi^2 n [ e^{-R/2} + e^{-alpha R} ( alpha R/2 (pi/4 alpha^-2
//             - (pi-1) alpha^-1 + (pi-2)) - 1 ) ],   xi = alpha / (alpha - 1/2).
double kbar_of_radius(double n, double alpha, double R) {
  const double pi = 3.14159265358979323846;
  const double xi = alpha / (alpha - 0.5);
  const double inv = 1.0 / alpha;
  const double poly = (pi / 4.0) * inv * inv - (pi - 1.0) * inv + (pi - 2.0);
  return (2.0 / pi) * xi * xi * n *
         (std::exp(-R / 2.0) + std::exp(-alpha * R) * (alpha * R / 2.0 * poly - 1.0));
}

// getTargetRadius.  kbar(R) rises from 0 at R = 0 to one peak
// and then falls (Z5); locate the peak by golden-section search, then
// bisect the falling branch down to adjacent doubles.
rhg_status target_radius(double n, double kbar, double alpha, double* R) {
  if (!(alpha > 0.5) || !(kbar > 0.0) || !std::isfinite(kbar) || !(n >= 2.0)) return RHG_ERR_INVALID;
  double a = 0.0, b = 50.0;
  const double g = 0.6180339887498949;
  double x1 = b - g * (b - a), x2 = a + g * (b - a);
  double f1 = kbar_of_radius(n, alpha, x1), f2 = kbar_of_radius(n, alpha, x2);
  for (int it = 0; it < 200; ++it) {
    if (f1 < f2) {
      a = x1; x1 = x2; f1 = f2; x2 = a + g * (b - a); f2 = kbar_of_radius(n, alpha, x2);
    } else {
      b = x2; x2 = x1; f2 = f1; x1 = b - g * (b - a); f1 = kbar_of_radius(n, alpha, x1);
    }
  }
  double lo = 0.5 * (a + b), hi = 10.0 * std::log(n) + 50.0;
  if (kbar > kbar_of_radius(n, alpha, lo) || kbar < kbar_of_radius(n, alpha, hi))
    return RHG_ERR_CALIBRATION;
  while (true) {
    double mid = lo + 0.5 * (hi - lo);
    if (!(mid > lo && mid < hi)) break;
    if (kbar_of_radius(n, alpha, mid) > kbar) lo = mid; else hi = mid;
  }
  *R = lo + 0.5 * (hi - lo);
  return RHG_OK;
}

// Layout defaults (Z7): L <= 16 slabs; width ratio p = 0.85 while
// ceil(ln n) <= 17, rising by 0.04 per further unit of ceil(ln n) up to 0.95 (the
// paper settled on p = 0.9 by experiment; with L capped at 16 the
// measured optimum is 0.85 at n = 1e7 and 0.93 at n = 1e8, profiles/r02_layout_sweep.log).
constexpr int kDefaultMaxBands = 16;
double default_band_ratio(uint64_t n) {
  const double lg = std::ceil(std::log((double)(n < 2 ? 2 : n)));
  const double p = 0.85 + 0.04 * (lg - 17.0);
  return p < 0.85 ? 0.85 : (p > 0.95 ? 0.95 : p);
}

// "log n" slabs (base unstated; Z7): ceil(ln n), capped at
// 16 so that one warp evaluates all windows of two vertices at once (k_query).
// The edge set does not depend on L or p.
int default_bands(uint64_t n) {
  int L = (int)std::ceil(std::log((double)n));
  if (L < 1) L = 1;
  return L > kDefaultMaxBands ? kDefaultMaxBands : L;
}

// Slab boundaries: c_0 = 0, c_1 = (1-p)R/(1-p^L),
// c_{k+1} - c_k = p (c_k - c_{k-1}), c_L = R.
void make_boundaries(double R, int L, double p, double* c) {
  const double c1 = (1.0 - p) * R / (1.0 - std::pow(p, L));
  double w = c1;
  c[0] = 0.0;
  for (int k = 1; k < L; ++k) {
    c[k] = c[k - 1] + w;
    w *= p;
  }
  c[L] = R;
}

uint64_t heavy_cap_for(uint64_t n) {
  uint64_t c = n / 128 + 4096;
  return c < n ? c : n;
}

rhg_status make_band_const(uint64_t n, double R, const rhg_options* opt, BandConst* bc) {
  int L = (opt && opt->num_bands > 0) ? opt->num_bands : default_bands(n);
  double p = (opt && opt->band_ratio > 0.0) ? opt->band_ratio : default_band_ratio(n);
  if (L < 1 || L > kMaxBands || !(p > 0.0 && p < 1.0)) return RHG_ERR_INVALID;
  memset(bc, 0, sizeof(*bc));
  bc->L = L;
  bc->R = R;
  const double h = std::sinh(R / 2.0);
  bc->T4 = 4.0 * h * h;
  make_boundaries(R, L, p, bc->c);
  for (int j = 0; j <= L; ++j) {
    bc->A[j] = std::exp(0.5 * bc->c[j]);
    bc->B[j] = std::exp(-0.5 * bc->c[j]);
    bc->invS[j] = bc->c[j] > 0.0 ? 1.0 / std::sinh(bc->c[j]) : 0.0;
    bc->padS[j] = bc->T4 * 0x1.0p-48 * bc->invS[j];
  }
  bc->T4min = bc->T4 * 0x1.0p-10;
  bc->heavy_threshold = (opt && opt->heavy_threshold) ? (double)opt->heavy_threshold : 1024.0;
  bc->heavy_cap = (uint32_t)heavy_cap_for(n);
  const int ns = (opt && opt->shard_count > 1) ? opt->shard_count : 1;
  const int si = (opt && ns > 1) ? opt->shard_index : 0;
  if (si < 0 || si >= ns || ns > 4096) return RHG_ERR_INVALID;
  bc->shard = (uint32_t)si;
  bc->nshards = (uint32_t)ns;
  return RHG_OK;
}

// ------------------------------------------------------------------ workspace
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t theta, r, keys_a, vals_a, keys_b, vals_b, sort_tmp, hist, lay, pts, sid2, dir, deg, cdeg, offs,
      scan_tmp, heavy_scan_tmp, sc, st_rowptr, st_edges, st_in_theta, st_in_r, bits, total;
  size_t h_pstart, h_plen, h_poff, h_np, h_vtot, h_vtot_off, h_cc,
      h_choff, h_cvtx, h_cpiece, h_chits, h_cpos, h_meta, h_bits;
  size_t b_bits, b_over, q_order, q_cell_lo, q_cell_cnt, q_cell_off;
  size_t s_work, s_prefix, s_plan, s_hub;
  uint64_t vcap, nslots_cap, chunk_cap, hbits_cap, light_warps, dir_cap, item_cap;
};

constexpr uint64_t kChunkExtra = 1ull << 21;
#ifndef RHG_CHUNK_MIN
#define RHG_CHUNK_MIN 1024
#endif
constexpr uint64_t kChunkMin = RHG_CHUNK_MIN;

int bands_for(uint64_t n, const rhg_options* opt) {
  return (opt && opt->num_bands > 0) ? opt->num_bands : default_bands(n);
}

Layout plan_layout(uint64_t n, rhg_format f, uint64_t cap, int host, int nbands) {
  Layout L{};
  if (nbands < 1) nbands = 1;
  if (nbands > kMaxBands) nbands = kMaxBands;
  L.vcap = heavy_cap_for(n);
  L.nslots_cap = L.vcap * (uint64_t)kRangesPerSlab * (uint64_t)nbands;
  L.chunk_cap = L.vcap + kChunkExtra;
  // Hub ballot words (k_heavy) are sized from the output capacity (~1.1-1.4 tests
  // per directed CSR entry); light warps get kLightBitRows x 32 words each.
  const uint64_t cap_tests = (f == RHG_CSR) ? cap + cap / 2 : 2 * cap;
  L.light_warps = (n + 31) / 32;
  L.item_cap = L.vcap + L.light_warps + 1;  // shard plan: hub vertices + light groups
  L.hbits_cap = cap_tests / 32 + L.vcap * 48 + 1024;  // >= nchunks (CH/32 + 8) when hubs fit
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += al(bytes);
    return at;
  };
  L.theta = take(8 * n);
  L.r = take(8 * n);
  L.keys_a = take(4 * n);
  L.vals_a = take(4 * n);
  L.keys_b = take(4 * n);
  L.vals_b = take(4 * n);
  L.sort_tmp = take(radix_sort_tmp_bytes(n));
  L.hist = take(4 * kMaxBands);
  L.lay = take(sizeof(BandLayout));
  L.pts = take(2 * sizeof(PointRec) * n);  // doubled SoA
  L.sid2 = take(2 * 4 * n);
  L.dir_cap = 2 * RHG_DIR_PER_PT * n + 4 * kMaxBands + 8;  // <= 2 RHG_DIR_PER_PT n_j + 1 per band
  L.dir = take(4 * L.dir_cap);
  L.deg = take(4 * n);
  L.cdeg = take(4 * n);
  L.offs = take(8 * (n + 1));
  {
    uint64_t m = n;
    if (L.vcap > m) m = L.vcap;
    if ((uint64_t)kQuerySectors * kMaxBands > m) m = (uint64_t)kQuerySectors * kMaxBands;
    if (L.chunk_cap > m) m = L.chunk_cap;
    if (L.item_cap > m) m = L.item_cap;
    L.scan_tmp = take(scan_tmp_bytes(m));
    L.heavy_scan_tmp = take(scan_tmp_bytes(m));
  }
  L.h_pstart = take(4 * L.nslots_cap);
  L.h_plen = take(4 * L.nslots_cap);
  L.h_poff = take(4 * L.nslots_cap);
  L.h_np = take(4 * L.vcap);
  L.h_vtot = take(4 * L.vcap);
  L.h_vtot_off = take(8 * (L.vcap + 1));
  L.h_cc = take(4 * L.vcap);
  L.h_choff = take(8 * (L.vcap + 1));
  L.h_cvtx = take(4 * L.chunk_cap);
  L.h_cpiece = take(4 * L.chunk_cap);
  L.h_chits = take(4 * L.chunk_cap);
  L.h_cpos = take(8 * (L.chunk_cap + 1));
  L.h_bits = take(4 * L.hbits_cap);
  L.b_bits = take(4ull * kLightBitRows * 32 * L.light_warps);
  L.b_over = take(4 * L.light_warps);
  L.q_order = take(4 * n);
  L.q_cell_lo = take(4 * kQuerySectors * kMaxBands);
  L.q_cell_cnt = take(4 * kQuerySectors * kMaxBands);
  L.q_cell_off = take(8 * (kQuerySectors * kMaxBands + 1));
  L.s_work = take(4 * L.item_cap);
  L.s_prefix = take(8 * (L.item_cap + 1));
  L.s_plan = take(sizeof(ShardPlan));
  L.s_hub = take(8 * 4096);  // per-shard hub work (shard_count <= 4096)
  L.h_meta = take(sizeof(HeavyMeta));
  L.sc = take(sizeof(DevScalars));
  L.st_rowptr = host && f == RHG_CSR ? take(8 * (n + 1)) : o;
  L.st_edges = host ? take(f == RHG_CSR ? 4 * cap : 8 * cap) : o;
  L.st_in_theta = o;  // host-mode inputs reuse theta / r
  L.st_in_r = o;
  L.bits = o;
  L.total = o;
  return L;
}

cudaError_t& last_cuda_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}
int& last_cuda_error_line() {
  static thread_local int l = 0;
  return l;
}

// Page-locked readback slot, one per host thread (a process-wide slot
// let concurrent callers read each other's totals).  Its address is stable per
// thread, so the CUDA graphs cached per thread (graph_cache) stay valid.
struct PinnedSlot {
  DevScalars* p = nullptr;
  ~PinnedSlot() {
    if (p) cudaFreeHost(p);
  }
};
DevScalars* pinned_scalars() {
  static thread_local PinnedSlot slot;
  if (!slot.p && cudaMallocHost(&slot.p, sizeof(DevScalars)) != cudaSuccess) slot.p = nullptr;
  return slot.p;
}

#define CK(x)                                  \
  do {                                         \
    cudaError_t e__ = (x);                     \
    if (e__ != cudaSuccess) {                  \
      last_cuda_error() = e__;                 \
      last_cuda_error_line() = __LINE__;       \
      return RHG_ERR_CUDA;                     \
    }                                          \
  } while (0)

// Side stream for the hub path: the hub count / emit kernels run next to the light
// kernels (they touch disjoint vertices and rows), forked from and joined back to
// the caller's stream with events, so the caller still sees one stream.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool ok = false;
  SideStream() {
    ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
};
// one side stream (and its events) per thread and device: the caller's stream
// belongs to the current device
constexpr int kMaxDevices = 64;
SideStream& side_stream() {
  static thread_local SideStream* ss[kMaxDevices] = {};
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  if (!ss[d]) ss[d] = new SideStream();
  return *ss[d];
}

struct Timer {
  bool on = false;
  cudaEvent_t ev[9];
  cudaStream_t st;
  int n = 0;
  void init(bool enable, cudaStream_t s) {
    on = enable;
    st = s;
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark() {
    if (on && n < 9) cudaEventRecord(ev[n++], st);
  }
  float between(int a, int b) {
    float ms = 0;
    if (on && b < n) cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return ms;
  }
  ~Timer() {
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
};

// CUDA-graph replay of the two halves of a call (rhg_options.graph): one cached
// executable per half and thread, re-captured whenever the arguments change.
struct GraphSlot {
  std::vector<char> key;
  cudaGraphExec_t exec = nullptr;
};
struct GraphCache {
  GraphSlot a, b;
};
GraphCache& graph_cache() {
  static thread_local GraphCache gc;
  return gc;
}
template <typename F>
rhg_status graph_run(GraphSlot& g, const std::vector<char>& key, cudaStream_t st, F&& fn) {
  if (!g.exec || g.key != key) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.key.clear();
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const rhg_status s = fn();
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (s != RHG_OK) {
      if (graph) cudaGraphDestroy(graph);
      return s;
    }
    CK(e);
    const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(ei);
    g.key = key;
  }
  CK(cudaGraphLaunch(g.exec, st));
  return RHG_OK;
}

// The full pipeline.  sample == true: Philox points (alpha, seed); else the
// caller's points (theta_in, r_in).
rhg_status run(uint64_t n, bool sample, double alpha, uint64_t seed, const double* theta_in,
               const double* r_in, double R, const rhg_output* out, cudaStream_t st) {
  if (!out || !out->num_edges) return RHG_ERR_INVALID;
  if (n < 2 || n >= (1ull << 31)) return RHG_ERR_INVALID;  // doubled positions < 2^32
  if (!(R >= 0.0) || !std::isfinite(R)) return RHG_ERR_INVALID;
  if (sample && (!(alpha > 0.5) || !std::isfinite(std::cosh(alpha * R)))) return RHG_ERR_INVALID;
  if (!std::isfinite(std::sinh(R / 2.0) * std::sinh(R / 2.0) * 4.0)) return RHG_ERR_INVALID;
  const rhg_format f = out->format;
  if (f != RHG_CSR && f != RHG_EDGES_UNDIRECTED) return RHG_ERR_INVALID;
  const int host = out->host_buffers ? 1 : 0;
  if (f == RHG_CSR && (!out->row_ptr || (!out->col && out->capacity_edges))) return RHG_ERR_INVALID;
  if (f == RHG_EDGES_UNDIRECTED && !out->pairs && out->capacity_edges) return RHG_ERR_INVALID;
  // device outputs are written in whole 32-byte sectors (k_query): 32-byte alignment
  if (!host && (((uintptr_t)out->col | (uintptr_t)out->pairs) & 31)) return RHG_ERR_INVALID;
  if (!sample && (!theta_in || !r_in)) return RHG_ERR_INVALID;
  const int order = out->options ? out->options->vertex_order : 0;
  if (order != 0 && order != 1) return RHG_ERR_INVALID;
  BandConst bc;
  rhg_status s = make_band_const(n, R, out->options, &bc);
  if (s != RHG_OK) return s;
  const Layout Lw = plan_layout(n, f, out->capacity_edges, host, bc.L);
  if (!out->workspace || out->workspace_bytes < Lw.total) return RHG_ERR_WORKSPACE;
  DevScalars* pin = pinned_scalars();
  if (!pin) return RHG_ERR_CUDA;

  char* ws = (char*)out->workspace;
  double* theta = (double*)(ws + Lw.theta);
  double* r = (double*)(ws + Lw.r);
  uint32_t* keys_a = (uint32_t*)(ws + Lw.keys_a);
  uint32_t* vals_a = (uint32_t*)(ws + Lw.vals_a);
  uint32_t* keys_b = (uint32_t*)(ws + Lw.keys_b);
  uint32_t* vals_b = (uint32_t*)(ws + Lw.vals_b);
  uint32_t* hist = (uint32_t*)(ws + Lw.hist);
  BandLayout* lay = (BandLayout*)(ws + Lw.lay);
  PointRec* pts = (PointRec*)(ws + Lw.pts);
  uint32_t* sid2 = (uint32_t*)(ws + Lw.sid2);
  uint32_t* dir = (uint32_t*)(ws + Lw.dir);
  uint32_t* deg = (uint32_t*)(ws + Lw.deg);
  uint64_t* offs_ws = (uint64_t*)(ws + Lw.offs);
  DevScalars* sc = (DevScalars*)(ws + Lw.sc);
  uint64_t* row_ptr_dev = host ? (uint64_t*)(ws + Lw.st_rowptr) : out->row_ptr;
  uint32_t* col_dev = host ? (uint32_t*)(ws + Lw.st_edges) : out->col;
  uint32_t* pairs_dev = host ? (uint32_t*)(ws + Lw.st_edges) : out->pairs;
  // Generate path: K1 stores the points only if the caller asked for them (the
  // index build re-derives them from Philox); device-mode callers get them directly.
  PhiloxPoints gen{};
  if (sample) {
    gen.seed = seed;
    gen.two_over_alpha = 2.0 / alpha;
    gen.half_span = (std::cosh(alpha * R) - 1.0) / 2.0;
    gen.R = R;
    set_band_cuts(gen, alpha, bc);
    if (host) {
      if (!out->theta_out) theta = nullptr;
      if (!out->r_out) r = nullptr;
    } else {
      theta = out->theta_out;
      r = out->r_out;
    }
  }

  Timer tm;
  tm.init(out->timing != nullptr, st);
  int launches = 0;
  float ms_h2d = 0;
  HeavyMeta* hmeta = (HeavyMeta*)(ws + Lw.h_meta);
  QueryArgs qa{};
  HeavyArgs ha{};
  uint64_t* offs = nullptr;
  SideStream& ss = side_stream();
  if (!ss.ok) return RHG_ERR_CUDA;
  CK(radix_sort_prepare());
  // part A: sampling through the degree scan, ending with the 8-byte readback
  auto partA = [&]() -> rhg_status {
  tm.mark();  // 0
  CK(cudaMemsetAsync(hist, 0, 4 * kMaxBands, st));
  CK(cudaMemsetAsync(sc, 0, sizeof(DevScalars), st));
  if (sample) {
    CK(launch_sample(n, gen, bc, theta, r, keys_a, vals_a, hist, st));
    ++launches;
  } else {
    const double* th_src = theta_in;
    const double* r_src = r_in;
    if (host) {
      CK(cudaMemcpyAsync(theta, theta_in, 8 * n, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(r, r_in, 8 * n, cudaMemcpyHostToDevice, st));
      th_src = theta;
      r_src = r;
    } else {
      theta = const_cast<double*>(theta_in);
      r = const_cast<double*>(r_in);
    }
    CK(launch_keys_from_points(n, th_src, r_src, bc, keys_a, vals_a, hist, sc, st));
    ++launches;
  }
  CK(launch_band_layout(bc, hist, lay, hmeta, st));
  ++launches;
  tm.mark();  // 1
  CK(radix_sort((uint32_t)n, keys_a, vals_a, keys_b, vals_b, ws + Lw.sort_tmp, 0, 32, st,
                &launches));
  tm.mark();  // 2
  CK(launch_build_index((uint32_t)n, theta, r, keys_a, vals_a, lay, bc.L, pts, sid2, dir,
                        sample ? &gen : nullptr, order, st, &launches));
  CK(launch_query_order(keys_a, lay, bc.L, (uint32_t*)(ws + Lw.q_cell_lo),
                        (uint32_t*)(ws + Lw.q_cell_cnt), (uint64_t*)(ws + Lw.q_cell_off),
                        (uint32_t*)(ws + Lw.q_order), ws + Lw.scan_tmp, st, &launches));
  tm.mark();  // 3

  if (order == 1 && out->perm_out)  // id (sorted position) -> sample / input index
    CK(cudaMemcpyAsync(out->perm_out, vals_a, 4 * n,
                       host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
  qa = QueryArgs{};
  qa.n = (uint32_t)n;
  qa.labels = (uint32_t)order;
  qa.poff = f == RHG_EDGES_UNDIRECTED ? 1u : 0u;  // rows of the list need no id order
  qa.force_wide = (out->options && out->options->wide_positions == 1) ? 1u : 0u;
  qa.stats = out->timing ? 1u : 0u;
  qa.pts = pts;
  qa.skey = keys_a;
  qa.sid = vals_a;
  qa.sid2 = sid2;
  qa.dir = dir;
  qa.lay = lay;
  qa.order = (const uint32_t*)(ws + Lw.q_order);
  qa.bits = (uint32_t*)(ws + Lw.b_bits);
  qa.warp_over = (uint32_t*)(ws + Lw.b_over);
  qa.deg = deg;
  qa.cdeg = (uint32_t*)(ws + Lw.cdeg);
  qa.sc = sc;
  if (bc.nshards > 1) {
    CK(cudaMemsetAsync(deg, 0, 4 * n, st));  // rows of other shards stay empty
    qa.shard_plan = (const ShardPlan*)(ws + Lw.s_plan);
    CK(launch_shard_plan((uint32_t)n, qa, bc, f == RHG_EDGES_UNDIRECTED ? 1 : 0,
                         (uint32_t*)(ws + Lw.s_work), (uint64_t*)(ws + Lw.s_prefix), Lw.item_cap,
                         ws + Lw.scan_tmp, (unsigned long long*)(ws + Lw.s_hub),
                         (ShardPlan*)(ws + Lw.s_plan), st, &launches));
  }
  ha = HeavyArgs{};
  ha.pstart = (uint32_t*)(ws + Lw.h_pstart);
  ha.plen = (uint32_t*)(ws + Lw.h_plen);
  ha.poff = (uint32_t*)(ws + Lw.h_poff);
  ha.np = (uint32_t*)(ws + Lw.h_np);
  ha.vtot = (uint32_t*)(ws + Lw.h_vtot);
  ha.vtot_off = (uint64_t*)(ws + Lw.h_vtot_off);
  ha.cc = (uint32_t*)(ws + Lw.h_cc);
  ha.choff = (uint64_t*)(ws + Lw.h_choff);
  ha.chunk_vtx = (uint32_t*)(ws + Lw.h_cvtx);
  ha.chunk_piece = (uint32_t*)(ws + Lw.h_cpiece);
  ha.chunk_hits = (uint32_t*)(ws + Lw.h_chits);
  ha.chunk_pos = (uint64_t*)(ws + Lw.h_cpos);
  ha.bits = (uint32_t*)(ws + Lw.h_bits);
  ha.bits_cap = Lw.hbits_cap;
  ha.meta = hmeta;
  ha.vcap = Lw.vcap;
  ha.chunk_cap = Lw.chunk_cap;
  ha.chunk_min = kChunkMin;
  // hub path on the side stream, light vertices on the caller's stream
  CK(cudaEventRecord(ss.fork, st));
  CK(cudaStreamWaitEvent(ss.s, ss.fork, 0));
  CK(launch_heavy_plan(f, qa, ha, bc, ws + Lw.heavy_scan_tmp, ss.s, &launches));
  CK(launch_heavy(QM_COUNT, f, qa, ha, bc, ss.s));
  ++launches;
  CK(exclusive_scan_u32_u64_dev(ha.chunk_cap, &hmeta->nchunks, ha.chunk_hits, ha.chunk_pos,
                                ws + Lw.heavy_scan_tmp, &hmeta->hits, ss.s, &launches));
  CK(cudaEventRecord(ss.join, ss.s));
  CK(launch_query(QM_COUNT, f, qa, bc, st));
  ++launches;
  CK(cudaStreamWaitEvent(st, ss.join, 0));
  tm.mark();  // 4
  offs = (f == RHG_CSR) ? row_ptr_dev : offs_ws;
  if (f == RHG_CSR)
    CK(exclusive_scan_u32_u64((uint32_t)n, deg, offs, ws + Lw.scan_tmp, &sc->total, st, &launches));
  else  // list: hub rows, then one entry per light warp (k_query)
    CK(exclusive_scan_u32_u64_dev(std::min<uint64_t>(n, bc.heavy_cap + (n + 31) / 32 + 1),
                                  &hmeta->list_len, deg, offs, ws + Lw.scan_tmp, &sc->total, st,
                                  &launches));
  tm.mark();  // 5
  CK(cudaMemcpyAsync(pin, sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
  return RHG_OK;
  };
  // graph mode (rhg_options.graph): both parts are captured once per argument set
  // and replayed as CUDA graphs; the legacy default stream cannot be captured
  const bool use_graph = out->options && out->options->graph == 1 && !out->timing && st != nullptr;
  std::vector<char> key;
  if (use_graph) {
    auto add = [&](const void* p, size_t b) {
      key.insert(key.end(), (const char*)p, (const char*)p + b);
    };
    const uint64_t hdr[4] = {n, (uint64_t)sample, seed, (uint64_t)(uintptr_t)st};
    add(hdr, sizeof(hdr));
    add(&alpha, 8);
    add(&R, 8);
    add(&theta_in, sizeof(theta_in));
    add(&r_in, sizeof(r_in));
    rhg_output o = *out;
    o.num_edges = nullptr; o.R_used = nullptr; o.options = nullptr; o.timing = nullptr;
    add(&o, sizeof(o));
    add(out->options, sizeof(rhg_options));
  }
  // part B: the emit passes (and host copies).  Device buffers: enqueued right
  // behind part A -- the emit kernels read the edge total on the device and write
  // nothing if it exceeds the capacity -- so the call synchronises once, at the end.
  // Host buffers: the copies are sized by the total, read back in between.
  uint64_t copy_total = 0;
  auto partB = [&]() -> rhg_status {
  qa.offs = offs;
  qa.col = col_dev;
  qa.pairs = pairs_dev;
  qa.total_dev = &sc->total;
  qa.cap = out->capacity_edges;
  qa.out_cap = out->capacity_edges;
  // hub chunks replay their bits unless the hub bit buffer was too small (checked
  // on the device); light warps replay theirs unless they ran out of bit words.
  CK(cudaEventRecord(ss.fork, st));
  CK(cudaStreamWaitEvent(ss.s, ss.fork, 0));
  CK(launch_heavy(QM_EMIT_BITS, f, qa, ha, bc, ss.s));
  CK(cudaEventRecord(ss.join, ss.s));
#ifdef RHG_BOUNDS
  CK(cudaStreamSynchronize(ss.s));
#endif
  CK(launch_query(QM_EMIT_BITS, f, qa, bc, st));  // warps whose bits overflowed re-test
  CK(cudaStreamWaitEvent(st, ss.join, 0));
#ifdef RHG_BOUNDS
  {
    cudaError_t e = cudaStreamSynchronize(st);
    DevScalars d;
    cudaMemcpy(&d, sc, sizeof(d), cudaMemcpyDeviceToHost);
    fprintf(stderr, "RHG_BOUNDS: sync %s, check line %u block %llu thread %llu\n",
            cudaGetErrorString(e), d.dbg_line, d.dbg[0], d.dbg[1]);
    CK(e);
  }
#endif
  launches += 2;
  tm.mark();  // 6
  if (host) {
    if (f == RHG_CSR) {
      CK(cudaMemcpyAsync(out->row_ptr, row_ptr_dev, 8 * (n + 1), cudaMemcpyDeviceToHost, st));
      if (copy_total)
        CK(cudaMemcpyAsync(out->col, col_dev, 4 * copy_total, cudaMemcpyDeviceToHost, st));
    } else if (copy_total) {
      CK(cudaMemcpyAsync(out->pairs, pairs_dev, 8 * copy_total, cudaMemcpyDeviceToHost, st));
    }
    if (sample && out->theta_out)
      CK(cudaMemcpyAsync(out->theta_out, theta, 8 * n, cudaMemcpyDeviceToHost, st));
    if (sample && out->r_out)
      CK(cudaMemcpyAsync(out->r_out, r, 8 * n, cudaMemcpyDeviceToHost, st));
  }
  tm.mark();  // 7
  return RHG_OK;
  };
  GraphCache& gc = graph_cache();
  rhg_status s2 = RHG_OK;
  DevScalars hs;
  if (!host) {
    auto both = [&]() -> rhg_status {
      const rhg_status sa = partA();
      return sa != RHG_OK ? sa : partB();
    };
    s2 = use_graph ? graph_run(gc.a, key, st, both) : both();
    if (s2 != RHG_OK) return s2;
    CK(cudaStreamSynchronize(st));
    hs = *pin;
    if (hs.domain_error) return RHG_ERR_DOMAIN;
    *out->num_edges = hs.total;
    if (out->R_used) *out->R_used = R;
    if (hs.total > out->capacity_edges) return RHG_ERR_CAPACITY;  // the emit wrote nothing
  } else {
    s2 = use_graph ? graph_run(gc.a, key, st, partA) : partA();
    if (s2 != RHG_OK) return s2;
    CK(cudaStreamSynchronize(st));
    hs = *pin;
    if (hs.domain_error) return RHG_ERR_DOMAIN;
    *out->num_edges = hs.total;
    if (out->R_used) *out->R_used = R;
    if (hs.total > out->capacity_edges) return RHG_ERR_CAPACITY;
    copy_total = hs.total;
    if (use_graph) {
      key.insert(key.end(), (const char*)&hs.total, (const char*)&hs.total + sizeof(hs.total));
      s2 = graph_run(gc.b, key, st, partB);
    } else {
      s2 = partB();
    }
  }
  if (s2 != RHG_OK) return s2;
  if (host || out->timing) CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (out->timing) {
    rhg_timing* t = out->timing;
    t->ms_sample = tm.between(0, 1);
    t->ms_sort = tm.between(1, 2);
    t->ms_index = tm.between(2, 3);
    t->ms_count = tm.between(3, 4);
    t->ms_scan = tm.between(4, 5);
    t->ms_emit = tm.between(5, 6);
    t->ms_copy = tm.between(6, 7) + ms_h2d;
    t->ms_total = tm.between(0, 7);
    t->candidates = hs.candidates;
    t->certain = hs.certain;
    t->launches = (uint64_t)launches;
    t->emit_retested = hs.bit_overflow;
  }
  return RHG_OK;
}

// ------------------------------------------------------------------ dynamic update
// Workspace of rhg_update_moved: the generator's layout (no hub scratch, no output
// staging) plus the update's arrays.
struct UpdLayout {
  Layout base;
  size_t pm, mbits, flag, fpos, qorder, morder, nlm, new_col, units, uoff, unit_j, mlist, mcount,
      n_rem, n_add, off_rem, off_add, rbits, abits, total;
  uint64_t rbits_words, abits_words;
  uint64_t unit_cap;
};

// delta work units: one per moved vertex, plus 512-entry chunks of long rows
uint64_t update_unit_cap(uint64_t n, uint64_t row_capacity, uint64_t old_entries) {
  return 2 * n + (row_capacity + old_entries) / 512 + 2;
}

UpdLayout plan_update(uint64_t n, uint64_t row_capacity, uint64_t old_entries, int nbands) {
  UpdLayout U{};
  U.base = plan_layout(n, RHG_CSR, 0, 0, nbands);
  U.unit_cap = update_unit_cap(n, row_capacity, old_entries);
  size_t o = U.base.total;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += al(bytes);
    return at;
  };
  U.pm = take(8 * n);
  U.mbits = take(4 * ((n + 31) / 32));
  U.flag = take(4 * n);
  U.fpos = take(8 * (n + 1));
  U.qorder = take(4 * n);
  U.morder = take(4 * n);
  U.nlm = take(8);
  U.new_col = take(4 * (row_capacity ? row_capacity : 1));
  U.units = take(4 * n);
  U.uoff = take(8 * (n + 1));
  U.unit_j = take(4 * U.unit_cap);
  U.mlist = take(4 * n);
  U.mcount = take(8);
  U.n_rem = take(4 * U.unit_cap);
  U.n_add = take(4 * U.unit_cap);
  U.off_rem = take(8 * (U.unit_cap + 1));
  U.off_add = take(8 * (U.unit_cap + 1));
  U.rbits_words = old_entries / 32 + 2;
  U.abits_words = row_capacity / 32 + 2;
  U.rbits = take(4 * U.rbits_words);
  U.abits = take(4 * U.abits_words);
  U.total = o;
  return U;
}

// SURVEY §8(f) f1 (k_update.cu): index the new points, query the moved vertices'
// new rows (count -> scan -> emit, as in run()), compare them with the old rows.
rhg_status run_update(uint64_t n, const double* theta, const double* r, double R,
                      const uint32_t* moved, uint64_t m, const double* theta_old,
                      const double* r_old, const uint64_t* old_rp, const uint32_t* old_col,
                      const rhg_update* out, cudaStream_t st) {
  if (!out || !out->num_added || !out->num_removed) return RHG_ERR_INVALID;
  if (n < 2 || n >= (1ull << 31) || m > n) return RHG_ERR_INVALID;
  if (!theta || !r || !old_rp || (m && (!moved || !theta_old || !r_old))) return RHG_ERR_INVALID;
  if (!(R >= 0.0) || !std::isfinite(R) || !std::isfinite(std::sinh(R / 2.0) * std::sinh(R / 2.0) * 4.0))
    return RHG_ERR_INVALID;
  if (out->capacity && (!out->added || !out->removed)) return RHG_ERR_INVALID;
  rhg_options opt{};
  if (out->options) {
    opt.num_bands = out->options->num_bands;
    opt.band_ratio = out->options->band_ratio;
    opt.heavy_threshold = out->options->heavy_threshold;
  }
  BandConst bc;
  rhg_status s = make_band_const(n, R, &opt, &bc);
  if (s != RHG_OK) return s;
  uint64_t old_entries = 0;
  CK(cudaMemcpyAsync(&old_entries, old_rp + n, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const UpdLayout U = plan_update(n, out->row_capacity, old_entries, bc.L);
  const Layout& Lw = U.base;
  if (!out->workspace || out->workspace_bytes < U.total) return RHG_ERR_WORKSPACE;
  DevScalars* pin = pinned_scalars();
  if (!pin) return RHG_ERR_CUDA;
  char* ws = (char*)out->workspace;
  uint32_t* keys_a = (uint32_t*)(ws + Lw.keys_a);
  uint32_t* vals_a = (uint32_t*)(ws + Lw.vals_a);
  uint32_t* hist = (uint32_t*)(ws + Lw.hist);
  BandLayout* lay = (BandLayout*)(ws + Lw.lay);
  PointRec* pts = (PointRec*)(ws + Lw.pts);
  uint32_t* sid2 = (uint32_t*)(ws + Lw.sid2);
  uint32_t* dir = (uint32_t*)(ws + Lw.dir);
  uint32_t* deg = (uint32_t*)(ws + Lw.deg);
  uint64_t* offs = (uint64_t*)(ws + Lw.offs);
  DevScalars* sc = (DevScalars*)(ws + Lw.sc);
  uint64_t* fpos = (uint64_t*)(ws + U.fpos);
  uint32_t* new_col = (uint32_t*)(ws + U.new_col);
  Timer tm;
  tm.init(out->timing != nullptr, st);
  int launches = 0;
  CK(radix_sort_prepare());
  tm.mark();  // 0
  CK(cudaMemsetAsync(hist, 0, 4 * kMaxBands, st));
  CK(cudaMemsetAsync(sc, 0, sizeof(DevScalars), st));
  CK(launch_keys_from_points(n, theta, r, bc, keys_a, vals_a, hist, sc, st));
  CK(launch_band_layout(bc, hist, lay, (HeavyMeta*)(ws + Lw.h_meta), st));
  CK(radix_sort((uint32_t)n, keys_a, vals_a, (uint32_t*)(ws + Lw.keys_b), (uint32_t*)(ws + Lw.vals_b),
                ws + Lw.sort_tmp, 0, 32, st, &launches));
  tm.mark();  // 1
  CK(launch_build_index((uint32_t)n, theta, r, keys_a, vals_a, lay, bc.L, pts, sid2, dir, nullptr, 0,
                        st, &launches));
  CK(launch_query_order(keys_a, lay, bc.L, (uint32_t*)(ws + Lw.q_cell_lo),
                        (uint32_t*)(ws + Lw.q_cell_cnt), (uint64_t*)(ws + Lw.q_cell_off),
                        (uint32_t*)(ws + Lw.q_order), ws + Lw.scan_tmp, st, &launches));
  // the moved vertices in processing order: light ones for the light kernels, hubs
  // through hub_mask for the chunked path
  CK(launch_update_select((uint32_t)n, m, moved, lay, (const uint32_t*)(ws + Lw.q_order), vals_a,
                          (uint2*)(ws + U.pm), (uint32_t*)(ws + U.mbits), (uint32_t*)(ws + U.flag),
                          fpos, (uint32_t*)(ws + U.qorder), (uint32_t*)(ws + U.morder),
                          (unsigned long long*)(ws + U.nlm), ws + Lw.scan_tmp, st, &launches));
  tm.mark();  // 2
  QueryArgs qa{};
  qa.n = (uint32_t)n;
  qa.nquery = (const unsigned long long*)(ws + U.nlm);
  qa.nquery_max = (uint32_t)m;
  qa.hub_mask = (const uint32_t*)(ws + U.flag);  // items [0, heavy_end) = hub positions
  qa.stats = out->timing ? 1u : 0u;
  qa.pts = pts;
  qa.skey = keys_a;
  qa.sid = vals_a;
  qa.sid2 = sid2;
  qa.dir = dir;
  qa.lay = lay;
  qa.order = (const uint32_t*)(ws + U.qorder);
  qa.bits = (uint32_t*)(ws + Lw.b_bits);
  qa.warp_over = (uint32_t*)(ws + Lw.b_over);
  qa.deg = deg;
  qa.cdeg = (uint32_t*)(ws + Lw.cdeg);
  qa.sc = sc;
  CK(cudaMemsetAsync(deg, 0, 4 * n, st));  // rows of vertices that did not move stay empty
  HeavyMeta* hmeta = (HeavyMeta*)(ws + Lw.h_meta);
  HeavyArgs ha{};
  ha.pstart = (uint32_t*)(ws + Lw.h_pstart);
  ha.plen = (uint32_t*)(ws + Lw.h_plen);
  ha.poff = (uint32_t*)(ws + Lw.h_poff);
  ha.np = (uint32_t*)(ws + Lw.h_np);
  ha.vtot = (uint32_t*)(ws + Lw.h_vtot);
  ha.vtot_off = (uint64_t*)(ws + Lw.h_vtot_off);
  ha.cc = (uint32_t*)(ws + Lw.h_cc);
  ha.choff = (uint64_t*)(ws + Lw.h_choff);
  ha.chunk_vtx = (uint32_t*)(ws + Lw.h_cvtx);
  ha.chunk_piece = (uint32_t*)(ws + Lw.h_cpiece);
  ha.chunk_hits = (uint32_t*)(ws + Lw.h_chits);
  ha.chunk_pos = (uint64_t*)(ws + Lw.h_cpos);
  ha.bits = (uint32_t*)(ws + Lw.h_bits);
  ha.bits_cap = Lw.hbits_cap;
  ha.meta = hmeta;
  ha.vcap = Lw.vcap;
  ha.chunk_cap = Lw.chunk_cap;
  ha.chunk_min = kChunkMin;
  if (m) {
    // moved hubs: the chunked hub path (hub_mask), the rest: light warps
    CK(launch_heavy_plan(RHG_CSR, qa, ha, bc, ws + Lw.heavy_scan_tmp, st, &launches));
    CK(launch_heavy(QM_COUNT, RHG_CSR, qa, ha, bc, st));
    CK(exclusive_scan_u32_u64_dev(ha.chunk_cap, &hmeta->nchunks, ha.chunk_hits, ha.chunk_pos,
                                  ws + Lw.heavy_scan_tmp, &hmeta->hits, st, &launches));
    CK(launch_query(QM_COUNT, RHG_CSR, qa, bc, st));
  }
  CK(exclusive_scan_u32_u64((uint32_t)n, deg, offs, ws + Lw.scan_tmp, &sc->total, st, &launches));
  tm.mark();  // 3
  CK(cudaMemcpyAsync(pin, sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const DevScalars hs = *pin;
  if (hs.domain_error) return RHG_ERR_DOMAIN;
  if (out->rows_needed) *out->rows_needed = hs.total;
  if (hs.total > out->row_capacity) return RHG_ERR_WORKSPACE;
  qa.offs = offs;
  qa.col = new_col;
  qa.out_cap = out->row_capacity;
  if (m) {
    CK(launch_heavy(QM_EMIT_BITS, RHG_CSR, qa, ha, bc, st));
    CK(launch_query(QM_EMIT_BITS, RHG_CSR, qa, bc, st));
  }
  uint32_t* n_rem = (uint32_t*)(ws + U.n_rem);
  uint32_t* n_add = (uint32_t*)(ws + U.n_add);
  uint64_t* off_rem = (uint64_t*)(ws + U.off_rem);
  uint64_t* off_add = (uint64_t*)(ws + U.off_add);
  const uint2* pm = (const uint2*)(ws + U.pm);
  const uint32_t* morder = (const uint32_t*)(ws + U.morder);
  const uint32_t* mbits = (const uint32_t*)(ws + U.mbits);
  uint64_t* uoff = (uint64_t*)(ws + U.uoff);
  uint32_t* unit_j = (uint32_t*)(ws + U.unit_j);
  if (m == 0) CK(cudaMemsetAsync(uoff, 0, 8, st));  // no units
  uint32_t* mlist = (uint32_t*)(ws + U.mlist);
  unsigned int* mcount = (unsigned int*)(ws + U.mcount);
  CK(launch_delta_plan(m, morder, old_rp, offs, (uint32_t*)(ws + U.units), uoff, unit_j, mlist,
                       mcount, ws + Lw.scan_tmp, st, &launches));
  uint32_t* rbits = (uint32_t*)(ws + U.rbits);
  uint32_t* abits = (uint32_t*)(ws + U.abits);
  CK(cudaMemsetAsync(rbits, 0, 4 * U.rbits_words, st));
  CK(cudaMemsetAsync(abits, 0, 4 * U.abits_words, st));
  CK(launch_delta_decide(m, U.unit_cap, uoff, unit_j, mlist, mcount, morder, pm, mbits, pts, keys_a,
                         lay, bc.L, theta_old, r_old, old_rp, old_col, offs, new_col, bc.T4, n_rem,
                         n_add, rbits, abits, st));
  // unit counts -> offsets (uoff[m] units, counted on the device)
  CK(exclusive_scan_u32_u64_dev(U.unit_cap, (const unsigned long long*)(uoff + m), n_rem, off_rem,
                                ws + Lw.scan_tmp, &sc->candidates, st, &launches));
  CK(exclusive_scan_u32_u64_dev(U.unit_cap, (const unsigned long long*)(uoff + m), n_add, off_add,
                                ws + Lw.scan_tmp, &sc->certain, st, &launches));
  CK(cudaMemcpyAsync(pin, sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const uint64_t nrem = m ? pin->candidates : 0, nadd = m ? pin->certain : 0;
  *out->num_removed = nrem;
  *out->num_added = nadd;
  if (nrem > out->capacity || nadd > out->capacity) return RHG_ERR_CAPACITY;
  CK(launch_delta_write(m, U.unit_cap, uoff, unit_j, morder, old_rp, old_col, offs, new_col, rbits,
                        abits, off_rem, off_add, out->removed, out->added, st));
  tm.mark();  // 4
  if (out->timing) {
    CK(cudaStreamSynchronize(st));
    rhg_timing* t = out->timing;
    memset(t, 0, sizeof(*t));
    t->ms_sort = tm.between(0, 1);
    t->ms_index = tm.between(1, 2);
    t->ms_count = tm.between(2, 3);
    t->ms_emit = tm.between(3, 4);
    t->ms_total = tm.between(0, 4);
    t->candidates = hs.candidates;
    t->certain = hs.certain;
    t->launches = (uint64_t)launches;
    t->emit_retested = hs.bit_overflow;
  }
  CK(cudaGetLastError());
  return RHG_OK;
}

}  // namespace

namespace rhg {
int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  int v = cache[d].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0)
      v = 148;
    cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // namespace rhg

#define RHG_EXPORT __attribute__((visibility("default")))

extern "C" {

RHG_EXPORT rhg_status rhg_target_radius(uint64_t n, double kbar, double gamma, double* R) {
  if (!R || !(gamma > 2.0) || !std::isfinite(gamma) || n < 2) return RHG_ERR_INVALID;
  return target_radius((double)n, kbar, (gamma - 1.0) / 2.0, R);
}

RHG_EXPORT rhg_status rhg_band_boundaries(uint64_t n, double R, const rhg_options* opt, int* L, double* c) {
  if (!L || !c || n < 2 || !(R >= 0.0) || !std::isfinite(R)) return RHG_ERR_INVALID;
  BandConst bc;
  rhg_status s = make_band_const(n, R, opt, &bc);
  if (s != RHG_OK) return s;
  *L = bc.L;
  for (int j = 0; j <= bc.L; ++j) c[j] = bc.c[j];
  return RHG_OK;
}

RHG_EXPORT size_t rhg_workspace_bytes(uint64_t n, rhg_format format, uint64_t capacity_edges,
                           int host_buffers, const rhg_options* options) {
  return plan_layout(n, format, capacity_edges, host_buffers ? 1 : 0, bands_for(n, options)).total;
}

RHG_EXPORT rhg_status rhg_generate_with_radius(uint64_t n, double R, double alpha, uint64_t seed,
                                    const rhg_output* out, rhg_stream stream) {
  if (!(alpha > 0.5) || !std::isfinite(alpha)) return RHG_ERR_INVALID;
  return run(n, true, alpha, seed, nullptr, nullptr, R, out, (cudaStream_t)stream);
}

RHG_EXPORT rhg_status rhg_generate(uint64_t n, double kbar, double gamma, uint64_t seed,
                        const rhg_output* out, rhg_stream stream) {
  double R = 0.0;
  rhg_status s = rhg_target_radius(n, kbar, gamma, &R);
  if (s != RHG_OK) return s;
  return rhg_generate_with_radius(n, R, (gamma - 1.0) / 2.0, seed, out, stream);
}

RHG_EXPORT rhg_status rhg_generate_with_C(uint64_t n, double C, double alpha, uint64_t seed,
                                          const rhg_output* out, rhg_stream stream) {
  if (!std::isfinite(C) || n < 2) return RHG_ERR_INVALID;
  const double R = 2.0 * std::log((double)n) + C;
  if (!(R >= 0.0)) return RHG_ERR_INVALID;
  return rhg_generate_with_radius(n, R, alpha, seed, out, stream);
}

RHG_EXPORT rhg_status rhg_movement_init(uint64_t n, uint64_t seed, double phi_lo, double phi_hi,
                                        double r_lo, double r_hi, double* tau_phi, double* tau_r,
                                        rhg_stream stream) {
  if (!tau_phi || !tau_r || !std::isfinite(phi_lo) || !std::isfinite(phi_hi) ||
      !std::isfinite(r_lo) || !std::isfinite(r_hi) || !(phi_hi >= phi_lo) || !(r_hi >= r_lo) ||
      !(phi_lo > -6.283185307179586) || !(phi_hi < 6.283185307179586))
    return RHG_ERR_INVALID;
  if (n == 0) return RHG_OK;
  CK(launch_movement_init(n, seed, phi_lo, phi_hi, r_lo, r_hi, tau_phi, tau_r, (cudaStream_t)stream));
  return RHG_OK;
}

RHG_EXPORT rhg_status rhg_move_points(uint64_t n, double* theta, double* r, const double* tau_phi,
                                      double* tau_r, double R, double alpha, rhg_stream stream) {
  if (!theta || !r || !tau_phi || !tau_r || !(alpha > 0.5) || !std::isfinite(alpha) ||
      !(R > 0.0) || !std::isfinite(std::sinh(alpha * R)))
    return RHG_ERR_INVALID;
  if (n == 0) return RHG_OK;
  CK(launch_move(n, theta, r, tau_phi, tau_r, R, alpha, (cudaStream_t)stream));
  return RHG_OK;
}

RHG_EXPORT size_t rhg_stats_workspace_bytes(uint64_t n) { return stats_workspace_bytes(n); }

RHG_EXPORT rhg_status rhg_graph_stats(uint64_t n, rhg_format format, const uint64_t* row_ptr,
                                      const uint32_t* col, const uint32_t* pairs, uint64_t m,
                                      const double* theta, const double* r, double R, double k_min,
                                      void* workspace, size_t workspace_bytes, rhg_stats* out,
                                      rhg_stream stream) {
  if (!out || n == 0 || n > (1ull << 31) || !workspace ||
      workspace_bytes < stats_workspace_bytes(n) || !(k_min >= 1.0) || !std::isfinite(R))
    return RHG_ERR_INVALID;
  if (format == RHG_CSR && (!row_ptr || (!col && (theta || r)))) return RHG_ERR_INVALID;
  if (format == RHG_EDGES_UNDIRECTED && !pairs && m) return RHG_ERR_INVALID;
  if (format != RHG_CSR && format != RHG_EDGES_UNDIRECTED) return RHG_ERR_INVALID;
  CK(launch_graph_stats((uint32_t)n, format, row_ptr, col, pairs, m, theta, r, R, k_min, workspace,
                        out, (cudaStream_t)stream));
  return RHG_OK;
}

RHG_EXPORT size_t rhg_update_workspace_bytes(uint64_t n, uint64_t row_capacity, uint64_t old_entries,
                                             const rhg_options* options) {
  return plan_update(n, row_capacity, old_entries, bands_for(n, options)).total;
}

RHG_EXPORT rhg_status rhg_update_moved(uint64_t n, const double* theta, const double* r, double R,
                                       const uint32_t* moved, uint64_t m, const double* theta_old,
                                       const double* r_old, const uint64_t* old_row_ptr,
                                       const uint32_t* old_col, const rhg_update* out,
                                       rhg_stream stream) {
  return run_update(n, theta, r, R, moved, m, theta_old, r_old, old_row_ptr, old_col, out,
                    (cudaStream_t)stream);
}

RHG_EXPORT rhg_status rhg_generate_from_points(uint64_t n, const double* theta, const double* r, double R,
                                    const rhg_output* out, rhg_stream stream) {
  return run(n, false, 0.0, 0, theta, r, R, out, (cudaStream_t)stream);
}

RHG_EXPORT rhg_status rhg_sample_points(uint64_t n, double alpha, double R, uint64_t seed, double* theta,
                             double* r, rhg_stream stream) {
  if (n == 0 || !theta || !r || !(alpha > 0.5) || !(R >= 0.0) || !std::isfinite(std::cosh(alpha * R)))
    return RHG_ERR_INVALID;
  BandConst bc;
  rhg_status s = make_band_const(n < 2 ? 2 : n, R, nullptr, &bc);
  if (s != RHG_OK) return s;
  PhiloxPoints gen{};
  gen.seed = seed;
  gen.two_over_alpha = 2.0 / alpha;
  gen.half_span = (std::cosh(alpha * R) - 1.0) / 2.0;
  gen.R = R;
  CK(launch_sample(n, gen, bc, theta, r, nullptr, nullptr, nullptr, (cudaStream_t)stream));
  return RHG_OK;
}

RHG_EXPORT rhg_status rhg_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t* out,
                            rhg_stream stream) {
  if (!out) return RHG_ERR_INVALID;
  if (count == 0) return RHG_OK;
  CK(launch_philox_words(seed, i0, count, out, (cudaStream_t)stream));
  return RHG_OK;
}

RHG_EXPORT const char* rhg_status_string(rhg_status s) {
  switch (s) {
    case RHG_OK: return "ok";
    case RHG_ERR_INVALID: return "invalid argument";
    case RHG_ERR_CALIBRATION: return "calibration failed: kbar cannot be reached by Eq. 22";
    case RHG_ERR_WORKSPACE: return "workspace too small";
    case RHG_ERR_CAPACITY: return "output capacity too small (required count in *num_edges)";
    case RHG_ERR_DOMAIN: return "input point outside the disk";
    case RHG_ERR_CUDA: return "CUDA error";
  }
  return "unknown status";
}

RHG_EXPORT const char* rhg_version(void) { return RHG_VERSION; }

RHG_EXPORT const char* rhg_last_cuda_error(void) {
  static thread_local char buf[160];
  snprintf(buf, sizeof(buf), "%s (rhg_abi.cu:%d)", cudaGetErrorString(last_cuda_error()),
           last_cuda_error_line());
  return buf;
}

}  // extern "C"
