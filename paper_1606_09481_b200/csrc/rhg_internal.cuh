// rhg_internal.cuh -- shared definitions of the B200 product path (kernels + host
// orchestration).  Nothing here is shared with oracle/ (see DESIGN.md).
#pragma once
#include <cuda_runtime.h>
#include <cmath>
#include <stdint.h>

#include "../../include/rhg.h"

namespace rhg {

constexpr int kMaxBands = 32;          // L <= 32: n < 2^32 => ceil(log2 n) <= 32
constexpr int kBandShift = 27;         // sort key = band << 27 | q27(theta)
constexpr uint32_t kQBits = 27;
#ifndef RHG_DIR_PER_PT
#define RHG_DIR_PER_PT 4u  // directory buckets per point (at least; power of two per slab)
#endif
constexpr uint32_t kQMax = (1u << kQBits) - 1u;
constexpr uint32_t kQMask = kQMax;
constexpr uint32_t kLightBitRows = 8;   // bit words per lane of a light warp (256 tests)
constexpr int kQuerySectorBits = 8;    // light queries run sector-major over 2^8 angular sectors
constexpr int kQuerySectors = 1 << kQuerySectorBits;  // light-warp bit blocks come from 64 sub-pools
constexpr uint32_t kRangesPerSlab = 6;  // hub slots per (vertex, slab): 4 pieces to test + 2 certain
constexpr uint32_t kTestPieces = 4;

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
  double A[kMaxBands + 1];   // e^{c_j/2}, j = 0..L
  double B[kMaxBands + 1];   // e^{-c_j/2}
  double invS[kMaxBands + 1];// 1/sinh(c_j)   (0 for c_j = 0 -> full circle)
  double padS[kMaxBands + 1];// T4 2^-48 / sinh(c_j): absolute upward pad of the window ratio
  double T4min;              // 2^-10 T4: certain windows need T4 - h^2 above this at both ends
  double heavy_threshold;    // expected candidates per vertex above which a slab's vertices are hubs
  uint32_t heavy_cap;        // at most this many hub vertices (workspace bound)
  uint32_t shard, nshards;   // this call owns shard `shard` of `nshards` (1: everything)
};

// Device-computed band layout after the band histogram.
struct BandLayout {
  uint32_t count[kMaxBands];       // n_j
  uint32_t start[kMaxBands + 1];   // first sorted index of band j
  uint32_t dir_off[kMaxBands + 1]; // offset of band j's bucket directory
  uint32_t shift[kMaxBands];       // bucket(q) = q >> shift[j]
  uint32_t nb[kMaxBands];          // buckets in band j (power of two)
  uint32_t heavy_end;              // sorted positions [0, heavy_end) are hub vertices
  float expected[kMaxBands];       // upper bound of E[candidates] for a vertex of band j
};

// Hub ("heavy") vertices: their (slab, piece) candidate ranges are materialised
// as compacted pieces per vertex, and each vertex's concatenated candidate
// sequence is cut into fixed-size chunks that are spread over the whole GPU.
struct HeavyMeta {
  unsigned long long nvtx;     // hub vertices (= heavy_end)
  unsigned long long cand;     // total candidates (tested + certain) of hub vertices
  unsigned long long nchunks;  // total chunks
  unsigned long long chunk;    // chunk size (candidates, multiple of 32)
  unsigned long long hits;     // total edges of hub vertices (directed / outward)
  unsigned long long list_len; // list output: hub rows + one entry per light warp (degree scan)
};

constexpr uint32_t kCertainPiece = 0x80000000u;  // plen flag: every candidate is an edge

struct HeavyArgs {
  // per hub vertex i, pieces [i * LS, i * LS + np[i]) (LS = kRangesPerSlab * L)
  uint32_t* pstart;         // first doubled position of the piece
  uint32_t* plen;           // candidates | kCertainPiece
  uint32_t* poff;           // offset of the piece in the vertex's candidate sequence
  uint32_t* np;             // [vcap] pieces
  uint32_t* vtot;           // [vcap] candidates
  uint64_t* vtot_off;       // [vcap + 1] scan of vtot (total -> meta->cand)
  uint32_t* cc;             // [vcap] chunks per vertex
  uint64_t* choff;          // [vcap + 1] scan of cc
  uint32_t* chunk_vtx;      // [chunk_cap]
  uint32_t* chunk_piece;    // [chunk_cap] first piece the chunk touches
  uint32_t* chunk_hits;     // [chunk_cap]
  uint64_t* chunk_pos;      // [chunk_cap + 1] scan of chunk_hits
  uint32_t* bits;           // [bits_cap] hub ballot words, (CH / 32 + 8) per chunk; if they do
                            // not fit, both passes test (same output)
  uint64_t bits_cap;
  HeavyMeta* meta;
  uint64_t vcap;
  uint64_t chunk_cap;
  uint64_t chunk_min;       // minimum chunk size
};

// Scalars the host reads back once per call.
struct DevScalars {
  unsigned long long total;        // edges (directed for CSR, undirected for pairs)
  unsigned long long candidates;   // tests performed by the count pass
  unsigned long long certain;      // edges accepted by the certified inner window (no test)
  unsigned long long bit_words;    // candidate-bit words allocated by the count pass
  unsigned int domain_error;       // a point outside the disk
  unsigned int bit_overflow;       // light warps whose bit buffer was too small (emit re-tests)
  unsigned int dbg_line;           // RHG_BOUNDS builds: first failed check (line, values)
  unsigned long long dbg[3];
};

// One point in the query SoA, 32 B: theta, sinh r, e^{r/2}, e^{-r/2}.
struct __align__(16) PointRec {
  double theta, s, a, b;
};

// Sharding (k_shard.cu): hub vertex i belongs to shard snake(i); the
// light groups [grp_beg, grp_end) of the sector-major order to this shard.
struct ShardPlan {
  uint32_t grp_beg, grp_end;      // this shard's light groups
  unsigned long long work_total;  // estimated candidates of all query items
  unsigned long long hub_work;    // estimated candidates of this shard's hubs
};
__host__ __device__ __forceinline__ uint32_t snake(uint64_t c, uint32_t N) {
  const uint32_t m = (uint32_t)(c % (2ull * N));
  return m < N ? m : 2u * N - 1u - m;
}

struct QueryArgs {
  uint32_t n;
  const unsigned long long* nquery;   // device: light query items in `order` (null: n - heavy_end)
  uint32_t nquery_max;                // host bound of *nquery for the grid (0: n)
  const uint32_t* hub_mask;           // non-null: only hubs i with hub_mask[i] != 0 are queried
  const ShardPlan* shard_plan;        // nshards > 1: this shard's items (k_shard.cu), else null
  const PointRec* __restrict__ pts;   // doubled SoA: slab j at [2 start_j, 2 start_j + 2 n_j), two copies
  const uint32_t* __restrict__ skey;  // sorted keys [n]
  const uint32_t* __restrict__ sid;   // sorted position -> vertex id [n]
  const uint32_t* __restrict__ sid2;  // doubled position -> vertex id [2n]
  const uint32_t* __restrict__ dir;   // bucket directory
  const BandLayout* __restrict__ lay;
  const uint32_t* __restrict__ order; // light query order: sorted positions, sector-major [n - heavy_end]
  uint32_t* deg;                      // count pass: degree per vertex id
  uint32_t* cdeg;                     // count pass: certain (untested) edges per light vertex id
  const uint64_t* __restrict__ offs;  // emit pass: output offset per vertex id
  uint32_t* col;                      // CSR output
  uint32_t* pairs;                    // undirected output
  unsigned long long out_cap;         // elements col / pairs hold (debug bounds checks)
  uint32_t* bits;                     // light test bits: kLightBitRows x 32 words per light warp
  uint32_t* warp_over;                // per light warp: 1 if its bits did not fit (emit re-tests)
  DevScalars* sc;
  uint32_t labels;                    // 0: ids = sample / input indices; 1: sorted positions
  uint32_t poff;                      // 1 (list output): deg / cdeg / offs indexed by processing
                                      // position (hub i, then heavy_end + light order index)
  uint32_t force_wide;                // 64-bit slab positions in the light kernels
  uint32_t stats;                     // accumulate candidate / certain totals (timing)
  const unsigned long long* total_dev;  // emit: skip everything if *total_dev > cap
  unsigned long long cap;
};

// ---- K1 device code shared by the sampler and the generate-path gather ----
// Philox4x32-10 (Salmon et al. 2011): counter (i_lo, i_hi, 0, 0), key = seed.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint4 vertex_words(uint64_t seed, uint64_t i) {
  return philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0u, 0u),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// theta = fl(2pi) * u1, u1 = (w1:w0 >> 11) 2^-53  (Z10, Z12)
// r = (2/alpha) asinh(sqrt(u2 * (cosh(alpha R) - 1)/2)), clamped to R (Z11)
__device__ __forceinline__ void words_to_point(uint4 w, double two_over_alpha, double half_span,
                                               double R, double& theta, double& r) {
  uint64_t a = ((uint64_t)w.y << 32) | w.x;
  uint64_t b = ((uint64_t)w.w << 32) | w.z;
  double u1 = __dmul_rn((double)(a >> 11), 0x1.0p-53);
  double u2 = __dmul_rn((double)(b >> 11), 0x1.0p-53);
  theta = __dmul_rn(RHG_TWO_PI_HI, u1);
  double rr = __dmul_rn(two_over_alpha, asinh(sqrt(__dmul_rn(u2, half_span))));
  r = rr > R ? R : rr;
}


// Parameters to re-derive the Philox points (generate path).
struct PhiloxPoints {
  uint64_t seed;
  double two_over_alpha, half_span, R;
  // ucut[j] = sinh^2(alpha c_j / 2) / half_span (j = 1..L-1): the u2 at which
  // words_to_point's r reaches c_j, so the band of a point follows from u2 alone
  // (k_sample); 0 = not set (every band from r)
  double ucut[kMaxBands + 1];
};
// the slab boundaries' u2 thresholds (host)
void set_band_cuts(PhiloxPoints& gen, double alpha, const BandConst& bc);

// Streaming multiprocessors of the current device (cudaDevAttrMultiProcessorCount,
// cached per device): grids are sized in multiples of it.
int num_sms();

// ---- launch wrappers (each returns cudaError_t of the launch) ----
cudaError_t launch_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t* out,
                                cudaStream_t st);
// theta / r may be nullptr (not stored); keys == nullptr: sample the points only.
cudaError_t launch_sample(uint64_t n, const PhiloxPoints& gen, const BandConst& bc, double* theta,
                          double* r, uint32_t* keys, uint32_t* idx, uint32_t* band_hist,
                          cudaStream_t st);
cudaError_t launch_keys_from_points(uint64_t n, const double* theta, const double* r,
                                    const BandConst& bc, uint32_t* keys, uint32_t* idx,
                                    uint32_t* band_hist, DevScalars* sc, cudaStream_t st);
cudaError_t launch_band_layout(const BandConst& bc, const uint32_t* band_hist, BandLayout* lay,
                               HeavyMeta* meta, cudaStream_t st);
// LSD radix sort of (key, val) pairs, 32-bit keys, stable.  Result lands in
// (keys_a, vals_a).  tmp must hold radix_sort_tmp_bytes(n).
size_t radix_sort_tmp_bytes(uint64_t n);
cudaError_t radix_sort_prepare();
cudaError_t radix_sort(uint32_t n, uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b,
                       uint32_t* vals_b, void* tmp, int begin_bit, int end_bit, cudaStream_t st,
                       int* launches);
// gen != nullptr: re-derive the points from Philox instead of reading theta / r.
// pts / sid2: the doubled SoA (2n entries; slab j stored twice back to back at
// [2 start_j, 2 start_j + 2 n_j), so any arc of the slab is one index range).
cudaError_t launch_build_index(uint32_t n, const double* theta, const double* r,
                               const uint32_t* skey, const uint32_t* sidx, const BandLayout* lay,
                               int L, PointRec* pts, uint32_t* sid2, uint32_t* dir,
                               const PhiloxPoints* gen, int seq_ids, cudaStream_t st,
                               int* launches);
// Sector-major order of the light queries (k_index.cu); cell arrays hold
// kQuerySectors * L entries (cell_off: + 1).
cudaError_t launch_query_order(const uint32_t* skey, const BandLayout* lay, int L,
                               uint32_t* cell_lo, uint32_t* cell_cnt, uint64_t* cell_off,
                               uint32_t* order, void* scan_tmp, cudaStream_t st, int* launches);
// Exclusive scan of n uint32 counts into n+1 uint64 offsets (out[n] = total);
// also writes the total into *total_out.  tmp: scan_tmp_bytes(n).
size_t scan_tmp_bytes(uint64_t n);
cudaError_t exclusive_scan_u32_u64(uint32_t n, const uint32_t* in, uint64_t* out, void* tmp,
                                   unsigned long long* total_out, cudaStream_t st, int* launches);
// Same with the element count read on the device (n_dev, clamped to n_cap).
cudaError_t exclusive_scan_u32_u64_dev(uint64_t n_cap, const unsigned long long* n_dev,
                                       const uint32_t* in, uint64_t* out, void* tmp,
                                       unsigned long long* total_out, cudaStream_t st,
                                       int* launches);

enum QueryMode { QM_COUNT = 0, QM_EMIT = 1, QM_EMIT_BITS = 2 };
cudaError_t launch_query(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const BandConst& bc,
                         cudaStream_t st);
// Hub path: ranges -> slot scan -> chunking -> count (mode QM_COUNT) / emit.
cudaError_t launch_heavy_plan(rhg_format fmt, const QueryArgs& qa, const HeavyArgs& ha,
                              const BandConst& bc, void* scan_tmp, cudaStream_t st, int* launches);
cudaError_t launch_heavy(QueryMode mode, rhg_format fmt, const QueryArgs& qa, const HeavyArgs& ha,
                         const BandConst& bc, cudaStream_t st);

// Shard plan (k_shard.cu): estimated work per query item (launch_shard_work, in
// k_query.cu), its scan, the hubs' work per shard and this shard's light range.
// work / prefix hold item_cap (+1) entries, item_cap >= heavy_end + ceil(light / 32).
cudaError_t launch_shard_work(const QueryArgs& qa, const BandConst& bc, int outward, uint32_t* work,
                              cudaStream_t st);
cudaError_t launch_shard_plan(uint32_t n, const QueryArgs& qa, const BandConst& bc, int outward,
                              uint32_t* work, uint64_t* prefix, uint64_t item_cap, void* scan_tmp,
                              unsigned long long* hub_work, ShardPlan* plan, cudaStream_t st,
                              int* launches);

// Incremental update of the dynamic model (k_update.cu)
// pm[id] = (sorted position, index in moved or ~0); flag[t] = 1 if query item t (hub
// position t < heavy_end, else light order entry) moved; morder = the moved vertices
// in processing order; qorder = the moved light entries, *nlight_moved their count
cudaError_t launch_update_select(uint32_t n, uint64_t m, const uint32_t* moved, const BandLayout* lay,
                                 const uint32_t* order, const uint32_t* sid, uint2* pm,
                                 uint32_t* mbits, uint32_t* flag, uint64_t* fpos, uint32_t* qorder,
                                 uint32_t* morder, unsigned long long* nlight_moved, void* scan_tmp,
                                 cudaStream_t st, int* launches);
// delta work units (k_update.cu): units[j], uoff (m + 1), unit_j (uoff[m] entries)
cudaError_t launch_delta_plan(uint64_t m, const uint32_t* morder, const uint64_t* old_rp,
                              const uint64_t* new_rp, uint32_t* units, uint64_t* uoff,
                              uint32_t* unit_j, uint32_t* mlist, unsigned int* mcount,
                              void* scan_tmp, cudaStream_t st, int* launches);
// decide: per-unit counts + decision bits over old_col (rbits) / new_col (abits),
// both zeroed by the caller; write: replay at the scanned per-unit offsets
cudaError_t launch_delta_decide(uint64_t m, uint64_t unit_cap, const uint64_t* uoff,
                                const uint32_t* unit_j, const uint32_t* mlist,
                                const unsigned int* mcount, const uint32_t* morder, const uint2* pm,
                                const uint32_t* mbits, const PointRec* pts, const uint32_t* skey,
                                const BandLayout* lay, int L, const double* theta_old,
                                const double* r_old, const uint64_t* old_rp, const uint32_t* old_col,
                                const uint64_t* new_rp, const uint32_t* new_col, double T4,
                                uint32_t* n_rem, uint32_t* n_add, uint32_t* rbits, uint32_t* abits,
                                cudaStream_t st);
cudaError_t launch_delta_write(uint64_t m, uint64_t unit_cap, const uint64_t* uoff,
                               const uint32_t* unit_j, const uint32_t* morder,
                               const uint64_t* old_rp, const uint32_t* old_col,
                               const uint64_t* new_rp, const uint32_t* new_col,
                               const uint32_t* rbits, const uint32_t* abits,
                               const uint64_t* off_rem, const uint64_t* off_add, uint32_t* removed,
                               uint32_t* added, cudaStream_t st);

// Validation statistics (k_stats.cu)
size_t stats_workspace_bytes(uint64_t n);
cudaError_t launch_graph_stats(uint32_t n, int fmt, const uint64_t* row_ptr, const uint32_t* col,
                               const uint32_t* pairs, uint64_t m, const double* theta,
                               const double* r, double R, double kmin, void* ws,
                               rhg_stats* host_out, cudaStream_t st);

// Dynamic model (k_dynamic.cu)
cudaError_t launch_movement_init(uint64_t n, uint64_t seed, double phi_lo, double phi_hi,
                                 double r_lo, double r_hi, double* tau_phi, double* tau_r,
                                 cudaStream_t st);
cudaError_t launch_move(uint64_t n, double* theta, double* r, const double* tau_phi, double* tau_r,
                        double R, double alpha, cudaStream_t st);

}  // namespace rhg
