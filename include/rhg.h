/*
 * rhg.h -- C-ABI of the B200-native threshold random-hyperbolic-graph generator
 *          (hot path of Algorithm 1, arXiv 1606.09481).
 *
 * Model: n points in the hyperbolic disk D_R, angle
 * phi ~ U[0, 2pi), radius with density
 * f(r) = alpha sinh(alpha r) / (cosh(alpha R) - 1) (Eq. 1),
 * alpha = (gamma - 1)/2.  Vertices u != v are adjacent iff their
 * hyperbolic distance (Eq. 3) is <= R (T = 0).
 *
 * Everything below is plain C: pointers, sizes, status codes.  No torch types.
 * A `rhg_stream` is a `cudaStream_t` (both are `struct CUstream_st *`); NULL is
 * the legacy default stream.
 *
 * Error behaviour: every entry point validates its arguments first and returns
 * a status without touching any buffer on RHG_ERR_INVALID / RHG_ERR_CALIBRATION /
 * RHG_ERR_WORKSPACE.  CUDA failures return RHG_ERR_CUDA; the stream may then hold
 * partially written outputs.  No entry point allocates device or host memory
 * beyond a few bytes of pinned host scratch held for the library's lifetime;
 * all large buffers are caller-owned.
 */
#ifndef RHG_H
#define RHG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *rhg_stream;

typedef enum {
  RHG_OK = 0,
  RHG_ERR_INVALID = 2,     /* bad argument: n < 2 or n >= 2^31 (the doubled point SoA is indexed
                              with 32 bits; 2^31 points need > 180 GB anyway), kbar <= 0, gamma <= 2 (alpha <= 1/2,
                              PAPER.md:78), non-finite input, NULL required pointer */
  RHG_ERR_CALIBRATION = 3, /* getTargetRadius could not bracket kbar on the decreasing branch of
                              Eq. 22 */
  RHG_ERR_WORKSPACE = 4,   /* workspace smaller than rhg_workspace_bytes() asks for */
  RHG_ERR_CAPACITY = 5,    /* output capacity too small; *num_edges holds the required count and
                              col / pairs are untouched (CSR row_ptr holds the offsets).  Output
                              is deterministic, so the caller may reallocate and call again. */
  RHG_ERR_DOMAIN = 6,      /* an input point has r outside [0, R] or theta outside [0, 2pi)
                              (SPEC.md:199), detected on the device; output buffers unspecified */
  RHG_ERR_CUDA = 7         /* a CUDA launch or runtime call failed */
} rhg_status;

typedef enum {
  /* Compressed sparse rows over vertex ids 0..n-1: row_ptr[n+1] (uint64),
     col[row_ptr[n]] (uint32).  Both directions of every edge, no self-loops.
     Row order is deterministic but unspecified (sort a row to canonicalise). */
  RHG_CSR = 0,
  /* Undirected list: pairs[2k], pairs[2k+1] = (u, v), u < v, each edge once.
     Order deterministic but unspecified. */
  RHG_EDGES_UNDIRECTED = 1
} rhg_format;

/* Tuning knobs.  The edge set does not depend on them (DESIGN.md "Why parity is
   layout-free"); they only move work between window evaluations and tests. */
typedef struct {
  int num_bands;     /* L, number of slabs (1..32); 0 -> min(16, ceil(ln n)) ("log n" slabs,
                        PAPER.md:108, base unstated; Z7) */
  double band_ratio; /* p, geometric width ratio in (0, 1); 0 -> 0.85 for ceil(ln n) <= 17,
                        + 0.04 per further unit, at most 0.95 (the paper's 0.9 was its own
                        measured choice; Z7) */
  uint32_t heavy_threshold; /* hub selection: a slab's vertices whose expected candidate
                               count (upper bound over the slab, all slabs' windows) exceeds
                               this are hubs, whose candidate sequences are cut into chunks
                               spread over all warps (DESIGN.md §1 a7); 0 -> 1024 */
  /* Sharding: with shard_count = N > 1 the call emits only
     the edges owned by shard shard_index: the rows (CSR) or the outward edges (list)
     of the query vertices it owns.  Ownership balances the estimated work (expected
     candidates per vertex): hub vertices are dealt in snake order, the light
     vertices go in N contiguous ranges of the sector-major order whose work makes up
     each shard's share (k_shard.cu).  Every shard samples
     and indexes the whole point set; rows of vertices owned by other shards are
     empty, so the N outputs are disjoint and their union is the graph.  Output
     (row contents included) is identical to the unsharded call's for owned vertices.
     0 / 1 -> one shard. */
  int shard_index;
  int shard_count;
  /* Vertex ids.  0 (default): vertex i is the i-th sample (Philox counter i) or
     the i-th input point.  1: ids in the order of Alg. 1 lines 9-12 (PAPER.md:
     150-155): slab by slab (inner to outer), by angular key within a slab
     (floor(theta 2^27 / 2pi), ties by sample index).  Same graph, relabelled;
     rows are then written without gathering ids (faster emit).
     rhg_output.perm_out, if set, receives perm[id] = sample / input index.
     theta_out / r_out stay in sample order. */
  int vertex_order;
  /* 1: run the light query kernels with 64-bit slab positions even when every slab
     holds < 2^30 points (the path n >= 2^30 takes; a test knob, same output). */
  int wide_positions;
  /* 1: record the call's kernels as two CUDA graphs (before / after the edge-count
     readback) and replay them while the arguments (sizes, pointers, seed, options,
     stream) stay the same; re-captured when they change.  Needs a non-default
     stream; ignored when timing is requested.  Same output. */
  int graph;
} rhg_options;

/* Per-phase device times (CUDA events on the caller's stream), filled when
   rhg_output.timing != NULL (adds event records and one extra sync). */
typedef struct {
  float ms_sample;   /* K1: Philox point sampling + band assignment            */
  float ms_sort;     /* K3: segmented radix sort by (band, angle)               */
  float ms_index;    /* K4: SoA gather + per-band bucket directory              */
  float ms_count;    /* K5/K7: windows, ranges, certified tests, degrees        */
  float ms_scan;     /* K6: degree scan -> row offsets                          */
  float ms_emit;     /* K8: edge emission                                       */
  float ms_copy;     /* host-buffer mode: device <-> host copies                */
  float ms_total;    /* first to last event                                     */
  uint64_t candidates;     /* candidate (vertex, point) pairs tested exactly in the count pass */
  uint64_t certain;        /* edges accepted by the certified inner window, without a test */
  uint64_t launches;       /* kernels launched by this call                                 */
  uint64_t emit_retested;  /* light warps (32 vertices each) whose test bits did not fit and
                              whose emit pass re-runs their tests                             */
} rhg_timing;

typedef struct {
  rhg_format format;
  /* 0: row_ptr/col/pairs/theta_out/r_out (and the input points of
     rhg_generate_from_points) are DEVICE pointers.
     1: they are HOST pointers (page-locked recommended); the library stages the
        graph in `workspace` and copies it with cudaMemcpyAsync on `stream`. */
  int host_buffers;
  uint64_t *row_ptr;       /* CSR: n+1 entries (row_ptr[n] = number of directed edges)        */
  uint32_t *col;           /* CSR: capacity_edges entries; device buffers 32-byte aligned       */
  uint32_t *pairs;         /* EDGES_UNDIRECTED: 2*capacity_edges entries; device: 32-byte aligned */
  uint64_t capacity_edges; /* CSR: directed entries col can hold; pairs: undirected edges      */
  void *workspace;         /* device scratch, caller-owned, >= rhg_workspace_bytes(...)        */
  size_t workspace_bytes;
  double *theta_out;       /* optional n-array: the sampled angles (generate calls only)       */
  double *r_out;           /* optional n-array: the sampled radii                              */
  uint64_t *num_edges;     /* HOST, required: directed count (CSR) or undirected count (pairs);
                              on RHG_ERR_CAPACITY the required count                          */
  double *R_used;          /* HOST, optional: the disk radius used                             */
  const rhg_options *options; /* optional, NULL -> defaults                                    */
  rhg_timing *timing;      /* HOST, optional                                                  */
  uint32_t *perm_out;      /* optional n-array, written when options->vertex_order = 1:
                              perm_out[id] = sample / input index of vertex id            */
} rhg_output;

/* getTargetRadius: R such that Eq. 22 (zeta = 1) gives kbar,
   on the decreasing branch (Z5).  Host only. */
rhg_status rhg_target_radius(uint64_t n, double kbar, double gamma, double *R);

/* Radial slab boundaries c_0..c_L (Eq. 4) the generator uses
   for n points and disk radius R: writes *L and c[0..L] (c must hold >= 65
   doubles).  Host only. */
rhg_status rhg_band_boundaries(uint64_t n, double R, const rhg_options *opt, int *L, double *c);

/* Device scratch needed by the generate calls for n points, output `format`,
   `capacity_edges` (as in rhg_output) and buffer kind (host_buffers as in
   rhg_output).  Includes a candidate-bit buffer sized from capacity_edges; if it
   proves too small at run time the emit pass re-runs the tests instead
   (slower, same output). */
size_t rhg_workspace_bytes(uint64_t n, rhg_format format, uint64_t capacity_edges,
                           int host_buffers, const rhg_options *options);

/* Algorithm 1 end to end: alpha from gamma (line 1), R from
   getTargetRadius (line 2), then on `stream`: Philox point sampling (lines 7-8;
   vertex i uses counter i, key = seed, Z12), band assignment (line 9),
   angular sort per band (lines 11-12), range queries with exact tests (lines
   13-21), and emission into `out`.  Device buffers: the emit kernels compare the
   edge total with capacity_edges on the device (nothing is written if it does not
   fit) and the call synchronises once, at the end; host buffers: one readback of
   the 8-byte total sizes the copies.  Deterministic for fixed (n, kbar, gamma, seed,
   options). */
rhg_status rhg_generate(uint64_t n, double kbar, double gamma, uint64_t seed,
                        const rhg_output *out, rhg_stream stream);

/* Same with the disk radius given directly ("or even accept R directly",
   PAPER.md:186); alpha > 1/2. */
rhg_status rhg_generate_with_radius(uint64_t n, double R, double alpha, uint64_t seed,
                                    const rhg_output *out, rhg_stream stream);

/* Same with the disk radius from the parameter C: R = 2 ln n + C ("accept the
   commonly used parameter C"); alpha > 1/2. */
rhg_status rhg_generate_with_C(uint64_t n, double C, double alpha, uint64_t seed,
                               const rhg_output *out, rhg_stream stream);

/* Dynamic model (Sec. 3.3).
   rhg_movement_init: per-vertex step values drawn uniformly from
   [phi_lo, phi_hi) and [r_lo, r_hi) (Appendix B uses (-1, 1) and (-10, 1),
   PAPER.md:526-529) by Philox(key = seed, counter = (i, 1)) -- independent of the
   point sample (counter (i, 0)).  Device arrays tau_phi[n], tau_r[n]; |phi_*| < 2pi.
   rhg_move_points: one movement step of every vertex, in place on device arrays:
   theta <- (theta + tau_phi) mod 2pi; r <- Algorithm 2
   (x = sinh(alpha r), y = x + tau_r, r = asinh(y)/alpha) with the
   reflection of PAPER.md:254 applied in y at 0 and sinh(alpha R): tau_r changes
   sign once per reflection.  The graph of the moved points is rebuilt with
   rhg_generate_from_points (the exact edge set of the new positions). */
rhg_status rhg_movement_init(uint64_t n, uint64_t seed, double phi_lo, double phi_hi, double r_lo,
                             double r_hi, double *tau_phi, double *tau_r, rhg_stream stream);
rhg_status rhg_move_points(uint64_t n, double *theta, double *r, const double *tau_phi,
                           double *tau_r, double R, double alpha, rhg_stream stream);

/* On-device validation statistics. */
#define RHG_STATS_BINS 40
typedef struct {
  uint64_t num_edges;      /* undirected edges                                           */
  uint64_t max_degree;
  double mean_degree;      /* 2m / n                                                     */
  uint64_t tail_count;     /* vertices with degree >= k_min                              */
  double tail_exponent;    /* discrete MLE 1 + N / sum ln(k / (k_min - 1/2)) over k >= k_min
                              (compare with gamma = 2 alpha + 1); 0 if no tail */
  uint64_t near_ties;      /* emitted edges with |cosh d - cosh R| <= 1e-12 cosh R
                              (the north star's excused window); ~0 if no points given      */
  uint64_t degree_hist[RHG_STATS_BINS]; /* [0]: degree 0; [b]: degree in [2^(b-1), 2^b)   */
} rhg_stats;

/* Scratch for rhg_graph_stats (device, caller-owned). */
size_t rhg_stats_workspace_bytes(uint64_t n);

/* Statistics of a graph produced by this library, computed on the device:
   format RHG_CSR: row_ptr[n+1], col (device); RHG_EDGES_UNDIRECTED: pairs[2m]
   (device), m undirected edges.  theta/r (device, vertex-id order, optional):
   the points, for the near-tie count.  Synchronises `stream` once. */
rhg_status rhg_graph_stats(uint64_t n, rhg_format format, const uint64_t *row_ptr,
                           const uint32_t *col, const uint32_t *pairs, uint64_t m,
                           const double *theta, const double *r, double R, double k_min,
                           void *workspace, size_t workspace_bytes, rhg_stats *out,
                           rhg_stream stream);

/* ---- Dynamic model: incremental edge update ----
   PAPER.md:387-389 (§4): "Our implementation allows updating a graph without
   rebuilding it from scratch.  Moving up to 12% of nodes and updating an existing
   graph is still faster than a new static generation."  (Movement: rhg_move_points,
   PAPER.md:223-254.)
   Inputs (device pointers): the NEW positions theta[n], r[n] of all points (domain as
   in rhg_generate_from_points); moved[m]: the ids of the vertices whose position
   changed (distinct, < n); theta_old[m], r_old[m]: their OLD positions (same order);
   old_row_ptr[n+1], old_col: the graph of the old positions as a CSR over vertex ids
   (both directions), e.g. rhg_generate_from_points' output with vertex_order 0.
   Output: the undirected edges (u < v) to remove from and to add to the old graph so
   that it becomes the graph of the new positions (each list deterministic, order
   unspecified).  The new points are indexed once (band assignment, sort, SoA,
   directory), the range queries of Alg. 1 run for the moved vertices only, and each
   moved vertex's old and new rows are compared with the certified test of Eq. 3.
   Errors: RHG_ERR_INVALID (arguments), RHG_ERR_DOMAIN (a new point outside the disk),
   RHG_ERR_WORKSPACE (workspace smaller than rhg_update_workspace_bytes(n, row_capacity,
   old_row_ptr[n])
   or the moved vertices' new rows need more than row_capacity entries; the required
   number is written to *rows_needed when given), RHG_ERR_CAPACITY (added or removed
   exceeds capacity; both counts are written, nothing else), RHG_ERR_CUDA.
   Synchronises `stream` three times (old graph size, row total, delta totals). */
typedef struct {
  uint32_t *added;         /* device, 2*capacity entries: (u, v) pairs, u < v                */
  uint32_t *removed;       /* device, 2*capacity entries                                    */
  uint64_t capacity;       /* pairs each list can hold                                      */
  uint64_t *num_added;     /* HOST, required                                                */
  uint64_t *num_removed;   /* HOST, required                                                */
  uint64_t row_capacity;   /* directed entries the moved vertices' new rows may take        */
  uint64_t *rows_needed;   /* HOST, optional: the entries the new rows took / need          */
  void *workspace;         /* device scratch, >= rhg_update_workspace_bytes(...)            */
  size_t workspace_bytes;
  const rhg_options *options; /* slab layout knobs (num_bands, band_ratio); NULL: defaults  */
  rhg_timing *timing;      /* HOST, optional: ms_sort, ms_index, ms_count, ms_emit (rows +
                              delta), ms_total, candidates, certain                        */
} rhg_update;

/* old_entries = old_row_ptr[n] (directed entries of the old graph) */
size_t rhg_update_workspace_bytes(uint64_t n, uint64_t row_capacity, uint64_t old_entries,
                                  const rhg_options *options);
rhg_status rhg_update_moved(uint64_t n, const double *theta, const double *r, double R,
                            const uint32_t *moved, uint64_t m, const double *theta_old,
                            const double *r_old, const uint64_t *old_row_ptr,
                            const uint32_t *old_col, const rhg_update *out, rhg_stream stream);

/* Edges of a given point set (Alg. 1 lines 9-21): theta[n] in [0, 2pi),
   r[n] in [0, R], fp64, device pointers (host if out->host_buffers).  Ids are
   the input indices.  Out-of-domain points -> RHG_ERR_DOMAIN. */
rhg_status rhg_generate_from_points(uint64_t n, const double *theta, const double *r, double R,
                                    const rhg_output *out, rhg_stream stream);

/* K1 alone: write the n sampled points (device pointers) exactly as
   rhg_generate_with_radius would sample them. */
rhg_status rhg_sample_points(uint64_t n, double alpha, double R, uint64_t seed, double *theta,
                             double *r, rhg_stream stream);

/* Raw Philox4x32-10 words for counters i0..i0+count-1 under key = seed
   (out: device, 4*count uint32).  Exposed for parity tests of the sampler. */
rhg_status rhg_philox_words(uint64_t seed, uint64_t i0, uint64_t count, uint32_t *out,
                            rhg_stream stream);

const char *rhg_status_string(rhg_status s);

/* Library version string (build id). */
const char *rhg_version(void);

/* Text of the CUDA error behind the calling thread's last RHG_ERR_CUDA. */
const char *rhg_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RHG_H */
