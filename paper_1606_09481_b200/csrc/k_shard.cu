// k_shard.cu -- SURVEY.md §8(e): one graph sharded over N GPUs.  Every shard samples,
// sorts and indexes all points (identical on every GPU), then emits only the rows
// of the query items it owns.  Items in processing order: the hub vertices (chunked
// path), then the 32-vertex groups of the sector-major light order.
//
// Ownership balances the expected work, not the vertex count (hubs
// sorted by slab put the heaviest work on shard 0):
//  * work of an item = the candidates its queries visit (k_shard_work in k_query.cu):
//    a hub's exact count (its windows, one slab per lane); for a light group the sum
//    of the expected counts E(r_v) = sum_k n_k min(1, W(r_v, c_k) / pi) of its
//    vertices (W = the outer window of slab k, getMinMaxPhi at c_k, PAPER.md:199-209
//    Eqs. 6-9; k over all slabs for CSR, over the slabs >= v's own for the outward
//    list), scaled by exact / E of the group's first vertex -- E captures the heavy
//    tail of the per-vertex work (gamma = 2.2: work ~ degree), the exact count the
//    lumpy angular distribution of the few inner-slab points an arc sees;
//  * hub vertices (few, heavy, sorted inner to outer so consecutive hubs have
//    similar work) are dealt in snake order (0..N-1, N-1..0, ...), giving hub work
//    H_s per shard;
//  * the light groups are cut into N contiguous ranges of the light-work prefix
//    with quotas proportional to max(0, W/N - H_s), so hub and light work together
//    are W/N per shard.  Contiguous ranges keep each GPU's reads in its own arc of
//    the circle (L2 locality); the realised point set makes the work of an arc
//    deviate from E by ~2 % at 1/16 of the circle.  (Cutting the whole item prefix
//    into equal chunks let single hubs larger than a chunk unbalance the shards by
//    up to 12 % at N = 8.)
// The partition never changes the edge set; every GPU computes the same numbers.
#include "rhg_internal.cuh"

namespace rhg {

// hub work per shard (snake order), then this shard's light group range
__global__ void __launch_bounds__(256)
    k_shard_hubs(const BandLayout* __restrict__ lay, const uint32_t* __restrict__ work,
                 uint32_t nshards, unsigned long long* __restrict__ hub_work) {
  const uint32_t he = lay->heavy_end;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < he; i += gridDim.x * blockDim.x)
    atomicAdd(hub_work + snake(i, nshards), (unsigned long long)work[i]);
}

__device__ __forceinline__ uint32_t first_group_at(const uint64_t* prefix, uint32_t he,
                                                   uint32_t ngroups, unsigned long long target) {
  uint32_t lo = 0, hi = ngroups;  // first light group whose prefix >= target
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (prefix[he + mid] < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_shard_bounds(uint32_t n, const BandLayout* __restrict__ lay,
                               const uint64_t* __restrict__ prefix,
                               const unsigned long long* __restrict__ hub_work, uint32_t shard,
                               uint32_t nshards, ShardPlan* plan) {
  const uint32_t he = lay->heavy_end, ngroups = (n - he + 31u) / 32u;
  const unsigned long long W = prefix[he + ngroups], H = prefix[he], WL = W - H;
  // quotas q_s = max(0, W/N - H_s); shard s takes light work [WL Q_<s / Q, WL Q_<=s / Q)
  const double share = (double)W / nshards;
  double Q = 0.0, Qlo = 0.0, Qhi = 0.0;
  for (uint32_t s = 0; s < nshards; ++s) {
    const double q = fmax(0.0, share - (double)hub_work[s]);
    if (s < shard) Qlo += q;
    if (s <= shard) Qhi += q;
    Q += q;
  }
  const double scale = Q > 0.0 ? (double)WL / Q : 0.0;
  const unsigned long long t0 = H + (unsigned long long)(Qlo * scale);
  const unsigned long long t1 = shard + 1 == nshards ? W : H + (unsigned long long)(Qhi * scale);
  plan->grp_beg = shard == 0 ? 0u : first_group_at(prefix, he, ngroups, t0);
  plan->grp_end = shard + 1 == nshards ? ngroups : first_group_at(prefix, he, ngroups, t1);
  plan->work_total = W;
  plan->hub_work = hub_work[shard];
}

cudaError_t launch_shard_plan(uint32_t n, const QueryArgs& qa, const BandConst& bc, int outward,
                              uint32_t* work, uint64_t* prefix, uint64_t item_cap, void* scan_tmp,
                              unsigned long long* hub_work, ShardPlan* plan, cudaStream_t st,
                              int* launches) {
  cudaError_t e = launch_shard_work(qa, bc, outward, work, st);
  if (e != cudaSuccess) return e;
  // items = heavy_end + ceil((n - heavy_end) / 32) <= item_cap, counted on the device
  e = exclusive_scan_u32_u64(item_cap, work, prefix, scan_tmp, nullptr, st, launches);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(hub_work, 0, 8ull * bc.nshards, st);
  if (e != cudaSuccess) return e;
  k_shard_hubs<<<num_sms(), 256, 0, st>>>(qa.lay, work, bc.nshards, hub_work);
  k_shard_bounds<<<1, 1, 0, st>>>(n, qa.lay, prefix, hub_work, bc.shard, bc.nshards, plan);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

}  // namespace rhg
