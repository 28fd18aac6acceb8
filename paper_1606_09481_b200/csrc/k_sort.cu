// k_sort.cu -- K3: stable LSD radix sort of 32-bit keys (band << 27 | q27(theta))
// with a 32-bit payload, plus the generic exclusive scans (K6).
//
// Paper: "sort points in b by their angular coordinates" (Alg. 1 lines 11-12,
// PAPER.md:153-155).  One global sort by (band, angle) yields every band as a
// contiguous, angle-sorted segment (the slabs b_i of PAPER.md:192-197).
#include <atomic>

#include "rhg_internal.cuh"

namespace rhg {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef RHG_RS_ITEMS
#define RHG_RS_ITEMS 16
#endif
constexpr int RS_ITEMS = RHG_RS_ITEMS;             // per thread
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;     // keys per tile
constexpr int RS_RADIX = 256;

// One read of the keys: the digit histograms of all passes (shift 8 p, p < P).
__global__ void __launch_bounds__(RS_THREADS)
    k_rs_hist_all(uint32_t n, const uint32_t* __restrict__ keys, int P, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[4][RS_RADIX];
  for (int p = 0; p < 4; ++p) h[p][threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * RS_THREADS + threadIdx.x; i < n; i += gridDim.x * RS_THREADS) {
    const uint32_t k = __ldg(keys + i);
    for (int p = 0; p < P; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFFu], 1u);
  }
  __syncthreads();
  for (int p = 0; p < P; ++p)
    if (h[p][threadIdx.x]) atomicAdd(&ghist[p * RS_RADIX + threadIdx.x], h[p][threadIdx.x]);
}

// exclusive scan of each pass's 256 digit counts -> digit start positions
__global__ void __launch_bounds__(RS_RADIX) k_rs_digit_start(int P, const uint32_t* __restrict__ ghist,
                                                             uint32_t* __restrict__ dstart) {
  __shared__ uint32_t ws[RS_RADIX / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int p = 0; p < P; ++p) {
    const uint32_t c = ghist[p * RS_RADIX + threadIdx.x];
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    uint32_t pre = 0;
    for (int ww = 0; ww < w; ++ww) pre += ws[ww];
    dstart[p * RS_RADIX + threadIdx.x] = pre + inc - c;
    __syncthreads();
  }
}

#ifndef RHG_RS_MINB
#define RHG_RS_MINB 5
#endif
// Look-back status of (tile, digit): bits 62-63 flag (0 not yet, 1 tile count,
// 2 inclusive prefix over tiles), bits 0-61 the value.
#ifndef RHG_RS_SPIN_NS
#define RHG_RS_SPIN_NS 0
#endif
#ifndef RHG_RS_VAL_SMEM
#define RHG_RS_VAL_SMEM 1
#endif
#ifndef RHG_RS_BALLOT_MATCH
#define RHG_RS_BALLOT_MATCH 1
#endif
constexpr unsigned long long kRsAgg = 1ull << 62, kRsIncl = 2ull << 62;
constexpr unsigned long long kRsVal = (1ull << 62) - 1ull;

// One LSD pass ("onesweep"): tiles take tickets in the order they start; each
// ranks its keys by digit (warp w of the tile owns items [w*512, +512) and walks
// them in 16 rounds of 32; 8 bit ballots find the lanes of equal digit in a round,
// whose leader reserves their slots with one shared-memory atomic, so the order is
// stable), publishes its per-digit counts, and finds the count of
// every digit in all earlier tiles by decoupled look-back (thread d walks back over
// the tiles' (tile, d) words until an inclusive prefix).  The tile is then
// re-ordered by digit in shared memory and written out so that consecutive threads
// store consecutive addresses of one digit run (coalesced).  A tile waits only on
// tiles that took earlier tickets, so every wait ends.
__global__ void __launch_bounds__(RS_THREADS, RHG_RS_MINB)
    k_rs_onesweep(uint32_t n, const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                  uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int shift,
                  const uint32_t* __restrict__ dstart, unsigned long long* status,
                  uint32_t* ticket) {
  __shared__ uint32_t wcnt[RS_WARPS][RS_RADIX];
  __shared__ uint32_t tstart[RS_RADIX];
  __shared__ uint32_t gbase[RS_RADIX];
  __shared__ uint32_t wsum[RS_WARPS];
  extern __shared__ uint32_t rs_dyn[];  // RS_TILE keys then RS_TILE values
  uint32_t* skey = rs_dyn;
  uint32_t* sval = rs_dyn + RS_TILE;
  __shared__ uint32_t tile_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) tile_s = atomicAdd(ticket, 1u);
  for (int d = lane; d < RS_RADIX; d += 32) wcnt[w][d] = 0;
  __syncthreads();
  const uint32_t tile = tile_s;
  const uint32_t tbase = tile * RS_TILE;
  const uint32_t wbase = tbase + w * (32 * RS_ITEMS);
  static_assert(RS_ITEMS % 2 == 0 && 32 * RS_ITEMS <= 65536, "two 16-bit ranks per register");
  uint32_t key[RS_ITEMS], loc2[RS_ITEMS / 2];  // rank in the warp's digit run
  const uint32_t lt = (1u << lane) - 1u;
#if RHG_RS_VAL_SMEM
  // values parked in shared memory at their input slots until the scatter (fewer
  // live registers through the ranking and the look-back)
  uint32_t* vpark = sval + w * (32 * RS_ITEMS);
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    key[it] = i < n ? __ldg(kin + i) : 0u;
    vpark[it * 32 + lane] = i < n ? __ldg(vin + i) : 0u;
  }
#else
  uint32_t val[RS_ITEMS];
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {  // all loads in flight before the ranking chain
    const uint32_t i = wbase + it * 32 + lane;
    key[it] = i < n ? __ldg(kin + i) : 0u;
    val[it] = i < n ? __ldg(vin + i) : 0u;
  }
#endif
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? ((key[it] >> shift) & 0xFFu) : (RS_RADIX + lane);
#if RHG_RS_BALLOT_MATCH
    // equal-digit peers from 8 bit ballots (+ validity), instead of match.any
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
    if (!valid) peers = ~peers;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
#else
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#endif
    // the group leader reserves the group's slots with one shared-memory atomic
    // (same-address atomics of one warp execute in issue order: stable)
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && leader == lane) old = atomicAdd(&wcnt[w][d], (uint32_t)__popc(peers));
    const uint32_t rk = __shfl_sync(0xffffffffu, old, leader) + __popc(peers & lt);
    if (it & 1) loc2[it >> 1] |= rk << 16; else loc2[it >> 1] = rk;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (warp order = item order => stable),
  // the digit's start inside the tile (block scan over the 256 digit totals), and
  // its start in the output (digit start + counts of earlier tiles, look-back)
  {
    const int d = threadIdx.x;  // RS_THREADS == RS_RADIX
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
      const uint32_t c = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += c;
    }
    volatile unsigned long long* my = status + (size_t)tile * RS_RADIX + d;
    *my = (tile == 0 ? kRsIncl : kRsAgg) | run;
    // look back over up to kLb earlier tiles per round (their words loaded together),
    // summing tile counts until an inclusive prefix
#ifndef RHG_RS_LOOKBACK
#define RHG_RS_LOOKBACK 1
#endif
    constexpr uint32_t kLb = RHG_RS_LOOKBACK;
    unsigned long long excl = 0;
    for (uint32_t t2 = tile; t2 > 0;) {
      const uint32_t k = t2 < kLb ? t2 : kLb;
      unsigned long long v[kLb];
#pragma unroll
      for (uint32_t j = 0; j < kLb; ++j)
        v[j] = j < k ? *(const volatile unsigned long long*)(status + (size_t)(t2 - 1 - j) * RS_RADIX + d) : 0ull;
      bool done = false;
#pragma unroll
      for (uint32_t j = 0; j < kLb; ++j) {
        if (done || j >= k) continue;
        const volatile unsigned long long* o = status + (size_t)(t2 - 1 - j) * RS_RADIX + d;
        while ((v[j] & ~kRsVal) == 0ull) {
#if RHG_RS_SPIN_NS
          __nanosleep(RHG_RS_SPIN_NS);  // back off: the spinning warps' polls take issue slots
#endif
          v[j] = *o;
        }
        excl += v[j] & kRsVal;
        done = (v[j] & ~kRsVal) == kRsIncl;
      }
      if (done) break;
      t2 -= k;
    }
    if (tile) *my = kRsIncl | (excl + run);
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) wpre += (ww < w) ? wsum[ww] : 0u;
    tstart[d] = wpre + inc - run;
    gbase[d] = dstart[d] + (uint32_t)excl;
  }
  __syncthreads();
#if RHG_RS_VAL_SMEM
  uint32_t val[RS_ITEMS];
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) val[it] = vpark[it * 32 + lane];
  __syncthreads();
#endif
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    if (i < n) {
      const uint32_t d = (key[it] >> shift) & 0xFFu;
      const uint32_t lp = tstart[d] + wcnt[w][d] + ((loc2[it >> 1] >> (16 * (it & 1))) & 0xFFFFu);
      skey[lp] = key[it];
      sval[lp] = val[it];
    }
  }
  __syncthreads();
  const uint32_t tn = (n - tbase) < (uint32_t)RS_TILE ? (n - tbase) : (uint32_t)RS_TILE;
  for (uint32_t i = threadIdx.x; i < tn; i += RS_THREADS) {
    const uint32_t k = skey[i];
    const uint32_t d = (k >> shift) & 0xFFu;
    const uint32_t gp = gbase[d] + (i - tstart[d]);
    kout[gp] = k;
    vout[gp] = sval[i];
  }
}

// ----------------------------------------------------------------- scans
constexpr int SC_THREADS = 1024;
constexpr int SC_ITEMS = 8;
constexpr int SC_CHUNK = SC_THREADS * SC_ITEMS;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T a = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += a;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive prefix,
// writes the block total to *total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : T(0);
    T si = warp_incl_scan(s);
    sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  T res = inc - v + sh[w];
  if (total) *total = sh[32];
  __syncthreads();
  return res;
}

__device__ __forceinline__ uint64_t dev_count(uint64_t n, const unsigned long long* n_dev) {
  if (!n_dev) return n;
  uint64_t d = *n_dev;
  return d < n ? d : n;
}

template <typename TIn, typename TAcc>
__global__ void __launch_bounds__(SC_THREADS)
    k_scan_reduce(uint64_t n, const TIn* __restrict__ in, TAcc* __restrict__ partial,
                  const unsigned long long* n_dev) {
  __shared__ TAcc sh[33];
  n = dev_count(n, n_dev);
  uint64_t base = (uint64_t)blockIdx.x * SC_CHUNK;
  TAcc s = 0;
#pragma unroll
  for (int it = 0; it < SC_ITEMS; ++it) {
    uint64_t i = base + (uint64_t)it * SC_THREADS + threadIdx.x;
    if (i < n) s += (TAcc)in[i];
  }
  TAcc tot;
  block_excl_scan<TAcc>(s, sh, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// single block: exclusive scan of the partials in place; total -> *total
template <typename TAcc, typename TOut>
__global__ void __launch_bounds__(SC_THREADS)
    k_scan_partials(uint32_t m, TAcc* partial, TOut* out_base, uint64_t n,
                    const unsigned long long* n_dev, unsigned long long* total_out) {
  __shared__ TAcc sh[33];
  TAcc carry = 0;
  for (uint32_t base = 0; base < m; base += SC_THREADS) {
    uint32_t i = base + threadIdx.x;
    TAcc v = i < m ? partial[i] : TAcc(0);
    TAcc tot;
    TAcc ex = block_excl_scan<TAcc>(v, sh, &tot);
    if (i < m) partial[i] = ex + carry;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    if (out_base) out_base[dev_count(n, n_dev)] = (TOut)carry;
    if (total_out) *total_out = (unsigned long long)carry;
  }
}

// Each thread owns SC_ITEMS consecutive elements (blocked), exclusive scan.
template <typename TIn, typename TOut, typename TAcc>
__global__ void __launch_bounds__(SC_THREADS)
    k_scan_down(uint64_t n, const TIn* __restrict__ in, TOut* __restrict__ out,
                const TAcc* __restrict__ partial, const unsigned long long* n_dev) {
  __shared__ TAcc sh[33];
  n = dev_count(n, n_dev);
  if ((uint64_t)blockIdx.x * SC_CHUNK >= n) return;
  uint64_t base = (uint64_t)blockIdx.x * SC_CHUNK + (uint64_t)threadIdx.x * SC_ITEMS;
  // whole 32-byte runs of the input (and 16-byte aligned output) move as vectors
  const bool vec = sizeof(TIn) == 4 && base + SC_ITEMS <= n && ((uintptr_t)(in + base) & 15) == 0 &&
                   ((uintptr_t)(out + base) & 15) == 0;
  TAcc v[SC_ITEMS];
  TAcc s = 0;
  if (vec) {
    const uint4 a = reinterpret_cast<const uint4*>(in + base)[0];
    const uint4 b = reinterpret_cast<const uint4*>(in + base)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int it = 0; it < SC_ITEMS; ++it) {
      uint64_t i = base + it;
      v[it] = i < n ? (TAcc)in[i] : TAcc(0);
    }
  }
#pragma unroll
  for (int it = 0; it < SC_ITEMS; ++it) s += v[it];
  TAcc ex = block_excl_scan<TAcc>(s, sh, (TAcc*)nullptr) + partial[blockIdx.x];
  TOut o[SC_ITEMS];
#pragma unroll
  for (int it = 0; it < SC_ITEMS; ++it) {
    o[it] = (TOut)ex;
    ex += v[it];
  }
  if (vec) {
    uint4* d = reinterpret_cast<uint4*>(out + base);
#pragma unroll
    for (int q = 0; q < (int)(SC_ITEMS * sizeof(TOut) / 16); ++q) d[q] = reinterpret_cast<const uint4*>(o)[q];
  } else {
#pragma unroll
    for (int it = 0; it < SC_ITEMS; ++it) {
      uint64_t i = base + it;
      if (i < n) out[i] = o[it];
    }
  }
}

static uint32_t sc_blocks(uint64_t n) { return (uint32_t)((n + SC_CHUNK - 1) / SC_CHUNK); }

size_t scan_tmp_bytes(uint64_t n) { return (size_t)(sc_blocks(n) + 2) * sizeof(uint64_t) + 256; }

cudaError_t exclusive_scan_u32_u64(uint32_t n, const uint32_t* in, uint64_t* out, void* tmp,
                                   unsigned long long* total_out, cudaStream_t st, int* launches) {
  return exclusive_scan_u32_u64_dev(n, nullptr, in, out, tmp, total_out, st, launches);
}

cudaError_t exclusive_scan_u32_u64_dev(uint64_t n_cap, const unsigned long long* n_dev,
                                       const uint32_t* in, uint64_t* out, void* tmp,
                                       unsigned long long* total_out, cudaStream_t st,
                                       int* launches) {
  uint32_t B = sc_blocks(n_cap);
  if (B == 0) B = 1;
  uint64_t* partial = (uint64_t*)tmp;
  k_scan_reduce<uint32_t, uint64_t><<<B, SC_THREADS, 0, st>>>(n_cap, in, partial, n_dev);
  k_scan_partials<uint64_t, uint64_t><<<1, SC_THREADS, 0, st>>>(B, partial, out, n_cap, n_dev,
                                                                total_out);
  k_scan_down<uint32_t, uint64_t, uint64_t><<<B, SC_THREADS, 0, st>>>(n_cap, in, out, partial,
                                                                      n_dev);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

// tmp: digit counts and starts (4 passes x 256), tickets, look-back words
size_t radix_sort_tmp_bytes(uint64_t n) {
  uint64_t G = (n + RS_TILE - 1) / RS_TILE;
  if (G == 0) G = 1;
  return (size_t)(2 * 4 * RS_RADIX + 8) * sizeof(uint32_t) + 4 * G * RS_RADIX * 8ull + 256;
}

// opt in to > 48 KB of dynamic shared memory once (outside any stream capture)
// (the attribute is per device: one flag per device, set atomically)
cudaError_t radix_sort_prepare() {
  static std::atomic<bool> done[64];
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) d = 0;
  if (done[d].load(std::memory_order_acquire)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(k_rs_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             2 * RS_TILE * (int)sizeof(uint32_t));
  if (e == cudaSuccess) done[d].store(true, std::memory_order_release);
  return e;
}

cudaError_t radix_sort(uint32_t n, uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b,
                       uint32_t* vals_b, void* tmp, int begin_bit, int end_bit, cudaStream_t st,
                       int* launches) {
  uint32_t G = (n + RS_TILE - 1) / RS_TILE;
  if (G == 0) return cudaSuccess;
  const int P = (end_bit - begin_bit + 7) / 8;
  if (begin_bit != 0 || P < 1 || P > 4) return cudaErrorInvalidValue;
  uint32_t* ghist = (uint32_t*)tmp;
  uint32_t* dstart = ghist + 4 * RS_RADIX;
  uint32_t* tickets = dstart + 4 * RS_RADIX;
  unsigned long long* status = (unsigned long long*)(tickets + 8);  // 32-byte aligned
  // counts, starts, tickets and the look-back words of the P passes that run
  const size_t zero = (size_t)((char*)(status + (size_t)P * G * RS_RADIX) - (char*)tmp);
  cudaError_t e = cudaMemsetAsync(tmp, 0, zero, st);
  if (e != cudaSuccess) return e;
  uint32_t hb = (n + RS_THREADS * 16 - 1) / (RS_THREADS * 16);
  if (hb > (uint32_t)num_sms() * 8) hb = (uint32_t)num_sms() * 8;
  k_rs_hist_all<<<hb, RS_THREADS, 0, st>>>(n, keys_a, P, ghist);
  k_rs_digit_start<<<1, RS_RADIX, 0, st>>>(P, ghist, dstart);
  uint32_t *ki = keys_a, *vi = vals_a, *ko = keys_b, *vo = vals_b;
  constexpr int dyn = 2 * RS_TILE * (int)sizeof(uint32_t);
  e = radix_sort_prepare();
  if (e != cudaSuccess) return e;
  for (int p = 0; p < P; ++p) {
    k_rs_onesweep<<<G, RS_THREADS, dyn, st>>>(n, ki, vi, ko, vo, 8 * p, dstart + p * RS_RADIX,
                                              status + (size_t)p * G * RS_RADIX, tickets + p);
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
  }
  if (launches) *launches += 2 + P;
  if (P & 1) {  // result must land in (keys_a, vals_a)
    e = cudaMemcpyAsync(keys_a, ki, (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(vals_a, vi, (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace rhg
