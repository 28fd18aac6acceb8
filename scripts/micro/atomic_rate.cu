// Microbenchmark: throughput of scattered 32-bit atomicAdd (RED) into an n-entry
// array on B200 -- the cost model of an outward-only count pass.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_red(uint32_t* a, uint32_t n, uint64_t m, uint32_t seed, int local) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12;
    uint32_t p = local ? ((uint32_t)(i >> 5) * 37u + (x & 1023u)) % n : x % n;  // local: nearby addresses
    atomicAdd(&a[p], 1u);
  }
}
int main() {
  const uint32_t n = 10000000; const uint64_t m = 130000000;
  uint32_t* a; cudaMalloc(&a, 4ull * n); cudaMemset(a, 0, 4ull * n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int local = 0; local < 2; ++local)
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      k_red<<<148 * 16, 256>>>(a, n, m, 12345 + rep, local);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%s: %llu atomics into %u entries: %.3f ms = %.2f G/s\n", local ? "local " : "random",
             (unsigned long long)m, n, ms, m / ms / 1e6);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
