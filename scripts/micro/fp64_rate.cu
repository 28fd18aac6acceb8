// Microbenchmark: FP64 / FP32 pipe throughput on B200 (sm_100a).
// Independent FMA chains per thread so the pipe, not latency, is the limit.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void fma_chain(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)123.456) out[0] = s;
}
__global__ void dmul_chain(double* out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = __dmul_rn(x[c], a);
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 123.456) out[0] = s;
}
__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpsm : {4, 8}) {
      int blocks = sms * bpsm, threads = 256, iters = 20000;
      fma_chain<double, 8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      fma_chain<double, 8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8;
      printf("DFMA  bpsm=%d: %.3f ms  %.2f Tfma/s  %.1f fma/clk/SM@1965\n", bpsm, ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
      fma_chain<float, 8><<<blocks, threads>>>((float*)d, 100, 1.0000001f, 1e-9f);
      cudaEventRecord(e0);
      fma_chain<float, 8><<<blocks, threads>>>((float*)d, iters, 1.0000001f, 1e-9f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("FFMA  bpsm=%d: %.3f ms  %.2f Tfma/s  %.1f fma/clk/SM@1965\n", bpsm, ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
      cudaEventRecord(e0);
      dmul_chain<<<blocks, threads>>>(d, iters, 1.0000001);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("DMUL  bpsm=%d: %.3f ms  %.2f Tmul/s  %.1f /clk/SM@1965\n", bpsm, ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  size_t bytes = 2ull << 30; float4 *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copyk<<<sms * 8, 512>>>(a, b, bytes / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 2 GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
