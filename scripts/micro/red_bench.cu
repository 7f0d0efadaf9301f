// Microbenchmark: float2 RED throughput at random rows of a 64 MB table
// (the backward scatter's access pattern), vs active lanes per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_red(float2* table, uint32_t rows, int iters, int active_lanes, uint32_t seed) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (lane >= active_lanes) return;
  uint32_t s = hash32(tid ^ seed);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s = hash32(s + k);
      atomicAdd(table + (s % rows), make_float2(1e-3f, 2e-3f));
    }
  }
}

int main() {
  const uint32_t rows = 1u << 23;  // 8M float2 = 64 MB
  float2* t;
  cudaMalloc(&t, rows * sizeof(float2));
  cudaMemset(t, 0, rows * sizeof(float2));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (uint32_t nrows : {1u << 23, 1u << 19, 10648u, 4913u, 1024u}) {
    const int active = 16, bps = 8;
    const int blocks = sms * bps, threads = 256, iters = 64;
    k_red<<<blocks, threads>>>(t, nrows, 4, active, 1);
    cudaEventRecord(a);
    k_red<<<blocks, threads>>>(t, nrows, iters, active, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = (double)blocks * threads / 32 * active * iters * 8;
    printf("rows %8u: %.3e float2 REDs in %.3f ms = %.1f G/s\n", nrows, n, ms, n / ms / 1e6);
  }
  return 0;
}
