// Measurement tool (not product code): L2 atomic throughput on this GPU for the bucket-append
// pattern (atomicAdd returning the old value on one of K counters, then a dependent 8-byte store).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_append(unsigned* fill, uint64_t* out, uint64_t n, unsigned K, unsigned cap, int store, int ret) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t h = i * 0x9E3779B97F4A7C15ULL;
    unsigned b = (unsigned)((h >> 32) % K);
    if (ret) {
      unsigned pos = atomicAdd(fill + b, 1u);
      if (store && pos < cap) out[(uint64_t)b * cap + pos] = h;
    } else {
      atomicAdd(fill + b, 1u);  // RED (no return)
    }
  }
}

int main() {
  const uint64_t n = 64ull << 20;
  unsigned* fill;
  uint64_t* out;
  cudaMalloc(&fill, (1u << 22) * 4);
  const unsigned cap = 64;
  cudaMalloc(&out, 8ull << 30);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (unsigned K : {1u, 64u, 3584u, 65536u, 1u << 20}) {
    const unsigned capk = (unsigned)((8ull << 30) / 8 / K < 1000000000ull ? (8ull << 30) / 8 / K : 1000000000u);
    for (int mode = 0; mode < 3; ++mode) {  // 0 RED, 1 atomic w/ return, 2 atomic + store
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(fill, 0, (uint64_t)K * 4);
        cudaEventRecord(a);
        k_append<<<sms * 8, 256>>>(fill, out, n, K, capk, mode == 2, mode >= 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("K=%8u %-16s %8.3f ms  %7.1f G atomics/s\n", K, mode == 0 ? "red" : mode == 1 ? "atomic-return" : "atomic+store",
             best, n / best / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
