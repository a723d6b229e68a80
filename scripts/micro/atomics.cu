// Micro-benchmark: what bounds 1M scattered atomics on a 16 MB counter array? (scratch; not product code)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2306_08252_b200/csrc/dg_kernels.cuh"
using namespace dg;

template <int kVar>
__global__ void __launch_bounds__(256) k(const uint32_t* __restrict__ src, uint32_t n, uint32_t* cnt, uint32_t* rank, uint32_t mask) {
  const uint32_t base = blockIdx.x * 1024 + threadIdx.x;
  uint32_t s[4], r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) { const uint32_t i = base + q * 256; s[q] = i < n ? src[i] : 0; }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t i = base + q * 256;
    if (i >= n) continue;
    uint32_t idx = s[q];
    if (kVar == 2) idx = (idx * 0x9E3779B1u) & mask;          // permuted index
    if (kVar == 0 || kVar == 2 || kVar == 4) r[q] = atomicAdd(&cnt[idx], 1u);
    if (kVar == 1) atomicAdd(&cnt[idx], 1u);                   // RED
    if (kVar == 3) cnt[idx] = 1;                               // plain store
    if (kVar == 5) r[q] = cnt[idx];                            // plain load
  }
  if (kVar == 0 || kVar == 2 || kVar == 4 || kVar == 5) {
#pragma unroll
    for (int q = 0; q < 4; ++q) { const uint32_t i = base + q * 256; if (i < n) rank[i] = r[q]; }
  }
}
__global__ void uniform_kernel(uint32_t* s, uint32_t n, uint32_t mask) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s[i] = (uint32_t)rmat_mix64(i * 7919ull + 1) & mask;
}
int main() {
  const uint32_t n = 1000000, V = 1u << 22;
  uint32_t *src, *dst, *usrc, *cnt, *rank;
  cudaMalloc(&src, n * 4); cudaMalloc(&dst, n * 4); cudaMalloc(&usrc, n * 4); cudaMalloc(&cnt, (V + 2) * 4); cudaMalloc(&rank, n * 4);
  rmat_kernel<<<1024, 256>>>(22, 2, 0, n, 2448131358u, 3264175144u, 4080218931u, src, dst);
  uniform_kernel<<<1024, 256>>>(usrc, n, V - 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"atomic+return rmat", "red rmat", "atomic+return permuted rmat", "plain store rmat", "atomic+return uniform", "plain load rmat"};
  for (int var = 0; var < 6; ++var) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemsetAsync(cnt, 0, (V + 2) * 4);
      cudaEventRecord(a);
      const uint32_t* s = var == 4 ? usrc : src;
      switch (var) {
        case 0: k<0><<<(n + 1023) / 1024, 256>>>(s, n, cnt, rank, V - 1); break;
        case 1: k<1><<<(n + 1023) / 1024, 256>>>(s, n, cnt, rank, V - 1); break;
        case 2: k<2><<<(n + 1023) / 1024, 256>>>(s, n, cnt, rank, V - 1); break;
        case 3: k<3><<<(n + 1023) / 1024, 256>>>(s, n, cnt, rank, V - 1); break;
        case 4: k<4><<<(n + 1023) / 1024, 256>>>(s, n, cnt, rank, V - 1); break;
        case 5: k<5><<<(n + 1023) / 1024, 256>>>(s, n, cnt, rank, V - 1); break;
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-32s %8.2f us\n", names[var], best * 1000);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
