// Global red.add throughput on B200: random words of a small table (the
// next-pass range histogram, G x 256 words) vs a private smem histogram.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_red(uint32_t* tab, uint32_t words, uint32_t iters, uint32_t local_words) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  // local_words: the addresses a CTA hits are confined to a window (a few ranges x 256)
  const uint32_t base = local_words ? (blockIdx.x * 977u) % (words - local_words) : 0;
  const uint32_t span = local_words ? local_words : words;
  for (uint32_t i = 0; i < iters; ++i) {
    const uint32_t a = base + hash32(t * 131071u + i) % span;
    atomicAdd(&tab[a], 1u);
  }
}

int main() {
  const uint32_t G = 296, words = G * 256;
  uint32_t* tab;
  cudaMalloc(&tab, words * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, threads = 512;
  const uint32_t iters = 512;
  for (uint32_t lw : {0u, 512u, 2048u, 256u}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(tab, 0, words * 4);
      cudaEventRecord(e0);
      k_red<<<blocks, threads>>>(tab, words, iters, lw);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters;
      if (rep) printf("window %u words: %.3f ms, %.1f G red/s\n", lw, ms, ops / ms / 1e6);
    }
  }
  return 0;
}
