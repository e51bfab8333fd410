// What limits the direct-address generate (profiles/r1h_*): global red.or
// throughput on B200 by width and table size, coalesced warp patterns
// (lane i -> cell base + i, the 5a stencil's mapping).
//   b32:  one red.or.b32 per access (4 B payload)
//   b64:  one red.or.b64 covering two adjacent cells (two accesses per lane)
//   st32: plain 4 B stores (no atomics), same addresses
// Table sizes: 32 MiB (L2-resident) and 2 GiB (DRAM-resident, 5a's table).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/red_width_microbench.cu -o scripts/red_width_microbench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// n_acc accesses; access a -> cell (a * 2654435761 >> 5 ... no: sweep) cell = (a % cells)
// with rows of 1024 cells visited 3 times each (stencil-like reuse): access a in
// [row r, col c, rep k] -> cell = ((r + k) % rows) * 1024 + c
template <int MODE>
__global__ void k_red(void* tab, uint64_t rows, uint64_t n_tuples) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tuples; t += stride) {
    if (MODE == 1) {
      // each lane covers 2 adjacent cells: tuple t -> cells 2t, 2t+1 of row (t*2 / 1024)
      const uint64_t cell = 2 * t;
      const uint64_t r = cell >> 10, c = cell & 1023;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t idx = ((r + k) % rows) * 1024 + c;
        atomicOr(reinterpret_cast<unsigned long long*>(tab) + idx / 2, 0x0000030100000301ull);
      }
    } else {
      const uint64_t r = t >> 10, c = t & 1023;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t idx = ((r + k) % rows) * 1024 + c;
        if (MODE == 0) atomicOr(reinterpret_cast<uint32_t*>(tab) + idx, 0x301u);
        else reinterpret_cast<uint32_t*>(tab)[idx] = 0x301u;
      }
    }
  }
}

int main() {
  void* tab;
  const uint64_t big = 1ull << 31;
  cudaMalloc(&tab, big);
  cudaMemset(tab, 0, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t acc = 1ull << 30;   // accesses per launch (4 per tuple for b32/st, 8 per tuple for b64)
  const uint64_t sizes[2] = {32ull << 20, big};
  for (uint64_t bytes : sizes) {
    const uint64_t rows = bytes / 4 / 1024;
    for (int mode = 0; mode < 3; ++mode) {
      for (int threads : {256}) {
        const uint64_t tuples = mode == 1 ? acc / 8 : acc / 4;
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          if (mode == 0) k_red<0><<<148 * 8, threads>>>(tab, rows, tuples);
          if (mode == 1) k_red<1><<<148 * 8, threads>>>(tab, rows, tuples);
          if (mode == 2) k_red<2><<<148 * 8, threads>>>(tab, rows, tuples);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep && ms < best) best = ms;
        }
        printf("table %5llu MiB  %-5s: %.3f ms per 2^30 accesses = %.1f G acc/s (%.2f TB/s payload)\n",
               (unsigned long long)(bytes >> 20), mode == 0 ? "b32" : mode == 1 ? "b64" : "st32", best,
               acc / best / 1e6, acc * 4.0 / best / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
