// MIO-pipe microbenchmark on sm_100a: cycles per warp-instruction per SM for
// the primitives a radix rank can be built from.  Build & run:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/mio_microbench.cu -o /tmp/mio && /tmp/mio
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void bench(unsigned* out, unsigned seed) {
  __shared__ unsigned sm[8192];
  __shared__ unsigned long long sm64[4096];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm64[i] = 0;
  __syncthreads();
  unsigned x = seed ^ (threadIdx.x * 2654435761u);
  unsigned acc = 0;
  long long t0 = clock64();
#pragma unroll 8
  for (int it = 0; it < ITERS; ++it) {
    x = x * 1664525u + 1013904223u;
    const unsigned d = (x >> 24);                // pseudo-random 8-bit digit
    if (OP == 0) acc += atomicAdd(&sm[(threadIdx.x >> 5) * 256 + d], 1u);          // ATOMS.ADD w/ return, random
    if (OP == 1) atomicAdd(&sm[(threadIdx.x >> 5) * 256 + d], 1u);                 // ATOMS no return (POPC.INC form)
    if (OP == 2) acc += __match_any_sync(0xffffffffu, d);                           // MATCH.ANY
    if (OP == 3) {                                                                  // 8 ballots multisplit
      unsigned p = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) { bool bit = (d >> b) & 1; unsigned m = __ballot_sync(0xffffffffu, bit); p &= bit ? m : ~m; }
      acc += p;
    }
    if (OP == 4) sm64[(d * 16 + (threadIdx.x & 15)) & 4095] = x;                    // STS.64 scattered
    if (OP == 5) acc += __shfl_sync(0xffffffffu, x, d & 31);                         // SHFL
    if (OP == 6) acc += sm[(threadIdx.x >> 5) * 256 + d];                           // LDS random
    if (OP == 7) acc += atomicAdd(&sm[(threadIdx.x >> 5) * 256 + (threadIdx.x & 31) * 8], 1u);  // ATOMS distinct, no conflicts
    if (OP == 8) sm64[threadIdx.x * 4 % 4096 + (it & 3)] = x;                       // STS.64 conflict-free
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x * 2] = (unsigned)(t1 - t0);
  out[blockIdx.x * 2 + 1] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* d;
  cudaMalloc(&d, 8 * 1024 * 1024);
  const char* names[] = {"ATOMS.ADD ret, random digit", "ATOMS no-ret, random digit", "MATCH.ANY", "8x ballot multisplit",
                         "STS.64 scattered", "SHFL", "LDS random", "ATOMS ret, distinct banks", "STS.64 conflict-free"};
  void (*k[])(unsigned*, unsigned) = {bench<0>, bench<1>, bench<2>, bench<3>, bench<4>, bench<5>, bench<6>, bench<7>, bench<8>};
  for (int op = 0; op < 9; ++op) {
    for (int warps : {4, 16, 32}) {
      bench<0><<<sms, 32 * warps>>>(d, 1);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k[op]<<<sms, 32 * warps>>>(d, 7);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      unsigned cyc;
      cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
      double per_warp_instr_sm = (double)cyc / ((double)ITERS * warps);   // SM cycles per warp-instruction (all warps share the SM)
      printf("%-32s warps/SM=%2d  cycles=%10u  SM-cycles per warp-op=%6.2f  (%.3f ms)\n", names[op], warps, cyc,
             per_warp_instr_sm, ms);
    }
  }
  return 0;
}
