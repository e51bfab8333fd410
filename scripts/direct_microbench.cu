// Sort-free direct-address detect, feasibility on B200: global red.or into a
// 2^29-cell table (one phase of the 5a stencil: 2^30 accesses), cell =
// OR(tid) | OR(~tid) << 10 | write << 20, then a scan of the table.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/direct_microbench.cu -o scripts/direct_microbench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s\n", cudaGetErrorString(e_)); return 1; } } while (0)

// tuple t = (tid, r, c), c fastest; R rows per thread, C cols, H = 1024*R rows
__global__ void k_stencil_red(uint32_t* tab, uint32_t R, uint32_t C, uint32_t H, uint32_t t_phase, uint64_t n_tuples,
                              int mode) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tuples; t += stride) {
    const uint32_t c = (uint32_t)(t % C);
    const uint32_t r = (uint32_t)((t / C) % R);
    const uint32_t tid = (uint32_t)(t / ((uint64_t)C * R));
    const uint64_t HC = (uint64_t)H * C;
    const uint64_t rb = (uint64_t)(t_phase % 2) * HC, wb = (uint64_t)((t_phase + 1) % 2) * HC;
    const uint32_t row = tid * R + r;
    const uint32_t enc_r = tid | ((~tid & 1023u) << 10);
    const uint32_t enc_w = enc_r | (1u << 20);
    uint64_t i0 = rb + (uint64_t)((row + H - 1) % H) * C + c;
    uint64_t i1 = rb + (uint64_t)row * C + c;
    uint64_t i2 = rb + (uint64_t)((row + 1) % H) * C + c;
    uint64_t i3 = wb + (uint64_t)row * C + c;
    if (mode == 0) {
      atomicOr(&tab[i0], enc_r); atomicOr(&tab[i1], enc_r); atomicOr(&tab[i2], enc_r); atomicOr(&tab[i3], enc_w);
    } else {  // plain stores (upper bound: no atomics)
      tab[i0] = enc_r; tab[i1] = enc_r; tab[i2] = enc_r; tab[i3] = enc_w;
    }
  }
}

__global__ void k_scan(const uint4* __restrict__ tab, uint64_t n4, unsigned long long* racy) {
  uint32_t cnt = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 v = tab[i];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) cnt += ((w[j] >> 20) & 1u) && ((w[j] & (w[j] >> 10) & 1023u) != 0);
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(racy, (unsigned long long)cnt);
}

int main() {
  const uint32_t R = 256, C = 1024, H = 1024 * R;
  const uint64_t cells = 2ull * H * C;  // 2^29
  const uint64_t n_tuples = 1024ull * R * C;  // 2^28 tuples, 4 accesses each
  uint32_t* tab;
  unsigned long long* racy;
  CK(cudaMalloc(&tab, cells * 4));
  CK(cudaMalloc(&racy, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  for (int mode = 0; mode < 2; ++mode)
    for (int threads : {256, 512}) {
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemset(tab, 0, cells * 4));
        cudaEventRecord(e0);
        k_stencil_red<<<sms * (2048 / threads), threads>>>(tab, R, C, H, 0, n_tuples, mode);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2)
          printf("%s threads %d: %.3f ms per 2^30 accesses, %.1f G acc/s\n", mode ? "store " : "red.or", threads, ms,
                 n_tuples * 4 / ms / 1e6);
      }
    }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    CK(cudaMemsetAsync(tab, 0, cells * 4));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) printf("memset 2 GiB: %.3f ms (%.0f GB/s)\n", ms, cells * 4 / ms / 1e6);
  }
  k_stencil_red<<<sms * 8, 256>>>(tab, R, C, H, 0, n_tuples, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(racy, 0, 8);
    cudaEventRecord(e0);
    k_scan<<<sms * 8, 256>>>((const uint4*)tab, cells / 4, racy);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h;
    cudaMemcpy(&h, racy, 8, cudaMemcpyDeviceToHost);
    if (rep == 2) printf("scan 2 GiB: %.3f ms (%.0f GB/s), racy %llu\n", ms, cells * 4 / ms / 1e6, h);
  }
  return 0;
}
