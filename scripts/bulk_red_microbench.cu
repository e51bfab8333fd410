// TMA bulk reductions (cp.reduce.async.bulk .or.b32) vs per-lane red.or.b64
// for the 5a stencil pattern: a CTA tile of 512 consecutive c of one row
// stages the codes of each of the 4 sites in shared memory (2 KB each) and one
// thread reduces each 2 KB run into the HBM-resident table.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/bulk_red_microbench.cu -o scripts/bulk_red_microbench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tile = 512 tuples = (tid, r, c0..c0+511); 128 threads x 4 tuples
template <int NBUF>
__global__ void __launch_bounds__(128)
k_bulk(uint32_t* tab, uint32_t R, uint32_t C, uint32_t H, uint64_t half, uint64_t n_tiles) {
  __shared__ __align__(128) uint32_t stage[NBUF][4][512];
  const int me = threadIdx.x;
  int buf = 0;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t t0 = tile * 512;
    const uint32_t c0 = (uint32_t)(t0 % C);
    const uint32_t r = (uint32_t)((t0 / C) % R);
    const uint32_t tid = (uint32_t)(t0 / ((uint64_t)C * R));
    const uint32_t row = tid * R + r;
    const uint32_t code = tid | ((~tid & 1023u) << 10);
    // the buffer we are about to overwrite must have been read by its bulk ops
    if (me == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
    __syncthreads();
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = v * 128 + me;
      stage[buf][0][j] = code;
      stage[buf][1][j] = code;
      stage[buf][2][j] = code;
      stage[buf][3][j] = code | (1u << 20);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (me == 0) {
      const uint64_t base[4] = {(uint64_t)((row + H - 1) % H) * C + c0, (uint64_t)row * C + c0,
                                (uint64_t)((row + 1) % H) * C + c0, half + (uint64_t)row * C + c0};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b32 [%0], [%1], %2;" ::"l"(tab + base[k]),
                     "r"(smem_u32(&stage[buf][k][0])), "r"(2048)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    buf = (buf + 1) % NBUF;
  }
  if (me == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_check(const uint32_t* tab, uint64_t cells, unsigned long long* nz) {
  unsigned long long c = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += (uint64_t)gridDim.x * blockDim.x)
    c += tab[i] != 0;
  atomicAdd(nz, c);
}

int main() {
  const uint32_t R = 256, C = 1024, H = 1024 * R;
  const uint64_t cells = 2ull << 28;
  uint32_t* tab;
  unsigned long long* nz;
  cudaMalloc(&tab, cells * 4);
  cudaMalloc(&nz, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t n_tiles = 1024ull * R * C / 512;
  for (int grid_per_sm : {8, 12, 16}) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(tab, 0, cells * 4);
      cudaEventRecord(e0);
      k_bulk<2><<<148 * grid_per_sm, 128>>>(tab, R, C, H, 1ull << 28, n_tiles);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    cudaMemset(nz, 0, 8);
    k_check<<<148 * 8, 256>>>(tab, cells, nz);
    unsigned long long h = 0;
    cudaMemcpy(&h, nz, 8, cudaMemcpyDeviceToHost);
    printf("bulk or.b32, %2d CTAs/SM: %.3f ms per 2^30 accesses (%.1f G acc/s), nonzero cells %llu of %llu\n",
           grid_per_sm, best, 1073741824.0 / best / 1e6, h, (unsigned long long)cells);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
