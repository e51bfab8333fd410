// Why does the direct generate move 1.36x its algorithmic DRAM bytes on 5a?
// The 5a phase pattern with paired red.or.b64 (2 consecutive c per thread):
// rows r-1, r, r+1 of the read half, row r of the write half; halves HALF
// cells apart.  Variants: HALF = 2^28 cells (the 5a table, halves 1 GiB apart),
// HALF = 2^28 + 4096 cells (skewed), and an L2 evict_last / evict_first hint.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/stencil_red_microbench.cu -o scripts/stencil_red_microbench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void red64(unsigned long long* p, unsigned long long v, int hint, uint64_t pol) {
  if (hint == 0) atomicOr(p, v);
  else asm volatile("red.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// tuple pair t: tid = t / (R*C/2), r, c2 ; cells base + 2*c2
__global__ void __launch_bounds__(128, 12)
k_stencil(unsigned long long* tab, uint32_t R, uint32_t C, uint32_t H, uint64_t half, uint64_t n_pairs, int hint,
          int evict_last) {
  uint64_t pol;
  if (evict_last)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t C2 = C / 2;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_pairs; t += stride) {
    const uint32_t c2 = (uint32_t)(t % C2);
    const uint32_t r = (uint32_t)((t / C2) % R);
    const uint32_t tid = (uint32_t)(t / ((uint64_t)C2 * R));
    const uint32_t row = tid * R + r;
    const uint64_t code = tid | ((~tid & 1023u) << 10);
    const unsigned long long v = code | (code << 32);
    const unsigned long long w = v | (1ull << 20) | (1ull << 52);
    red64(tab + (((uint64_t)((row + H - 1) % H) * C) >> 1) + c2, v, hint, pol);
    red64(tab + (((uint64_t)row * C) >> 1) + c2, v, hint, pol);
    red64(tab + (((uint64_t)((row + 1) % H) * C) >> 1) + c2, v, hint, pol);
    red64(tab + ((half + (uint64_t)row * C) >> 1) + c2, w, hint, pol);
  }
}

// Packed cells: K = 3 cells of 21 bits per u64 word; a thread's two consecutive
// cells merge into one red when they share a word, else two reds.
__device__ __forceinline__ void red_pair_packed(unsigned long long* tab, uint64_t sf0, uint64_t code) {
  const uint64_t w0 = sf0 / 3, w1 = (sf0 + 1) / 3;
  const uint32_t s0 = (uint32_t)(sf0 - w0 * 3) * 21, s1 = (uint32_t)(sf0 + 1 - w1 * 3) * 21;
  if (w0 == w1) {
    atomicOr(tab + w0, (code << s0) | (code << s1));
  } else {
    atomicOr(tab + w0, code << s0);
    atomicOr(tab + w1, code << s1);
  }
}
__global__ void __launch_bounds__(128, 12)
k_stencil_packed(unsigned long long* tab, uint32_t R, uint32_t C, uint32_t H, uint64_t half, uint64_t n_pairs) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t C2 = C / 2;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_pairs; t += stride) {
    const uint32_t c2 = (uint32_t)(t % C2);
    const uint32_t r = (uint32_t)((t / C2) % R);
    const uint32_t tid = (uint32_t)(t / ((uint64_t)C2 * R));
    const uint32_t row = tid * R + r;
    const uint64_t code = tid | ((~tid & 1023u) << 10);
    red_pair_packed(tab, (uint64_t)((row + H - 1) % H) * C + 2 * c2, code);
    red_pair_packed(tab, (uint64_t)row * C + 2 * c2, code);
    red_pair_packed(tab, (uint64_t)((row + 1) % H) * C + 2 * c2, code);
    red_pair_packed(tab, half + (uint64_t)row * C + 2 * c2, code | (1ull << 20));
  }
}

// Same as k_stencil (no hints) but every CTA walks a CONTIGUOUS block of the
// pair space (blocked instead of grid-stride tile order).
__global__ void __launch_bounds__(128, 12)
k_stencil_blocked(unsigned long long* tab, uint32_t R, uint32_t C, uint32_t H, uint64_t half, uint64_t n_pairs) {
  const uint32_t C2 = C / 2;
  const uint64_t per_cta = (n_pairs + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * per_cta, hi = min(n_pairs, lo + per_cta);
  for (uint64_t t = lo + threadIdx.x; t < hi; t += blockDim.x) {
    const uint32_t c2 = (uint32_t)(t % C2);
    const uint32_t r = (uint32_t)((t / C2) % R);
    const uint32_t tid = (uint32_t)(t / ((uint64_t)C2 * R));
    const uint32_t row = tid * R + r;
    const uint64_t code = tid | ((~tid & 1023u) << 10);
    const unsigned long long v = code | (code << 32);
    const unsigned long long w = v | (1ull << 20) | (1ull << 52);
    atomicOr(tab + (((uint64_t)((row + H - 1) % H) * C) >> 1) + c2, v);
    atomicOr(tab + (((uint64_t)row * C) >> 1) + c2, v);
    atomicOr(tab + (((uint64_t)((row + 1) % H) * C) >> 1) + c2, v);
    atomicOr(tab + ((half + (uint64_t)row * C) >> 1) + c2, w);
  }
}

// k_stencil + L2 prefetch of the cells DIST grid-strides ahead
template <int DIST>
__global__ void __launch_bounds__(128, 12)
k_stencil_pf(unsigned long long* tab, uint32_t R, uint32_t C, uint32_t H, uint64_t half, uint64_t n_pairs) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t C2 = C / 2;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_pairs; t += stride) {
    {
      const uint64_t tp = t + DIST * stride;
      if (tp < n_pairs) {
        const uint32_t c2 = (uint32_t)(tp % C2);
        const uint32_t r = (uint32_t)((tp / C2) % R);
        const uint32_t tid = (uint32_t)(tp / ((uint64_t)C2 * R));
        const uint32_t row = tid * R + r;
        if ((c2 & 15) == 0) {   // one prefetch per 128-B line
          asm volatile("prefetch.global.L2 [%0];" ::"l"(tab + (((uint64_t)((row + 1) % H) * C) >> 1) + c2));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(tab + ((half + (uint64_t)row * C) >> 1) + c2));
        }
      }
    }
    const uint32_t c2 = (uint32_t)(t % C2);
    const uint32_t r = (uint32_t)((t / C2) % R);
    const uint32_t tid = (uint32_t)(t / ((uint64_t)C2 * R));
    const uint32_t row = tid * R + r;
    const uint64_t code = tid | ((~tid & 1023u) << 10);
    const unsigned long long v = code | (code << 32);
    const unsigned long long w = v | (1ull << 20) | (1ull << 52);
    atomicOr(tab + (((uint64_t)((row + H - 1) % H) * C) >> 1) + c2, v);
    atomicOr(tab + (((uint64_t)row * C) >> 1) + c2, v);
    atomicOr(tab + (((uint64_t)((row + 1) % H) * C) >> 1) + c2, v);
    atomicOr(tab + ((half + (uint64_t)row * C) >> 1) + c2, w);
  }
}

int main() {
  const uint32_t R = 256, C = 1024, H = 1024 * R;
  const uint64_t cells_max = (2ull << 28) + 8192;
  unsigned long long* tab;
  cudaMalloc(&tab, cells_max * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t n_pairs = 1024ull * R * C / 2;   // 2^30 accesses
  struct V { const char* name; uint64_t half; int hint, el; } vs[] = {
      {"halves 2^28 apart", 1ull << 28, 0, 0},
      {"halves 2^28+4096 apart", (1ull << 28) + 4096, 0, 0},
      {"evict_last hint", 1ull << 28, 1, 1},
      {"evict_first hint", 1ull << 28, 1, 0},
  };
  for (auto& v : vs) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(tab, 0, cells_max * 4);
      cudaEventRecord(e0);
      k_stencil<<<148 * 12, 128>>>(tab, R, C, H, v.half, n_pairs, v.hint, v.el);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    printf("%-26s %.3f ms per 2^30 accesses (%.1f G acc/s)\n", v.name, best, 1073741824.0 / best / 1e6);
  }
  {
    const uint64_t words = ((2ull << 28) + 2) / 3;
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(tab, 0, words * 8);
      cudaEventRecord(e0);
      k_stencil_packed<<<148 * 12, 128>>>(tab, R, C, H, 1ull << 28, n_pairs);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    printf("%-26s %.3f ms per 2^30 accesses (%.1f G acc/s)\n", "packed 3 x 21 bits", best, 1073741824.0 / best / 1e6);
  }
  {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(tab, 0, cells_max * 4);
      cudaEventRecord(e0);
      k_stencil_blocked<<<148 * 12, 128>>>(tab, R, C, H, 1ull << 28, n_pairs);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    printf("%-26s %.3f ms per 2^30 accesses (%.1f G acc/s)\n", "blocked CTA ranges", best, 1073741824.0 / best / 1e6);
  }
  for (int dist : {1, 2, 4}) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(tab, 0, cells_max * 4);
      cudaEventRecord(e0);
      if (dist == 1) k_stencil_pf<1><<<148 * 12, 128>>>(tab, R, C, H, 1ull << 28, n_pairs);
      if (dist == 2) k_stencil_pf<2><<<148 * 12, 128>>>(tab, R, C, H, 1ull << 28, n_pairs);
      if (dist == 4) k_stencil_pf<4><<<148 * 12, 128>>>(tab, R, C, H, 1ull << 28, n_pairs);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    printf("prefetch L2 %d strides ahead  %.3f ms per 2^30 accesses (%.1f G acc/s)\n", dist, best, 1073741824.0 / best / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
