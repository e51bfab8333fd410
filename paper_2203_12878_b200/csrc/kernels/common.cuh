// common.cuh -- small device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../devabi.h"

namespace mapk {

__device__ __forceinline__ uint32_t fastdiv(uint32_t n, const MapcFastDiv& f) {
  if (f.pow2) return n >> f.s;
  uint32_t hi = __umulhi(f.m, n);
  return (hi + ((n - hi) >> 1)) >> f.s;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Streaming 16-byte load that does not allocate in L1 (keys are read once per pass).
__device__ __forceinline__ ulonglong2 ld_stream2(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned long long ld_stream(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Exclusive scan across the block; `tmp` holds >= NW elements.  Returns the
// exclusive prefix of the calling thread; *total receives the block sum.
template <int THREADS, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* tmp, T* total) {
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) tmp[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < NW ? tmp[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < NW) tmp[lane] = xi - x;
    if (lane == NW - 1) tmp[NW] = xi;
  }
  __syncthreads();
  T r = tmp[w] + inc - v;
  *total = tmp[NW];
  __syncthreads();
  return r;
}

}  // namespace mapk
