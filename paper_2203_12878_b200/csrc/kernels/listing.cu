// listing.cu -- full race listing (SPEC.md:434-437
// races_of, reported per racy segment): the canonical witness of EVERY racy
// segment, in sort-field order, over fully sorted keys.
//
// Two passes over the keys with the same warp ranges as the detect
// (detect_unit): k_list_racy(count) counts, per warp, the racy segments whose
// FIRST key lies in the warp's range (a segment is walked to its end even
// past the range); one CTA scans the counts; k_list_racy(write) walks again
// and stores each racy segment's packed witness at its rank.  The output is
// in sort-field order by construction; entries at rank >= cap are dropped
// (the count stays exact).
#include <algorithm>

#include "common.cuh"
#include "segstate.cuh"

namespace mapk {

constexpr int LS_THREADS = 256;

__device__ __forceinline__ unsigned long long list_unit(unsigned long long n, unsigned long long nw) {
  unsigned long long u = (n + nw - 1) / nw;
  u = (u + 31ull) & ~31ull;
  return u < 32ull ? 32ull : u;
}

// Fold the segment starting at position i (its first key) and return its packed
// witness (~0 when race-free).  Walks keys i, i+1, ... while the sort field holds.
__device__ unsigned long long segment_witness(const unsigned long long* __restrict__ keys, unsigned long long n,
                                              unsigned long long i, uint32_t pay_bits, uint32_t w_tid,
                                              uint32_t tmask) {
  const unsigned long long sf = keys[i] >> pay_bits;
  St s;
  st_init(s);
  unsigned long long j = i;
  for (; j + 4 <= n; j += 4) {                         // 4 loads in flight
    unsigned long long k[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = keys[j + u];
    bool done = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!done && (k[u] >> pay_bits) == sf) st_add(s, (uint32_t)(k[u] >> 1) & tmask, 1u << (k[u] & 1u));
      else done = true;
    }
    if (done) return st_witness(s, sf, w_tid);
  }
  for (; j < n; ++j) {
    const unsigned long long k = keys[j];
    if ((k >> pay_bits) != sf) break;
    st_add(s, (uint32_t)(k >> 1) & tmask, 1u << (k & 1u));
  }
  return st_witness(s, sf, w_tid);
}

// mode 0: counts[gw] = racy segments headed in warp gw's range.
// mode 1: write each one's packed witness to out[offsets[gw] + rank] (rank < cap).
__global__ void __launch_bounds__(LS_THREADS)
k_list_racy(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
            const MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid, int mode,
            unsigned long long* __restrict__ counts, unsigned long long* __restrict__ out, unsigned long long cap) {
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const uint32_t lane = threadIdx.x & 31;
  const unsigned long long nw = (unsigned long long)gridDim.x * (LS_THREADS / 32);
  const unsigned long long gw = (unsigned long long)blockIdx.x * (LS_THREADS / 32) + (threadIdx.x >> 5);
  const unsigned long long unit = list_unit(n, nw);
  const unsigned long long start = gw * unit, end = min(n, start + unit);
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  unsigned long long rank = mode ? counts[gw] : 0ull;    // mode 1: counts holds the exclusive offsets
  for (unsigned long long b = start; b < end; b += 32) {
    const unsigned long long i = b + lane;
    bool head = false;
    if (i < end) head = i == 0 || (keys[i] >> pay_bits) != (keys[i - 1] >> pay_bits);
    unsigned long long w = ~0ull;
    if (head) w = segment_witness(keys, n, i, pay_bits, w_tid, tmask);
    const uint32_t racy = __ballot_sync(0xFFFFFFFFu, w != ~0ull);
    if (mode && w != ~0ull) {
      const unsigned long long r = rank + __popc(racy & ((1u << lane) - 1u));
      if (r < cap) out[r] = w;
    }
    rank += __popc(racy);
  }
  if (!mode && lane == 0) counts[gw] = rank;
}

// Exclusive scan of the per-warp counts in place (one CTA); total -> *total.
__global__ void __launch_bounds__(1024) k_list_scan(unsigned long long* __restrict__ counts, unsigned int nw,
                                                   unsigned long long* __restrict__ total) {
  __shared__ unsigned long long part[1024];
  const unsigned int per = (nw + 1023) / 1024;
  const unsigned int lo = threadIdx.x * per, hi = min(nw, lo + per);
  unsigned long long sum = 0;
  for (unsigned int i = lo; i < hi; ++i) sum += counts[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int t = 0; t < 1024; ++t) { const unsigned long long v = part[t]; part[t] = acc; acc += v; }
    *total = acc;
  }
  __syncthreads();
  unsigned long long acc = part[threadIdx.x];
  for (unsigned int i = lo; i < hi; ++i) { const unsigned long long v = counts[i]; counts[i] = acc; acc += v; }
}

}  // namespace mapk

// Lists the packed witnesses of all racy segments of the chunk whose sorted keys
// are in bufA/bufB (ctrl->sel[n_passes]); out[cap] (device), *total (device).
extern "C" cudaError_t mapc_launch_list_racy(const unsigned long long* bufA, const unsigned long long* bufB,
                                             const MapcCtrl* ctrl, uint32_t n_passes, uint32_t pay_bits,
                                             uint32_t w_tid, unsigned long long* counts, unsigned int max_warps,
                                             unsigned long long* out, unsigned long long cap,
                                             unsigned long long* total, unsigned long long max_keys, int n_sms,
                                             cudaStream_t s) {
  unsigned long long warps = (max_keys + 31) / 32;
  const unsigned long long cap_w = std::min<unsigned long long>((unsigned long long)n_sms * 64, max_warps);
  if (warps > cap_w) warps = cap_w;
  if (warps < 8) warps = 8;
  const int grid = (int)(warps / 8);
  const unsigned int nw = (unsigned int)grid * 8;
  mapk::k_list_racy<<<grid, mapk::LS_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid, 0, counts,
                                                      out, cap);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mapk::k_list_scan<<<1, 1024, 0, s>>>(counts, nw, total);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mapk::k_list_racy<<<grid, mapk::LS_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid, 1, counts,
                                                      out, cap);
  return cudaGetLastError();
}
