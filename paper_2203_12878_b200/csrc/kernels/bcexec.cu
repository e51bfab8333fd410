// bcexec.cu -- device helpers of the Theorem-1 differential check (NEXT-2,
// DESIGN.md §5.12): re-pack access keys between key layouts, and compare two
// fully sorted key sets.
//
// The MAP side's keys (Lambda) come out of the generate in a
// chunk's local layout [lphase | array | lblock | index - idx_lo | tid | kind];
// the executor's (alpha in^ P) in the global layout [phase | array | block |
// index | tid | kind].  k_bc_repack maps the former onto the latter so both sides
// can be sorted on all 64 bits and compared as sets (Theorem 1: alpha in^ P iff
// alpha in Lambda).
#include <cuda_runtime.h>

#include <cstdint>

#include "../devabi.h"

namespace {

typedef unsigned long long u64;

struct Repack {
  uint32_t ip, ia, ib, ii, pay;          // input field widths (phase, array, block, index) and payload
  uint32_t op, oa, ob, oi;               // output widths
  u64 phase_lo, b_lo, idx_lo;            // input offsets
};

__device__ __forceinline__ u64 lowbits(u64 v, uint32_t w) { return w >= 64 ? v : (v & ((1ull << w) - 1ull)); }

__global__ void k_bc_repack(const u64* __restrict__ in, u64 n, Repack R, u64* __restrict__ out,
                            unsigned long long* __restrict__ n_outside) {
  unsigned long long outside = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 k = in[i];
    const u64 tk = lowbits(k, R.pay);
    u64 sf = R.pay >= 64 ? 0 : k >> R.pay;
    const u64 idx = lowbits(sf, R.ii) + R.idx_lo;
    sf = R.ii >= 64 ? 0 : sf >> R.ii;
    const u64 blk = lowbits(sf, R.ib) + R.b_lo;
    sf = R.ib >= 64 ? 0 : sf >> R.ib;
    const u64 arr = lowbits(sf, R.ia);
    sf = R.ia >= 64 ? 0 : sf >> R.ia;
    const u64 ph = sf + R.phase_lo;
    // an index the output layout cannot hold (beyond the executor's array
    // extents): counted, written as the all-ones key (never an executed access)
    if (R.oi < 64 && (idx >> R.oi) != 0) {
      ++outside;
      out[i] = ~0ull;
      continue;
    }
    out[i] = ((((((ph << R.oa) | arr) << R.ob | blk) << R.oi) | idx) << R.pay) | tk;
  }
  if (outside) atomicAdd(n_outside, outside);
}

// Distinct keys of sorted a[0..na) (counted into res[0]) that are absent from
// sorted b[0..nb) (counted into res[1], the smallest into res[2] by atomicMin).
// The sorted keys sit in the buffer ctrl->sel[n_passes] picks.
__global__ void k_bc_setdiff(const u64* __restrict__ a0, const u64* __restrict__ a1, const MapcCtrl* __restrict__ ca,
                             uint32_t pa, u64 na, const u64* __restrict__ b0, const u64* __restrict__ b1,
                             const MapcCtrl* __restrict__ cb, uint32_t pb, u64 nb, unsigned long long* __restrict__ res) {
  const u64* a = (ca && ca->sel[pa]) ? a1 : a0;
  const u64* b = (cb && cb->sel[pb]) ? b1 : b0;
  unsigned long long uniq = 0, only = 0, first = ~0ull;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < na; i += (u64)gridDim.x * blockDim.x) {
    const u64 k = a[i];
    if (i > 0 && a[i - 1] == k) continue;
    if (k == ~0ull) continue;                      // a re-packed key outside the layout (k_bc_repack)
    ++uniq;
    u64 lo = 0, hi = nb;                           // lower bound of k in b
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (b[mid] < k) lo = mid + 1; else hi = mid;
    }
    if (lo == nb || b[lo] != k) {
      ++only;
      first = k < first ? k : first;
    }
  }
  if (uniq) atomicAdd(&res[0], uniq);
  if (only) {
    atomicAdd(&res[1], only);
    atomicMin(&res[2], first);
  }
}

}  // namespace

extern "C" cudaError_t mapc_launch_bc_repack(const unsigned long long* in, unsigned long long n, const uint32_t* w_in,
                                             const unsigned long long* offs, const uint32_t* w_out,
                                             unsigned long long* out, unsigned long long* n_outside, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  Repack R{w_in[0], w_in[1], w_in[2], w_in[3], w_in[4], w_out[0], w_out[1], w_out[2], w_out[3], offs[0], offs[1], offs[2]};
  const u64 blocks = (n + 255) / 256;
  k_bc_repack<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(in, n, R, out, n_outside);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_bc_setdiff(const unsigned long long* a0, const unsigned long long* a1,
                                              const MapcCtrl* ca, uint32_t pa, unsigned long long na,
                                              const unsigned long long* b0, const unsigned long long* b1,
                                              const MapcCtrl* cb, uint32_t pb, unsigned long long nb,
                                              unsigned long long* res, cudaStream_t s) {
  if (na == 0) return cudaSuccess;
  const u64 blocks = (na + 255) / 256;
  k_bc_setdiff<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(a0, a1, ca, pa, na, b0, b1, cb, pb, nb, res);
  return cudaGetLastError();
}
