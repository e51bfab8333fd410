// segstate.cuh -- the order-independent per-segment state of the canonical
// witness: m1 = smallest tid with kind mask k1, m2 = second
// smallest distinct tid with mask k2, w = smallest writer tid.  The merge is
// associative and commutative; st_witness gives the segment's canonical
// witness in closed form, packed so that unsigned order = lexicographic order.
#pragma once
#include "common.cuh"

namespace mapk {

constexpr uint32_t NONE = 0xFFFFFFFFu;

struct St {
  uint32_t m1, m2, w;
  uint32_t k1, k2;
};

__device__ __forceinline__ void st_init(St& s) {
  s.m1 = s.m2 = s.w = NONE;
  s.k1 = s.k2 = 0;
}

__device__ __forceinline__ void st_add(St& s, uint32_t t, uint32_t mask) {
  if (t == s.m1) {
    s.k1 |= mask;
  } else if (t < s.m1) {
    s.m2 = s.m1; s.k2 = s.k1;
    s.m1 = t; s.k1 = mask;
  } else if (t == s.m2) {
    s.k2 |= mask;
  } else if (t < s.m2) {
    s.m2 = t; s.k2 = mask;
  }
  if ((mask & 2u) && t < s.w) s.w = t;
}

__device__ __forceinline__ void st_merge(St& s, const St& o) {
  if (o.m1 != NONE) st_add(s, o.m1, o.k1);
  if (o.m2 != NONE) st_add(s, o.m2, o.k2);
  if (o.w < s.w) s.w = o.w;
}

// Packed witness (UINT64_MAX if the segment is race-free).
__device__ __forceinline__ unsigned long long st_witness(const St& s, unsigned long long sf, uint32_t wt) {
  uint32_t thi, klo, khi;
  if (s.k1 & 2u) {                       // m1 writes: partner is m2 (any kind)
    if (s.m2 == NONE) return ~0ull;
    thi = s.m2;
    if ((s.k1 & 1u) && (s.k2 & 2u)) { klo = 0; khi = 1; }
    else if (s.k2 & 1u) { klo = 1; khi = 0; }
    else { klo = 1; khi = 1; }
  } else {                               // m1 only reads: partner is the smallest writer
    if (s.w == NONE) return ~0ull;
    thi = s.w; klo = 0; khi = 1;
  }
  return (sf << (2 * wt + 2)) | ((unsigned long long)s.m1 << (wt + 2)) | ((unsigned long long)thi << 2) |
         (klo << 1) | khi;
}

}  // namespace mapk
