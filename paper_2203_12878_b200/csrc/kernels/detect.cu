// detect.cu -- K4/K5: segmented conflict scan over sorted keys + min witness.
//
// A segment is a maximal run of keys with equal sort field, i.e. all access
// values of one (phase, array, block, index) cell.  A segment is racy iff it
// holds two DISTINCT tids and at least one write (
// SPEC.md:423-426, 490), i.e. iff it holds a write and min tid != max tid.
//
// Pass 1 (k_detect + k_detect_fixup) folds only (has write, min tid, max tid)
// per segment, counts racy segments and keeps the smallest racy sort field.
// The canonical witness order is lexicographic with the sort field first, so
// the witness lies in that one segment: pass 2 (k_witness, one CTA) folds the
// full order-independent state (m1, k1, m2, k2, w) over it -- smallest tid and
// its kind mask, second smallest distinct tid and its mask, smallest writer --
// whose witness has a closed form: t_lo = m1; if m1 writes,
// t_hi = m2 with kinds the first feasible of (rd,wr),(wr,rd),(wr,wr), else
// t_hi = w with kinds (rd,wr).  Nothing depends on launch or arrival order.
//
// Segments spanning tiles: each tile records the state of its leading
// continuation fragment and of its trailing open segment; k_detect_fixup lets
// the tile that owns an open segment's head fold the following fragments.
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

// ---- pass 1: racy test per segment ------------------------------------------
// racy(segment) <=> it holds a write and two distinct tids <=> it holds a write
// and two ADJACENT keys with different tids (if all adjacent tids agree, all
// agree).  A CTA stages a tile of sorted keys in shared memory; each head
// position folds (first tid, last tid, adjacent-diff, write) over its segment,
// counts racy segments and keeps the smallest racy sort field (keys are sorted,
// and the witness order is lexicographic with the sort field first).
constexpr int DW_CHUNK = 4096;          // keys per tile (and per fragment record)
constexpr int DT_THREADS = 256;

struct Frag {
  uint32_t first_tid, last_tid, wr, diff;
  unsigned long long sf;
};

__device__ __forceinline__ void put_frag(MapcSegState* f, const Frag& c, bool ends) {
  MapcSegState o;
  o.first_tid = c.first_tid; o.last_tid = c.last_tid;
  o.wr = (uint8_t)(c.wr != 0); o.diff = (uint8_t)(c.diff != 0);
  o.valid = 1; o.ends = ends ? 1 : 0;
  o.sf = c.sf;
  *f = o;
}

__global__ void __launch_bounds__(DT_THREADS)
k_detect(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
         MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid,
         MapcSegState* __restrict__ first_frag, MapcSegState* __restrict__ last_frag) {
  __shared__ unsigned long long K[DW_CHUNK + 2];
  __shared__ unsigned long long red_s[DT_THREADS / 32];
  __shared__ unsigned long long red_c[DT_THREADS / 32];
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const unsigned long long n_tiles = (n + DW_CHUNK - 1) / DW_CHUNK;
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  unsigned long long best = ~0ull, racy = 0;

  for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const unsigned long long tb = tile * DW_CHUNK;
    const uint32_t tn = (uint32_t)min((unsigned long long)DW_CHUNK, n - tb);
    for (uint32_t i = threadIdx.x; i < tn; i += DT_THREADS) K[i + 1] = ld_stream(keys + tb + i);
    if (threadIdx.x == 0) {
      K[0] = tb > 0 ? keys[tb - 1] : 0ull;
      K[tn + 1] = tb + tn < n ? keys[tb + tn] : 0ull;
      first_frag[tile].valid = 0;
      last_frag[tile].valid = 0;
    }
    __syncthreads();
    const bool has_prev = tb > 0, has_next = tb + tn < n;
    const unsigned long long sf_next = K[tn + 1] >> pay_bits;
    for (uint32_t i = threadIdx.x; i < tn; i += DT_THREADS) {
      const unsigned long long key0 = K[i + 1];
      const unsigned long long sf = key0 >> pay_bits;
      const bool head = (i == 0) ? (!has_prev || (K[0] >> pay_bits) != sf) : ((K[i] >> pay_bits) != sf);
      if (!head && i != 0) continue;
      Frag f;
      f.first_tid = f.last_tid = (uint32_t)(key0 >> 1) & tmask;
      f.wr = (uint32_t)key0 & 1u;
      f.diff = 0;
      f.sf = sf;
      uint32_t j = i + 1;
      for (; j < tn; ++j) {
        const unsigned long long key = K[j + 1];
        if ((key >> pay_bits) != sf) break;
        const uint32_t t = (uint32_t)(key >> 1) & tmask;
        f.diff |= (uint32_t)(t != f.last_tid);
        f.last_tid = t;
        f.wr |= (uint32_t)key & 1u;
      }
      const bool ends = j < tn || !has_next || sf_next != sf;
      if (head && ends) {
        if (f.wr && f.diff) { ++racy; best = min(best, sf); }
      } else if (head) {
        put_frag(&last_frag[tile], f, false);
      } else {
        put_frag(&first_frag[tile], f, ends);
      }
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    best = min(best, __shfl_down_sync(0xffffffffu, best, o));
    racy += __shfl_down_sync(0xffffffffu, racy, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { red_s[w] = best; red_c[w] = racy; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < DT_THREADS / 32; ++i) { best = min(best, red_s[i]); racy += red_c[i]; }
    if (best != ~0ull) atomicMin(&ctrl->racy_sf, best);
    if (racy) atomicAdd(&ctrl->racy, racy);
  }
}

// One thread per chunk that owns an open segment head: fold continuation fragments.
__global__ void k_detect_fixup(MapcCtrl* __restrict__ ctrl, const MapcSegState* __restrict__ first_frag,
                               const MapcSegState* __restrict__ last_frag, uint32_t chunk) {
  const unsigned long long n = ctrl->n;
  const unsigned long long n_chunks = (n + chunk - 1) / chunk;
  unsigned long long best = ~0ull, racy = 0;
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < n_chunks;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const MapcSegState lf = last_frag[t];
    if (!lf.valid) continue;
    uint32_t wr = lf.wr, diff = lf.diff, last = lf.last_tid;
    for (unsigned long long u = t + 1; u < n_chunks; ++u) {
      const MapcSegState ff = first_frag[u];
      if (!ff.valid || ff.sf != lf.sf) { atomicOr(&ctrl->err, MAPC_ERR_LAYOUT); break; }
      diff |= ff.diff | (uint32_t)(ff.first_tid != last);
      wr |= ff.wr;
      last = ff.last_tid;
      if (ff.ends) break;
    }
    if (wr && diff) { ++racy; best = min(best, lf.sf); }
  }
  if (best != ~0ull) atomicMin(&ctrl->racy_sf, best);
  if (racy) atomicAdd(&ctrl->racy, racy);
}

// ---- pass 2: canonical witness of the first racy segment ----------------------
// One CTA: lower_bound of the segment in the sorted keys, then a parallel fold
// of the full state (m1, k1, m2, k2, w) over the segment, closed-form witness.
constexpr int WT_THREADS = 256;
__global__ void __launch_bounds__(WT_THREADS)
k_witness(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
          MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid) {
  const unsigned long long target = ctrl->racy_sf;
  if (target == ~0ull) return;
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  __shared__ unsigned long long s_lo;
  __shared__ St part[WT_THREADS];
  if (threadIdx.x == 0) {
    unsigned long long lo = 0, hi = n;                  // first index with sf >= target
    while (lo < hi) {
      const unsigned long long mid = (lo + hi) >> 1;
      if ((keys[mid] >> pay_bits) < target) lo = mid + 1; else hi = mid;
    }
    s_lo = lo;
  }
  __syncthreads();
  St s;
  st_init(s);
  for (unsigned long long i = s_lo + threadIdx.x; i < n; i += WT_THREADS) {
    const unsigned long long key = keys[i];
    if ((key >> pay_bits) != target) break;
    st_add(s, (uint32_t)(key >> 1) & tmask, 1u << (key & 1u));
  }
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < WT_THREADS; ++t) st_merge(s, part[t]);
    ctrl->witness = st_witness(s, target, w_tid);
  }
}

__global__ void k_chunk_init(MapcCtrl* __restrict__ ctrl, unsigned long long n0) {
  unsigned int* p = reinterpret_cast<unsigned int*>(ctrl);
  const int words = (int)(sizeof(MapcCtrl) / 4);
  for (int i = threadIdx.x; i < words; i += blockDim.x) p[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->witness = ~0ull;
    ctrl->racy_sf = ~0ull;
    ctrl->n = n0;            // dense keys are placed directly; compaction appends after them
  }
}

__global__ void k_chunk_finish(const MapcCtrl* __restrict__ ctrl, uint32_t n_passes, MapcChunkResult* __restrict__ out) {
  MapcChunkResult r;
  r.n = ctrl->n;
  r.witness = ctrl->witness;
  r.racy = ctrl->racy;
  r.err = ctrl->err;
  r.active_passes = 0;
  for (uint32_t p = 0; p < n_passes; ++p) r.active_passes += ctrl->active[p] ? 1u : 0u;
  *out = r;
}

}  // namespace mapk

extern "C" unsigned long long mapc_detect_tile() { return mapk::DW_CHUNK; }

extern "C" cudaError_t mapc_launch_chunk_init(MapcCtrl* ctrl, unsigned long long n0, cudaStream_t s) {
  mapk::k_chunk_init<<<1, 256, 0, s>>>(ctrl, n0);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_detect(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                                          uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid, MapcSegState* first_frag,
                                          MapcSegState* last_frag, unsigned long long max_keys, int n_sms,
                                          cudaStream_t s) {
  const unsigned long long tiles = (max_keys + mapk::DW_CHUNK - 1) / mapk::DW_CHUNK;
  const unsigned long long cap = (unsigned long long)n_sms * 8;
  const int grid = (int)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
  mapk::k_detect<<<grid, mapk::DT_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid, first_frag, last_frag);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int g2 = (int)((tiles + 255) / 256);
  if (g2 < 1) g2 = 1;
  if (g2 > n_sms * 4) g2 = n_sms * 4;
  mapk::k_detect_fixup<<<g2, 256, 0, s>>>(ctrl, first_frag, last_frag, (unsigned)mapk::DW_CHUNK);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mapk::k_witness<<<1, mapk::WT_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_chunk_finish(const MapcCtrl* ctrl, uint32_t n_passes, MapcChunkResult* out,
                                                cudaStream_t s) {
  mapk::k_chunk_finish<<<1, 1, 0, s>>>(ctrl, n_passes, out);
  return cudaGetLastError();
}
