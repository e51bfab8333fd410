// detect.cu -- K4/K5: segmented conflict scan over sorted keys + min witness.
//
// A segment is a maximal run of keys with equal sort field, i.e. all access
// values of one (phase, array, block, index) cell.  A segment is racy iff it
// holds two DISTINCT tids and at least one write (
// SPEC.md:423-426, 490).  Per segment the kernel folds an order-independent
// state (m1, k1, m2, k2, w): smallest tid and its kind mask, second smallest
// distinct tid and its mask, smallest writer tid.  Its canonical witness has a
// closed form: t_lo = m1 always; if m1 writes, t_hi = m2 with
// kinds the first feasible of (rd,wr),(wr,rd),(wr,wr); otherwise t_hi = w with
// kinds (rd,wr).  Witnesses are packed so that unsigned order = lexicographic
// order and combined with atomicMin, so the result does not depend on launch
// or arrival order.
//
// Segments spanning tiles: each tile records the state of its leading
// continuation fragment and of its trailing open segment; k_detect_fixup lets
// the tile that owns an open segment's head fold the following fragments.
#include "common.cuh"

namespace mapk {

constexpr int DT_THREADS = 256;
constexpr int DT_ITEMS = 16;
constexpr int DT_TILE = DT_THREADS * DT_ITEMS;
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

__device__ __forceinline__ void to_frag(MapcSegState* f, const St& s, unsigned long long sf, bool ends) {
  MapcSegState o;
  o.m1 = s.m1; o.m2 = s.m2; o.w = s.w;
  o.k1 = (uint8_t)s.k1; o.k2 = (uint8_t)s.k2;
  o.valid = 1; o.ends = ends ? 1 : 0;
  o.sf = sf;
  *f = o;
}

__device__ __forceinline__ St from_frag(const MapcSegState& f) {
  St s;
  s.m1 = f.m1; s.m2 = f.m2; s.w = f.w; s.k1 = f.k1; s.k2 = f.k2;
  return s;
}

__global__ void __launch_bounds__(DT_THREADS)
k_detect(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
         MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid,
         MapcSegState* __restrict__ first_frag, MapcSegState* __restrict__ last_frag) {
  __shared__ unsigned long long K[DT_TILE + 2];
  __shared__ unsigned long long red_w[DT_THREADS / 32];
  __shared__ unsigned long long red_c[DT_THREADS / 32];
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const unsigned long long n_tiles = (n + DT_TILE - 1) / DT_TILE;
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  unsigned long long best = ~0ull, racy = 0;

  for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const unsigned long long tb = tile * DT_TILE;
    const uint32_t tn = (uint32_t)min((unsigned long long)DT_TILE, n - tb);
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
    // thread-strided positions: a warp touches consecutive shared-memory words
    for (uint32_t i = threadIdx.x; i < tn; i += DT_THREADS) {
      const unsigned long long sf = K[i + 1] >> pay_bits;
      const bool head = (i == 0) ? (!has_prev || (K[0] >> pay_bits) != sf) : ((K[i] >> pay_bits) != sf);
      if (!head && i != 0) continue;
      St s;
      st_init(s);
      uint32_t j = i;
      for (; j < tn; ++j) {
        const unsigned long long key = K[j + 1];
        if ((key >> pay_bits) != sf) break;
        st_add(s, (uint32_t)(key >> 1) & tmask, 1u << (key & 1u));
      }
      const bool ends = j < tn || !has_next || sf_next != sf;
      if (head && ends) {
        const unsigned long long wv = st_witness(s, sf, w_tid);
        if (wv != ~0ull) { ++racy; if (wv < best) best = wv; }
      } else if (head) {
        to_frag(&last_frag[tile], s, sf, false);
      } else {
        to_frag(&first_frag[tile], s, sf, ends);
      }
    }
    __syncthreads();
  }
  // block reduction: min witness, sum of racy segments
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_down_sync(0xffffffffu, best, o);
    const unsigned long long oc = __shfl_down_sync(0xffffffffu, racy, o);
    best = ob < best ? ob : best;
    racy += oc;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { red_w[w] = best; red_c[w] = racy; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < DT_THREADS / 32; ++i) { best = red_w[i] < best ? red_w[i] : best; racy += red_c[i]; }
    if (best != ~0ull) atomicMin(&ctrl->witness, best);
    if (racy) atomicAdd(&ctrl->racy, racy);
  }
}

// One thread per tile that owns an open segment head: fold continuation fragments.
__global__ void k_detect_fixup(MapcCtrl* __restrict__ ctrl, uint32_t w_tid, const MapcSegState* __restrict__ first_frag,
                               const MapcSegState* __restrict__ last_frag, uint32_t tile) {
  const unsigned long long n = ctrl->n;
  const unsigned long long n_tiles = (n + tile - 1) / tile;
  unsigned long long best = ~0ull, racy = 0;
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const MapcSegState lf = last_frag[t];
    if (!lf.valid) continue;
    St s = from_frag(lf);
    for (unsigned long long u = t + 1; u < n_tiles; ++u) {
      const MapcSegState ff = first_frag[u];
      if (!ff.valid || ff.sf != lf.sf) { atomicOr(&ctrl->err, MAPC_ERR_LAYOUT); break; }
      st_merge(s, from_frag(ff));
      if (ff.ends) break;
    }
    const unsigned long long wv = st_witness(s, lf.sf, w_tid);
    if (wv != ~0ull) { ++racy; if (wv < best) best = wv; }
  }
  if (best != ~0ull) atomicMin(&ctrl->witness, best);
  if (racy) atomicAdd(&ctrl->racy, racy);
}

__global__ void k_chunk_init(MapcCtrl* __restrict__ ctrl, unsigned long long n0) {
  unsigned int* p = reinterpret_cast<unsigned int*>(ctrl);
  const int words = (int)(sizeof(MapcCtrl) / 4);
  for (int i = threadIdx.x; i < words; i += blockDim.x) p[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->witness = ~0ull;
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

extern "C" unsigned long long mapc_detect_tile() { return mapk::DT_TILE; }

extern "C" cudaError_t mapc_launch_chunk_init(MapcCtrl* ctrl, unsigned long long n0, cudaStream_t s) {
  mapk::k_chunk_init<<<1, 256, 0, s>>>(ctrl, n0);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_detect(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                                          uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid, MapcSegState* first_frag,
                                          MapcSegState* last_frag, unsigned long long max_keys, int n_sms,
                                          cudaStream_t s) {
  const unsigned long long tiles = (max_keys + mapk::DT_TILE - 1) / mapk::DT_TILE;
  const unsigned long long cap = (unsigned long long)n_sms * 8;
  const int grid = (int)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
  mapk::k_detect<<<grid, mapk::DT_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid, first_frag, last_frag);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int g2 = (int)((tiles + 255) / 256);
  if (g2 < 1) g2 = 1;
  if (g2 > n_sms * 4) g2 = n_sms * 4;
  mapk::k_detect_fixup<<<g2, 256, 0, s>>>(ctrl, w_tid, first_frag, last_frag, (unsigned)mapk::DT_TILE);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_chunk_finish(const MapcCtrl* ctrl, uint32_t n_passes, MapcChunkResult* out,
                                                cudaStream_t s) {
  mapk::k_chunk_finish<<<1, 1, 0, s>>>(ctrl, n_passes, out);
  return cudaGetLastError();
}
