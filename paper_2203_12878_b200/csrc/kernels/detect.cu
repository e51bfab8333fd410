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
#include <cstdlib>

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

// ---- warp-streaming detect: registers + shuffles, no shared-memory tiles ----
// Each warp owns a contiguous chunk of DW_CHUNK sorted keys and walks it 32 keys
// per step (coalesced 256-byte loads).  Segment heads come from comparing each
// key's sort field with its left neighbour (shfl_up); every head lane folds its
// segment's (tid, kind) values by gathering the following lanes; the segment
// still open at lane 31 is carried into the next step.  Chunk-spanning
// segments use the same first/last fragment records as the tile version.
constexpr int DW_CHUNK = 4096;
constexpr int DW_WARPS = 8;

__device__ __forceinline__ St shfl_st(const St& s, int src) {
  St o;
  o.m1 = __shfl_sync(0xffffffffu, s.m1, src);
  o.m2 = __shfl_sync(0xffffffffu, s.m2, src);
  o.w = __shfl_sync(0xffffffffu, s.w, src);
  o.k1 = __shfl_sync(0xffffffffu, s.k1, src);
  o.k2 = __shfl_sync(0xffffffffu, s.k2, src);
  return o;
}

__global__ void __launch_bounds__(DW_WARPS * 32)
k_detect_warp(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
              MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid,
              MapcSegState* __restrict__ first_frag, MapcSegState* __restrict__ last_frag) {
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const unsigned long long n_chunks = (n + DW_CHUNK - 1) / DW_CHUNK;
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  unsigned long long best = ~0ull, racy = 0;
  const unsigned long long gw = (unsigned long long)blockIdx.x * DW_WARPS + (threadIdx.x >> 5);
  const unsigned long long nw = (unsigned long long)gridDim.x * DW_WARPS;

  for (unsigned long long c = gw; c < n_chunks; c += nw) {
    const unsigned long long cs = c * DW_CHUNK;
    const unsigned long long ce = min(cs + DW_CHUNK, n);
    // state of the segment open at the start of the step (uniform across lanes)
    St carry;
    st_init(carry);
    unsigned long long carry_sf = 0;
    bool carry_is_first = false;    // carry is the chunk's leading continuation fragment
    bool have_carry = false;
    unsigned long long prev_sf = 0;
    bool has_prev = cs > 0;
    if (has_prev) prev_sf = keys[cs - 1] >> pay_bits;
    if (lane == 0) { first_frag[c].valid = 0; last_frag[c].valid = 0; }
    for (unsigned long long base = cs; base < ce; base += 32) {
      const unsigned long long pos = base + lane;
      const bool valid = pos < ce;
      const unsigned long long key = valid ? ld_stream(keys + pos) : 0ull;
      const unsigned long long sf = key >> pay_bits;
      unsigned long long left = __shfl_up_sync(0xffffffffu, sf, 1);
      if (lane == 0) left = prev_sf;
      const bool head = valid && (((base == cs) && lane == 0) ? (!has_prev || sf != prev_sf) : (sf != left));
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
      const uint32_t hmask = __ballot_sync(0xffffffffu, head);
      // pseudo-heads: real heads plus lane 0 (continuation of the carried segment)
      const uint32_t pmask = hmask | 1u;
      const bool phead = (pmask >> lane) & 1u;
      const uint32_t after = pmask & ~((2u << lane) - 1u) & vmask;     // pseudo-heads after me
      const int nxt = after ? __ffs(after) - 1 : (32 - __clz(vmask));   // end of my run (exclusive)
      St f;
      st_init(f);
      const uint32_t tk = (uint32_t)(key >> 1) & tmask;
      const uint32_t km = 1u << (key & 1u);
      // gather-fold [lane, nxt) for pseudo-head lanes
      int len = phead ? nxt - lane : 0;
      int maxlen = len;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
      for (int o = 0; o < maxlen; ++o) {
        const uint32_t t2 = __shfl_sync(0xffffffffu, tk, (lane + o) & 31);
        const uint32_t k2 = __shfl_sync(0xffffffffu, km, (lane + o) & 31);
        if (o < len) st_add(f, t2, k2);
      }
      const bool lane0_head = hmask & 1u;
      // lane 0's run either continues the carry or starts a new segment
      const St f0 = shfl_st(f, 0);
      if (lane0_head) {
        if (have_carry) {                         // carried segment ended at this step's start
          if (carry_is_first) {
            if (lane == 0) to_frag(&first_frag[c], carry, carry_sf, true);
          } else if (lane == 0) {
            const unsigned long long wv = st_witness(carry, carry_sf, w_tid);
            if (wv != ~0ull) { ++racy; if (wv < best) best = wv; }
          }
        }
        carry = f0;
        carry_sf = __shfl_sync(0xffffffffu, sf, 0);
        carry_is_first = false;
        have_carry = true;
      } else if (vmask & 1u) {
        if (!have_carry) {                        // chunk starts inside a segment
          carry = f0;
          carry_sf = __shfl_sync(0xffffffffu, sf, 0);
          carry_is_first = true;
          have_carry = true;
        } else {
          st_merge(carry, f0);
        }
      }
      // segments headed at lanes > 0: complete ones are finalised here, the last (open) one becomes the carry
      const uint32_t heads_hi = hmask & ~1u;
      const int last_head = heads_hi ? 31 - __clz(heads_hi) : -1;
      if (head && lane > 0 && lane != last_head) {
        const unsigned long long wv = st_witness(f, sf, w_tid);
        if (wv != ~0ull) { ++racy; if (wv < best) best = wv; }
      }
      if (last_head > 0) {
        // the carried segment (lane 0's run) ended before last_head's... if lane 0 did not run to the end
        if (have_carry) {
          if (carry_is_first) {
            if (lane == 0) to_frag(&first_frag[c], carry, carry_sf, true);
          } else if (lane == 0) {
            const unsigned long long wv = st_witness(carry, carry_sf, w_tid);
            if (wv != ~0ull) { ++racy; if (wv < best) best = wv; }
          }
        }
        carry = shfl_st(f, last_head);
        carry_sf = __shfl_sync(0xffffffffu, sf, last_head);
        carry_is_first = false;
        have_carry = true;
      }
      prev_sf = __shfl_sync(0xffffffffu, sf, 31 - __clz(vmask));
    }
    // close the chunk: the carry continues into the next chunk iff its first key has the same sort field
    if (have_carry) {
      const bool cont = ce < n && (keys[ce] >> pay_bits) == carry_sf;
      if (carry_is_first) {
        if (lane == 0) to_frag(&first_frag[c], carry, carry_sf, !cont);
      } else if (cont) {
        if (lane == 0) to_frag(&last_frag[c], carry, carry_sf, false);
      } else if (lane == 0) {
        const unsigned long long wv = st_witness(carry, carry_sf, w_tid);
        if (wv != ~0ull) { ++racy; if (wv < best) best = wv; }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_down_sync(0xffffffffu, best, o);
    const unsigned long long oc = __shfl_down_sync(0xffffffffu, racy, o);
    best = ob < best ? ob : best;
    racy += oc;
  }
  if (lane == 0) {
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

extern "C" unsigned long long mapc_detect_tile() { return mapk::DW_CHUNK < mapk::DT_TILE ? mapk::DW_CHUNK : mapk::DT_TILE; }

extern "C" cudaError_t mapc_launch_chunk_init(MapcCtrl* ctrl, unsigned long long n0, cudaStream_t s) {
  mapk::k_chunk_init<<<1, 256, 0, s>>>(ctrl, n0);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_detect(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                                          uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid, MapcSegState* first_frag,
                                          MapcSegState* last_frag, unsigned long long max_keys, int n_sms,
                                          cudaStream_t s) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("MAPC_DETECT");
    mode = e ? atoi(e) : 0;
  }
  const unsigned tile = mode == 1 ? (unsigned)mapk::DW_CHUNK : (unsigned)mapk::DT_TILE;
  unsigned long long tiles = (max_keys + tile - 1) / tile;
  if (mode == 1) {
    unsigned long long blocks = (tiles + mapk::DW_WARPS - 1) / mapk::DW_WARPS;
    unsigned long long cap = (unsigned long long)n_sms * 8;
    int grid = (int)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
    mapk::k_detect_warp<<<grid, mapk::DW_WARPS * 32, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid, first_frag,
                                                            last_frag);
  } else {
    unsigned long long cap = (unsigned long long)n_sms * 8;
    int grid = (int)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
    mapk::k_detect<<<grid, mapk::DT_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid, first_frag, last_frag);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int g2 = (int)((tiles + 255) / 256);
  if (g2 < 1) g2 = 1;
  if (g2 > n_sms * 4) g2 = n_sms * 4;
  mapk::k_detect_fixup<<<g2, 256, 0, s>>>(ctrl, w_tid, first_frag, last_frag, tile);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_chunk_finish(const MapcCtrl* ctrl, uint32_t n_passes, MapcChunkResult* out,
                                                cudaStream_t s) {
  mapk::k_chunk_finish<<<1, 1, 0, s>>>(ctrl, n_passes, out);
  return cudaGetLastError();
}
