// rsweep.cu -- look-back-free LSD radix passes over static key ranges.
//
// Each radix pass is still ONE launch that reads and writes every key once
// (16 B per key), ranks a tile in shared memory and scatters runs of equal
// digit -- but the inter-tile prefix comes from a per-range histogram instead
// of a decoupled look-back (measured as the limiter of the radix pass on B200,
// DESIGN.md §6.1):
//   * CTA c of G owns the contiguous key range [c*L, (c+1)*L) (L a multiple of
//     the tile), walks its tiles in order and keeps running per-digit output
//     cursors, so the pass is stable;
//   * its starting cursors are base[c][d] = offs[d] + sum_{c' < c} rhist[c'][d],
//     where rhist[c'][d] counts the keys of range c' with digit d;
//   * rhist for the NEXT active pass is accumulated by this pass's scatter:
//     every key's output position fixes its next-pass range, so the CTA counts
//     (position / L, next digit) in a G x 256 shared-memory table and flushes it
//     once at the end.  The first pass's table comes from k_hist_ranges.
#include <cstdlib>

#include "common.cuh"

namespace mapk {

constexpr int RS_TILE = 4096;        // range lengths are multiples of this
constexpr int RH_THREADS = 1024;

__device__ __forceinline__ uint32_t range_len(unsigned long long n, uint32_t G) {
  unsigned long long per = (n + G - 1) / G;
  per = (per + RS_TILE - 1) / RS_TILE * RS_TILE;
  return (uint32_t)(per ? per : RS_TILE);
}

__device__ MapcFastDiv dev_fastdiv(uint32_t d) {
  MapcFastDiv f;
  f.d = d ? d : 1u;
  d = f.d;
  const uint32_t l = 31 - __clz(d);
  if ((d & (d - 1)) == 0) { f.pow2 = 1; f.s = l; f.m = 0; return f; }
  // m = floor(2^32 * (2^(l+1) - d) / d) + 1
  const unsigned long long num_hi = ((1ull << (l + 1)) - d);        // times 2^32
  const unsigned long long q = (num_hi << 32) / d;                     // fits: num_hi < d*2
  f.m = (uint32_t)(q + 1);
  f.s = l;
  f.pow2 = 0;
  return f;
}

// Global digit histograms of all passes + the per-range table of pass 0.
// Grid = G CTAs; CTA c reads exactly its range.
__global__ void __launch_bounds__(RH_THREADS)
k_hist_ranges(const unsigned long long* __restrict__ keys, MapcCtrl* __restrict__ ctrl, unsigned int* __restrict__ rhist0,
              uint32_t pay_bits, uint32_t n_passes) {
  __shared__ uint32_t h[MAPC_MAX_PASSES][MAPC_RADIX];
  for (int i = threadIdx.x; i < MAPC_MAX_PASSES * MAPC_RADIX; i += RH_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  const unsigned long long n = ctrl->n;
  const uint32_t G = gridDim.x;
  const uint32_t L = range_len(n, G);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctrl->rng_L = L;
    ctrl->rng_div = dev_fastdiv(L);
  }
  const unsigned long long r0 = (unsigned long long)blockIdx.x * L;
  const unsigned long long r1 = min(r0 + L, n);
  if (r0 < r1) {
    const unsigned long long cnt = r1 - r0;
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys + r0);   // r0 % 2 == 0
    const unsigned long long n2 = cnt >> 1;
    constexpr int U = 4;                                 // loads in flight per thread
    unsigned long long i = threadIdx.x;
    for (; i + (U - 1) * RH_THREADS < n2; i += U * RH_THREADS) {
      ulonglong2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream2(k2 + i + u * RH_THREADS);
#pragma unroll
      for (int u = 0; u < U; ++u)
        for (uint32_t p = 0; p < n_passes; ++p) {
          atomicAdd(&h[p][(v[u].x >> (pay_bits + 8 * p)) & 0xFF], 1u);
          atomicAdd(&h[p][(v[u].y >> (pay_bits + 8 * p)) & 0xFF], 1u);
        }
    }
    for (; i < n2; i += RH_THREADS) {
      const ulonglong2 v = ld_stream2(k2 + i);
      for (uint32_t p = 0; p < n_passes; ++p) {
        atomicAdd(&h[p][(v.x >> (pay_bits + 8 * p)) & 0xFF], 1u);
        atomicAdd(&h[p][(v.y >> (pay_bits + 8 * p)) & 0xFF], 1u);
      }
    }
    if ((cnt & 1) && threadIdx.x == 0) {
      const unsigned long long v = keys[r1 - 1];
      for (uint32_t p = 0; p < n_passes; ++p) atomicAdd(&h[p][(v >> (pay_bits + 8 * p)) & 0xFF], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)n_passes * MAPC_RADIX; i += RH_THREADS) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&(&ctrl->hist[0][0])[i], c);
  }
  if (threadIdx.x < MAPC_RADIX) rhist0[blockIdx.x * MAPC_RADIX + threadIdx.x] = h[0][threadIdx.x];
}

// Per-range table of pass p, read from the pass's input buffer (pass 0's table
// comes from k_hist_ranges).  Used when the scatter does not fuse the next
// pass's table (2 CTAs per SM).
// Per-range table of pass p, read from the pass's input buffer (pass 0's table
// comes from k_hist_ranges; fused variants get later tables from the scatter).
__global__ void __launch_bounds__(RH_THREADS)
k_range_hist(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
             MapcCtrl* __restrict__ ctrl, unsigned int* __restrict__ rhist, uint32_t p, uint32_t pay_bits,
             uint32_t fused) {
  if (p == 0 || !ctrl->active[p]) return;
  if (ctrl->rt_done[p] && !ctrl->rt_bad[p]) return;  // accumulated by the previous pass's scatter
  (void)fused;
  const unsigned long long* __restrict__ keys = ctrl->sel[p] ? bufB : bufA;
  __shared__ uint32_t h[MAPC_RADIX];
  for (int i = threadIdx.x; i < MAPC_RADIX; i += RH_THREADS) h[i] = 0;
  __syncthreads();
  const unsigned long long n = ctrl->n;
  const uint32_t L = ctrl->rng_L;
  const unsigned long long r0 = (unsigned long long)blockIdx.x * L;
  const unsigned long long r1 = min(r0 + L, n);
  const uint32_t sh = pay_bits + 8 * p;
  if (r0 < r1) {
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys + r0);
    const unsigned long long n2 = (r1 - r0) >> 1;
    constexpr int U = 4;                                 // loads in flight per thread
    for (unsigned long long i0 = threadIdx.x; i0 < n2; i0 += U * RH_THREADS) {
      ulonglong2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned long long i = i0 + u * RH_THREADS;
        v[u] = i < n2 ? ld_stream2(k2 + i) : make_ulonglong2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u * RH_THREADS >= n2) break;
        atomicAdd(&h[(v[u].x >> sh) & 0xFF], 1u);
        atomicAdd(&h[(v[u].y >> sh) & 0xFF], 1u);
      }
    }
    if (((r1 - r0) & 1) && threadIdx.x == 0) atomicAdd(&h[(keys[r1 - 1] >> sh) & 0xFF], 1u);
  }
  __syncthreads();
  if (threadIdx.x < MAPC_RADIX)
    rhist[((size_t)p * MAPC_MAX_RANGES + blockIdx.x) * MAPC_RADIX + threadIdx.x] = h[threadIdx.x];
}

// Tile buffer index with one 8-byte pad slot per 16 keys: digit regions of a
// tile start ~16 keys (128 B = one full bank cycle) apart, so an unpadded
// scatter puts the lanes of a warp into the same bank (measured: ~16
// wavefronts per STS.64, 80% of the shared-memory pipe).
__device__ __forceinline__ uint32_t kslot(uint32_t p) { return p + (p >> 4); }

template <int THREADS, int ITEMS>
struct RsSmem {
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr int WARPS = THREADS / 32;
  unsigned long long keys[TILE + TILE / 16];
  uint32_t pos[WARPS][MAPC_RADIX];                 // running tile position per (warp, digit)
  uint32_t mask[WARPS][MAPC_RADIX];                // early counts, then peer masks
  unsigned long long running[MAPC_RADIX];          // global output cursor per digit
  unsigned long long gbase[MAPC_RADIX];           // output index of tile position 0 for digit d
  unsigned long long gaddr[MAPC_RADIX];           // the same as a byte address in dst (mod 2^64)
  uint32_t scan_tmp[WARPS + 1];
};

// RED_NEXT: the scatter also accumulates the NEXT active pass's range table:
// an output position fixes its range, so each warp row of 32 consecutive
// outputs adds (range, next digit) to rhist -- once, +32, when the row is
// uniform (bucket digits of dense MAPs: the common case), else per key.  A CTA
// whose rows turn out mostly non-uniform abandons (rt_bad) and k_range_hist
// recomputes the table from one read, as without fusion.
template <int THREADS, int ITEMS, bool RED_NEXT, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
k_rsweep(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
         unsigned int* __restrict__ rhist, uint32_t pass, uint32_t pay_bits) {
  using Sm = RsSmem<THREADS, ITEMS>;
  constexpr int TILE = Sm::TILE, WARPS = Sm::WARPS;
  if (!ctrl->active[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sm& S = *reinterpret_cast<Sm*>(smem_raw);
  const uint32_t shift = pay_bits + 8 * pass;
  const uint32_t nxt = ctrl->next_active[pass];
  bool fuse_on = RED_NEXT && nxt < MAPC_MAX_PASSES && !ctrl->rt_bad[nxt];
  unsigned int* __restrict__ next_tab = rhist + (size_t)(nxt < MAPC_MAX_PASSES ? nxt : 0) * MAPC_MAX_RANGES * MAPC_RADIX;
  if (RED_NEXT && fuse_on && blockIdx.x == 0 && threadIdx.x == 0) ctrl->rt_done[nxt] = 1;
  uint32_t rows = 0, nonuni = 0;
  uint32_t vcur = 0xFFFFFFFFu, vcnt = 0;                 // warp-uniform running (range, next digit) count
  const uint32_t nshift = pay_bits + 8 * (nxt < MAPC_MAX_PASSES ? nxt : 0);
  const unsigned long long* __restrict__ src = ctrl->sel[pass] ? bufB : bufA;
  unsigned long long* __restrict__ dst = ctrl->sel[pass] ? bufA : bufB;
  const unsigned long long n = ctrl->n;
  const uint32_t L = ctrl->rng_L;
  const MapcFastDiv rdiv = ctrl->rng_div;
  bool stable = false;                                   // first active pass: any order of equal digits
  for (uint32_t q = 0; q < pass; ++q) stable |= ctrl->active[q] != 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t wbase = (uint32_t)w * ITEMS * 32;
  const unsigned long long r0 = (unsigned long long)blockIdx.x * L;
  const unsigned long long r1 = min(r0 + L, n);

  if (threadIdx.x < MAPC_RADIX) {
    const int d = threadIdx.x;
    const unsigned int* col = rhist + (size_t)pass * MAPC_MAX_RANGES * MAPC_RADIX + d;
    uint32_t acc[4] = {0, 0, 0, 0};
    uint32_t c = 0;
    for (; c + 4 <= blockIdx.x; c += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += col[(size_t)(c + u) * MAPC_RADIX];
    for (; c < blockIdx.x; ++c) acc[0] += col[(size_t)c * MAPC_RADIX];
    S.running[d] = ctrl->offs[pass][d] + acc[0] + acc[1] + acc[2] + acc[3];
  }
  auto load_tile = [&](unsigned long long tb, unsigned long long* kk) {
    if (tb >= r1) return;
    const uint32_t tn = (uint32_t)min((unsigned long long)TILE, r1 - tb);
    if (tn == TILE) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) kk[j] = ld_stream(src + tb + wbase + j * 32 + lane);
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t li = wbase + j * 32 + lane;
        kk[j] = li < tn ? ld_stream(src + tb + li) : 0ull;
      }
    }
  };
  unsigned long long k[ITEMS];
  load_tile(r0, k);
  const uint32_t lt = lanemask_lt();
  // the per-(warp, digit) words hold early counts, then peer masks; ranking
  // leaves them zero, so they are cleared once here, not per tile
  for (int i = threadIdx.x; i < WARPS * MAPC_RADIX; i += THREADS) (&S.mask[0][0])[i] = 0;
  __syncthreads();
  static_assert(MAPC_RADIX == 256 && THREADS >= MAPC_RADIX, "one thread per digit in the tile scan");
  for (unsigned long long tb = r0; tb < r1; tb += TILE) {
    const uint32_t tile_n = (uint32_t)min((unsigned long long)TILE, r1 - tb);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (wbase + j * 32 + lane < tile_n) atomicAdd(&S.mask[w][(uint32_t)(k[j] >> shift) & 0xFFu], 1u);
    __syncthreads();
    // tile scan: thread d < 256 owns digit d; 8 warps scan 32 digits each
    uint32_t count = 0, incl = 0;
    uint32_t wpre[WARPS];
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww) {
        wpre[ww] = count;
        count += S.mask[ww][d];
      }
      incl = warp_incl_scan(count);
      if (lane == 31) S.scan_tmp[w] = incl;
    }
    __syncthreads();
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
      uint32_t dex = incl - count;
      for (int ww = 0; ww < w; ++ww) dex += S.scan_tmp[ww];
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww) {
        S.pos[ww][d] = dex + wpre[ww];
        S.mask[ww][d] = 0;
      }
      S.gbase[d] = S.running[d] - dex;
      S.gaddr[d] = reinterpret_cast<unsigned long long>(dst) + 8ull * (S.running[d] - dex);
      S.running[d] += count;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const bool valid = wbase + j * 32 + lane < tile_n;
      const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
      if (vmask == 0) continue;
      const int first = __ffs(vmask) - 1;
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, first);
      if (__all_sync(0xffffffffu, !valid || d == d0)) {
        const uint32_t v = S.pos[w][d0];
        __syncwarp();
        if (valid) S.keys[kslot(v + __popc(vmask & lt))] = k[j];
        if (lane == first) S.pos[w][d0] = v + __popc(vmask);
        __syncwarp();
      } else if (!stable) {
        if (valid) S.keys[kslot(atomicAdd(&S.pos[w][d], 1u))] = k[j];
        __syncwarp();
      } else {
        if (valid) atomicOr(&S.mask[w][d], 1u << lane);
        __syncwarp();
        const uint32_t peers = S.mask[w][d];
        const uint32_t v = S.pos[w][d];
        __syncwarp();
        const uint32_t before = peers & lt;
        if (valid) {
          if (before == 0) { S.pos[w][d] = v + __popc(peers); S.mask[w][d] = 0; }
          S.keys[kslot(v + __popc(before))] = k[j];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    load_tile(tb + TILE, k);                             // in flight during the write-out
    if (tile_n == TILE) {
      // full tile: key i of the tile goes to byte address gaddr[digit] + 8 i
#pragma unroll
      for (int u = 0; u < ITEMS; ++u) {
        const uint32_t i = u * THREADS + threadIdx.x;
        const unsigned long long key = S.keys[kslot(i)];
        const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
        const unsigned long long a = S.gaddr[d] + 8ull * i;
        *reinterpret_cast<unsigned long long*>(a) = key;
        if (RED_NEXT && fuse_on) {
          const uint32_t pidx = (uint32_t)((a - reinterpret_cast<unsigned long long>(dst)) >> 3);
          const uint32_t v = (fastdiv(pidx, rdiv) << 8) | ((uint32_t)(key >> nshift) & 0xFFu);
          const uint32_t v0 = __shfl_sync(0xffffffffu, v, 0);
          ++rows;
          if (__all_sync(0xffffffffu, v == v0)) {     // uniform row: into the warp's running entry
            if (v0 != vcur) {
              if (vcnt && lane == 0) atomicAdd(&next_tab[vcur], vcnt);
              vcur = v0;
              vcnt = 0;
            }
            vcnt += 32;
          } else {
            atomicAdd(&next_tab[v], 1u);
            ++nonuni;
          }
        }
      }
    } else {
      for (uint32_t i = threadIdx.x; i < tile_n; i += THREADS) {
        const unsigned long long key = S.keys[kslot(i)];
        const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
        const unsigned long long p = S.gbase[d] + i;
        dst[p] = key;
        if (RED_NEXT && fuse_on)
          atomicAdd(&next_tab[(fastdiv((uint32_t)p, rdiv) << 8) | ((uint32_t)(key >> nshift) & 0xFFu)], 1u);
      }
    }
    if (RED_NEXT && fuse_on && nonuni > 8 + rows / 8) {   // mostly non-uniform rows: give the table up
      fuse_on = false;
      atomicOr(&ctrl->rt_bad[nxt], 1u);
    }
  }
  if (RED_NEXT && vcnt && lane == 0) atomicAdd(&next_tab[vcur], vcnt);
}

struct RsVariant {
  const void* fn;          // plain pass
  const void* fn_next;     // pass that also accumulates the next pass's range table
  int threads;
  size_t smem;
  int per_sm;
};

template <int T, int I, int B>
RsVariant rs_variant() {
  return RsVariant{(const void*)k_rsweep<T, I, false, B>, (const void*)k_rsweep<T, I, true, B>, T,
                   sizeof(RsSmem<T, I>), B};
}

RsVariant rs_pick() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MAPC_RS_VARIANT");
    v = e ? atoi(e) : 7;
  }
  // 7 (default): 256 threads x 12 keys, 4 CTAs/SM (592 ranges) -- measured best
  //    on B200 (5.46 TB/s per pass on 5a vs 4.83 for 2: 512 x 8, 2 CTAs/SM)
  if (v == 2) return rs_variant<512, 8, 2>();
  if (v == 3) return rs_variant<512, 12, 2>();
  if (v == 6) return rs_variant<256, 8, 4>();
  return rs_variant<256, 12, 4>();
}

}  // namespace mapk

extern "C" unsigned long long mapc_rsweep_tile() { return mapk::RS_TILE; }

extern "C" int mapc_rsweep_ranges(int n_sms) {
  const int g = n_sms * mapk::rs_pick().per_sm;
  return g < MAPC_MAX_RANGES ? g : MAPC_MAX_RANGES;
}

extern "C" cudaError_t mapc_launch_hist_ranges(const unsigned long long* keys, MapcCtrl* ctrl, unsigned int* rhist,
                                               uint32_t pay_bits, uint32_t n_passes, int G, cudaStream_t s) {
  mapk::k_hist_ranges<<<G, mapk::RH_THREADS, 0, s>>>(keys, ctrl, rhist, pay_bits, n_passes);
  return cudaGetLastError();
}

// Per-pass range table when the variant does not fuse it into the previous scatter.
extern "C" cudaError_t mapc_launch_range_hist(const unsigned long long* bufA, const unsigned long long* bufB,
                                              MapcCtrl* ctrl, unsigned int* rhist, uint32_t pass, uint32_t pay_bits,
                                              int G, cudaStream_t s) {
  mapk::k_range_hist<<<G, mapk::RH_THREADS, 0, s>>>(bufA, bufB, ctrl, rhist, pass, pay_bits, 0u);
  return cudaGetLastError();
}

extern "C" int mapc_rsweep_fused() { return 0; }

extern "C" cudaError_t mapc_launch_rsweep(unsigned long long* bufA, unsigned long long* bufB, MapcCtrl* ctrl,
                                          unsigned int* rhist, uint32_t pass, uint32_t pay_bits, int G, int red_next,
                                          cudaStream_t s) {
  const mapk::RsVariant V = mapk::rs_pick();
  const void* fn = red_next ? V.fn_next : V.fn;
  const size_t smem = V.smem;
  static size_t attr[2] = {0, 0};
  if (attr[red_next ? 1 : 0] < smem) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[red_next ? 1 : 0] = smem;
  }
  void* args[] = {&bufA, &bufB, &ctrl, &rhist, &pass, &pay_bits};
  return cudaLaunchKernel(fn, dim3(G), dim3(V.threads), args, smem, s);
}
