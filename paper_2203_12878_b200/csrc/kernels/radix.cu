// radix.cu -- K2 (all-digit histogram), digit scan, K3 (onesweep LSD pass).
//
// Stable LSD radix sort of u64 keys on the chunk's sort-field bits
// [pay_bits, pay_bits + S), 8-bit digits, P = ceil(S/8) passes (SURVEY.md §8a,
// "a2").  One pass = one launch of k_onesweep: a persistent grid takes tiles in
// order from an atomic ticket (forward progress for the look-back), ranks the
// tile's keys per digit with warp ballots (stable: warp-striped order, j-major
// then lane), publishes the tile's per-digit counts, resolves its global
// per-digit offsets by DECOUPLED LOOK-BACK over earlier tiles (Merrill &
// Garland), reorders the tile in shared memory and writes runs of equal digit
// contiguously.  Passes whose digit has a single non-empty bin are skipped on
// the device (ctrl->active), so the host never synchronises between passes.
#include <cstdlib>

#include "common.cuh"

namespace mapk {

// --------------------------------------------------------------- histogram --
constexpr int HIST_THREADS = 512;

__global__ void __launch_bounds__(HIST_THREADS)
k_hist(const unsigned long long* __restrict__ keys, MapcCtrl* __restrict__ ctrl, uint32_t pay_bits, uint32_t n_passes) {
  __shared__ uint32_t h[MAPC_MAX_PASSES][MAPC_RADIX];
  for (int i = threadIdx.x; i < MAPC_MAX_PASSES * MAPC_RADIX; i += HIST_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  const unsigned long long n = ctrl->n;
  const unsigned long long n2 = n >> 1;
  const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
  for (unsigned long long i = (unsigned long long)blockIdx.x * HIST_THREADS + threadIdx.x; i < n2;
       i += (unsigned long long)gridDim.x * HIST_THREADS) {
    ulonglong2 v = ld_stream2(k2 + i);
    for (uint32_t p = 0; p < n_passes; ++p) {
      atomicAdd(&h[p][(v.x >> (pay_bits + 8 * p)) & 0xFF], 1u);
      atomicAdd(&h[p][(v.y >> (pay_bits + 8 * p)) & 0xFF], 1u);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v = keys[n - 1];
    for (uint32_t p = 0; p < n_passes; ++p) atomicAdd(&h[p][(v >> (pay_bits + 8 * p)) & 0xFF], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)n_passes * MAPC_RADIX; i += HIST_THREADS) {
    uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&(&ctrl->hist[0][0])[i], c);
  }
}

// One block of 256 threads: exclusive scans, active passes, buffer selection.
__global__ void __launch_bounds__(MAPC_RADIX) k_digit_scan(MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t tile) {
  __shared__ uint32_t tmp[MAPC_RADIX / 32 + 1];
  __shared__ unsigned long long tmp64[MAPC_RADIX / 32 + 1];
  const int d = threadIdx.x;
  for (uint32_t p = 0; p < n_passes; ++p) {
    const uint32_t c = ctrl->hist[p][d];
    uint32_t nz_total;
    block_excl_scan<MAPC_RADIX>(c != 0 ? 1u : 0u, tmp, &nz_total);
    unsigned long long tot;
    unsigned long long ex = block_excl_scan<MAPC_RADIX>((unsigned long long)c, tmp64, &tot);
    ctrl->offs[p][d] = ex;
    if (d == 0) ctrl->active[p] = nz_total > 1 ? 1u : 0u;
  }
  __syncthreads();
  if (d == 0) {
    uint32_t s = 0;
    ctrl->sel[0] = 0;
    for (uint32_t p = 0; p < n_passes; ++p) {
      if (ctrl->active[p]) s ^= 1u;
      ctrl->sel[p + 1] = s;
    }
    ctrl->n_sort_tiles = (uint32_t)((ctrl->n + tile - 1) / tile);
    uint32_t nxt = MAPC_MAX_PASSES;
    for (int p = MAPC_MAX_PASSES - 1; p >= 0; --p) {
      ctrl->next_active[p] = nxt;
      if ((uint32_t)p < n_passes && ctrl->active[p]) nxt = (uint32_t)p;
    }
    ctrl->first_active = nxt;
  }
}

// --------------------------------------------------------------- onesweep --
// Decoupled look-back variant (kept for comparison: MAPC_SORT=onesweep).
// look-back word: [epoch:16][inclusive:1][count:47]
constexpr unsigned long long LB_INCL = 1ull << 47;
constexpr unsigned long long LB_MASK = (1ull << 47) - 1;
constexpr int OS_MIN_TILE = 2048;     // sizes the look-back array

// Tile buffer slot with one pad per 16 keys (see rsweep.cu: digit regions start
// one bank cycle apart, an unpadded scatter is a ~16-way bank conflict).
__device__ __forceinline__ uint32_t os_slot(uint32_t p) { return p + (p >> 4); }

// ---- v6: MATCH-free stable ranking ---------------------------------------
// Peers of a (warp, digit) are found with one shared-memory atomicOr of the
// lane bit into a 64-bit word [peer mask:32 | running tile position:32]
// (3 MIO ops per item; MATCH.ANY measures ~61 SM-cycles per warp instruction
// on B200 and an 8-ballot multisplit ~24, profiles/r1_mio_microbench.txt).
// The first LSD pass needs no stability: rank = atomicAdd (1 MIO op).
template <int THREADS, int ITEMS>
struct Os6Smem {
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr int WARPS = THREADS / 32;
  unsigned long long keys[TILE + TILE / 16];
  unsigned long long wctr[WARPS][MAPC_RADIX];   // [peer mask | position]
  uint32_t whist[WARPS][MAPC_RADIX];            // early counts
  unsigned long long gbase[MAPC_RADIX];
  uint32_t scan_tmp[WARPS + 1];
  uint32_t tile, next;
};

template <int THREADS, int ITEMS, int MINB, int LBW = 4>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep6(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
            unsigned long long* __restrict__ lookback, uint32_t pass, uint32_t shift, unsigned long long epoch) {
  using Sm = Os6Smem<THREADS, ITEMS>;
  constexpr int TILE = Sm::TILE, WARPS = Sm::WARPS;
  static_assert(THREADS >= MAPC_RADIX, "one thread per digit");
  if (!ctrl->active[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sm& S = *reinterpret_cast<Sm*>(smem_raw);
  const unsigned long long* __restrict__ src = ctrl->sel[pass] ? bufB : bufA;
  unsigned long long* __restrict__ dst = ctrl->sel[pass] ? bufA : bufB;
  const unsigned long long n = ctrl->n;
  const uint32_t n_tiles = (uint32_t)((n + TILE - 1) / TILE);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long ep = epoch << 48;
  const uint32_t wbase = (uint32_t)w * ITEMS * 32;
  // pass 0 sees keys in generation order: any order of equal digits is valid
  bool stable = false;
  for (uint32_t q = 0; q < pass; ++q) stable |= ctrl->active[q] != 0;

  auto load_tile = [&](uint32_t t, unsigned long long* kk) {
    if (t >= n_tiles) return;
    const unsigned long long tb = (unsigned long long)t * TILE;
    const uint32_t tn = (uint32_t)min((unsigned long long)TILE, n - tb);
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

  if (threadIdx.x == 0) S.tile = atomicAdd(&ctrl->tickets[pass], 1u);
  __syncthreads();
  uint32_t tile = S.tile;
  unsigned long long k[ITEMS];
  load_tile(tile, k);
  while (tile < n_tiles) {
    for (int i = threadIdx.x; i < WARPS * MAPC_RADIX; i += THREADS) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    const unsigned long long tbase = (unsigned long long)tile * TILE;
    const uint32_t tile_n = (uint32_t)min((unsigned long long)TILE, n - tbase);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (wbase + j * 32 + lane < tile_n) atomicAdd(&S.whist[w][(uint32_t)(k[j] >> shift) & 0xFFu], 1u);
    __syncthreads();
    uint32_t count = 0;
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww) {
        const uint32_t v = S.whist[ww][d];
        S.whist[ww][d] = count;
        count += v;
      }
      st_relaxed(lookback + (unsigned long long)tile * MAPC_RADIX + d,
                 ep | (tile == 0 ? LB_INCL : 0ull) | (unsigned long long)count);
    }
    uint32_t tot;
    const uint32_t dex = block_excl_scan<THREADS>(threadIdx.x < MAPC_RADIX ? count : 0u, S.scan_tmp, &tot);
    if (threadIdx.x < MAPC_RADIX) {
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww)
        S.wctr[ww][threadIdx.x] = (unsigned long long)(dex + S.whist[ww][threadIdx.x]);
    }
    if (threadIdx.x == 0) S.next = atomicAdd(&ctrl->tickets[pass], 1u);
    __syncthreads();
    auto rank_and_place = [&]() {
      const uint32_t lt = lanemask_lt();
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const bool valid = wbase + j * 32 + lane < tile_n;
        const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        if (vmask == 0) continue;
        const int first = __ffs(vmask) - 1;
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, first);
        if (__all_sync(0xffffffffu, !valid || d == d0)) {
          // warp-uniform digit (typical once the low digits are sorted): no atomics
          const unsigned long long v = S.wctr[w][d0];
          __syncwarp();
          if (valid) S.keys[os_slot((uint32_t)v + __popc(vmask & lt))] = k[j];
          if (lane == first) S.wctr[w][d0] = v + (unsigned long long)__popc(vmask);
          __syncwarp();
        } else if (!stable) {
          if (valid) S.keys[os_slot((uint32_t)atomicAdd(&S.wctr[w][d], 1ull))] = k[j];
          __syncwarp();
        } else {
          if (valid) atomicOr(&S.wctr[w][d], (unsigned long long)(1u << lane) << 32);
          __syncwarp();
          const unsigned long long v = S.wctr[w][d];
          __syncwarp();
          const uint32_t peers = (uint32_t)(v >> 32), before = peers & lt;
          if (valid) {
            if (before == 0) S.wctr[w][d] = (unsigned long long)((uint32_t)v + __popc(peers));
            S.keys[os_slot((uint32_t)v + __popc(before))] = k[j];
          }
          __syncwarp();
        }
      }
    };
    if (threadIdx.x >= MAPC_RADIX) {
      rank_and_place();
    } else {
      const int d = threadIdx.x;
      unsigned long long excl = 0;
      if (tile > 0) {
        uint32_t spins = 0;
        int64_t t = (int64_t)tile - 1;
        for (;;) {
          unsigned long long v[LBW];
#pragma unroll
          for (int i = 0; i < LBW; ++i)
            v[i] = (t - i >= 0) ? ld_relaxed(lookback + (unsigned long long)(t - i) * MAPC_RADIX + d) : (ep | LB_INCL);
          int i = 0;
          bool done = false;
#pragma unroll
          for (int q = 0; q < LBW; ++q) {
            if (i != q) continue;
            if ((v[q] >> 48) != epoch) break;
            excl += v[q] & LB_MASK;
            ++i;
            if (v[q] & LB_INCL) { done = true; break; }
          }
          if (done) break;
          t -= i;
          if (i == 0 && ++spins > (1u << 26)) { atomicOr(&ctrl->err, MAPC_ERR_WATCHDOG); break; }
        }
        st_relaxed(lookback + (unsigned long long)tile * MAPC_RADIX + d, ep | LB_INCL | (excl + count));
      }
      S.gbase[d] = ctrl->offs[pass][d] + excl - dex;
      rank_and_place();
    }
    __syncthreads();
    const uint32_t next = S.next;
    load_tile(next, k);
    for (uint32_t i = threadIdx.x; i < tile_n; i += THREADS) {
      const unsigned long long key = S.keys[os_slot(i)];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      dst[S.gbase[d] + i] = key;
    }
    tile = next;
    __syncthreads();
  }
}

struct OsVariant {
  const void* fn;
  int threads, tile;
  size_t smem;
};

OsVariant pick_variant() {
  return OsVariant{(const void*)k_onesweep6<512, 8, 2>, 512, 4096, sizeof(Os6Smem<512, 8>)};
}

}  // namespace mapk

extern "C" cudaError_t mapc_launch_hist(const unsigned long long* keys, MapcCtrl* ctrl, uint32_t pay_bits,
                                        uint32_t n_passes, unsigned long long max_keys, int n_sms, cudaStream_t s) {
  if (n_passes == 0) return cudaSuccess;
  unsigned long long want = (max_keys / 2 + mapk::HIST_THREADS - 1) / mapk::HIST_THREADS;
  unsigned long long cap = (unsigned long long)n_sms * 4;
  int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  mapk::k_hist<<<grid, mapk::HIST_THREADS, 0, s>>>(keys, ctrl, pay_bits, n_passes);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_digit_scan(MapcCtrl* ctrl, uint32_t n_passes, cudaStream_t s) {
  mapk::k_digit_scan<<<1, MAPC_RADIX, 0, s>>>(ctrl, n_passes, (uint32_t)mapk::pick_variant().tile);
  return cudaGetLastError();
}

extern "C" unsigned long long mapc_sort_tile() { return mapk::OS_MIN_TILE; }

extern "C" cudaError_t mapc_launch_onesweep(unsigned long long* bufA, unsigned long long* bufB, MapcCtrl* ctrl,
                                            unsigned long long* lookback, uint32_t pass, uint32_t shift,
                                            unsigned long long epoch, unsigned long long max_keys, int n_sms,
                                            cudaStream_t s) {
  static int occ = -1;
  const mapk::OsVariant V = mapk::pick_variant();
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(V.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V.smem);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, V.fn, V.threads, V.smem);
    if (occ < 1) occ = 1;
  }
  unsigned long long tiles = (max_keys + V.tile - 1) / V.tile;
  unsigned long long cap = (unsigned long long)n_sms * occ;
  dim3 grid((unsigned)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap))), block(V.threads);
  void* args[] = {&bufA, &bufB, &ctrl, &lookback, &pass, &shift, &epoch};
  return cudaLaunchKernel(V.fn, grid, block, args, V.smem, s);
}

