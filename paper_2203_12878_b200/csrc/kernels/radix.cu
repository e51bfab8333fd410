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
  }
}

// --------------------------------------------------------------- onesweep --
constexpr int OS_THREADS = 512;
constexpr int OS_ITEMS = 16;
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;
constexpr int OS_WARPS = OS_THREADS / 32;

// look-back word: [epoch:16][inclusive:1][count:47]
constexpr unsigned long long LB_INCL = 1ull << 47;
constexpr unsigned long long LB_MASK = (1ull << 47) - 1;

struct OsSmem {
  unsigned long long keys[OS_TILE];
  uint32_t whist[OS_WARPS][MAPC_RADIX];
  uint32_t dstart[MAPC_RADIX];
  unsigned long long gbase[MAPC_RADIX];
  uint32_t scan_tmp[OS_WARPS + 1];
  uint32_t tile;
};

__global__ void __launch_bounds__(OS_THREADS, 1)
k_onesweep(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
           unsigned long long* __restrict__ lookback, uint32_t pass, uint32_t shift, unsigned long long epoch) {
  if (!ctrl->active[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OsSmem& S = *reinterpret_cast<OsSmem*>(smem_raw);
  const unsigned long long* __restrict__ src = ctrl->sel[pass] ? bufB : bufA;
  unsigned long long* __restrict__ dst = ctrl->sel[pass] ? bufA : bufB;
  const unsigned long long n = ctrl->n;
  const uint32_t n_tiles = ctrl->n_sort_tiles;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long ep = epoch << 48;

  for (;;) {
    if (threadIdx.x == 0) S.tile = atomicAdd(&ctrl->tickets[pass], 1u);
    for (int i = threadIdx.x; i < OS_WARPS * MAPC_RADIX; i += OS_THREADS) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = S.tile;
    if (tile >= n_tiles) break;
    const unsigned long long tbase = (unsigned long long)tile * OS_TILE;
    const uint32_t tile_n = (uint32_t)min((unsigned long long)OS_TILE, n - tbase);

    // load (warp-striped) + digits
    unsigned long long k[OS_ITEMS];
    uint32_t dg[OS_ITEMS];
    const uint32_t wbase = (uint32_t)w * OS_ITEMS * 32;
#pragma unroll
    for (int j = 0; j < OS_ITEMS; ++j) {
      const uint32_t li = wbase + j * 32 + lane;
      k[j] = li < tile_n ? ld_stream(src + tbase + li) : 0ull;
      dg[j] = (uint32_t)(k[j] >> shift) & 0xFFu;
    }
    // stable warp-level ranking
    uint32_t rk[OS_ITEMS];
#pragma unroll
    for (int j = 0; j < OS_ITEMS; ++j) {
      const uint32_t li = wbase + j * 32 + lane;
      const bool valid = li < tile_n;
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool bit = (dg[j] >> b) & 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
      }
      const uint32_t before = peers & lanemask_lt();
      const uint32_t cnt = __popc(peers);
      uint32_t basev = 0;
      if (valid) basev = S.whist[w][dg[j]];
      rk[j] = basev + __popc(before);
      __syncwarp();
      if (valid && before == 0 && peers != 0) S.whist[w][dg[j]] = basev + cnt;   // lowest peer updates
      __syncwarp();
    }
    __syncthreads();
    // per-digit: exclusive prefix over warps, tile count, publish aggregate
    uint32_t count = 0;
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < OS_WARPS; ++ww) {
        const uint32_t v = S.whist[ww][d];
        S.whist[ww][d] = count;
        count += v;
      }
      unsigned long long* slot = lookback + (unsigned long long)tile * MAPC_RADIX + d;
      if (tile == 0) st_relaxed(slot, ep | LB_INCL | (unsigned long long)count);
      else st_relaxed(slot, ep | (unsigned long long)count);
    }
    // tile-local exclusive digit scan (all threads take part; digits >= 256 contribute 0)
    uint32_t tot;
    const uint32_t dex = block_excl_scan<OS_THREADS>(threadIdx.x < MAPC_RADIX ? count : 0u, S.scan_tmp, &tot);
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
      S.dstart[d] = dex;
      unsigned long long excl = 0;
      if (tile > 0) {
        uint32_t spins = 0;
        for (int64_t t = (int64_t)tile - 1; t >= 0;) {
          const unsigned long long v = ld_relaxed(lookback + (unsigned long long)t * MAPC_RADIX + d);
          if ((v >> 48) != epoch) {                // not published yet: spin (with a watchdog)
            if (++spins > (1u << 26)) { atomicOr(&ctrl->err, MAPC_ERR_WATCHDOG); break; }
            continue;
          }
          excl += v & LB_MASK;
          if (v & LB_INCL) break;
          --t;
        }
        st_relaxed(lookback + (unsigned long long)tile * MAPC_RADIX + d, ep | LB_INCL | (excl + count));
      }
      S.gbase[d] = ctrl->offs[pass][d] + excl - dex;
    }
    __syncthreads();
    // scatter into shared memory in sorted order
#pragma unroll
    for (int j = 0; j < OS_ITEMS; ++j) {
      const uint32_t li = wbase + j * 32 + lane;
      if (li < tile_n) S.keys[S.dstart[dg[j]] + S.whist[w][dg[j]] + rk[j]] = k[j];
    }
    __syncthreads();
    // write out: consecutive i with equal digit land on consecutive addresses
    for (uint32_t i = threadIdx.x; i < tile_n; i += OS_THREADS) {
      const unsigned long long key = S.keys[i];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      dst[S.gbase[d] + i] = key;
    }
    __syncthreads();
  }
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
  mapk::k_digit_scan<<<1, MAPC_RADIX, 0, s>>>(ctrl, n_passes, mapk::OS_TILE);
  return cudaGetLastError();
}

extern "C" unsigned long long mapc_sort_tile() { return mapk::OS_TILE; }

extern "C" cudaError_t mapc_launch_onesweep(unsigned long long* bufA, unsigned long long* bufB, MapcCtrl* ctrl,
                                            unsigned long long* lookback, uint32_t pass, uint32_t shift,
                                            unsigned long long epoch, unsigned long long max_keys, int n_sms,
                                            cudaStream_t s) {
  static bool attr_set = false;
  const int smem = (int)sizeof(mapk::OsSmem);
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(mapk::k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  unsigned long long tiles = (max_keys + mapk::OS_TILE - 1) / mapk::OS_TILE;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mapk::k_onesweep, mapk::OS_THREADS, smem);
  if (occ < 1) occ = 1;
  unsigned long long cap = (unsigned long long)n_sms * occ;
  int grid = (int)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
  mapk::k_onesweep<<<grid, mapk::OS_THREADS, smem, s>>>(bufA, bufB, ctrl, lookback, pass, shift, epoch);
  return cudaGetLastError();
}
