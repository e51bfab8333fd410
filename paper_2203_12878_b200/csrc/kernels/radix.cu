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
  }
}

// --------------------------------------------------------------- onesweep --
// look-back word: [epoch:16][inclusive:1][count:47]
constexpr unsigned long long LB_INCL = 1ull << 47;
constexpr unsigned long long LB_MASK = (1ull << 47) - 1;
constexpr int OS_MIN_TILE = 2048;     // smallest tile of any variant (sizes the look-back array)

template <int THREADS, int ITEMS>
struct OsSmem {
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr int WARPS = THREADS / 32;
  unsigned long long keys[TILE];
  uint32_t whist[WARPS][MAPC_RADIX];
  uint32_t dstart[MAPC_RADIX];
  unsigned long long gbase[MAPC_RADIX];
  uint32_t scan_tmp[WARPS + 1];
  uint32_t tile;
};

// Warp peers with the same 8-bit digit.  MATCH: MATCH.ANY; else 8 ballots.
template <bool MATCH>
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid) {
  if (MATCH) {
    const uint32_t key = valid ? d : (0x100u | (threadIdx.x & 31));
    return __match_any_sync(0xffffffffu, key) & __ballot_sync(0xffffffffu, valid);
  }
  uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// MODE (experiments only; the product uses 0): 1 = skip look-back, 2 = skip ranking too.
template <int THREADS, int ITEMS, bool MATCH, int MINB, int MODE = 0>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
           unsigned long long* __restrict__ lookback, uint32_t pass, uint32_t shift, unsigned long long epoch) {
  using Sm = OsSmem<THREADS, ITEMS>;
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

  for (;;) {
    if (threadIdx.x == 0) S.tile = atomicAdd(&ctrl->tickets[pass], 1u);
    for (int i = threadIdx.x; i < WARPS * MAPC_RADIX; i += THREADS) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = S.tile;
    if (tile >= n_tiles) break;
    const unsigned long long tbase = (unsigned long long)tile * TILE;
    const uint32_t tile_n = (uint32_t)min((unsigned long long)TILE, n - tbase);

    // load (warp-striped: warp w owns [w*ITEMS*32, (w+1)*ITEMS*32) of the tile)
    unsigned long long k[ITEMS];
    const uint32_t wbase = (uint32_t)w * ITEMS * 32;
    if (tile_n == TILE) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) k[j] = ld_stream(src + tbase + wbase + j * 32 + lane);
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t li = wbase + j * 32 + lane;
        k[j] = li < tile_n ? ld_stream(src + tbase + li) : 0ull;
      }
    }
    // stable warp-level ranking (j-major, lane-minor = original order)
    uint32_t rk[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if (MODE == 2) { rk[j] = j * 32 + lane; continue; }
      const bool valid = wbase + j * 32 + lane < tile_n;
      const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
      const uint32_t peers = digit_peers<MATCH>(d, valid);
      const uint32_t before = peers & lanemask_lt();
      uint32_t basev = 0;
      if (valid) basev = S.whist[w][d];
      rk[j] = basev + __popc(before);
      __syncwarp();
      if (valid && before == 0) S.whist[w][d] = basev + __popc(peers);   // lowest peer updates
      __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, tile count, publish aggregate
    uint32_t count = 0;
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww) {
        const uint32_t v = S.whist[ww][d];
        S.whist[ww][d] = count;
        count += v;
      }
      unsigned long long* slot = lookback + (unsigned long long)tile * MAPC_RADIX + d;
      st_relaxed(slot, ep | (tile == 0 ? LB_INCL : 0ull) | (unsigned long long)count);
    }
    uint32_t tot;
    const uint32_t dex = block_excl_scan<THREADS>(threadIdx.x < MAPC_RADIX ? count : 0u, S.scan_tmp, &tot);
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
      S.dstart[d] = dex;
      unsigned long long excl = 0;
      if (MODE == 0 && tile > 0) {
        // windowed decoupled look-back: LBW independent loads in flight per digit
        constexpr int LBW = 8;
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
            if (i != q) continue;                            // stopped earlier
            if ((v[q] >> 48) != epoch) break;               // not published yet: re-poll from here
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
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if (wbase + j * 32 + lane < tile_n) {
        const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
        if (MODE == 2) S.keys[wbase + rk[j]] = k[j];
        else S.keys[S.dstart[d] + S.whist[w][d] + rk[j]] = k[j];
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tile_n; i += THREADS) {
      const unsigned long long key = S.keys[i];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      unsigned long long pos = S.gbase[d] + i;
      if (MODE != 0) pos = pos < n ? pos : n - 1;
      dst[pos] = key;
    }
    __syncthreads();
  }
}

// ---- v3: persistent CTAs, next tile prefetched by a TMA bulk copy ----------
// Double-buffered: while tile t is ranked, look-back-resolved and scattered,
// the bulk-copy engine streams tile t+1 into the other buffer (mbarrier
// completion).  The tile is permuted in place in its buffer for the
// coalesced write-out, so shared memory is 2 x TILE keys + per-warp counters.
template <int THREADS, int ITEMS>
struct Os3Smem {
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr int WARPS = THREADS / 32;
  unsigned long long buf[2][TILE];
  uint32_t whist[WARPS][MAPC_RADIX];
  uint32_t dstart[MAPC_RADIX];
  unsigned long long gbase[MAPC_RADIX];
  uint32_t scan_tmp[WARPS + 1];
  uint32_t tile[2];
  unsigned long long bar[2];
};

template <int THREADS, int ITEMS, bool MATCH, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep3(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
            unsigned long long* __restrict__ lookback, uint32_t pass, uint32_t shift, unsigned long long epoch) {
  using Sm = Os3Smem<THREADS, ITEMS>;
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

  auto issue = [&](int b) {   // thread 0: take the next ticket and start its load
    const uint32_t t = atomicAdd(&ctrl->tickets[pass], 1u);
    S.tile[b] = t;
    if (t < n_tiles) {
      const unsigned long long tb = (unsigned long long)t * TILE;
      const uint32_t cnt = (uint32_t)min((unsigned long long)TILE, n - tb);
      const uint32_t bytes = (cnt * 8u + 15u) & ~15u;       // key buffers carry >= 8 B of slack
      fence_proxy_async();
      mbar_expect_tx(&S.bar[b], bytes);
      bulk_g2s(S.buf[b], src + tb, bytes, &S.bar[b]);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
    issue(0);
  }
  __syncthreads();
  uint32_t parity[2] = {0, 0};
  int b = 0;
  for (;;) {
    const uint32_t tile = S.tile[b];
    if (tile >= n_tiles) break;
    if (threadIdx.x == 0) issue(b ^ 1);                     // prefetch the next tile
    for (int i = threadIdx.x; i < WARPS * MAPC_RADIX; i += THREADS) (&S.whist[0][0])[i] = 0;
    const unsigned long long tbase = (unsigned long long)tile * TILE;
    const uint32_t tile_n = (uint32_t)min((unsigned long long)TILE, n - tbase);
    mbar_wait(&S.bar[b], parity[b]);
    parity[b] ^= 1u;
    __syncthreads();                                        // whist zeroed for everyone

    unsigned long long k[ITEMS];
    const uint32_t wbase = (uint32_t)w * ITEMS * 32;
    uint32_t rk[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t li = wbase + j * 32 + lane;
      const bool valid = li < tile_n;
      k[j] = S.buf[b][li];
      const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
      const uint32_t peers = digit_peers<MATCH>(d, valid);
      const uint32_t before = peers & lanemask_lt();
      uint32_t basev = 0;
      if (valid) basev = S.whist[w][d];
      rk[j] = basev + __popc(before);
      __syncwarp();
      if (valid && before == 0) S.whist[w][d] = basev + __popc(peers);
      __syncwarp();
    }
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
      const int d = threadIdx.x;
      S.dstart[d] = dex;
      unsigned long long excl = 0;
      if (tile > 0) {
        constexpr int LBW = 8;
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
    }
    __syncthreads();
    // permute the tile in place (all keys are in registers)
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if (wbase + j * 32 + lane < tile_n) {
        const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
        S.buf[b][S.dstart[d] + S.whist[w][d] + rk[j]] = k[j];
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tile_n; i += THREADS) {
      const unsigned long long key = S.buf[b][i];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      dst[S.gbase[d] + i] = key;
    }
    __syncthreads();
    b ^= 1;
  }
}

// ---- v4: early counts -> publish -> look-back -> stable ranking ----------
// The tile's digit counts come from an unordered pass of shared-memory
// atomics, so its aggregate is published right after the load and its
// inclusive prefix right after the look-back (short dependency chain between
// consecutive tiles).  Warps >= 8 start the stable ranking while warps 0..7
// (one thread per digit) do the look-back.
template <int THREADS, int ITEMS>
struct Os4Smem {
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr int WARPS = THREADS / 32;
  unsigned long long keys[TILE];
  uint32_t whist[WARPS][MAPC_RADIX];
  uint32_t dstart[MAPC_RADIX];
  unsigned long long gbase[MAPC_RADIX];
  uint32_t scan_tmp[WARPS + 1];
  uint32_t tile;
};

__device__ unsigned long long g_os_dbg[16];

template <int THREADS, int ITEMS, bool MATCH, int MINB, bool DBG = false>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep4(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
            unsigned long long* __restrict__ lookback, uint32_t pass, uint32_t shift, unsigned long long epoch) {
  using Sm = Os4Smem<THREADS, ITEMS>;
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

  unsigned long long T[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long c0 = DBG ? clock64() : 0ull;
  auto mark = [&](int i) {
    if (DBG && (threadIdx.x == 0 || threadIdx.x == THREADS - 1)) {
      unsigned long long c = clock64();
      T[i] += c - c0;
      c0 = c;
    }
  };
  for (;;) {
    mark(7);
    if (threadIdx.x == 0) S.tile = atomicAdd(&ctrl->tickets[pass], 1u);
    for (int i = threadIdx.x; i < WARPS * MAPC_RADIX; i += THREADS) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    mark(0);
    const uint32_t tile = S.tile;
    if (tile >= n_tiles) break;
    const unsigned long long tbase = (unsigned long long)tile * TILE;
    const uint32_t tile_n = (uint32_t)min((unsigned long long)TILE, n - tbase);
    const uint32_t wbase = (uint32_t)w * ITEMS * 32;
    unsigned long long k[ITEMS];
    if (tile_n == TILE) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) k[j] = ld_stream(src + tbase + wbase + j * 32 + lane);
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t li = wbase + j * 32 + lane;
        k[j] = li < tile_n ? ld_stream(src + tbase + li) : 0ull;
      }
    }
    // early counts (order-free)
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (wbase + j * 32 + lane < tile_n) atomicAdd(&S.whist[w][(uint32_t)(k[j] >> shift) & 0xFFu], 1u);
    mark(1);
    __syncthreads();
    mark(2);
    uint32_t count = 0;
    if (threadIdx.x < MAPC_RADIX) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < WARPS; ++ww) {
        const uint32_t v = S.whist[ww][d];
        S.whist[ww][d] = count;                 // -> per-warp running counter base
        count += v;
      }
      st_relaxed(lookback + (unsigned long long)tile * MAPC_RADIX + d,
                 ep | (tile == 0 ? LB_INCL : 0ull) | (unsigned long long)count);
    }
    uint32_t tot;
    const uint32_t dex = block_excl_scan<THREADS>(threadIdx.x < MAPC_RADIX ? count : 0u, S.scan_tmp, &tot);
    if (threadIdx.x < MAPC_RADIX) S.dstart[threadIdx.x] = dex;
    __syncthreads();
    mark(3);
    auto rank_and_place = [&]() {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const bool valid = wbase + j * 32 + lane < tile_n;
        const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
        const uint32_t peers = digit_peers<MATCH>(d, valid);
        const uint32_t before = peers & lanemask_lt();
        uint32_t basev = 0;
        if (valid) basev = S.whist[w][d];
        __syncwarp();
        if (valid) {
          if (before == 0) S.whist[w][d] = basev + __popc(peers);
          S.keys[S.dstart[d] + basev + __popc(before)] = k[j];
        }
        __syncwarp();
      }
    };
    if (threadIdx.x >= MAPC_RADIX) {
      rank_and_place();                          // overlaps the digit warps' look-back
    } else {
      const int d = threadIdx.x;
      unsigned long long excl = 0;
      if (tile > 0) {
        constexpr int LBW = 4;
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
      mark(4);
      rank_and_place();
    }
    mark(5);
    __syncthreads();
    mark(6);
    for (uint32_t i = threadIdx.x; i < tile_n; i += THREADS) {
      const unsigned long long key = S.keys[i];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      dst[S.gbase[d] + i] = key;
    }
    __syncthreads();
  }
  if (DBG && threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&g_os_dbg[i], T[i]);
  if (DBG && threadIdx.x == THREADS - 1)
    for (int i = 0; i < 8; ++i) atomicAdd(&g_os_dbg[8 + i], T[i]);
}

// ---- v5: v4 + hoisted peer masks + next tile's loads under the write-out ---
template <int THREADS, int ITEMS, bool MATCH, int MINB, bool ATOMIC_RANK>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep5(unsigned long long* __restrict__ bufA, unsigned long long* __restrict__ bufB, MapcCtrl* __restrict__ ctrl,
            unsigned long long* __restrict__ lookback, uint32_t pass, uint32_t shift, unsigned long long epoch) {
  using Sm = Os4Smem<THREADS, ITEMS>;
  constexpr int TILE = Sm::TILE, WARPS = Sm::WARPS;
  static_assert(THREADS >= MAPC_RADIX, "one thread per digit");
  if (!ctrl->active[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sm& S = *reinterpret_cast<Sm*>(smem_raw);
  __shared__ uint32_t s_next;
  const unsigned long long* __restrict__ src = ctrl->sel[pass] ? bufB : bufA;
  unsigned long long* __restrict__ dst = ctrl->sel[pass] ? bufA : bufB;
  const unsigned long long n = ctrl->n;
  const uint32_t n_tiles = (uint32_t)((n + TILE - 1) / TILE);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long ep = epoch << 48;
  const uint32_t wbase = (uint32_t)w * ITEMS * 32;

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
    // early counts (order-free)
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
    if (threadIdx.x < MAPC_RADIX) S.dstart[threadIdx.x] = dex;
    if (threadIdx.x == 0) s_next = atomicAdd(&ctrl->tickets[pass], 1u);   // next tile (loaded under the write-out)
    __syncthreads();
    auto rank_and_place = [&]() {
      uint32_t peers[ITEMS];
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {       // independent: pipelined
        const bool valid = wbase + j * 32 + lane < tile_n;
        peers[j] = digit_peers<MATCH>((uint32_t)(k[j] >> shift) & 0xFFu, valid);
      }
      if (ATOMIC_RANK) {
        uint32_t old[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {     // issued back to back; same-warp shared atomics apply in order
          const uint32_t before = peers[j] & lanemask_lt();
          const bool lead = peers[j] != 0 && before == 0;
          old[j] = lead ? atomicAdd(&S.whist[w][(uint32_t)(k[j] >> shift) & 0xFFu], (uint32_t)__popc(peers[j])) : 0u;
        }
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
          const uint32_t leader = peers[j] ? (uint32_t)(__ffs(peers[j]) - 1) : (uint32_t)lane;
          const uint32_t basev = __shfl_sync(0xffffffffu, old[j], leader);
          if (peers[j]) {
            const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
            S.keys[S.dstart[d] + basev + __popc(peers[j] & lanemask_lt())] = k[j];
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
          const uint32_t d = (uint32_t)(k[j] >> shift) & 0xFFu;
          const uint32_t before = peers[j] & lanemask_lt();
          uint32_t basev = 0;
          if (peers[j]) basev = S.whist[w][d];
          __syncwarp();
          if (peers[j]) {
            if (before == 0) S.whist[w][d] = basev + __popc(peers[j]);
            S.keys[S.dstart[d] + basev + __popc(before)] = k[j];
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
        constexpr int LBW = 4;
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
    const uint32_t next = s_next;
    load_tile(next, k);                       // in flight during the write-out
    for (uint32_t i = threadIdx.x; i < tile_n; i += THREADS) {
      const unsigned long long key = S.keys[i];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      dst[S.gbase[d] + i] = key;
    }
    tile = next;
    __syncthreads();
  }
}

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
  unsigned long long keys[TILE];
  unsigned long long wctr[WARPS][MAPC_RADIX];   // [peer mask | position]
  uint32_t whist[WARPS][MAPC_RADIX];            // early counts
  unsigned long long gbase[MAPC_RADIX];
  uint32_t scan_tmp[WARPS + 1];
  uint32_t tile, next;
};

template <int THREADS, int ITEMS, int MINB, int WMODE = 0, bool NO_LB = false, int LBW = 4>
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
          if (valid) S.keys[(uint32_t)v + __popc(vmask & lt)] = k[j];
          if (lane == first) S.wctr[w][d0] = v + (unsigned long long)__popc(vmask);
          __syncwarp();
        } else if (!stable) {
          if (valid) S.keys[(uint32_t)atomicAdd(&S.wctr[w][d], 1ull)] = k[j];
          __syncwarp();
        } else {
          if (valid) atomicOr(&S.wctr[w][d], (unsigned long long)(1u << lane) << 32);
          __syncwarp();
          const unsigned long long v = S.wctr[w][d];
          __syncwarp();
          const uint32_t peers = (uint32_t)(v >> 32), before = peers & lt;
          if (valid) {
            if (before == 0) S.wctr[w][d] = (unsigned long long)((uint32_t)v + __popc(peers));
            S.keys[(uint32_t)v + __popc(before)] = k[j];
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
      if (!NO_LB && tile > 0) {
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
      const unsigned long long key = S.keys[i];
      const uint32_t d = (uint32_t)(key >> shift) & 0xFFu;
      if (WMODE == 0) dst[S.gbase[d] + i] = key;                    // product
      if (WMODE == 1) dst[tbase + i] = key + S.gbase[d];           // experiment: linear write
      if (WMODE == 2 && key == 0x123456789ull) dst[i] = S.gbase[d];  // experiment: no write
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

template <int T, int I, bool M, int B, int MODE = 0>
OsVariant os_variant() {
  return OsVariant{(const void*)k_onesweep<T, I, M, B, MODE>, T, T * I, sizeof(OsSmem<T, I>)};
}

OsVariant pick_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MAPC_OS_VARIANT");
    v = e ? atoi(e) : 52;
  }
  switch (v) {
    case 0: return os_variant<512, 16, false, 1>();
    case 2: return os_variant<256, 16, true, 3>();
    case 3: return os_variant<256, 8, false, 4>();
    case 4: return os_variant<512, 8, false, 2>();
    case 5: return os_variant<256, 12, false, 3>();
    case 6: return os_variant<256, 16, false, 2>();
    case 7: return os_variant<256, 16, true, 2>();
    case 8: return os_variant<512, 16, true, 1>();
    case 20: return OsVariant{(const void*)k_onesweep3<256, 16, false, 2>, 256, 4096, sizeof(Os3Smem<256, 16>)};
    case 21: return OsVariant{(const void*)k_onesweep3<256, 16, true, 2>, 256, 4096, sizeof(Os3Smem<256, 16>)};
    case 22: return OsVariant{(const void*)k_onesweep3<512, 16, true, 1>, 512, 8192, sizeof(Os3Smem<512, 16>)};
    case 23: return OsVariant{(const void*)k_onesweep3<256, 8, true, 3>, 256, 2048, sizeof(Os3Smem<256, 8>)};
    case 24: return OsVariant{(const void*)k_onesweep3<256, 12, true, 2>, 256, 3072, sizeof(Os3Smem<256, 12>)};
    case 30: return OsVariant{(const void*)k_onesweep4<512, 16, false, 1>, 512, 8192, sizeof(Os4Smem<512, 16>)};
    case 31: return OsVariant{(const void*)k_onesweep4<512, 16, true, 1>, 512, 8192, sizeof(Os4Smem<512, 16>)};
    case 32: return OsVariant{(const void*)k_onesweep4<384, 16, true, 1>, 384, 6144, sizeof(Os4Smem<384, 16>)};
    case 33: return OsVariant{(const void*)k_onesweep4<512, 8, true, 2>, 512, 4096, sizeof(Os4Smem<512, 8>)};
    case 34: return OsVariant{(const void*)k_onesweep4<256, 16, true, 2>, 256, 4096, sizeof(Os4Smem<256, 16>)};
    case 35: return OsVariant{(const void*)k_onesweep4<768, 8, true, 1>, 768, 6144, sizeof(Os4Smem<768, 8>)};
    case 36: return OsVariant{(const void*)k_onesweep4<1024, 8, true, 1>, 1024, 8192, sizeof(Os4Smem<1024, 8>)};
    case 39: return OsVariant{(const void*)k_onesweep4<512, 16, true, 1, true>, 512, 8192, sizeof(Os4Smem<512, 16>)};
    case 40: return OsVariant{(const void*)k_onesweep5<512, 16, true, 1, false>, 512, 8192, sizeof(Os4Smem<512, 16>)};
    case 41: return OsVariant{(const void*)k_onesweep5<512, 16, true, 1, true>, 512, 8192, sizeof(Os4Smem<512, 16>)};
    case 42: return OsVariant{(const void*)k_onesweep5<512, 16, false, 1, true>, 512, 8192, sizeof(Os4Smem<512, 16>)};
    case 43: return OsVariant{(const void*)k_onesweep5<512, 8, true, 2, true>, 512, 4096, sizeof(Os4Smem<512, 8>)};
    case 44: return OsVariant{(const void*)k_onesweep5<256, 16, true, 2, true>, 256, 4096, sizeof(Os4Smem<256, 16>)};
    case 45: return OsVariant{(const void*)k_onesweep5<1024, 8, true, 1, true>, 1024, 8192, sizeof(Os4Smem<1024, 8>)};
    case 60: return OsVariant{(const void*)k_onesweep6<512, 8, 2, 0, false, 8>, 512, 4096, sizeof(Os6Smem<512, 8>)};
    case 61: return OsVariant{(const void*)k_onesweep6<512, 8, 2, 0, false, 16>, 512, 4096, sizeof(Os6Smem<512, 8>)};
    case 62: return OsVariant{(const void*)k_onesweep6<512, 8, 2, 0, false, 32>, 512, 4096, sizeof(Os6Smem<512, 8>)};
    case 63: return OsVariant{(const void*)k_onesweep6<512, 16, 1, 0, false, 16>, 512, 8192, sizeof(Os6Smem<512, 16>)};
    case 58: return OsVariant{(const void*)k_onesweep6<512, 16, 1, 0, true>, 512, 8192, sizeof(Os6Smem<512, 16>)};
    case 59: return OsVariant{(const void*)k_onesweep6<512, 8, 2, 0, true>, 512, 4096, sizeof(Os6Smem<512, 8>)};
    case 56: return OsVariant{(const void*)k_onesweep6<512, 16, 1, 1>, 512, 8192, sizeof(Os6Smem<512, 16>)};
    case 57: return OsVariant{(const void*)k_onesweep6<512, 16, 1, 2>, 512, 8192, sizeof(Os6Smem<512, 16>)};
    case 50: return OsVariant{(const void*)k_onesweep6<512, 16, 1>, 512, 8192, sizeof(Os6Smem<512, 16>)};
    case 51: return OsVariant{(const void*)k_onesweep6<256, 16, 2>, 256, 4096, sizeof(Os6Smem<256, 16>)};
    case 52: return OsVariant{(const void*)k_onesweep6<512, 8, 2>, 512, 4096, sizeof(Os6Smem<512, 8>)};
    case 53: return OsVariant{(const void*)k_onesweep6<1024, 8, 1>, 1024, 8192, sizeof(Os6Smem<1024, 8>)};
    case 54: return OsVariant{(const void*)k_onesweep6<256, 24, 1>, 256, 6144, sizeof(Os6Smem<256, 24>)};
    case 55: return OsVariant{(const void*)k_onesweep6<384, 16, 1>, 384, 6144, sizeof(Os6Smem<384, 16>)};
    case 10: return os_variant<256, 16, false, 3, 1>();   // experiment: no look-back
    case 11: return os_variant<256, 16, false, 3, 2>();   // experiment: no look-back, no ranking
    case 12: return os_variant<512, 16, false, 1, 1>();
    case 13: return os_variant<512, 16, false, 1, 2>();
    default: return os_variant<256, 16, false, 3>();
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

extern "C" void mapc_os_debug(unsigned long long* out16, int reset) {
  cudaMemcpyFromSymbol(out16, mapk::g_os_dbg, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(mapk::g_os_dbg, z, sizeof(z));
  }
}
