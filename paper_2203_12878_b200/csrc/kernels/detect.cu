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
#include <cstdlib>

#include "common.cuh"
#include "segstate.cuh"

namespace mapk {

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

// ---- pass 1, warp-streaming form (default) ----------------------------------
// Each warp owns a contiguous range of `unit` keys (a multiple of 512) and
// streams it 32 keys per step, one key per lane, coalesced.  Per step the
// segment structure is three ballots: H (lane starts a segment), D (lane's tid
// differs from its predecessor's inside one segment), W (lane writes).  A head
// lane whose segment closes inside the step owns it: racy <=> D and W meet the
// lanes [head, next head).  The segment still open at the end of a step is
// carried (its key, and whether it has seen a diff / a write) -- a uniform
// update from the masks, no per-segment serial walk.  Ranges are joined by the
// same fragment records as the tiled form (first_frag: the range's leading
// continuation; last_frag: its trailing open segment), folded by the fixup.
constexpr int DWS_THREADS = 256;
constexpr int DWS_V = 4;                        // 4-key steps per lane per batch (512 keys per warp)

__device__ __forceinline__ unsigned long long detect_unit(unsigned long long n, unsigned long long nw) {
  unsigned long long u = (n + nw - 1) / nw;
  u = (u + 511ull) & ~511ull;
  return u < 512ull ? 512ull : u;
}

struct WsCarry {
  unsigned long long key;      // key of the previous position
  bool lead, diff, wr;         // open segment: range's leading continuation? seen a tid diff? a write?
  bool lead_closed, lead_diff, lead_wr;
  uint32_t racy;
  unsigned long long best;
};

// One 32-key step; lanes >= nvalid hold no key.  Collectives run converged.
template <bool FULL>
__device__ __forceinline__ void ws_step(WsCarry& c, unsigned long long k, uint32_t nvalid, uint32_t lane,
                                        uint32_t pay_bits, unsigned long long tmask) {
  unsigned long long pk = __shfl_up_sync(0xFFFFFFFFu, k, 1);
  if (lane == 0) pk = c.key;
  const unsigned long long x = k ^ pk;
  const bool valid = FULL || lane < nvalid;
  const bool head = valid && (x >> pay_bits) != 0;
  const bool diff = valid && !head && ((x >> 1) & tmask) != 0;
  const uint32_t H = __ballot_sync(0xFFFFFFFFu, head);
  const uint32_t D = __ballot_sync(0xFFFFFFFFu, diff);
  const uint32_t W = __ballot_sync(0xFFFFFFFFu, valid && (k & 1ull));
  const uint32_t V = FULL ? 0xFFFFFFFFu : (nvalid == 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u));
  // the carried segment covers lanes [0, first head)
  const uint32_t m0 = H ? ((H & (0u - H)) - 1u) : V;
  const bool cd = c.diff || (D & m0) != 0, cw = c.wr || (W & m0) != 0;
  if (H) {
    if (c.lead) {
      c.lead_closed = true; c.lead_diff = cd; c.lead_wr = cw; c.lead = false;
    } else if (lane == 0 && cd && cw) {
      ++c.racy; c.best = min(c.best, c.key >> pay_bits);
    }
    // head lanes whose segment closes in this step own it
    const uint32_t upto = (2u << lane) - 1u;        // lanes <= lane (lane 31: all)
    const uint32_t later = H & ~upto;
    if (head && later) {
      const uint32_t m = ((later & (0u - later)) - 1u) & ~((1u << lane) - 1u);
      if ((D & m) && (W & m)) { ++c.racy; c.best = min(c.best, k >> pay_bits); }
    }
    const uint32_t o = 31u - __clz(H);            // the last segment becomes the carry
    const uint32_t m = V & ~((1u << o) - 1u);
    c.diff = (D & m) != 0;
    c.wr = (W & m) != 0;
  } else {
    c.diff = cd; c.wr = cw;
  }
  c.key = __shfl_sync(0xFFFFFFFFu, k, FULL ? 31 : nvalid - 1);
}

// Four consecutive keys per lane per step (128 keys per warp).  A lane turns
// its 4 keys into three 4-bit masks -- head (new segment), diff (tid differs
// from the predecessor inside a segment), write -- and one lookup in a 4 KiB
// shared table gives everything the in-lane segments decide: the lead part's
// (diff, write), the trailing part's (diff, write), how many segments close
// racy inside the lane and where the first one starts.  Only segments that
// cross lanes use the ballots.  Keys are sorted by sort field, so "new
// segment" is one 64-bit compare: sf(a) != sf(p) <=> a > (p | payload mask).
//   table entry: bit0 lead diff, bit1 lead write, bit2 trail diff, bit3 trail
//   write, bits4-5 racy in-lane segments, bits6-7 head position of the first.
__device__ void ws_fill_table(uint8_t* tab) {
  for (uint32_t idx = threadIdx.x; idx < 4096; idx += blockDim.x) {
    const uint32_t h = idx & 15u, d = (idx >> 4) & 15u, w = idx >> 8;
    uint32_t in_lead = 1, cd = 0, cw = 0, ld = 0, lw = 0, cnt = 0, first = 0, start = 0;
    for (uint32_t i = 0; i < 4; ++i) {
      const uint32_t hi = (h >> i) & 1u, di = (d >> i) & 1u, wi = (w >> i) & 1u;
      if (hi) {
        if (in_lead) { ld = cd; lw = cw; in_lead = 0; }
        else if (cd && cw) { if (!cnt) first = start; ++cnt; }
        start = i; cd = 0; cw = wi;
      } else {
        cd |= di; cw |= wi;
      }
    }
    if (in_lead) { ld = cd; lw = cw; }
    tab[idx] = (uint8_t)(ld | (lw << 1) | (cd << 2) | (cw << 3) | (cnt << 4) | (first << 6));
  }
}

template <bool P32>
__device__ __forceinline__ void ws_step4(WsCarry& c, const unsigned long long (&a)[4], const uint8_t* tab,
                                         uint32_t lane, uint32_t pay_bits, unsigned long long paymask,
                                         unsigned long long tmask) {
  unsigned long long prev = __shfl_up_sync(0xFFFFFFFFu, a[3], 1);
  if (lane == 0) prev = c.key;
  uint32_t h = 0, d = 0, w = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long p = i ? a[i - 1] : prev;
    h |= (uint32_t)(a[i] > (p | paymask)) << i;
    d |= (uint32_t)(P32 ? (((uint32_t)a[i] ^ (uint32_t)p) & ((uint32_t)tmask << 1)) != 0
                        : (((a[i] ^ p) >> 1) & tmask) != 0) << i;
    w |= ((uint32_t)a[i] & 1u) << i;
  }
  const uint32_t e = tab[h | ((d & ~h) << 4) | (w << 8)];
  const uint32_t HL = __ballot_sync(0xFFFFFFFFu, h != 0);
  const uint32_t LD = __ballot_sync(0xFFFFFFFFu, e & 1u);
  const uint32_t LW = __ballot_sync(0xFFFFFFFFu, e & 2u);
  if (e & 0x30u) {                               // racy segments closing inside the lane
    c.racy += (e >> 4) & 3u;
    const uint32_t f = e >> 6;
    const unsigned long long k = f == 0 ? a[0] : f == 1 ? a[1] : f == 2 ? a[2] : a[3];
    c.best = min(c.best, k >> pay_bits);
  }
  if (HL) {
    // the carried segment covers the lead parts of lanes [0, first head lane]
    const uint32_t m0 = ((HL & (0u - HL)) << 1) - 1u;
    const bool ccd = c.diff || (LD & m0) != 0, ccw = c.wr || (LW & m0) != 0;
    if (c.lead) {
      c.lead_closed = true; c.lead_diff = ccd; c.lead_wr = ccw; c.lead = false;
    } else if (lane == 0 && ccd && ccw) {
      ++c.racy; c.best = min(c.best, c.key >> pay_bits);
    }
    // a lane's trailing segment runs through the lead parts of lanes (lane, next head lane]
    const uint32_t upto = (2u << lane) - 1u;
    const uint32_t later = HL & ~upto;
    if (h && later) {
      const uint32_t m = (((later & (0u - later)) << 1) - 1u) & ~upto;
      if (((e & 4u) || (LD & m)) && ((e & 8u) || (LW & m))) { ++c.racy; c.best = min(c.best, a[3] >> pay_bits); }
    }
    const uint32_t TD = __ballot_sync(0xFFFFFFFFu, e & 4u);
    const uint32_t TW = __ballot_sync(0xFFFFFFFFu, e & 8u);
    const uint32_t o = 31u - __clz(HL);
    const uint32_t rest = ~((2u << o) - 1u);
    c.diff = ((TD >> o) & 1u) || (LD & rest);
    c.wr = ((TW >> o) & 1u) || (LW & rest);
  } else {
    c.diff = c.diff || LD != 0;
    c.wr = c.wr || LW != 0;
  }
  c.key = __shfl_sync(0xFFFFFFFFu, a[3], 31);
}

template <bool P32>
__global__ void __launch_bounds__(DWS_THREADS, 4)
k_detect_ws(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
            MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid,
            MapcSegState* __restrict__ first_frag, MapcSegState* __restrict__ last_frag) {
  __shared__ uint8_t tab[4096];
  ws_fill_table(tab);
  __syncthreads();
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const uint32_t lane = threadIdx.x & 31;
  const unsigned long long nw = (unsigned long long)gridDim.x * (DWS_THREADS / 32);
  const unsigned long long gw = (unsigned long long)blockIdx.x * (DWS_THREADS / 32) + (threadIdx.x >> 5);
  const unsigned long long unit = detect_unit(n, nw);
  const unsigned long long start = gw * unit;
  if (lane == 0) { first_frag[gw].valid = 0; last_frag[gw].valid = 0; }
  if (start >= n) return;
  const unsigned long long end = min(n, start + unit);
  const unsigned long long tmask = w_tid >= 32 ? 0xFFFFFFFFull : ((1ull << w_tid) - 1ull);

  WsCarry c;
  const unsigned long long k0 = keys[start];
  // at the chunk's first key: continuation of an empty segment, closed (and
  // counted) like any other by lane 0
  c.key = start > 0 ? keys[start - 1] : k0;
  c.lead = start > 0 && ((c.key ^ k0) >> pay_bits) == 0;
  if (c.lead) c.key = k0;                        // first position: same segment, no tid diff
  c.diff = c.wr = false;
  c.lead_closed = c.lead_diff = c.lead_wr = false;
  c.racy = 0;
  c.best = ~0ull;

  constexpr unsigned long long BATCH = 128ull * DWS_V;
  const unsigned long long paymask = (pay_bits >= 64) ? ~0ull : ((1ull << pay_bits) - 1ull);
  const unsigned long long full_end = start + ((end - start) / BATCH) * BATCH;
  const ulonglong2* __restrict__ p = reinterpret_cast<const ulonglong2*>(keys + start) + 2 * lane;
  for (unsigned long long b = start; b < full_end; b += BATCH, p += BATCH / 2) {
    ulonglong2 v[2 * DWS_V];
#pragma unroll
    for (int j = 0; j < DWS_V; ++j) {
      v[2 * j] = ld_stream2(p + j * 64);
      v[2 * j + 1] = ld_stream2(p + j * 64 + 1);
    }
#pragma unroll
    for (int j = 0; j < DWS_V; ++j) {
      const unsigned long long a4[4] = {v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y};
      ws_step4<P32>(c, a4, tab, lane, pay_bits, paymask, tmask);
    }
  }
#pragma unroll 1
  for (unsigned long long b = full_end; b < end; b += 32) {
    const uint32_t nvalid = (uint32_t)min(32ull, end - b);
    const unsigned long long k = lane < nvalid ? keys[b + lane] : 0ull;
    ws_step<false>(c, k, nvalid, lane, pay_bits, tmask);
  }
  if (lane == 0) {
    const uint32_t t0 = (uint32_t)((k0 >> 1) & tmask);
    if (c.lead_closed) {
      MapcSegState f;
      f.first_tid = t0; f.last_tid = 0;
      f.wr = c.lead_wr; f.diff = c.lead_diff; f.valid = 1; f.ends = 1; f.sf = k0 >> pay_bits;
      first_frag[gw] = f;
    }
    // the segment open at the range end
    const bool ends = end == n || ((keys[end] ^ c.key) >> pay_bits) != 0;
    MapcSegState f;
    f.first_tid = t0;
    f.last_tid = (uint32_t)((c.key >> 1) & tmask);
    f.wr = c.wr; f.diff = c.diff; f.valid = 1; f.ends = ends; f.sf = c.key >> pay_bits;
    if (c.lead) {
      first_frag[gw] = f;
    } else if (ends) {
      if (c.diff && c.wr) { ++c.racy; c.best = min(c.best, c.key >> pay_bits); }
    } else {
      last_frag[gw] = f;
    }
  }
  unsigned long long best = c.best, racy = c.racy;
  for (int o = 16; o > 0; o >>= 1) {
    best = min(best, __shfl_down_sync(0xffffffffu, best, o));
    racy += __shfl_down_sync(0xffffffffu, racy, o);
  }
  if (lane == 0) {
    if (best != ~0ull) atomicMin(&ctrl->racy_sf, best);
    if (racy) atomicAdd(&ctrl->racy, racy);
  }
}

// Fixup over warp ranges: one thread per range that owns an open segment head.
__global__ void k_detect_fixup_ws(MapcCtrl* __restrict__ ctrl, const MapcSegState* __restrict__ first_frag,
                                  const MapcSegState* __restrict__ last_frag, unsigned long long nw) {
  const unsigned long long n = ctrl->n;
  const unsigned long long unit = detect_unit(n, nw);
  const unsigned long long n_units = (n + unit - 1) / unit;
  unsigned long long best = ~0ull, racy = 0;
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < n_units;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const MapcSegState lf = last_frag[t];
    if (!lf.valid) continue;
    uint32_t wr = lf.wr, diff = lf.diff, last = lf.last_tid;
    for (unsigned long long u = t + 1; u < n_units; ++u) {
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
// With the bucket-table detect (table.cu) the keys are sorted only by bucket
// = sf >> tb: the fold then walks the target's bucket and takes its keys.
constexpr int WT_THREADS = 256;
__global__ void __launch_bounds__(WT_THREADS)
k_witness(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
          MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t tb, uint32_t w_tid) {
  const unsigned long long target = ctrl->racy_sf;
  if (target == ~0ull) return;
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  const uint32_t bsh = pay_bits + tb;
  const unsigned long long tbucket = target >> tb;
  __shared__ unsigned long long s_lo;
  __shared__ St part[WT_THREADS];
  if (threadIdx.x == 0) {
    unsigned long long lo = 0, hi = n;                  // first index with bucket >= target's
    while (lo < hi) {
      const unsigned long long mid = (lo + hi) >> 1;
      if ((keys[mid] >> bsh) < tbucket) lo = mid + 1; else hi = mid;
    }
    s_lo = lo;
  }
  __syncthreads();
  St s;
  st_init(s);
  for (unsigned long long i = s_lo + threadIdx.x; i < n; i += WT_THREADS) {
    const unsigned long long key = keys[i];
    if ((key >> bsh) != tbucket) break;
    if ((key >> pay_bits) == target) st_add(s, (uint32_t)(key >> 1) & tmask, 1u << (key & 1u));
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
    ctrl->wit_sf = ~0ull;
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
  r.table_reads = 0;
  r.active_mask = 0;
  for (uint32_t p = 0; p < n_passes; ++p) {
    if (!ctrl->active[p]) continue;
    r.active_passes += 1;
    r.active_mask |= 1u << p;
    // the first active pass's table comes from k_hist_ranges' read; a later one from
    // k_range_hist's, unless the previous scatter accumulated it
    if (p == ctrl->first_active || !(ctrl->rt_done[p] && !ctrl->rt_bad[p])) r.table_reads += 1;
  }
  if (n_passes && !r.active_passes) r.table_reads = 1;   // the histogram read found every pass single-bin
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
  static const int variant = [] { const char* e = getenv("MAPC_DETECT"); return e && e[0] == 't' ? 1 : 0; }();
  if (variant == 0) {
    // warp-streaming form: grid sized to the SMs (4 CTAs of 8 warps each), capped by the fragment arrays
    unsigned long long warps = (max_keys + 511) / 512;
    unsigned long long ctas = (warps + 7) / 8;
    unsigned long long cap = (unsigned long long)n_sms * 4;
    if (cap * 8 > MAPC_DETECT_MAX_UNITS) cap = MAPC_DETECT_MAX_UNITS / 8;
    const int grid = (int)(ctas < 1 ? 1 : (ctas < cap ? ctas : cap));
    if (pay_bits <= 32)
      mapk::k_detect_ws<true><<<grid, mapk::DWS_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid,
                                                                 first_frag, last_frag);
    else
      mapk::k_detect_ws<false><<<grid, mapk::DWS_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, w_tid,
                                                                  first_frag, last_frag);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const unsigned long long nw = (unsigned long long)grid * (mapk::DWS_THREADS / 32);
    mapk::k_detect_fixup_ws<<<(int)((nw + 255) / 256), 256, 0, s>>>(ctrl, first_frag, last_frag, nw);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
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
  return cudaGetLastError();
}

// Canonical witness of the smallest racy segment (no-op when the chunk is DRF).
extern "C" cudaError_t mapc_launch_witness(const unsigned long long* bufA, const unsigned long long* bufB,
                                           MapcCtrl* ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t tb,
                                           uint32_t w_tid, cudaStream_t s) {
  mapk::k_witness<<<1, mapk::WT_THREADS, 0, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, tb, w_tid);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_chunk_finish(const MapcCtrl* ctrl, uint32_t n_passes, MapcChunkResult* out,
                                                cudaStream_t s) {
  mapk::k_chunk_finish<<<1, 1, 0, s>>>(ctrl, n_passes, out);
  return cudaGetLastError();
}
