// table.cu -- bucket-table detect (direct-address detect).
//
// The race condition is per segment = per sort field sf:
// racy <=> the segment holds a write and two distinct tids <=> it holds a write
// and min tid != max tid.  None of that needs the segment's keys to be
// adjacent: it is an order-independent fold per sf value.  So the keys are
// radix-sorted only by the HIGH bits of sf -- the bucket b = sf >> tb -- and
// each bucket is folded into a direct-address table of 2^tb cells in shared
// memory (cell = sf & (2^tb - 1)): atomicMin / atomicMax of the tid and an
// atomicOr of the write bit.  A bucket's table is then scanned: racy cells are
// counted and the smallest racy sf is kept (atomicMin, so the result does not
// depend on launch or arrival order).  The LSD passes shrink from ceil(S/8)
// to ceil((S - tb)/8) and the final read of the keys does the detect.
//
// Work split: CTA c owns the key range [c*L, (c+1)*L).  Buckets are
// contiguous; a bucket crossing a range boundary leaves PARTIAL tables (the
// range's leading bucket when it started earlier: "head"; its trailing bucket
// when it continues: "tail"), which k_table_merge folds along the chain.
#include <cstdlib>

#include "common.cuh"

namespace mapk {

constexpr int TB_MAX = MAPC_TABLE_BITS_MAX;        // cells per table: 2^13
constexpr int TB_CELLS = 1 << TB_MAX;
constexpr int TB_THREADS = 512;
constexpr int TB_ITEMS = 8;
constexpr int TB_TILE = TB_THREADS * TB_ITEMS;
constexpr uint32_t TB_EMPTY = 0xFFFFFFFFu;

struct __align__(16) TableSmem {
  uint32_t mn[TB_CELLS];                           // min tid (TB_EMPTY = no access)
  uint32_t mx[TB_CELLS];                           // max tid
  uint32_t wf[TB_CELLS / 4];                       // write flags, one byte per cell (plain stores:
                                                   // a warp writing 32 neighbouring cells must not
                                                   // serialise on one word as atomicOr would)
  unsigned long long next_bucket;
  unsigned long long best;
  unsigned long long racy;
  unsigned long long b_first;
  uint32_t head_open;
};

// Cells are stored at a swizzled slot: the low 5 bits (the bank) are XORed
// with bits 5-9 and 10-14, a bijection that keeps cells one or more 1 KiB
// rows apart (stencil neighbours, transposes) out of each other's bank.
__device__ __forceinline__ uint32_t cell_slot(uint32_t cell) { return cell ^ (((cell >> 5) ^ (cell >> 10)) & 31u); }

__device__ __forceinline__ void table_reset(TableSmem& S) {
  for (int g = threadIdx.x; g < TB_CELLS / 4; g += TB_THREADS) {
    reinterpret_cast<uint4*>(S.mn)[g] = make_uint4(TB_EMPTY, TB_EMPTY, TB_EMPTY, TB_EMPTY);
    reinterpret_cast<uint4*>(S.mx)[g] = make_uint4(0, 0, 0, 0);
    S.wf[g] = 0;
  }
}

// Scan a complete bucket's table: racy cells -> count and smallest sf.  Resets it.
__device__ __forceinline__ void table_flush(TableSmem& S, unsigned long long bucket, uint32_t tb,
                                            unsigned long long& racy, unsigned long long& best) {
  // four consecutive slots per thread: 16-byte loads and stores, and one word of
  // write flags -- a group without writes cannot hold a race
  uint4* mn4 = reinterpret_cast<uint4*>(S.mn);
  uint4* mx4 = reinterpret_cast<uint4*>(S.mx);
  for (int g = threadIdx.x; g < TB_CELLS / 4; g += TB_THREADS) {
    const uint32_t wf = S.wf[g];
    if (wf) {
      const uint4 m = mn4[g], x = mx4[g];
      const uint32_t mm[4] = {m.x, m.y, m.z, m.w}, xx[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (((wf >> (8 * j)) & 0xFFu) && mm[j] != TB_EMPTY && mm[j] != xx[j]) {
          ++racy;
          best = min(best, (bucket << tb) | (unsigned long long)cell_slot(4 * g + j));   // slot -> cell
        }
      }
      S.wf[g] = 0;
    }
    mn4[g] = make_uint4(TB_EMPTY, TB_EMPTY, TB_EMPTY, TB_EMPTY);
    mx4[g] = make_uint4(0, 0, 0, 0);
  }
}

// One key into the table: two fire-and-forget shared reductions and, for a
// write, a byte store.  32-bit shared-window addresses computed once per CTA.
struct TableAddr {
  uint32_t mn, mx, wf;
};

__device__ __forceinline__ void table_add(const TableAddr& A, unsigned long long key, uint32_t pay_bits,
                                          uint32_t cmask, uint32_t tmask) {
  const uint32_t cell = cell_slot((uint32_t)(key >> pay_bits) & cmask);
  const uint32_t t = (uint32_t)(key >> 1) & tmask;
  asm volatile("red.shared.min.u32 [%0], %1;" :: "r"(A.mn + 4 * cell), "r"(t));
  asm volatile("red.shared.max.u32 [%0], %1;" :: "r"(A.mx + 4 * cell), "r"(t));
  if (key & 1ull) asm volatile("st.shared.u8 [%0], %1;" :: "r"(A.wf + cell), "r"(1u));
}

__device__ __forceinline__ void table_spill(TableSmem& S, MapcTablePart* part, uint32_t* store,
                                            unsigned long long bucket, uint32_t ends) {
  uint4* mn = reinterpret_cast<uint4*>(store);
  uint4* mx = reinterpret_cast<uint4*>(store + TB_CELLS);
  uint32_t* wf = store + 2 * TB_CELLS;
  for (int g = threadIdx.x; g < TB_CELLS / 4; g += TB_THREADS) {
    mn[g] = reinterpret_cast<const uint4*>(S.mn)[g];
    mx[g] = reinterpret_cast<const uint4*>(S.mx)[g];
    wf[g] = S.wf[g];
    reinterpret_cast<uint4*>(S.mn)[g] = make_uint4(TB_EMPTY, TB_EMPTY, TB_EMPTY, TB_EMPTY);
    reinterpret_cast<uint4*>(S.mx)[g] = make_uint4(0, 0, 0, 0);
    S.wf[g] = 0;
  }
  if (threadIdx.x == 0) { part->bucket = bucket; part->ends = ends; part->valid = 1; }
}

__global__ void __launch_bounds__(TB_THREADS, 3)
k_detect_table(const unsigned long long* __restrict__ bufA, const unsigned long long* __restrict__ bufB,
               MapcCtrl* __restrict__ ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t tb, uint32_t w_tid,
               MapcTablePart* __restrict__ parts, uint32_t* __restrict__ store) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TableSmem& S = *reinterpret_cast<TableSmem*>(smem_raw);
  const unsigned long long* __restrict__ keys = ctrl->sel[n_passes] ? bufB : bufA;
  const unsigned long long n = ctrl->n;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  if (threadIdx.x == 0) { parts[2 * c].valid = 0; parts[2 * c + 1].valid = 0; }
  unsigned long long L = (n + G - 1) / G;
  L = (L + TB_TILE - 1) / TB_TILE * TB_TILE;
  if (L == 0) L = TB_TILE;
  const unsigned long long r0 = (unsigned long long)c * L;
  if (r0 >= n) return;
  const unsigned long long r1 = min(r0 + L, n);
  const uint32_t bsh = pay_bits + tb;
  const uint32_t cmask = (1u << tb) - 1u;
  const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
  if (threadIdx.x == 0) {
    const unsigned long long bf = keys[r0] >> bsh;
    S.b_first = bf;
    S.head_open = r0 > 0 && (keys[r0 - 1] >> bsh) == bf;
  }
  table_reset(S);
  unsigned long long racy = 0, best = ~0ull;
  const TableAddr A{(uint32_t)__cvta_generic_to_shared(S.mn), (uint32_t)__cvta_generic_to_shared(S.mx),
                    (uint32_t)__cvta_generic_to_shared(S.wf)};
  __syncthreads();
  unsigned long long cur = S.b_first;

  // completes bucket `cur`: evaluate it, or spill it when it began in an earlier
  // range (head partial) or continues into the next one (tail partial)
  auto close_bucket = [&](bool ends_here) {
    if (cur == S.b_first && S.head_open)
      table_spill(S, parts + 2 * c, store + (size_t)(2 * c) * MAPC_TABLE_WORDS, cur, ends_here ? 1u : 0u);
    else if (!ends_here)
      table_spill(S, parts + 2 * c + 1, store + (size_t)(2 * c + 1) * MAPC_TABLE_WORDS, cur, 0u);
    else
      table_flush(S, cur, tb, racy, best);
  };

  for (unsigned long long t0 = r0; t0 < r1; t0 += TB_TILE) {
    const uint32_t tn = (uint32_t)min((unsigned long long)TB_TILE, r1 - t0);
    // the tile's keys and its first / last bucket are loaded together (one round trip)
    unsigned long long k[TB_ITEMS];
    if (tn == TB_TILE) {
#pragma unroll
      for (int j = 0; j < TB_ITEMS; ++j) k[j] = ld_stream(keys + t0 + j * TB_THREADS + threadIdx.x);
    } else {
#pragma unroll
      for (int j = 0; j < TB_ITEMS; ++j) {
        const uint32_t li = j * TB_THREADS + threadIdx.x;
        k[j] = li < tn ? ld_stream(keys + t0 + li) : 0ull;
      }
    }
    const unsigned long long bf = keys[t0] >> bsh, bl = keys[t0 + tn - 1] >> bsh;
    if (bf != cur) {
      // the open bucket ended exactly at the tile boundary
      __syncthreads();
      close_bucket(true);
      __syncthreads();
      cur = bf;
    }
    if (bl == cur) {
      // common case: the whole tile belongs to the open bucket
      if (tn == TB_TILE) {
#pragma unroll
        for (int j = 0; j < TB_ITEMS; ++j) table_add(A, k[j], pay_bits, cmask, tmask);
      } else {
#pragma unroll
        for (int j = 0; j < TB_ITEMS; ++j)
          if (j * TB_THREADS + threadIdx.x < tn) table_add(A, k[j], pay_bits, cmask, tmask);
      }
      continue;
    }
    // the tile closes one or more buckets: one sweep per bucket present (keys re-read from L2)
#pragma unroll 1
    while (true) {
      unsigned long long nb = ~0ull;
      {
        unsigned long long kk[TB_ITEMS];
#pragma unroll
        for (int j = 0; j < TB_ITEMS; ++j) {
          const uint32_t li = j * TB_THREADS + threadIdx.x;
          kk[j] = li < tn ? keys[t0 + li] : ~0ull;
        }
#pragma unroll
        for (int j = 0; j < TB_ITEMS; ++j) {
          const uint32_t li = j * TB_THREADS + threadIdx.x;
          const unsigned long long b = kk[j] >> bsh;
          if (li < tn) {
            if (b == cur) table_add(A, kk[j], pay_bits, cmask, tmask);
            else if (b > cur) nb = min(nb, b);
          }
        }
      }
      if (cur == bl) break;
      if (threadIdx.x == 0) S.next_bucket = ~0ull;
      __syncthreads();
      if (nb != ~0ull) atomicMin(&S.next_bucket, nb);
      close_bucket(true);
      __syncthreads();
      cur = S.next_bucket;
      __syncthreads();
      if (cur == ~0ull) {                 // no later bucket in the tile: unsorted input (flagged, not looped on)
        if (threadIdx.x == 0) atomicOr(&ctrl->err, MAPC_ERR_LAYOUT);
        break;
      }
    }
  }
  __syncthreads();
  close_bucket(!(r1 < n && (keys[r1] >> bsh) == cur));
  // block reduction of (racy, best)
  for (int o = 16; o > 0; o >>= 1) {
    best = min(best, __shfl_down_sync(0xffffffffu, best, o));
    racy += __shfl_down_sync(0xffffffffu, racy, o);
  }
  if (threadIdx.x == 0) { S.best = ~0ull; S.racy = 0; }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    if (best != ~0ull) atomicMin(&S.best, best);
    if (racy) atomicAdd(&S.racy, racy);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (S.best != ~0ull) atomicMin(&ctrl->racy_sf, S.best);
    if (S.racy) atomicAdd(&ctrl->racy, S.racy);
  }
}

// Range c's tail bucket continues into the following ranges' head partials:
// fold them cell by cell until one ends, then evaluate the merged table.
__global__ void __launch_bounds__(TB_THREADS)
k_table_merge(MapcCtrl* __restrict__ ctrl, const MapcTablePart* __restrict__ parts, const uint32_t* __restrict__ store,
              uint32_t G, uint32_t tb) {
  const uint32_t c = blockIdx.x;
  const MapcTablePart tp = parts[2 * c + 1];
  if (!tp.valid) return;
  __shared__ unsigned long long s_best, s_racy;
  if (threadIdx.x == 0) { s_best = ~0ull; s_racy = 0; }
  __syncthreads();
  const uint32_t* T = store + (size_t)(2 * c + 1) * MAPC_TABLE_WORDS;
  unsigned long long racy = 0, best = ~0ull;
  for (int i = threadIdx.x; i < TB_CELLS; i += TB_THREADS) {
    uint32_t m = T[i], x = T[TB_CELLS + i];
    bool w = reinterpret_cast<const uint8_t*>(T + 2 * TB_CELLS)[i] != 0;
    bool closed = false;
    for (uint32_t u = c + 1; u < G; ++u) {
      const MapcTablePart hp = parts[2 * u];
      if (!hp.valid || hp.bucket != tp.bucket) { if (i == threadIdx.x && threadIdx.x == 0) atomicOr(&ctrl->err, MAPC_ERR_LAYOUT); break; }
      const uint32_t* H = store + (size_t)(2 * u) * MAPC_TABLE_WORDS;
      m = min(m, H[i]);
      x = max(x, H[TB_CELLS + i]);
      w = w || reinterpret_cast<const uint8_t*>(H + 2 * TB_CELLS)[i] != 0;
      if (hp.ends) { closed = true; break; }
    }
    if (!closed) continue;
    if (m != TB_EMPTY && w && m != x) {
      ++racy;
      best = min(best, (tp.bucket << tb) | (unsigned long long)cell_slot(i));
    }
  }
  if (best != ~0ull) atomicMin(&s_best, best);
  if (racy) atomicAdd(&s_racy, racy);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_best != ~0ull) atomicMin(&ctrl->racy_sf, s_best);
    if (s_racy) atomicAdd(&ctrl->racy, s_racy);
  }
}

}  // namespace mapk

extern "C" uint32_t mapc_table_bits_max() { return mapk::TB_MAX; }

extern "C" unsigned long long mapc_table_tile() { return mapk::TB_TILE; }

extern "C" int mapc_table_ctas(int n_sms) {
  const int g = n_sms * 3;
  return g < MAPC_TABLE_MAX_CTAS ? g : MAPC_TABLE_MAX_CTAS;
}

// Grid: enough ranges of >= one tile each, at most mapc_table_ctas().
extern "C" cudaError_t mapc_launch_detect_table(const unsigned long long* bufA, const unsigned long long* bufB,
                                                MapcCtrl* ctrl, uint32_t n_passes, uint32_t pay_bits, uint32_t tb,
                                                uint32_t w_tid, MapcTablePart* parts, uint32_t* store,
                                                unsigned long long max_keys, int n_sms, cudaStream_t s) {
  const unsigned long long tiles = (max_keys + mapk::TB_TILE - 1) / mapk::TB_TILE;
  const unsigned long long cap = (unsigned long long)mapc_table_ctas(n_sms);
  uint32_t G = (uint32_t)(tiles < 1 ? 1 : (tiles < cap ? tiles : cap));
  static const int g_env = [] { const char* e = getenv("MAPC_TABLE_G"); return e ? atoi(e) : 0; }();
  if (g_env > 0 && (uint32_t)g_env < G) G = (uint32_t)g_env;     // testing: fewer, longer ranges
  const size_t smem = sizeof(mapk::TableSmem);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mapk::k_detect_table, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  mapk::k_detect_table<<<G, mapk::TB_THREADS, smem, s>>>(bufA, bufB, ctrl, n_passes, pay_bits, tb, w_tid, parts,
                                                          store);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mapk::k_table_merge<<<G, mapk::TB_THREADS, 0, s>>>(ctrl, parts, store, G, tb);
  return cudaGetLastError();
}
