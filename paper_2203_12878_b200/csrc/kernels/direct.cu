// direct.cu -- sort-free direct-address detect.
//
// The race condition of a cell (phase, array, block, index) is order-
// independent: racy <=> the cell holds a write and two
// distinct tids.  Both facts survive a bitwise OR, so every access can be
// folded into its cell with ONE fire-and-forget global red.or, and no key is
// ever materialised or sorted:
//
//   cell |= tid | (~tid & M) << wt | kind << 2wt        (M = 2^wt - 1)
//
// After all accesses, A = OR of the tids and B = OR of their complements.
// One tid t gives A & B = t & ~t = 0; two distinct tids differ in some bit k,
// one sets bit k of A and the other bit k of B, so A & B != 0.  Hence
//   racy(cell) <=> (cell >> 2wt) & 1  and  (cell & (cell >> wt) & M) != 0.
// The table index of a cell is the chunk's sort field sf,
// so sf order is cell order.  Generate (generate.cu / the JIT kernels, mode
// MAPC_MODE_DIRECT) does the red.or; k_direct_scan reads the table once
// (counts racy cells, atomicMin of the smallest racy sf); the canonical
// witness of that one cell is folded from its keys, which generate re-emits in
// mode MAPC_MODE_FILTER (k_witness_flat).  Cells are u32 when 2wt + 1 <= 32,
// else u64 -- except for blockDim <= 1024 (wt <= 10), where a shorter exact code
// fits 16 bits: each 5-bit digit of the tid becomes one of 32 seven-bit words
// with exactly three ones (the OR of two distinct such words has four or more),
// so "two distinct tids" <=> some digit's 7-bit field has popcount > 3
// (devabi.h code16; tests/test_direct_lemma.py).  Half the table bytes of the
// u32 code, two cells per 32-bit atomic word.
#include "common.cuh"
#include "segstate.cuh"

namespace mapk {

constexpr int DS_THREADS = 128;

template <typename C>
__device__ __forceinline__ bool cell_racy(C c, uint32_t wt) {
  if constexpr (sizeof(C) == 2) {     // constant-weight 16-bit code (devabi.h)
    const uint32_t x = c;
    return ((x >> 14) & 1u) && (__popc(x & 0x7Fu) > 3 || __popc((x >> 7) & 0x7Fu) > 3);
  } else {
    const C m = wt >= 8 * sizeof(C) ? ~C(0) : ((C(1) << wt) - 1);
    return ((c >> (2 * wt)) & 1) && ((c & (c >> wt) & m) != 0);
  }
}

// Two 16-bit cells of one 32-bit word at once, without POPC (a quarter-rate
// pipe: it bounded the scan at ~0.4 ms per 2^29 cells).  The four 7-bit digit
// fields are spread into the byte lanes of a word whose lane top bits are set
// as guards (no borrow leaves a lane); three rounds of "clear the lowest set
// bit" (x & (x - 1), guard restored) leave a nonzero field iff it had >= 4
// ones; a lane counts only if its cell's kind bit (14, 30) is set.  Nonzero
// result <=> some cell of the word is racy (same predicate as cell_racy;
// exhaustive CPU check via mapc_test_racy16_word, tests/test_direct_lemma.py).
__host__ __device__ __forceinline__ uint32_t racy16_word(uint32_t w) {
  const uint32_t g = 0x80808080u, one = 0x01010101u;
  uint32_t x = (w & 0x007F007Fu) | ((w << 1) & 0x7F007F00u) | g;
  x = (x & (x - one)) | g;
  x = (x & (x - one)) | g;
  x = (x & (x - one));
  const uint32_t k = (w >> 14) & 0x00010001u;        // kind bits of the two cells -> bits 0 and 16
  return x & (k * 0x7F7Fu);
}

// Grid-stride over 16-byte vectors of cells, DS_UNROLL vectors in flight per
// thread; each thread's first racy cell is its smallest (indices increase
// along the stride).  The common all-clean vector costs a few ALU ops per cell.
template <typename C, int DS_UNROLL = 8>
__global__ void __launch_bounds__(DS_THREADS)
k_direct_scan(const C* __restrict__ tab, unsigned long long cells, uint32_t wt, MapcCtrl* __restrict__ ctrl) {
  constexpr int PER = 16 / sizeof(C);
  const unsigned long long nvec = cells / PER;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long best = ~0ull, racy = 0;
  const uint4* __restrict__ v4 = reinterpret_cast<const uint4*>(tab);
  for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < nvec;
       i0 += stride * DS_UNROLL) {
    uint4 v[DS_UNROLL];
#pragma unroll
    for (int u = 0; u < DS_UNROLL; ++u) {
      const unsigned long long i = i0 + u * stride;
      if (i < nvec)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(v4 + i));
      else
        v[u] = make_uint4(0, 0, 0, 0);
    }

#pragma unroll
    for (int u = 0; u < DS_UNROLL; ++u) {
      C c[PER];
      memcpy(c, &v[u], 16);
      bool hit = false;
      if constexpr (sizeof(C) == 2)
        hit = (racy16_word(v[u].x) | racy16_word(v[u].y) | racy16_word(v[u].z) | racy16_word(v[u].w)) != 0;
      else {
#pragma unroll
        for (int j = 0; j < PER; ++j) hit |= cell_racy(c[j], wt);
      }
      if (hit) {
        const unsigned long long base = (i0 + u * stride) * PER;
        if constexpr (sizeof(C) == 2) {     // the SWAR lanes say which cell: bytes 0-1 low, 2-3 high
          const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t r = racy16_word(wv[q]);
            if (r & 0xFFFFu) { ++racy; best = min(best, base + 2 * q); }
            if (r >> 16) { ++racy; best = min(best, base + 2 * q + 1); }
          }
        } else {
#pragma unroll
          for (int j = 0; j < PER; ++j)
            if (cell_racy(c[j], wt)) {
              ++racy;
              best = min(best, base + j);
            }
        }
      }
    }
  }
  // ragged tail (cells not a multiple of PER)
  for (unsigned long long i = nvec * PER + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += stride)
    if (cell_racy(tab[i], wt)) {
      ++racy;
      best = min(best, i);
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    racy += __shfl_xor_sync(0xffffffffu, racy, o);
    best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (racy) atomicAdd(&ctrl->racy, racy);
    if (best != ~0ull) atomicMin(&ctrl->racy_sf, best);
  }
}

// Stride-compressed table (mapcheck.cpp Chunk::pcomp): the scan's smallest racy cell
// index back to its sort field -- local phase q = the last block base <= the index,
// (array, block) from the index's high bits within the block, index - idx_lo = the low
// bits * 2^sh + residue.  The map is monotone, so the smallest racy cell is the smallest
// racy sort field.
__device__ __forceinline__ void comp_to_sf(MapcCtrl* __restrict__ ctrl, const unsigned long long* __restrict__ pcomp,
                                           uint32_t nph, uint32_t wa, uint32_t wb, uint32_t wi) {
  const unsigned long long t = ctrl->racy_sf;
  if (t == ~0ull) return;
  uint32_t q = 0;
  for (uint32_t i = 1; i < nph; ++i)
    if (pcomp[2 * i] <= t) q = i;
  const unsigned long long off = t - pcomp[2 * q];
  const uint32_t sh = (uint32_t)(pcomp[2 * q + 1] & 255ull);
  const unsigned long long res = pcomp[2 * q + 1] >> 8;
  const uint32_t bits = wi - sh;
  const unsigned long long sub = off >> bits;                    // (array << wb) | local block
  const unsigned long long idx = ((off & ((1ull << bits) - 1ull)) << sh) + res;
  ctrl->racy_sf = ((unsigned long long)q << (wa + wb + wi)) | (sub << wi) | idx;
}

// Canonical witness of the smallest racy cell from its keys (all with sf =
// ctrl->racy_sf, in arrival order, ctrl->nf of them; filter-mode generate).
constexpr int WF_THREADS = 512;
__global__ void __launch_bounds__(WF_THREADS)
// (out != nullptr: then also the chunk's result record -- what k_chunk_finish writes for
// a chunk without radix passes -- one launch less per chunk)
k_witness_flat(const unsigned long long* __restrict__ keys, MapcCtrl* __restrict__ ctrl, uint32_t pay_bits,
               uint32_t w_tid, unsigned long long cap, MapcChunkResult* __restrict__ out) {
  const unsigned long long target = ctrl->wit_sf;
  const unsigned long long n = ctrl->nf;
  const bool work = target != ~0ull && n <= cap;            // uniform over the block
  if (target != ~0ull && n > cap && threadIdx.x == 0) atomicOr(&ctrl->err, MAPC_ERR_CAPACITY);
  if (work) {
    const uint32_t tmask = w_tid >= 32 ? 0xFFFFFFFFu : ((1u << w_tid) - 1u);
    __shared__ St part[WF_THREADS];
    St s;
    st_init(s);
    for (unsigned long long i = threadIdx.x; i < n; i += WF_THREADS) {
      const unsigned long long key = keys[i];
      if ((key >> pay_bits) != target) {          // library bug guard: the filter let a foreign key through
        atomicOr(&ctrl->err, MAPC_ERR_LAYOUT);
        continue;
      }
      st_add(s, (uint32_t)(key >> 1) & tmask, 1u << (key & 1u));
    }
    part[threadIdx.x] = s;
    __syncthreads();
    for (int h = WF_THREADS / 2; h; h >>= 1) {
      if (threadIdx.x < h) st_merge(part[threadIdx.x], part[threadIdx.x + h]);
      __syncthreads();
    }
    if (threadIdx.x == 0) ctrl->witness = st_witness(part[0], target, w_tid);
  }
  if (out) {
    __syncthreads();                              // every thread's err bits are in
    if (threadIdx.x == 0) {
      __threadfence_block();
      MapcChunkResult r;
      r.n = ctrl->n;
      r.witness = ctrl->witness;
      r.racy = ctrl->racy;
      r.err = atomicOr(&ctrl->err, 0u);
      r.active_passes = 0;
      r.table_reads = 0;
      r.active_mask = 0;
      *out = r;
    }
  }
}

// Which racy chunk folds a witness.  The canonical witness is the minimum over
// chunks, and phase is its most significant field: once a racy chunk whose
// phases end at ph_hi has been seen (on this stream, in chunk order), a later
// chunk whose phases all exceed ph_hi cannot hold the minimum, so its filter
// pass is skipped (its racy count still counts).  *gate = the smallest ph_hi
// of a racy chunk so far (UINT32_MAX = none; reset once per run).
// (pcomp != nullptr: the chunk's table was stride-compressed -- the scan's smallest racy
// cell is mapped back to its sort field first, comp_to_sf)
__global__ void k_witness_gate(MapcCtrl* __restrict__ ctrl, uint32_t* __restrict__ gate, uint32_t ph_lo,
                               uint32_t ph_hi, const unsigned long long* __restrict__ pcomp, uint32_t nph, uint32_t wa,
                               uint32_t wb, uint32_t wi) {
  if (pcomp) comp_to_sf(ctrl, pcomp, nph, wa, wb, wi);
  const unsigned long long sf = ctrl->racy_sf;
  if (sf == ~0ull) return;
  if (*gate < ph_lo) return;
  ctrl->wit_sf = sf;
  if (ph_hi < *gate) *gate = ph_hi;
}

// Table reset: 16-byte stores over the cells (the table region is 256-B aligned).
__global__ void k_table_clear(uint4* __restrict__ tab, unsigned long long n16) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    tab[i] = make_uint4(0, 0, 0, 0);
}

}  // namespace mapk

// ctas_per_sm: 0 = fill the GPU; k > 0 = k CTAs per SM (the overlapped pipeline
// runs these next to a generate that leaves room for them).
extern "C" cudaError_t mapc_launch_table_clear(void* tab, unsigned long long bytes, int n_sms, int ctas_per_sm,
                                               cudaStream_t s) {
  const unsigned long long n16 = (bytes + 15) / 16;
  if (n16 == 0) return cudaSuccess;
  const unsigned long long want = (n16 + 255) / 256;
  const unsigned long long cap = (unsigned long long)n_sms * (ctas_per_sm > 0 ? ctas_per_sm : 8);
  mapk::k_table_clear<<<(int)(want < cap ? want : cap), 256, 0, s>>>((uint4*)tab, n16);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_witness_gate(MapcCtrl* ctrl, uint32_t* gate, uint32_t ph_lo, uint32_t ph_hi,
                                                cudaStream_t s, const unsigned long long* pcomp, uint32_t nph,
                                                uint32_t wa, uint32_t wb, uint32_t wi) {
  mapk::k_witness_gate<<<1, 1, 0, s>>>(ctrl, gate, ph_lo, ph_hi, pcomp, nph, wa, wb, wi);
  return cudaGetLastError();
}

// unroll: 16-B vectors in flight per thread, 8 (default) or 4 (fewer registers:
// more scan CTAs fit next to the overlapped generate)
extern "C" cudaError_t mapc_launch_direct_scan(const void* tab, unsigned long long cells, uint32_t cell_bytes,
                                               uint32_t w_tid, MapcCtrl* ctrl, int n_sms, int ctas_per_sm,
                                               cudaStream_t s, int unroll) {
  if (cells == 0) return cudaSuccess;
  const unsigned long long vec = (cells * cell_bytes + 15) / 16;
  const unsigned long long want = (vec + mapk::DS_THREADS * 8 - 1) / (mapk::DS_THREADS * 8);
  const unsigned long long cap = (unsigned long long)n_sms * (ctas_per_sm > 0 ? ctas_per_sm : 16);
  const int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  if (cell_bytes == 2 && unroll == 4)
    mapk::k_direct_scan<uint16_t, 4><<<grid, mapk::DS_THREADS, 0, s>>>((const uint16_t*)tab, cells, w_tid, ctrl);
  else if (cell_bytes == 2)
    mapk::k_direct_scan<uint16_t><<<grid, mapk::DS_THREADS, 0, s>>>((const uint16_t*)tab, cells, w_tid, ctrl);
  else if (cell_bytes == 4)
    mapk::k_direct_scan<uint32_t><<<grid, mapk::DS_THREADS, 0, s>>>((const uint32_t*)tab, cells, w_tid, ctrl);
  else
    mapk::k_direct_scan<unsigned long long>
        <<<grid, mapk::DS_THREADS, 0, s>>>((const unsigned long long*)tab, cells, w_tid, ctrl);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_witness_flat(const unsigned long long* keys, MapcCtrl* ctrl, uint32_t pay_bits,
                                                uint32_t w_tid, unsigned long long cap, cudaStream_t s,
                                                MapcChunkResult* out) {
  mapk::k_witness_flat<<<1, mapk::WF_THREADS, 0, s>>>(keys, ctrl, pay_bits, w_tid, cap, out);
  return cudaGetLastError();
}

// Host-side check of the SWAR racy test (CPU tests): nonzero iff a cell of w is racy.
extern "C" uint32_t mapc_test_racy16_word(uint32_t w) { return mapk::racy16_word(w); }
