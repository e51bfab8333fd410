// generate.cu -- K1: enumerate the access values of a chunk as packed u64 keys.
//
// One GPU thread per tuple (block, tid, k_0..k_{L-1}) of a group's bounding
// box (north_star mapping).  The thread decodes its tuple by mixed radix
// (invariant-divisor multiplies), runs the group's straight-line program from
// __constant__ memory -- the data-free image of rules seq/if/for of
// PAPER.md:506-551 with the par union of PAPER.md:579-589 made explicit as the
// tid coordinate -- and emits one key per access whose guards hold:
//   key = [lphase | array | lblock | index - idx_lo][tid][kind]
// Dense segments store keys at precomputed slots; guarded segments compact
// their keys in shared memory and reserve space with one global atomicAdd per
// CTA iteration (block-aggregated compaction).
#include "common.cuh"

namespace mapk {

__constant__ MapcOp c_ops[MAPC_MAX_OPS];


template <typename W>
struct VmWidth;
template <>
struct VmWidth<uint32_t> { static constexpr uint32_t bits = 32; };
template <>
struct VmWidth<uint64_t> { static constexpr uint32_t bits = 64; };

// ---- v2: segment-uniform tiles, 4 tuples per thread per VM pass ------------
// A CTA iteration covers MAPC_GEN_TILE consecutive tuples of ONE segment, so the
// bytecode stream is uniform across the CTA; each op is decoded once and applied
// to V tuples per thread (dispatch cost amortised V-fold).  The shared register
// file holds only the registers the chunk's programs use.  Dense segments
// (no guard, no fault check: every tuple emits n_emits keys) store each key
// at key_begin + e * n_tuples + tuple (site-major, coalesced); other segments
// are compacted through shared memory with one global atomicAdd per tile.
template <typename W>
__global__ void __launch_bounds__(MAPC_GEN_THREADS)
k_generate2(const MapcSeg* __restrict__ segs, int n_segs, unsigned long long tile_lo, unsigned long long tile_hi,
            MapcLayout lay, unsigned long long* __restrict__ keys, MapcCtrl* __restrict__ ctrl, uint32_t nreg,
            uint32_t force_compact, uint32_t mode, void* __restrict__ tab, uint32_t cell_bytes) {
  constexpr int T = MAPC_GEN_THREADS, V = MAPC_GEN_V;
  constexpr uint32_t WB = VmWidth<W>::bits;
  extern __shared__ __align__(16) unsigned char gsm[];
  W* R = reinterpret_cast<W*>(gsm);                                    // [nreg][V][T]
  unsigned long long* stage = reinterpret_cast<unsigned long long*>(gsm + ((size_t)nreg * V * T * sizeof(W) + 15) / 16 * 16);
  __shared__ uint32_t scan_tmp[T / 32 + 1];
  __shared__ unsigned long long s_base;
  const int me = threadIdx.x;
  uint32_t err = 0;
  unsigned long long cnt_all = 0;                 // direct mode: guarded accesses, added once at the end
  // filter mode: only the keys of the witness cell (none if the chunk is DRF)
  const unsigned long long target = mode == MAPC_MODE_FILTER ? ctrl->wit_sf : ~0ull;
  if (mode == MAPC_MODE_FILTER && target == ~0ull) return;
  unsigned long long* const n_out = mode == MAPC_MODE_FILTER ? &ctrl->nf : &ctrl->n;
  // direct mode: cell code of (tid, kind) = tid | (~tid & M) << wt | kind << 2wt (direct.cu)
  const uint32_t wt = lay.w_tid;
  const unsigned long long tmask = wt >= 64 ? ~0ull : ((1ull << wt) - 1);
#define RG(r, v) R[((size_t)(r) * V + (v)) * T + me]

  for (unsigned long long tile = tile_lo + blockIdx.x; tile < tile_hi; tile += gridDim.x) {
    int lo = 0, hi = n_segs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
    }
    const MapcSeg& sg = segs[lo];
    // stage API and filter mode: every key goes through compaction
    const bool dense = sg.dense && !force_compact && mode != MAPC_MODE_FILTER;
    const uint32_t tl0 = (uint32_t)(tile - sg.tile_begin) * (uint32_t)(V * T);
    const uint32_t L = sg.n_levels;
    uint32_t tidv[V], lbv[V];
    bool act[V], valid[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t t = tl0 + v * T + me;
      valid[v] = t < sg.n_tuples;
      uint32_t rem = valid[v] ? t : 0u;
      // mixed radix: (block, tid, k_0..k_{L-1}) with k_{L-1} fastest, or
      // (block, k_0..k_{L-1}, tid) with tid fastest (sg.tid_inner)
      if (sg.tid_inner) {
        const uint32_t q = fastdiv(rem, sg.tid_div);
        tidv[v] = rem - q * sg.tid_div.d;
        rem = q;
      }
      for (int l = (int)L - 1; l >= 0; --l) {
        const uint32_t q = fastdiv(rem, sg.trip_div[l]);
        RG(MAPC_REG_K0 + l, v) = (W)(rem - q * sg.trip_div[l].d);
        rem = q;
      }
      if (!sg.tid_inner) {
        const uint32_t q = fastdiv(rem, sg.tid_div);
        tidv[v] = rem - q * sg.tid_div.d;
        rem = q;
      }
      RG(MAPC_REG_TID, v) = (W)tidv[v];
      RG(MAPC_REG_BID, v) = (W)(sg.b0 + rem);
      lbv[v] = sg.lb0 + rem;
      act[v] = true;
    }
    uint32_t cnt = 0, e = 0;
    for (uint32_t pc = sg.prog_begin; pc < sg.prog_end; ++pc) {
      const MapcOp op = c_ops[pc];
      const uint32_t code = op.code & MAPC_CODE_MASK;
      const bool ai = op.code & MAPC_A_IMM, bi = op.code & MAPC_B_IMM;
      const W im = (W)op.imm;
#define AV(v) (ai ? im : RG(op.a, v))
#define BV(v) (bi ? im : RG(op.b, v))
#define VLOOP(expr)                                       \
  _Pragma("unroll") for (int v = 0; v < V; ++v) {         \
    const W A = AV(v), B = BV(v);                         \
    (void)A; (void)B;                                     \
    RG(op.dst, v) = (W)(expr);                            \
  }                                                       \
  break;
      switch (code) {
        case VM_ADD: VLOOP(A + B)
        case VM_SUB: VLOOP(A > B ? A - B : W(0))
        case VM_MUL: VLOOP(A * B)
        case VM_DIV:
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const W A = AV(v), B = BV(v);
            if (B == 0 && act[v] && valid[v] && (op.aux & MAPC_AUX_FAULT)) err |= MAPC_ERR_DIV0;
            RG(op.dst, v) = B ? A / B : W(0);
          }
          break;
        case VM_MOD:
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const W A = AV(v), B = BV(v);
            if (B == 0 && act[v] && valid[v] && (op.aux & MAPC_AUX_FAULT)) err |= MAPC_ERR_DIV0;
            RG(op.dst, v) = B ? A % B : W(0);
          }
          break;
        case VM_SHL: VLOOP(B >= WB ? W(0) : W(A << B))
        case VM_SHR: VLOOP(B >= WB ? W(0) : W(A >> B))
        case VM_MIN: VLOOP(A < B ? A : B)
        case VM_MAX: VLOOP(A > B ? A : B)
        case VM_DIVM:
        case VM_MODM: {
          const uint32_t dv = (uint32_t)(op.imm >> 32), m = (uint32_t)op.imm;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const uint32_t a32 = (uint32_t)(ai ? im : RG(op.a, v));
            const uint32_t h = __umulhi(m, a32);
            const uint32_t qq = (h + ((a32 - h) >> 1)) >> op.aux;
            RG(op.dst, v) = code == VM_DIVM ? W(qq) : W(a32 - qq * dv);
          }
          break;
        }
        case VM_BAND: VLOOP(A & (W)op.imm)
        case VM_EQ: VLOOP(A == B)
        case VM_NE: VLOOP(A != B)
        case VM_LT: VLOOP(A < B)
        case VM_LE: VLOOP(A <= B)
        case VM_GT: VLOOP(A > B)
        case VM_GE: VLOOP(A >= B)
        case VM_LAND: VLOOP((A != 0) & (B != 0))
        case VM_LOR: VLOOP((A != 0) | (B != 0))
        case VM_LNOT: VLOOP(A == 0)
        case VM_TRIP:
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const W A = AV(v), B = BV(v);
            const W step = (op.aux & MAPC_AUX_CONST) ? (W)(op.aux & ~MAPC_AUX_CONST) : RG(op.aux, v);
            const W span = B > A ? B - A : W(0);
            RG(op.dst, v) = span == 0 ? W(0) : (step == 1 ? span : W((span - 1) / (step ? step : W(1)) + 1));
          }
          break;
        case VM_MADK: VLOOP(A + RG(op.aux, v) * B)
        case VM_MOVI: VLOOP(im)
        case VM_ACT:
#pragma unroll
          for (int v = 0; v < V; ++v) act[v] = AV(v) != 0;
          break;
        case VM_EMIT: {
          const unsigned long long arr = (unsigned long long)(op.aux >> 1) << (lay.w_block + lay.w_index);
          const unsigned long long kind = op.aux & 1u;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (!(act[v] && valid[v])) continue;
            unsigned long long idx = (unsigned long long)AV(v) - lay.idx_lo;
            // outside the layout (a compiler bug guard): flag it and fold into cell 0
            // of the chunk instead, so no reduction can leave the table
            if (lay.w_index < 64 && (idx >> lay.w_index) != 0) { err |= MAPC_ERR_LAYOUT; idx = 0; }
            const unsigned long long sf = sg.key_hi + arr + ((unsigned long long)lbv[v] << lay.w_index) + idx;
            if (mode == MAPC_MODE_DIRECT) {
              const unsigned long long code =
                  tidv[v] | ((~(unsigned long long)tidv[v] & tmask) << wt) | (kind << (2 * wt));
              if (cell_bytes == 2)   // two 16-bit cells per 32-bit word
                atomicOr(reinterpret_cast<uint32_t*>(tab) + (sf >> 1), code16(tidv[v], (uint32_t)kind) << (16 * (sf & 1)));
              else if (cell_bytes == 4) atomicOr(reinterpret_cast<uint32_t*>(tab) + sf, (uint32_t)code);
              else atomicOr(reinterpret_cast<unsigned long long*>(tab) + sf, code);
              cnt += dense ? 0u : 1u;
              continue;
            }
            const unsigned long long key = (sf << lay.pay_bits) | ((unsigned long long)tidv[v] << 1) | kind;
            if (mode == MAPC_MODE_FILTER && sf != target) continue;
            if (dense) {
              keys[sg.key_begin + (unsigned long long)e * sg.n_tuples + tl0 + v * T + me] = key;
            } else {
              stage[(size_t)cnt * T + me] = key;
              ++cnt;
            }
          }
          ++e;
          break;
        }
        default: break;
      }
#undef AV
#undef BV
#undef VLOOP
    }
    if (mode == MAPC_MODE_DIRECT) {                   // only the count: the accesses are in the table
      if (!dense) cnt_all += cnt;
    } else if (!dense) {                              // uniform across the CTA
      uint32_t total;
      const uint32_t excl = block_excl_scan<T>(cnt, scan_tmp, &total);
      if (me == 0) s_base = total ? atomicAdd(n_out, (unsigned long long)total) : 0ull;
      __syncthreads();
      const unsigned long long obase = s_base;
      for (uint32_t j = 0; j < cnt; ++j) {
        const unsigned long long pos = obase + excl + j;
        if (pos < lay.cap) keys[pos] = stage[(size_t)j * T + me];
        else err |= MAPC_ERR_CAPACITY;
      }
      __syncthreads();
    }
  }
#undef RG
  if (mode == MAPC_MODE_DIRECT) {
    // (one atomicAdd per warp and launch: per tile, they serialised in the counter's L2 slice)
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt_all += __shfl_xor_sync(0xffffffffu, cnt_all, o);
    if ((me & 31) == 0 && cnt_all) atomicAdd(&ctrl->n, cnt_all);
  }
  if (err) atomicOr(&ctrl->err, err);
}

}  // namespace mapk

// --------------------------------------------------------------- launchers --
extern "C" cudaError_t mapc_upload_ops(const MapcOp* host_ops, size_t n_ops, cudaStream_t s) {
  if (n_ops == 0) return cudaSuccess;
  return cudaMemcpyToSymbolAsync(mapk::c_ops, host_ops, n_ops * sizeof(MapcOp), 0, cudaMemcpyHostToDevice, s);
}

extern "C" cudaError_t mapc_launch_generate(const MapcSeg* segs, int n_segs, unsigned long long tile_lo,
                                            unsigned long long tile_hi, const MapcLayout* lay, int u32_mode,
                                            unsigned long long* keys, MapcCtrl* ctrl, int n_sms, uint32_t nreg,
                                            uint32_t max_emits, uint32_t force_compact, uint32_t mode, void* tab,
                                            uint32_t cell_bytes, cudaStream_t s) {
  if (tile_hi <= tile_lo) return cudaSuccess;
  const unsigned long long total_tiles = tile_hi - tile_lo;
  const size_t wb = u32_mode ? 4 : 8;
  const size_t smem = ((size_t)nreg * MAPC_GEN_V * MAPC_GEN_THREADS * wb + 15) / 16 * 16 +
                      (size_t)MAPC_GEN_V * max_emits * MAPC_GEN_THREADS * 8;
  const void* fn = u32_mode ? (const void*)mapk::k_generate2<uint32_t> : (const void*)mapk::k_generate2<uint64_t>;
  static size_t attr[2] = {0, 0};
  // opt in above 32 KiB: the default 48 KiB limit also covers the static shared variables
  if (smem > 32 * 1024 && attr[u32_mode ? 0 : 1] < smem) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[u32_mode ? 0 : 1] = smem;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, MAPC_GEN_THREADS, smem);
  if (occ < 1) occ = 1;
  unsigned long long cap = (unsigned long long)n_sms * occ;
  int grid = (int)(total_tiles < cap ? total_tiles : cap);
  void* args[] = {(void*)&segs, (void*)&n_segs, (void*)&tile_lo, (void*)&tile_hi, (void*)lay, (void*)&keys,
                  (void*)&ctrl, (void*)&nreg, (void*)&force_compact, (void*)&mode, (void*)&tab, (void*)&cell_bytes};
  return cudaLaunchKernel(fn, dim3(grid), dim3(MAPC_GEN_THREADS), args, smem, s);
}
