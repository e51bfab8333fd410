// generate.cu -- K1: enumerate the access values of a chunk as packed u64 keys.
//
// One GPU thread per tuple (block, tid, k_0..k_{L-1}) of a group's bounding
// box (north_star mapping).  The thread decodes its tuple by mixed radix
// (invariant-divisor multiplies), runs the group's straight-line program from
// __constant__ memory -- the data-free image of rules seq/if/for of
// PAPER.md:506-551 with the par union of PAPER.md:579-589 made explicit as the
// tid coordinate -- and emits one key per access whose guards hold:
//   key = [lphase | array | lblock | index - idx_lo][tid][kind]
// Keys of a CTA iteration are compacted in shared memory and reserved with one
// global atomicAdd per CTA iteration (block-aggregated compaction), then
// stored with coalesced 16-byte stores.
#include "common.cuh"

namespace mapk {

__constant__ MapcOp c_ops[MAPC_MAX_OPS];

constexpr int GEN_THREADS = 128;

template <typename W>
struct VmWidth;
template <>
struct VmWidth<uint32_t> { static constexpr uint32_t bits = 32; };
template <>
struct VmWidth<uint64_t> { static constexpr uint32_t bits = 64; };

template <typename W>
__global__ void __launch_bounds__(GEN_THREADS)
k_generate(const MapcSeg* __restrict__ segs, int n_segs, unsigned long long total_tuples, MapcLayout lay,
           unsigned long long* __restrict__ keys, MapcCtrl* __restrict__ ctrl) {
  __shared__ W R[MAPC_NREG][GEN_THREADS];
  __shared__ unsigned long long stage[GEN_THREADS * MAPC_MAX_EMITS];
  __shared__ uint32_t scan_tmp[GEN_THREADS / 32 + 1];
  __shared__ unsigned long long s_base;
  constexpr uint32_t WB = VmWidth<W>::bits;
  const int me = threadIdx.x;
  uint32_t err = 0;

  for (unsigned long long base = (unsigned long long)blockIdx.x * GEN_THREADS; base < total_tuples;
       base += (unsigned long long)gridDim.x * GEN_THREADS) {
    const unsigned long long t = base + me;
    uint32_t cnt = 0;
    if (t < total_tuples) {
      // segment lookup: last s with tuple_begin <= t
      int lo = 0, hi = n_segs - 1;
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (segs[mid].tuple_begin <= t) lo = mid; else hi = mid - 1;
      }
      const MapcSeg& sg = segs[lo];
      uint32_t rem = (uint32_t)(t - sg.tuple_begin);
      const uint32_t L = sg.n_levels;
      for (int l = (int)L - 1; l >= 0; --l) {
        uint32_t q = fastdiv(rem, sg.trip_div[l]);
        R[MAPC_REG_K0 + l][me] = (W)(rem - q * sg.trip_div[l].d);
        rem = q;
      }
      uint32_t q = fastdiv(rem, sg.tid_div);
      const uint32_t tid = rem - q * sg.tid_div.d;
      const uint32_t bid = sg.b0 + q;
      const uint32_t lb = sg.lb0 + q;
      R[MAPC_REG_TID][me] = (W)tid;
      R[MAPC_REG_BID][me] = (W)bid;
      bool act = true;
      for (uint32_t pc = sg.prog_begin; pc < sg.prog_end; ++pc) {
        const MapcOp op = c_ops[pc];
        const uint32_t code = op.code & MAPC_CODE_MASK;
        const W A = (op.code & MAPC_A_IMM) ? (W)op.imm : R[op.a][me];
        const W B = (op.code & MAPC_B_IMM) ? (W)op.imm : R[op.b][me];
        W d = 0;
        switch (code) {
          case VM_ADD: d = A + B; break;
          case VM_SUB: d = A > B ? A - B : W(0); break;
          case VM_MUL: d = A * B; break;
          case VM_DIV:
            if (B == 0) { if (act && (op.aux & MAPC_AUX_FAULT)) err |= MAPC_ERR_DIV0; d = 0; }
            else d = A / B;
            break;
          case VM_MOD:
            if (B == 0) { if (act && (op.aux & MAPC_AUX_FAULT)) err |= MAPC_ERR_DIV0; d = 0; }
            else d = A % B;
            break;
          case VM_SHL: d = B >= WB ? W(0) : W(A << B); break;
          case VM_SHR: d = B >= WB ? W(0) : W(A >> B); break;
          case VM_MIN: d = A < B ? A : B; break;
          case VM_MAX: d = A > B ? A : B; break;
          case VM_DIVM:
          case VM_MODM: {
            const uint32_t dv = (uint32_t)(op.imm >> 32), m = (uint32_t)op.imm;
            const uint32_t a32 = (uint32_t)A;
            const uint32_t h = __umulhi(m, a32);
            const uint32_t qq = (h + ((a32 - h) >> 1)) >> op.aux;
            d = code == VM_DIVM ? W(qq) : W(a32 - qq * dv);
            break;
          }
          case VM_BAND: d = A & (W)op.imm; break;
          case VM_EQ: d = A == B; break;
          case VM_NE: d = A != B; break;
          case VM_LT: d = A < B; break;
          case VM_LE: d = A <= B; break;
          case VM_GT: d = A > B; break;
          case VM_GE: d = A >= B; break;
          case VM_LAND: d = (A != 0) & (B != 0); break;
          case VM_LOR: d = (A != 0) | (B != 0); break;
          case VM_LNOT: d = A == 0; break;
          case VM_TRIP: {
            const W step = (op.aux & MAPC_AUX_CONST) ? (W)(op.aux & ~MAPC_AUX_CONST) : R[op.aux][me];
            const W span = B > A ? B - A : W(0);
            d = span == 0 ? W(0) : (step == 1 ? span : W((span - 1) / (step ? step : W(1)) + 1));
            break;
          }
          case VM_MADK: d = A + R[op.aux][me] * B; break;
          case VM_ACT: act = A != 0; break;
          case VM_MOVI: d = (W)op.imm; break;
          case VM_EMIT:
            if (act) {
              const unsigned long long idx = (unsigned long long)A - lay.idx_lo;
              if (lay.w_index < 64 && (idx >> lay.w_index) != 0) err |= MAPC_ERR_LAYOUT;
              const unsigned long long sf = sg.key_hi +
                                            ((unsigned long long)(op.aux >> 1) << (lay.w_block + lay.w_index)) +
                                            ((unsigned long long)lb << lay.w_index) + idx;
              stage[cnt * GEN_THREADS + me] = (sf << lay.pay_bits) | ((unsigned long long)tid << 1) | (op.aux & 1u);
              ++cnt;
            }
            break;
          default: break;
        }
        if (code != VM_EMIT && code != VM_ACT) R[op.dst][me] = d;
      }
    }
    // block-aggregated compaction
    uint32_t total;
    const uint32_t excl = block_excl_scan<GEN_THREADS>(cnt, scan_tmp, &total);
    if (me == 0) s_base = total ? atomicAdd(&ctrl->n, (unsigned long long)total) : 0ull;
    __syncthreads();
    const unsigned long long obase = s_base;
    // local keys -> compacted order in `stage` is per-thread strided; write directly
    for (uint32_t j = 0; j < cnt; ++j) {
      const unsigned long long pos = obase + excl + j;
      if (pos < lay.cap) keys[pos] = stage[j * GEN_THREADS + me];
      else err |= MAPC_ERR_CAPACITY;
    }
    __syncthreads();
  }
  if (err) atomicOr(&ctrl->err, err);
}

}  // namespace mapk

// --------------------------------------------------------------- launchers --
extern "C" cudaError_t mapc_upload_ops(const MapcOp* host_ops, size_t n_ops, cudaStream_t s) {
  if (n_ops == 0) return cudaSuccess;
  return cudaMemcpyToSymbolAsync(mapk::c_ops, host_ops, n_ops * sizeof(MapcOp), 0, cudaMemcpyHostToDevice, s);
}

extern "C" cudaError_t mapc_launch_generate(const MapcSeg* segs, int n_segs, unsigned long long total_tuples,
                                            const MapcLayout* lay, int u32_mode, unsigned long long* keys,
                                            MapcCtrl* ctrl, int n_sms, cudaStream_t s) {
  if (total_tuples == 0) return cudaSuccess;
  unsigned long long want = (total_tuples + mapk::GEN_THREADS - 1) / mapk::GEN_THREADS;
  unsigned long long cap = (unsigned long long)n_sms * 8;
  int grid = (int)(want < cap ? want : cap);
  if (u32_mode)
    mapk::k_generate<uint32_t><<<grid, mapk::GEN_THREADS, 0, s>>>(segs, n_segs, total_tuples, *lay, keys, ctrl);
  else
    mapk::k_generate<uint64_t><<<grid, mapk::GEN_THREADS, 0, s>>>(segs, n_segs, total_tuples, *lay, keys, ctrl);
  return cudaGetLastError();
}
