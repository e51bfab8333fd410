// jit.cpp -- specialised generate kernels: the chunk's bytecode lowered to
// straight-line CUDA C and compiled with NVRTC for sm_100a at first use.
//
// The bytecode stays the compiler's output and the VM
// (k_generate2) stays available (MAPC_GEN=vm).  The JIT removes the
// interpreter's per-op dispatch and shared-memory register file: constants
// (parameters, forS values, layout widths) become literals, divisions by
// constants become multiply-shift sequences chosen by the compiler, and each
// tuple's registers live in real registers.  Tuple -> key semantics, tile
// mapping, dense slots and guarded-segment compaction are exactly those of
// k_generate2 (generate.cu), so the key multiset is identical.
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdint>
#include <thread>
#include <cstring>
#include <map>
#include <set>
#include <tuple>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../compiler/compiler.h"
#include "../devabi.h"
#include "jit.h"

namespace mapj {
namespace {

std::string lit(uint64_t v, bool u32) {
  std::ostringstream o;
  o << "(W)" << v << (u32 ? "u" : "ull");
  return o.str();
}

std::string opnd(const MapcOp& op, bool a_side, bool u32) {
  const bool imm = a_side ? (op.code & MAPC_A_IMM) : (op.code & MAPC_B_IMM);
  if (imm) return lit(u32 ? (uint64_t)(uint32_t)op.imm : op.imm, u32);
  return "r[" + std::to_string(a_side ? op.a : op.b) + "]";
}

// Straight-line body of one group program for one tuple (variables in scope:
// W r[], bool act, bool valid, u32 tidv, u32 lbv, u32 e-counter, tuple index t).
// site_literal: EMIT expands to EMIT_SITE(k, index, array, kind) with the
// site's ordinal k as a literal (the paired direct mode keeps per-site state).
std::string program_body(const std::vector<MapcOp>& ops, bool u32, bool site_literal = false) {
  std::ostringstream s;
  int site = 0;
  const char* WB = u32 ? "32u" : "64u";
  for (const MapcOp& op : ops) {
    const uint32_t c = op.code & MAPC_CODE_MASK;
    const std::string A = opnd(op, true, u32), B = opnd(op, false, u32);
    const std::string D = "r[" + std::to_string(op.dst) + "]";
    switch (c) {
      case VM_ADD: s << D << " = " << A << " + " << B << ";\n"; break;
      case VM_SUB: s << "{ W a_ = " << A << ", b_ = " << B << "; " << D << " = a_ > b_ ? a_ - b_ : (W)0; }\n"; break;
      case VM_MUL: s << D << " = " << A << " * " << B << ";\n"; break;
      case VM_DIV:
      case VM_MOD: {
        const char* o = c == VM_DIV ? "/" : "%";
        s << "{ W a_ = " << A << ", b_ = " << B << "; ";
        if (op.aux & MAPC_AUX_FAULT) s << "if (b_ == 0 && act && valid) err |= " << MAPC_ERR_DIV0 << "u; ";
        s << D << " = b_ ? (W)(a_ " << o << " b_) : (W)0; }\n";
        break;
      }
      case VM_SHL: s << "{ W b_ = " << B << "; " << D << " = b_ >= " << WB << " ? (W)0 : (W)(" << A << " << b_); }\n"; break;
      case VM_SHR: s << "{ W b_ = " << B << "; " << D << " = b_ >= " << WB << " ? (W)0 : (W)(" << A << " >> b_); }\n"; break;
      case VM_MIN: s << "{ W a_ = " << A << ", b_ = " << B << "; " << D << " = a_ < b_ ? a_ : b_; }\n"; break;
      case VM_MAX: s << "{ W a_ = " << A << ", b_ = " << B << "; " << D << " = a_ > b_ ? a_ : b_; }\n"; break;
      case VM_BAND: s << D << " = " << A << " & " << lit(op.imm, u32) << ";\n"; break;
      case VM_EQ: s << D << " = (W)(" << A << " == " << B << ");\n"; break;
      case VM_NE: s << D << " = (W)(" << A << " != " << B << ");\n"; break;
      case VM_LT: s << D << " = (W)(" << A << " < " << B << ");\n"; break;
      case VM_LE: s << D << " = (W)(" << A << " <= " << B << ");\n"; break;
      case VM_GT: s << D << " = (W)(" << A << " > " << B << ");\n"; break;
      case VM_GE: s << D << " = (W)(" << A << " >= " << B << ");\n"; break;
      case VM_LAND: s << D << " = (W)((" << A << " != 0) & (" << B << " != 0));\n"; break;
      case VM_LOR: s << D << " = (W)((" << A << " != 0) | (" << B << " != 0));\n"; break;
      case VM_LNOT: s << D << " = (W)(" << A << " == 0);\n"; break;
      case VM_TRIP: {
        const std::string step = (op.aux & MAPC_AUX_CONST) ? lit(op.aux & ~MAPC_AUX_CONST, u32)
                                                           : "r[" + std::to_string(op.aux) + "]";
        s << "{ W a_ = " << A << ", b_ = " << B << ", st_ = " << step << "; W sp_ = b_ > a_ ? b_ - a_ : (W)0; "
          << D << " = sp_ == 0 ? (W)0 : (st_ == 1 ? sp_ : (W)((sp_ - 1) / (st_ ? st_ : (W)1) + 1)); }\n";
        break;
      }
      case VM_MADK: s << D << " = " << A << " + r[" << op.aux << "] * " << B << ";\n"; break;
      case VM_ACT: s << "act = " << A << " != 0;\n"; break;
      case VM_MOVI: s << D << " = " << lit(op.imm, u32) << ";\n"; break;
      case VM_EMIT:
        if (site_literal)
          s << "if (act && valid) { EMIT_SITE(" << site++ << ", " << A << ", " << (op.aux >> 1) << "ull, " << (op.aux & 1u)
            << "ull); }\n";
        else
          s << "if (act && valid) { EMIT_KEY(" << A << ", " << (op.aux >> 1) << "ull, " << (op.aux & 1u) << "ull); }\n"
            << "++e;\n";
        break;
      default: break;
    }
  }
  return s.str();
}

// Per EMIT site of a program: is its index "X + k" with X independent of the
// innermost loop coordinate k (register `inner`) and k entering once, additively?
// Then the cells of tuples t and t + h (k -> k + h, nothing else changed) are
// sf and sf + h (mod 2^32) and the paired generate needs no run-time test.
// Conservative taint walk over the straight-line program: 0 = independent of k,
// 1 = X + k, 2 = anything else.
std::vector<bool> unit_stride_sites(const std::vector<MapcOp>& ops, uint32_t inner) {
  uint8_t st[MAPC_NREG] = {};
  st[inner] = 1;
  std::vector<bool> out;
  for (const MapcOp& op : ops) {
    const uint32_t c = op.code & MAPC_CODE_MASK;
    const uint8_t a = (op.code & MAPC_A_IMM) ? 0 : st[op.a % MAPC_NREG];
    const uint8_t b = (op.code & MAPC_B_IMM) ? 0 : st[op.b % MAPC_NREG];
    uint8_t d;
    switch (c) {
      case VM_EMIT: out.push_back(a == 1); continue;
      case VM_ACT: continue;
      case VM_MOVI: d = 0; break;
      case VM_ADD: d = (a == 0 && b == 0) ? 0 : ((a == 1 && b == 0) || (a == 0 && b == 1)) ? 1 : 2; break;
      case VM_MADK: {
        const uint8_t x = st[op.aux % MAPC_NREG];
        d = (x == 0 && b == 0) ? a : 2;
        break;
      }
      case VM_TRIP: {
        const uint8_t x = (op.aux & MAPC_AUX_CONST) ? 0 : st[op.aux % MAPC_NREG];
        d = (a == 0 && b == 0 && x == 0) ? 0 : 2;
        break;
      }
      default: d = (a == 0 && b == 0) ? 0 : 2; break;
    }
    st[op.dst % MAPC_NREG] = d;
  }
  return out;
}

const char* kPrelude = R"(
typedef unsigned int u32;
typedef unsigned long long u64;
struct FD { u32 d, m, s, pow2; };
struct Seg {
  u64 tuple_begin, n_tuples, tile_begin, key_begin, key_hi;
  u32 prog_begin, prog_end, n_levels, b0, lb0, n_emits, dense, tid_inner;
  FD trip_div[8];
  FD tid_div;
};
__device__ __forceinline__ u32 fdiv(u32 n, const FD& f) {
  if (f.pow2) return n >> f.s;
  u32 hi = __umulhi(f.m, n);
  return (hi + ((n - hi) >> 1)) >> f.s;
}
// 16-bit cell code (devabi.h code16): constant-weight 3-of-7 codewords per 5-bit tid digit
__device__ __forceinline__ u32 cw7(u32 d) {
  const u64 w = d < 8 ? MAPC_CW7_W0_ : d < 16 ? MAPC_CW7_W1_ : d < 24 ? MAPC_CW7_W2_ : MAPC_CW7_W3_;
  return (u32)(w >> (7u * (d & 7u))) & 0x7Fu;
}
__device__ __forceinline__ u32 code16(u32 t, u32 kind) { return cw7(t & 31u) | (cw7((t >> 5) & 31u) << 7) | (kind << 14); }
// thread-block clusters: rank, barrier (all threads of every CTA), and a
// fire-and-forget OR into word `off` of CTA `rank`'s copy of `tab` (DSMEM)
__device__ __forceinline__ u32 cl_rank() { u32 r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_or(u32* tab, u32 rank, u32 off, u32 v) {
  const u32 local = (u32)__cvta_generic_to_shared(tab + off);
  u32 remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" :: "r"(remote), "r"(v) : "memory");
}
// nonzero iff a 16-bit cell of the word is racy (SWAR, same test as direct.cu racy16_word)
__device__ __forceinline__ u32 racy16w(u32 w) {
  const u32 g = 0x80808080u, one = 0x01010101u;
  u32 x = (w & 0x007F007Fu) | ((w << 1) & 0x7F007F00u) | g;
  x = (x & (x - one)) | g;
  x = (x & (x - one)) | g;
  x = (x & (x - one));
  return x & (((w >> 14) & 0x00010001u) * 0x7F7Fu);
}
// Block offset (within the segment) of tuple t: t / (blockDim * prod(trips)).
__device__ __forceinline__ u32 block_of(u32 t, const Seg& sg) {
  u32 rem = fdiv(t, sg.tid_div);
  for (u32 l = 0; l < sg.n_levels; ++l) rem = fdiv(rem, sg.trip_div[l]);
  return rem;
}
template <int T>
__device__ __forceinline__ u32 block_excl_scan(u32 v, u32* tmp, u32* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32 inc = v;
  for (int o = 1; o < 32; o <<= 1) { u32 x = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += x; }
  if (lane == 31) tmp[w] = inc;
  __syncthreads();
  if (w == 0) {
    u32 x = lane < T / 32 ? tmp[lane] : 0u, xi = x;
    for (int o = 1; o < 32; o <<= 1) { u32 y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
    if (lane < T / 32) tmp[lane] = xi - x;
    if (lane == T / 32 - 1) tmp[T / 32] = xi;
  }
  __syncthreads();
  u32 r = tmp[w] + inc - v;
  *total = tmp[T / 32];
  __syncthreads();
  return r;
}
)";

// The prelude with the 16-bit cell code's codeword constants (devabi.h).
std::string prelude() {
  std::ostringstream o;
  o << "#define MAPC_CW7_W0_ " << MAPC_CW7_W0 << "ull\n#define MAPC_CW7_W1_ " << MAPC_CW7_W1
    << "ull\n#define MAPC_CW7_W2_ " << MAPC_CW7_W2 << "ull\n#define MAPC_CW7_W3_ " << MAPC_CW7_W3 << "ull\n"
    << kPrelude;
  return o.str();
}

struct Module {
  cudaLibrary_t lib = nullptr;
  std::vector<cudaKernel_t> kernels;
};

std::mutex g_mu;
std::map<std::string, Module> g_cache;   // chunk_key -> loaded module (process-wide)

// Everything the generated source depends on, as raw bytes (cheaper than
// generating the source text to look a module up: e2e runs recompile per step).
template <typename T>
void put(std::string& k, const T& v) { k.append(reinterpret_cast<const char*>(&v), sizeof(T)); }
std::string chunk_key(const JitChunk& ch, bool u32, uint32_t mode, uint32_t cell_bytes) {
  std::string k;
  put(k, u32);
  put(k, mode);
  put(k, cell_bytes);
  put(k, ch.lay);
  put(k, ch.max_emits);
  put(k, ch.programs.size());
  for (const JitProgram& pg : ch.programs) {
    put(k, pg.prog_begin);
    put(k, pg.n_levels);
    put(k, pg.inner_range);
    put(k, pg.tid_inner);
    put(k, pg.ops.size());
    k.append(reinterpret_cast<const char*>(pg.ops.data()), pg.ops.size() * sizeof(MapcOp));
  }
  put(k, ch.segs.size());
  k.append(reinterpret_cast<const char*>(ch.segs.data()), ch.segs.size() * sizeof(MapcSeg));
  put(k, ch.comp);
  if (mode == MAPC_MODE_UNIT || mode == MAPC_MODE_UNITF) {
    put(k, ch.unit_cluster);
    put(k, ch.unit_threads);
    put(k, ch.n_blocks);
    put(k, ch.unit_segs.size());
    k.append(reinterpret_cast<const char*>(ch.unit_segs.data()), ch.unit_segs.size() * sizeof(MapcSeg));
  }
  return k;
}

// Mixed-radix decode of the tuple index `rem` (in scope) into r[tid], r[bid],
// r[k_l], tidv, lbv: (block, tid, k_0..k_{L-1}) with k_{L-1} fastest, or tid
// fastest when sg.tid_inner (a literal for baked segments, so one branch folds).
std::string decode_tuple(const JitProgram& pg, const std::string& ind) {
  std::ostringstream s;
  s << ind << "u32 tidv = 0;\n"
    << ind << "if (sg.tid_inner) { const u32 q = fdiv(rem, sg.tid_div); tidv = rem - q * sg.tid_div.d; rem = q; }\n";
  for (int l = (int)pg.n_levels - 1; l >= 0; --l)
    s << ind << "{ const u32 q = fdiv(rem, sg.trip_div[" << l << "]); r[" << MAPC_REG_K0 + l
      << "] = (W)(rem - q * sg.trip_div[" << l << "].d); rem = q; }\n";
  s << ind << "if (!sg.tid_inner) { const u32 q = fdiv(rem, sg.tid_div); tidv = rem - q * sg.tid_div.d; rem = q; }\n"
    << ind << "const u32 lbv = sg.lb0 + rem;\n"
    << ind << "r[" << MAPC_REG_TID << "] = (W)tidv; r[" << MAPC_REG_BID << "] = (W)(sg.b0 + rem);\n";
  return s.str();
}

// The tail of EMIT_KEY per generate mode (variables in scope: sf_, tidv, KIND,
// sg, e, t, cnt, stage, keys, me).
std::string emit_tail(uint32_t mode, uint32_t w_tid, int T) {
  std::ostringstream s;
  if (mode == MAPC_MODE_DIRECT) {
    // cell |= tid | (~tid & M) << wt | kind << 2wt  (direct.cu); fire-and-forget red.or
    s << "const u64 code_ = (u64)tidv | ((~(u64)tidv & TMASK) << " << w_tid << "u) | ((u64)(KIND) << " << 2 * w_tid
      << "u); atomicOr(reinterpret_cast<CELL*>(keys) + sf_, (CELL)code_); if (!sg.dense) ++cnt;";
  } else if (mode == MAPC_MODE_FILTER) {
    // matches are rare: warp-aggregated slot reservation, no staging, no CTA scan
    s << "{ const bool hit_ = sf_ == target; const u32 hm_ = __ballot_sync(__activemask(), hit_); "
         "if (hit_) { const u32 ln_ = me & 31u, ld_ = __ffs(hm_) - 1u; u64 b_ = 0; "
         "if (ln_ == ld_) b_ = atomicAdd(n_ctr, (u64)__popc(hm_)); b_ = __shfl_sync(hm_, b_, ld_); "
         "const u64 pos_ = b_ + __popc(hm_ & ((1u << ln_) - 1u)); "
         "if (pos_ < cap) keys[pos_] = (sf_ << PAY) | ((u64)tidv << 1) | (KIND); else err |= " << MAPC_ERR_CAPACITY
      << "u; } }";
  } else {
    s << "const u64 key_ = (sf_ << PAY) | ((u64)tidv << 1) | (KIND); "
         "if (sg.dense) keys[sg.key_begin + (u64)e * sg.n_tuples + t] = key_; "
         "else { stage[(size_t)cnt * " << T << " + me] = key_; ++cnt; }";
  }
  return s.str();
}

// Unit mode (MAPC_MODE_UNIT; SURVEY.md §8f NEXT-3 "detect in smem tables per
// unit ... fully on-chip"): races are intra-(phase, block) and
// shared arrays are per block (R10), so a (phase, block) unit whose
// cells (array, index) fit in shared memory is checked entirely on chip: one CTA
// clears the unit's table, runs every tuple of the unit's segments folding each
// access into its cell with a shared-memory atomicOr of the same cell code as the
// HBM table (direct.cu), scans the table (racy cells counted, the smallest racy
// sort field atomicMin-ed into ctrl->racy_sf) and moves to its next unit.  No
// table in HBM, no clear and no scan launch.  The witness cell's keys are
// re-emitted by the filter-mode kernel as on the HBM direct path.
std::string unit_kernel_source(const JitChunk& ch, int index, bool u32, uint32_t cell_bytes, bool filter) {
  // filter = MAPC_MODE_UNITF: re-emit the keys of the witness cell (sort field
  // *target_ptr) from the tuples of its unit only -- the unit-mode counterpart of
  // the filter generate, which would walk every tile of the chunk.
  std::ostringstream s;
  const MapcLayout& L = ch.lay;
  const uint32_t wu = L.w_array + L.w_index;
  const uint64_t cells = 1ull << wu;
  const uint64_t words = cell_bytes == 2 ? (cells + 1) / 2 : cells;
  const uint64_t nb = std::max<uint64_t>(ch.n_blocks, 1);
  const uint32_t wt = L.w_tid;
  const uint32_t hb = L.w_array + L.w_block + L.w_index;
  // cluster units (K > 1): the unit's table is spread over the shared memory of a
  // K-CTA thread-block cluster, CTA r holding words [r*WPC, (r+1)*WPC); an access
  // ORs into its word's owner through distributed shared memory (mapa +
  // red.shared::cluster); cluster barriers separate clear, fold and scan
  const uint32_t K = filter ? 1u : std::max(1u, ch.unit_cluster);
  const int T = filter ? MAPC_GEN_THREADS : (int)ch.unit_threads;
  const uint64_t wpc = words / K;
  const uint64_t words_k1 = (words + 31) / 32 * 32;   // K == 1: whole 32-word swizzle rows
  uint32_t log_wpc = 0;
  while ((1ull << log_wpc) < wpc) ++log_wpc;
  s << "extern \"C\" __global__ void __launch_bounds__(" << T << ") gen_" << index;
  if (filter)
    s << "(const unsigned long long* target_ptr, unsigned long long* keys, unsigned long long* n_ctr, "
         "unsigned long long cap, u32* err_flag) {\n";
  else
    s << "(unsigned long long n_units, unsigned long long* n_ctr, unsigned long long* racy_ctr, "
         "unsigned long long* racy_sf, u32* err_flag) {\n";
  s << "  typedef " << (u32 ? "u32" : "u64") << " W;\n"
    << "  const u32 WI = " << L.w_index << "u; (void)WI;\n"
    << "  const u64 IDX_LO = " << L.idx_lo << "ull;\n"
    << "  const u32 TMASK = " << (wt >= 32 ? 0xFFFFFFFFu : ((1u << wt) - 1u)) << "u; (void)TMASK;\n"
    << "  const int me = threadIdx.x;\n"
    << "  u32 err = 0, cnt = 0;\n";
  if (filter) {
    s << "  const unsigned long long target = *target_ptr;\n"
      << "  if (target == ~0ull) return;\n"
      << "  const u32 lph = " << (hb >= 64 ? "0u" : "(u32)(target >> " + std::to_string(hb) + "u)") << ";\n"
      << "  const u32 lb = (u32)((target >> WI) & " << ((1ull << L.w_block) - 1) << "ull);\n"
      << "  const u64 base_ = ((((u64)lph << " << L.w_array << "u) << " << L.w_block << "u) | lb) << " << L.w_index
      << "u;\n"
      << "  {\n";
  } else if (K == 1) {
    // one CTA per unit: the table's words are XOR-swizzled (word w lives at
    // w ^ ((w >> 5) & 31), a permutation inside each 32-word row, so the table is
    // padded to whole rows) -- column-wise sites (3a's transposed reads: lanes 16
    // words apart) spread over all 32 banks instead of 2; the scan zeroes each word
    // after reading it, so the table is cleared once per CTA, not per unit
    s << "  __shared__ __align__(16) u32 tab[" << words_k1 << "];\n"
      << "  const u32 crank_ = 0u; (void)crank_;\n"
      << "  unsigned long long racy = 0, best = ~0ull;\n"
      << "  for (u32 i = me; i < " << words_k1 << "u; i += " << T << "u) tab[i] = 0u;\n"
      << "  __syncthreads();\n"
      << "  for (unsigned long long u = blockIdx.x; u < n_units; u += gridDim.x) {\n"
      << "    const u32 lph = (u32)(u / " << nb << "ull), lb = (u32)(u % " << nb << "ull);\n";
  } else {
    s << "  extern __shared__ u32 tab[];        // this CTA's " << wpc << " words of the unit table\n"
      << "  const u32 crank_ = cl_rank();\n"
      << "  unsigned long long racy = 0, best = ~0ull;\n"
      << "  for (unsigned long long u = blockIdx.x / " << K << "u; u < n_units; u += gridDim.x / " << K << "u) {\n"
      << "    const u32 lph = (u32)(u / " << nb << "ull), lb = (u32)(u % " << nb << "ull);\n"
      << "    for (u32 i = me; i < " << wpc << "u; i += " << T << "u) tab[i] = 0u;\n"
      << "    cl_sync();\n";
  }
  s << "#define EMIT_KEY(IX, ARR, KIND) { u64 idx_ = (u64)(IX) - IDX_LO; "
       "if (WI < 64 && (idx_ >> WI) != 0) { err |= " << MAPC_ERR_LAYOUT << "u; idx_ = 0; } ";
  if (filter) {
    // the access's sort field; matches are appended (warp-aggregated slot reservation)
    s << "const u64 sf_ = base_ + ((u64)(ARR) << " << L.w_block + L.w_index << "u) + idx_; "
         "const bool hit_ = sf_ == target; const u32 hm_ = __ballot_sync(__activemask(), hit_); "
         "if (hit_) { const u32 ln_ = me & 31u, ld_ = __ffs(hm_) - 1u; u64 b_ = 0; "
         "if (ln_ == ld_) b_ = atomicAdd(n_ctr, (u64)__popc(hm_)); b_ = __shfl_sync(hm_, b_, ld_); "
         "const u64 pos_ = b_ + __popc(hm_ & ((1u << ln_) - 1u)); "
         "if (pos_ < cap) keys[pos_] = (sf_ << " << L.pay_bits << "u) | ((u64)tidv << 1) | (KIND); else err |= "
      << MAPC_ERR_CAPACITY << "u; } }\n";
  } else {
    // the unit-local cell of an access: (array, index - idx_lo)
    s << "const u32 c_ = ((u32)(ARR) << WI) | (u32)idx_; ";
    const std::string w = cell_bytes == 2 ? "(c_ >> 1)" : "c_";
    const std::string v = cell_bytes == 2 ? "(tcd_ | ((u32)(KIND) << 14)) << (16u * (c_ & 1u))"
                                          : "tidv | ((~tidv & TMASK) << " + std::to_string(wt) + "u) | ((u32)(KIND) << " +
                                                std::to_string(2 * wt) + "u)";
    if (K == 1)
      s << "{ const u32 w_ = " << w << "; atomicOr(&tab[w_ ^ ((w_ >> 5) & 31u)], " << v << "); } ";
    else
      s << "cl_or(tab, " << w << " >> " << log_wpc << "u, " << w << " & " << wpc - 1 << "u, " << v << "); ";
    s << "if (!sg.dense) ++cnt; }\n";
  }
  auto fd = [](const MapcFastDiv& f) {
    std::ostringstream o;
    o << "{" << f.d << "u, " << f.m << "u, " << f.s << "u, " << f.pow2 << "u}";
    return o.str();
  };
  for (const MapcSeg& g : ch.unit_segs) {
    const JitProgram* pg = nullptr;
    for (const JitProgram& p : ch.programs)
      if (p.prog_begin == g.prog_begin) pg = &p;
    if (!pg) continue;
    uint64_t tpb = g.tid_div.d;        // tuples per block of the segment: blockDim * prod(trips)
    for (uint32_t l = 0; l < g.n_levels; ++l) tpb *= g.trip_div[l].d;
    const uint64_t seg_nb = g.n_tuples / std::max<uint64_t>(tpb, 1);
    const uint32_t seg_lph = hb >= 64 ? 0u : (uint32_t)(g.key_hi >> hb);
    s << "    if (lph == " << seg_lph << "u && lb >= " << g.lb0 << "u && lb < " << (uint64_t)g.lb0 + seg_nb << "ull) {\n"
      << "      const Seg sg = {" << g.tuple_begin << "ull, " << g.n_tuples << "ull, " << g.tile_begin << "ull, "
      << g.key_begin << "ull, " << g.key_hi << "ull, " << g.prog_begin << "u, " << g.prog_end << "u, " << g.n_levels
      << "u, " << g.b0 << "u, " << g.lb0 << "u, " << g.n_emits << "u, " << g.dense << "u, " << g.tid_inner << "u, {";
    for (int l = 0; l < 8; ++l) s << (l ? ", " : "") << fd(g.trip_div[l]);
    s << "}, " << fd(g.tid_div) << "};\n"
      << "      const u32 t0 = (lb - " << g.lb0 << "u) * " << tpb << "u;\n";
    // Four consecutive tuples per thread when the innermost coordinate's range is a
    // multiple of 4: they differ only in that coordinate (no carry), so the tuple
    // is decoded once and NVRTC shares everything that does not depend on it.
    const bool tid_is_inner = pg->tid_inner || pg->n_levels == 0;
    const bool quad = pg->inner_range % 4 == 0 && tpb % 4 == 0;
    const uint32_t inner_reg = tid_is_inner ? MAPC_REG_TID : MAPC_REG_K0 + pg->n_levels - 1;
    const uint32_t step = quad ? 4 : 1;
    const std::string first = filter ? "(blockIdx.x * " + std::to_string(T) + "u + me) * " + std::to_string(step) + "u"
                                     : "(crank_ * " + std::to_string(T) + "u + me) * " + std::to_string(step) + "u";
    const std::string stride = filter ? "gridDim.x * " + std::to_string(T * step) + "u"
                                      : std::to_string((uint64_t)K * T * step) + "u";
    s << "#pragma unroll 1\n"
      << "      for (u32 k = " << first << "; k < " << tpb << "u; k += " << stride << ") {\n"
      << "        const u32 t = t0 + k; (void)t;\n"
      << "        const bool valid = true;\n"
      << "        u32 rem = t;\n"
      << "        W r[" << MAPC_NREG << "];\n"
      << decode_tuple(*pg, "        ");
    if (quad) {
      s << "        const W c0_ = r[" << inner_reg << "];\n"
        << "        const u32 tid0_ = tidv;\n"
        << "#pragma unroll\n"
        << "        for (u32 h_ = 0; h_ < 4u; ++h_) {\n";
      if (tid_is_inner) s << "        tidv = tid0_ + h_;\n";
      s << "        r[" << inner_reg << "] = c0_ + (W)h_;\n";
    } else {
      s << "        {\n";
    }
    if (cell_bytes == 2 && !filter) s << "        const u32 tcd_ = code16(tidv, 0u);\n";
    s << "        bool act = true;\n"
      << "        u32 e = 0;\n"
      << program_body(pg->ops, u32)
      << "        (void)act; (void)e; (void)lbv;\n"
      << (quad ? "        }\n        (void)tid0_;\n" : "        }\n")
      << "      }\n"
      << "    }\n";
  }
  s << "#undef EMIT_KEY\n";
  if (filter) {
    s << "  }\n"
      << "  (void)cnt;\n"
      << "  if (err) atomicOr(err_flag, err);\n"
      << "}\n";
    return s.str();
  }
  s << (K == 1 ? "    __syncthreads();\n" : "    cl_sync();\n")
    << "    const u64 base_ = ((((u64)lph << " << L.w_array << "u) << " << L.w_block << "u) | lb) << " << L.w_index
    << "u;\n"
    ;
  const bool pairs = K == 1 && cell_bytes == 2;   // two words per 8-byte shared load (and clear)
  if (pairs)
    s << "    for (u32 il2 = me; il2 < " << words_k1 / 2 << "u; il2 += " << T << "u) {\n"
      << "      const unsigned long long w2 = reinterpret_cast<unsigned long long*>(tab)[il2];\n"
      << "      reinterpret_cast<unsigned long long*>(tab)[il2] = 0ull;\n"
      << "      if (!(racy16w((u32)w2) | racy16w((u32)(w2 >> 32)))) continue;\n"
      << "#pragma unroll\n"
      << "      for (u32 p_ = 0; p_ < 2u; ++p_) {\n"
      << "      const u32 il = 2u * il2 + p_;\n"
      << "      const u32 i = il ^ ((il >> 5) & 31u);   // the word's index in the unit table (unswizzled)\n"
      << "      const u32 w = (u32)(w2 >> (32u * p_));\n";
  else
    s << "    for (u32 il = me; il < " << (K == 1 ? words_k1 : wpc) << "u; il += " << T << "u) {\n"
      << (K == 1 ? "      const u32 i = il ^ ((il >> 5) & 31u);   // the word's index in the unit table (unswizzled)\n"
                 : "      const u32 i = crank_ * " + std::to_string(wpc) + "u + il;      // the word's index in the unit table\n")
      << "      const u32 w = tab[il];\n"
      << (K == 1 ? "      tab[il] = 0u;\n" : "")
      << (cell_bytes == 2 ? "      if (!racy16w(w)) continue;\n" : "      if (!w) continue;\n");
  // cell c = (array, index) -> sort field base_ + (array << (wB + wI)) + index
  auto cell_sf = [&](const std::string& c) {
    return "(base_ + (((u64)(" + c + ") >> " + std::to_string(L.w_index) + "u) << " +
           std::to_string(L.w_block + L.w_index) + "u) + ((u64)(" + c + ") & " +
           std::to_string(L.w_index >= 32 ? 0xFFFFFFFFull : ((1ull << L.w_index) - 1)) + "ull))";
  };
  if (cell_bytes == 2) {
    // racy16w's byte lanes 0-1 belong to the word's first cell, 2-3 to its second
    s << "      const u32 rw_ = racy16w(w);\n"
      << "#pragma unroll\n"
      << "      for (u32 h = 0; h < 2u; ++h) {\n"
      << "        if ((rw_ >> (16u * h)) & 0xFFFFu) {\n"
      << "          ++racy; const u64 sf = " << cell_sf("2u * i + h") << "; best = sf < best ? sf : best; }\n"
      << "      }\n";
    if (pairs) s << "      }\n";   // p_
  } else {
    s << "      if (((w >> " << 2 * wt << "u) & 1u) && (w & (w >> " << wt << "u) & TMASK)) {\n"
      << "        ++racy; const u64 sf = " << cell_sf("i") << "; best = sf < best ? sf : best; }\n";
  }
  s << "    }\n"
    << (K == 1 ? "    __syncthreads();\n" : "")
    << "  }\n"
    << "#pragma unroll\n"
    << "  for (int o = 16; o; o >>= 1) {\n"
    << "    racy += __shfl_xor_sync(0xffffffffu, racy, o);\n"
    << "    const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, best, o); best = b2 < best ? b2 : best;\n"
    << "    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);\n"
    << "  }\n"
    << "  if ((me & 31) == 0) {\n"
    << "    if (racy) atomicAdd(racy_ctr, racy);\n"
    << "    if (best != ~0ull) atomicMin(racy_sf, best);\n"
    << "    if (cnt) atomicAdd(n_ctr, (unsigned long long)cnt);\n"
    << "  }\n"
    << "  if (err) atomicOr(err_flag, err);\n"
    << "}\n";
  return s.str();
}

// Row-jam rows per thread for a direct-mode chunk of 16-bit cells (paired_case):
// every baked segment's program has a second-innermost loop (rows) and a
// multiple-of-4 innermost range L dividing or divisible by the 512-tuple tile, the
// segment is whole super-tiles of JU tiles and its row count is a multiple of JU
// (a thread's rows never cross that loop's carry).  The largest JU in {16, 8, 4,
// 2} that holds for every segment, else 0.  MAPC_JAM=0 disables, MAPC_JAM=n caps.
// Site pairs (k, k2) of a program such that site k of row r + 1 is site k2 of
// row r (same array, same index) at every sampled tuple where both are active and
// at least one: the only pairs the row-jam compares at run time (the comparison
// itself keeps it exact -- a pair that does not hold at some tuple just does not
// merge there).  Sampled with the host evaluator of the bytecode.
std::vector<std::pair<int, int>> jam_pairs(const JitProgram& pg, const MapcSeg& g) {
  std::vector<std::pair<int, int>> out;
  std::vector<uint32_t> arr;
  for (const MapcOp& op : pg.ops)
    if ((op.code & MAPC_CODE_MASK) == VM_EMIT) arr.push_back(op.aux >> 1);
  const int ne = (int)arr.size();
  if (pg.n_levels < 2 || ne == 0) return out;
  const uint64_t nt = g.tid_div.d, rows = g.trip_div[pg.n_levels - 2].d, L = g.trip_div[pg.n_levels - 1].d;
  if (rows < 2) return out;
  std::vector<std::vector<int>> hold(ne, std::vector<int>(ne, 0));   // 0 unseen, 1 held, -1 broken
  const uint64_t tids[] = {0, 1, nt / 2, nt - 1};
  const uint64_t rs[] = {0, 1 % (rows - 1), (rows / 2) % (rows - 1), rows - 2};   // r + 1 < rows
  const uint64_t cs[] = {0, 4 % L, (L / 2) / 4 * 4, (L - 4) % L};
  std::vector<int64_t> a, b;
  for (uint64_t tid : tids)
    for (uint64_t r : rs)
      for (uint64_t c : cs) {
        uint64_t k0[MAPC_MAX_LEVELS] = {}, k1[MAPC_MAX_LEVELS] = {};
        k0[pg.n_levels - 2] = r;
        k1[pg.n_levels - 2] = r + 1;
        k0[pg.n_levels - 1] = k1[pg.n_levels - 1] = c;
        mapc::eval_ops_sites(pg.ops, pg.n_levels, tid % nt, g.b0, k0, &a);
        mapc::eval_ops_sites(pg.ops, pg.n_levels, tid % nt, g.b0, k1, &b);
        for (int k = 0; k < ne && k < (int)b.size(); ++k)
          for (int k2 = 0; k2 < ne && k2 < (int)a.size(); ++k2) {
            if (b[k] < 0 || a[k2] < 0 || hold[k][k2] < 0) continue;
            hold[k][k2] = (b[k] == a[k2] && arr[k] == arr[k2]) ? 1 : -1;
          }
      }
  for (int k = 0; k < ne; ++k)
    for (int k2 = 0; k2 < ne; ++k2)
      if (hold[k][k2] == 1) out.emplace_back(k, k2);
  return out;
}

uint32_t jam_rows(const JitChunk& ch) {
  static const int env = [] { const char* e = getenv("MAPC_JAM"); return e ? atoi(e) : 16; }();
  if (env < 2 || ch.segs.empty() || ch.lay.sort_bits > 31) return 0;
  for (uint32_t U = 16; U >= 2; U /= 2) {
    if ((int)U > env) continue;
    bool ok = true;
    for (const MapcSeg& g : ch.segs) {
      const JitProgram* pg = nullptr;
      for (const JitProgram& p : ch.programs)
        if (p.prog_begin == g.prog_begin) pg = &p;
      if (!pg || pg->n_levels < 2 || pg->tid_inner || g.tid_inner || g.n_levels != pg->n_levels) { ok = false; break; }
      const uint64_t L = pg->inner_range;
      const uint64_t rows = g.trip_div[pg->n_levels - 2].d;
      ok = L % 4 == 0 && g.trip_div[pg->n_levels - 1].d == L && (L <= MAPC_GEN_TILE ? MAPC_GEN_TILE % L == 0
                                                                                   : L % MAPC_GEN_TILE == 0) &&
           rows % U == 0 && g.n_tuples % ((uint64_t)MAPC_GEN_TILE * U) == 0 && g.tile_begin % U == 0 &&
           g.n_tuples < (1ull << 32) && !jam_pairs(*pg, g).empty();   // something to merge
      if (!ok) break;
    }
    if (ok) return U;
  }
  return 0;
}

}  // namespace

bool jam_active(const JitChunk& ch, uint32_t cell_bytes) {
  static const bool blocked_env = [] { const char* e = getenv("MAPC_BLOCKED_TILES"); return !(e && e[0] == '0'); }();
  return cell_bytes == 2 && blocked_env && jam_rows(ch) != 0;
}

std::string chunk_kernel_source(const JitChunk& ch, int index, bool u32, uint32_t mode, uint32_t cell_bytes) {
  static_assert(sizeof(MapcSeg) == 5 * 8 + 8 * 4 + 9 * 16, "Seg layout mirrored in the JIT prelude");
  if (mode == MAPC_MODE_UNIT || mode == MAPC_MODE_UNITF)
    return unit_kernel_source(ch, index, u32, cell_bytes, mode == MAPC_MODE_UNITF);
  std::ostringstream s;
  const int T = MAPC_GEN_THREADS, V = MAPC_GEN_V;
  // keys staged per thread per tile for compaction: the guarded segments' emits
  // (keys mode), every segment's (filter mode), none (direct mode)
  const bool paired = mode == MAPC_MODE_DIRECT && (cell_bytes == 4 || cell_bytes == 2);
  // Direct mode: every CTA walks a contiguous block of tiles (instead of a grid
  // stride), so the cells a CTA re-touches (stencil rows r-1, r, r+1) stay in L2
  // between its tiles: the table's DRAM traffic drops to the algorithmic read +
  // write of every cell (profiles/r1k_stencil_red_microbench.txt), which leaves
  // HBM bandwidth to the overlapped scans.  MAPC_BLOCKED_TILES=0 restores the stride.
  static const bool blocked_env = [] { const char* e = getenv("MAPC_BLOCKED_TILES"); return !(e && e[0] == '0'); }();
  const bool blocked = mode == MAPC_MODE_DIRECT && blocked_env;
  const uint32_t stage_emits = V * (mode == MAPC_MODE_DIRECT   ? 1u
                                    : mode == MAPC_MODE_FILTER ? 1u
                                                               : std::max(1u, ch.max_emits));
  // direct mode: minimum resident CTAs per SM (register cap 48): 10 measured best
  // on 5a with the blocked, carry-free paired generate (profiles/r1q_probe_minb.txt);
  // MAPC_JIT_MINB overrides (0 = none)
  static const int minb_env = [] { const char* e = getenv("MAPC_JIT_MINB"); return e ? atoi(e) : 10; }();
  // (A per-thread 4-entry cache of aligned quads, which halves 5a's global
  // red.or.b64 count by folding the three reads of a row in registers, was
  // measured 25% SLOWER: the direct generate is bound by the table's DRAM
  // read-modify-write traffic, not by the reduction count -- DESIGN.md §6.1.)
  const int minb = mode == MAPC_MODE_DIRECT ? minb_env : 0;
  const uint32_t JU = paired && blocked && cell_bytes == 2 ? jam_rows(ch) : 0u;   // row-jam (paired_case), 0 = off
  s << "extern \"C\" __global__ void __launch_bounds__(" << T;
  if (minb > 0) s << ", " << minb;
  s << ") gen_" << index
    << "(const Seg* __restrict__ segs, int n_segs, u64 total_tiles, u64* __restrict__ keys, u64* n_ctr, u32* err_flag, "
       "u64 cap, const u64* target_ptr, const u64* __restrict__ pcomp_) {\n"
    << "  (void)pcomp_;\n"
    << "  typedef " << (u32 ? "u32" : "u64") << " W;\n"
    << "  typedef " << (cell_bytes == 4 ? "u32" : "u64") << " CELL;\n"
    << "  const u32 WI = " << ch.lay.w_index << "u, WB_ = " << ch.lay.w_block << "u, PAY = " << ch.lay.pay_bits << "u;\n"
    << "  const u32 WA_ = " << ch.lay.w_array << "u; (void)WA_;\n"
    << "  const u64 IDX_LO = " << ch.lay.idx_lo << "ull;\n"
    << "  __shared__ u64 stage[" << stage_emits << " * " << T << "];\n"
    << "  __shared__ u32 scan_tmp[" << T / 32 + 1 << "];\n"
    << "  __shared__ u64 s_base;\n"
    << "  const int me = threadIdx.x;\n"
    << "  u32 err = 0;\n"
    << "  unsigned long long cnt_all_ = 0; (void)cnt_all_;\n"
    << "  const u64 TMASK = " << (ch.lay.w_tid >= 64 ? ~0ull : ((1ull << ch.lay.w_tid) - 1)) << "ull;\n"
    << "  (void)TMASK; (void)target_ptr;\n";
  // sort fields below 2^31 (5a: 29 bits): 32-bit cell arithmetic in the paired case
  const bool sf32 = ch.lay.sort_bits <= 31;
  if (paired)   // one set for every case: per-case arrays inflate the register allocation per switch case
    s << "  " << (sf32 ? "u32" : "u64") << " sfP[" << MAPC_MAX_EMITS << "]; u32 cdP[" << MAPC_MAX_EMITS
      << "]; bool okP[" << MAPC_MAX_EMITS << "]; u64 accP[" << MAPC_MAX_EMITS << "]; (void)cdP; (void)accP;\n";
  // row-jam: the previous row's quads.  Every slot is defined before the first row:
  // a site that does not emit leaves its slot unwritten, and the row-to-row copy
  // of an indeterminate value let NVRTC fold the loop-carried state wrongly
  // (random row MAPs lost or misplaced codes until these were initialised)
  if (JU)
    s << "  u32 sfQ[" << MAPC_MAX_EMITS << "]; bool okQ[" << MAPC_MAX_EMITS << "]; u64 accQ[" << MAPC_MAX_EMITS << "];\n"
      << "#pragma unroll\n"
      << "  for (int k = 0; k < " << MAPC_MAX_EMITS << "; ++k) { sfQ[k] = 0u; okQ[k] = false; accQ[k] = 0ull; "
         "sfP[k] = 0u; okP[k] = false; accP[k] = 0ull; }\n";
  if (mode == MAPC_MODE_FILTER)
    s << "  const u64 target = *target_ptr;\n"
      << "  if (target == ~0ull) return;\n";
  // (L2 eviction-priority hints -- evict-last on these reductions, evict-first on the
  // concurrent scan and clear -- were measured without effect: profiles/r2r_l2_hints_ab.jsonl)
  if (JU)   // row-jam: every CTA walks a contiguous block of super-tiles (JU tiles each)
    s << "  const u64 n_super_ = total_tiles / " << JU << "u;\n"
      << "  const u64 per_cta_ = (n_super_ + gridDim.x - 1) / gridDim.x;\n"
      << "  const u64 st_end_ = min(n_super_, (u64)(blockIdx.x + 1) * per_cta_);\n"
      << "  for (u64 st_ = (u64)blockIdx.x * per_cta_; st_ < st_end_; ++st_) {\n"
      << "    const u64 tile = st_ * " << JU << "u;\n";
  else
    s << (blocked ? "  const u64 per_cta_ = (total_tiles + gridDim.x - 1) / gridDim.x;\n"
                    "  const u64 tile_end_ = min(total_tiles, (u64)(blockIdx.x + 1) * per_cta_);\n"
                    "  for (u64 tile = (u64)blockIdx.x * per_cta_; tile < tile_end_; ++tile) {\n"
                  : "  for (u64 tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {\n");
  if (!ch.segs.empty()) {
    // baked segments: the tile's segment from the literal segment starts (no
    // dependent loads of segs[] per tile)
    s << "    int lo = 0";
    for (size_t i = 1; i < ch.segs.size(); ++i) s << " + (tile >= " << ch.segs[i].tile_begin << "ull)";
    s << "; (void)n_segs;\n";
  } else {
    s << "    int lo = 0, hi = n_segs - 1;\n"
      << "    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (segs[mid].tile_begin <= tile) lo = mid; else hi = mid - 1; }\n";
  }
  // Direct mode with u32 cells: every thread takes two CONSECUTIVE tuples
  // (t, t+1) of the tile; an access site whose two cells are adjacent and
  // 8-byte aligned (sf, sf + 1; sf even -- the unit-stride innermost loops of
  // row sweeps and stencils) is folded with ONE red.or.b64 of both codes,
  // otherwise with one red.or.b32 each.  The generate is bound by the rate of
  // memory instructions (profiles/r1h_red_width_microbench.txt: b32 2.9 TB/s of
  // payload, b64 4.0 TB/s with a DRAM-resident table), so pairing halves the
  // instructions on the common path.  Same cells, same codes: same table.
  auto paired_case = [&](std::ostringstream& s, const JitProgram& pg) {
    int ne = 0;
    for (const MapcOp& op : pg.ops) ne += (op.code & MAPC_CODE_MASK) == VM_EMIT;
    const int NE = std::max(ne, 1);
    // stride-compressed table (ch.comp, 16-bit cells, 32-bit cell indices): the
    // phase's block at cbase_, one cell per 2^csh_ indices of residue cres_
    const bool comp = ch.comp && cell_bytes == 2 && sf32 && mode == MAPC_MODE_DIRECT;
    const std::string cell =
        "u64 idx_ = (u64)(IX) - IDX_LO; if (WI < 64 && (idx_ >> WI) != 0) { err |= " +
        std::to_string(MAPC_ERR_LAYOUT) + "u; idx_ = 0; } " +
        (comp ? std::string("const u32 sf_ = cbase_ + ((((u32)(ARR) << WB_) | lbv) << (WI - csh_)) + "
                            "(((u32)idx_ - cres_) >> csh_); if (((u32)idx_ - cres_) & ((1u << csh_) - 1u)) err |= ") +
                    std::to_string(MAPC_ERR_LAYOUT) + "u; "
         : sf32 ? std::string("const u32 sf_ = (u32)sg.key_hi + ((u32)(ARR) << (WB_ + WI)) + (lbv << WI) + (u32)idx_; ")
                : std::string("const u64 sf_ = sg.key_hi + ((ARR) << (WB_ + WI)) + ((u64)lbv << WI) + idx_; ")) +
        (cell_bytes == 2 ? std::string("const u32 cd_ = tcd_ | ((u32)(KIND) << 14); ")
                         : "const u32 cd_ = tidv | ((~tidv & (u32)TMASK) << " + std::to_string(ch.lay.w_tid) +
                               "u) | ((u32)(KIND) << " + std::to_string(2 * ch.lay.w_tid) + "u); ") +
        "if (!sg.dense) ++cnt; ";
    // one cell's reduction: u32 cells are words; 16-bit cells are halves of a word
    auto red1 = [&](const std::string& sf, const std::string& cd) {
      return cell_bytes == 2 ? "atomicOr(reinterpret_cast<u32*>(keys) + (" + sf + " >> 1), " + cd + " << (16u * (u32)(" +
                                   sf + " & 1u)));"
                             : "atomicOr(reinterpret_cast<u32*>(keys) + " + sf + ", " + cd + ");";
    };
    // an aligned pair of adjacent cells: one 64-bit word of u32 cells, one 32-bit word of 16-bit cells
    const std::string red2 =
        cell_bytes == 2 ? "atomicOr(reinterpret_cast<u32*>(keys) + (sf_ >> 1), cdP[K] | (cd_ << 16));"
                        : "atomicOr(reinterpret_cast<u64*>(keys) + (sf_ >> 1), (u64)cdP[K] | ((u64)cd_ << 32));";
    // G consecutive tuples per thread: pairs of u32 cells (one red.or.b64), or
    // quads of 16-bit cells (one red.or.b64 over four cells)
    const int G = cell_bytes == 2 ? 4 : 2;
    // Row-jam (JU > 0, chunk-wide, jam_rows): a thread takes JU consecutive rows
    // (second-innermost coordinate) of one column quad instead of one quad per
    // tile; a cell the next row touches again (5a: a read-half row is read as
    // row r + 1, r and r - 1 of three successive rows) is ORed into that row's
    // quad in registers, and a quad is reduced into the table only when the next
    // row no longer touches it -- 5a: 0.25 -> (JU + 2 + JU) / (16 JU) global
    // red.or.b64 per access.  Same cells, same codes: the table is identical.
    const bool jam = JU != 0 && G == 4;
    const uint64_t L = pg.inner_range;
    const bool nocarry = pg.inner_range % (uint64_t)G == 0;
    const bool tid_is_inner = pg.tid_inner || pg.n_levels == 0;
    s << "    case " << pg.prog_begin << "u: {\n";
    if (comp)
      s << "      const u32 lphc_ = (u32)(sg.key_hi >> (WA_ + WB_ + WI));\n"
        << "      const u32 cbase_ = (u32)pcomp_[2 * lphc_];\n"
        << "      const u32 csh_ = (u32)(pcomp_[2 * lphc_ + 1] & 255ull), cres_ = (u32)(pcomp_[2 * lphc_ + 1] >> 8);\n";
    if (jam) {
      s << "      const u32 sl_ = (u32)((tile - sg.tile_begin) / " << JU << "u);\n";
      if (L <= 512)   // P = 512 / L rows per tile, L / 4 threads per row
        s << "      const u32 tq_ = (sl_ * " << JU * (512 / L) << "u + (u32)(me / " << L / 4 << ") * " << JU << "u) * " << L
          << "u + 4u * (u32)(me % " << L / 4 << ");\n";
      else            // S = L / 512 super-tiles per row block
        s << "      const u32 tq_ = (sl_ / " << L / 512 << "u) * " << JU * L << "u + (sl_ % " << L / 512
          << "u) * 512u + 4u * (u32)me;\n";
      s << "#pragma unroll\n"
        << "      for (int k = 0; k < " << NE << "; ++k) okQ[k] = false;\n"
        << "      bool valid0_; u32 tidv0_, lbv0_; W bid0_; W c0_[" << std::max(1u, pg.n_levels) << "];\n"
        << "      {\n"
        << "        const u32 t = tq_;\n"
        << "        const bool valid = true;\n"
        << "        u32 rem = t;\n"
        << "        W r[" << MAPC_NREG << "];\n"
        << decode_tuple(pg, "        ")
        << "        valid0_ = valid; tidv0_ = tidv; lbv0_ = lbv; bid0_ = r[" << MAPC_REG_BID << "];\n";
      for (uint32_t l = 0; l < pg.n_levels; ++l) s << "        c0_[" << l << "] = r[" << MAPC_REG_K0 + l << "];\n";
      s << "        (void)t;\n"
        << "      }\n"
        << "#pragma unroll 1\n"
        << "      for (u32 u_ = 0; u_ < " << JU << "u; ++u_) {\n"
        << "        const u32 tp = tq_ + u_ * " << L << "u; (void)tp;\n";
    } else {
      s << "#pragma unroll 1\n"
        << "      for (int v = 0; v < " << V / G << "; ++v) {\n"
        << "        const u32 tp = tl0 + v * " << G * T << "u + " << G << "u * me;\n";
    }
    s << "#pragma unroll\n"
      << "        for (int k = 0; k < " << NE << "; ++k) okP[k] = false;\n";
    // tuple t: remember each site's cell; tuple t + 1: one red.or.b64 when the
    // two cells are adjacent and aligned, else one red.or.b32 each
    // With an even innermost range, tuple t + 1 is tuple t with the innermost
    // coordinate + 1 (tp is even): its coordinates are copied, not decoded, so
    // NVRTC shares every value of the program that does not depend on that
    // coordinate between the two tuples.
    if (nocarry && !jam)
      s << "        bool valid0_; u32 tidv0_, lbv0_; W bid0_; W c0_[" << std::max(1u, pg.n_levels) << "];\n";
    // sites whose cell advances by exactly h from tuple 0 to tuple h (32-bit sort fields)
    std::vector<bool> us;
    if (G == 4 && nocarry && sf32)   // the coordinate that advances by h: tid or the innermost loop's
      us = unit_stride_sites(pg.ops, tid_is_inner ? MAPC_REG_TID : MAPC_REG_K0 + pg.n_levels - 1);
    us.resize(NE, false);
    // site pairs whose index is the same value (same register, not rewritten between
    // them, or the same literal) in the same array: their quads are merged in registers
    // before the flush, one red.or.b64 instead of two (4b/5b/2b: a read and a write of
    // the same cell by the same thread)
    std::vector<std::pair<int, int>> same_cell;
    if (G == 4) {
      std::vector<std::tuple<int, uint64_t, uint32_t, uint32_t>> site;   // (is_imm, reg/imm, version, array)
      std::vector<uint32_t> ver(MAPC_NREG, 0);
      for (const MapcOp& op : pg.ops) {
        const uint32_t c = op.code & MAPC_CODE_MASK;
        if (c == VM_EMIT) {
          const bool imm = op.code & MAPC_A_IMM;
          site.emplace_back(imm ? 1 : 0, imm ? op.imm : op.a, imm ? 0u : ver[op.a % MAPC_NREG], op.aux >> 1);
        } else if (c != VM_ACT) {
          ++ver[op.dst % MAPC_NREG];
        }
      }
      for (size_t a = 0; a < site.size(); ++a)
        for (size_t b = a + 1; b < site.size(); ++b)
          if (site[a] == site[b]) same_cell.emplace_back((int)a, (int)b);
    }
    s << "        constexpr bool US_[" << NE << "] = {";
    for (int k = 0; k < NE; ++k) s << (k ? ", " : "") << (us[k] ? "true" : "false");
    s << "}; (void)US_;\n";
    for (int h = 0; h < G; ++h) {
      s << "        {\n"
        << "          const u32 t = tp + " << h << "u;\n";
      if (jam || (h >= 1 && nocarry)) {
        s << "          const bool valid = valid0_;\n"
          << "          W r[" << MAPC_NREG << "];\n"
          << "          const u32 tidv = tidv0_" << (tid_is_inner ? " + " + std::to_string(h) + "u" : "") << ";\n"
          << "          const u32 lbv = lbv0_;\n"
          << "          r[" << MAPC_REG_TID << "] = (W)tidv; r[" << MAPC_REG_BID << "] = bid0_;\n";
        for (uint32_t l = 0; l < pg.n_levels; ++l)
          s << "          r[" << MAPC_REG_K0 + l << "] = c0_[" << l << "]"
            << (!tid_is_inner && l + 1 == pg.n_levels && h ? " + (W)" + std::to_string(h) : "")
            << (jam && l + 2 == pg.n_levels ? " + (W)u_" : "") << ";\n";
        s << "          (void)t;\n";
      } else {
        s << "          const bool valid = t < sg.n_tuples;\n"
          << "          u32 rem = valid ? t : 0u;\n"
          << "          W r[" << MAPC_NREG << "];\n"
          << decode_tuple(pg, "          ");
        if (h == 0 && nocarry) {
          s << "          valid0_ = valid; tidv0_ = tidv; lbv0_ = lbv; bid0_ = r[" << MAPC_REG_BID << "];\n";
          for (uint32_t l = 0; l < pg.n_levels; ++l) s << "          c0_[" << l << "] = r[" << MAPC_REG_K0 + l << "];\n";
        }
      }
      // the tid part of the 16-bit code once per tuple, outside the sites' guards
      // (inside them NVRTC re-derived it at every site: ~30 instructions each);
      // a 2 KB shared table of the codes instead made 3a/4b 20-30% slower (r1u)
      if (cell_bytes == 2) s << "          const u32 tcd_ = code16(tidv, 0u);\n";
      s << "          bool act = true;\n";
      if (G == 4) {      // quads of 16-bit cells: accumulate the run starting at tuple 0's cell
        if (h == 0)
          s << "#define EMIT_SITE(K, IX, ARR, KIND) { " << cell << "sfP[K] = sf_; accP[K] = (u64)cd_; okP[K] = true; }\n";
        else
          s << "#define EMIT_SITE(K, IX, ARR, KIND) { " << cell << "if (okP[K] && (US_[K] || sf_ == sfP[K] + " << h
            << "u)) accP[K] |= (u64)cd_ << " << 16 * h << "; else " << red1("sf_", "cd_") << " }\n";
      } else if (h == 0) {
        s << "#define EMIT_SITE(K, IX, ARR, KIND) { " << cell << "sfP[K] = sf_; cdP[K] = cd_; okP[K] = true; }\n";
      } else {
        s << "#define EMIT_SITE(K, IX, ARR, KIND) { " << cell
          << "if (okP[K] && sf_ == sfP[K] + 1 && !(sfP[K] & 1u)) { "
          << red2 << " okP[K] = false; } "
             "else " << red1("sf_", "cd_") << " }\n";
      }
      s << program_body(pg.ops, u32, true)
        << "#undef EMIT_SITE\n"
        << "          (void)act;\n"
        << "        }\n";
    }
    for (const auto& pr : same_cell)
      s << "        if (okP[" << pr.first << "] && okP[" << pr.second << "] && sfP[" << pr.first << "] == sfP["
        << pr.second << "]) { accP[" << pr.first << "] |= accP[" << pr.second << "]; okP[" << pr.second
        << "] = false; }\n";
    // one red.or.b64 over an aligned quad, else the run's cells one by one
    auto flush4 = [&](const std::string& ok, const std::string& sf, const std::string& acc) {
      return "#pragma unroll\n"
             "        for (int k = 0; k < " + std::to_string(ne) + "; ++k) {\n"
             "          if (" + ok + "[k]) {\n"
             "            if ((" + sf + "[k] & 3u) == 0) { atomicOr(reinterpret_cast<u64*>(keys) + (" + sf + "[k] >> 2), " +
             acc + "[k]); } else {\n"
             "#pragma unroll\n"
             "              for (int j = 0; j < 4; ++j) {\n"
             "                const u32 c_ = (u32)(" + acc + "[k] >> (16 * j)) & 0xFFFFu;\n"
             "                if (c_) { const u32 sj_ = " + sf + "[k] + (u32)j; " + red1("sj_", "c_") + " }\n"
             "              }\n"
             "            }\n"
             "          }\n"
             "        }\n";
    };
    if (jam) {
      // this row's quads absorb the previous row's quads on the same cells; the
      // previous row's others are final (the next row is compared with this one)
      const MapcSeg* g0 = nullptr;
      for (const MapcSeg& g : ch.segs)
        if (g.prog_begin == pg.prog_begin && !g0) g0 = &g;
      for (const auto& pr : g0 ? jam_pairs(pg, *g0) : std::vector<std::pair<int, int>>{})
        s << "        if (okP[" << pr.first << "] && okQ[" << pr.second << "] && sfP[" << pr.first << "] == sfQ["
          << pr.second << "]) { accP[" << pr.first << "] |= accQ[" << pr.second << "]; okQ[" << pr.second
          << "] = false; }\n";
      s << flush4("okQ", "sfQ", "accQ")
        << "#pragma unroll\n"
        << "        for (int k = 0; k < " << NE << "; ++k) { okQ[k] = okP[k]; sfQ[k] = sfP[k]; accQ[k] = accP[k]; }\n"
        << "      }\n"
        << flush4("okQ", "sfQ", "accQ")
        << "      break; }\n";
      return;
    }
    if (G == 4)
      s << flush4("okP", "sfP", "accP");
    else
      s << "#pragma unroll\n"
        << "        for (int k = 0; k < " << ne << "; ++k)\n"
        << "          if (okP[k]) " << red1("sfP[k]", "cdP[k]") << "\n";
    s << "      }\n"
      << "      break; }\n";
  };
  // the per-tile body, emitted once per baked segment (fields as literals) and
  // once generic (fields loaded from segs[])
  // (only_prog >= 0: a baked segment -- only its own program is emitted)
  auto tile_body = [&](std::ostringstream& s, int64_t only_prog) {
    s << "    const u32 tl0 = (u32)(tile - sg.tile_begin) * " << V * T << "u;\n";
    if (mode == MAPC_MODE_FILTER) {
      // the witness cell lies in one phase and one block: tiles of other phases
      // or whose blocks cannot contain it are skipped (uniform per CTA)
      const uint32_t hb = ch.lay.w_array + ch.lay.w_block + ch.lay.w_index;
      s << "    bool skip_ = false;\n";
      if (hb < 64) s << "    skip_ = (sg.key_hi >> " << hb << "u) != (target >> " << hb << "u);\n";
      if (ch.lay.w_block > 0)
        s << "    if (!skip_) {\n"
          << "      const u32 tlb_ = (u32)((target >> WI) & ((1ull << WB_) - 1ull));\n"
          << "      const u32 tl1_ = min(tl0 + " << V * T - 1 << "u, (u32)sg.n_tuples - 1u);\n"
          << "      skip_ = tlb_ < sg.lb0 + block_of(tl0, sg) || tlb_ > sg.lb0 + block_of(tl1_, sg);\n"
          << "    }\n";
      s << "    if (!skip_) {\n";
    }
    s << "    u32 cnt = 0;\n"
      << "#define EMIT_KEY(IX, ARR, KIND) { u64 idx_ = (u64)(IX) - IDX_LO; "
         "if (WI < 64 && (idx_ >> WI) != 0) { err |= " << MAPC_ERR_LAYOUT << "u; idx_ = 0; } "
         "const u64 sf_ = sg.key_hi + ((ARR) << (WB_ + WI)) + ((u64)lbv << WI) + idx_; "
         << emit_tail(mode, ch.lay.w_tid, T) << " }\n"
      << "    switch (sg.prog_begin) {\n";
    for (const JitProgram& pg : ch.programs) {
      if (only_prog >= 0 && pg.prog_begin != (uint32_t)only_prog) continue;
      if (paired) {
        paired_case(s, pg);
        continue;
      }
      s << "    case " << pg.prog_begin << "u: {\n"
        << "#pragma unroll 1\n"
        << "      for (int v = 0; v < " << V << "; ++v) {\n"
        << "        const u32 t = tl0 + v * " << T << " + me;\n"
        << "        const bool valid = t < sg.n_tuples;\n"
        << "        u32 rem = valid ? t : 0u;\n"
        << "        W r[" << MAPC_NREG << "];\n";
      s << decode_tuple(pg, "        ")
        << "        bool act = true;\n"
        << "        u32 e = 0;\n"
        << program_body(pg.ops, u32)
        << "        (void)act; (void)e;\n"
        << "      }\n"
        << "      break; }\n";
    }
    s << "    default: break;\n"
      << "    }\n"
      << "#undef EMIT_KEY\n";
    if (mode == MAPC_MODE_DIRECT) {
      // guarded accesses are counted per thread over all its tiles and added once
      // at the end: a per-tile atomicAdd on the one counter word serialised in its L2
      // slice (4b: one slice 30% busy with atomics, the others 2%)
      s << "    cnt_all_ += cnt;\n";
      return;
    }
    if (mode != MAPC_MODE_FILTER)   // keys mode: guarded segments compact through shared memory
      s << "    if (!sg.dense) {\n"
      << "      u32 total;\n"
      << "      const u32 excl = block_excl_scan<" << T << ">(cnt, scan_tmp, &total);\n"
      << "      if (me == 0) s_base = total ? atomicAdd(n_ctr, (u64)total) : 0ull;\n"
      << "      __syncthreads();\n"
      << "      const u64 obase = s_base;\n"
      << "      for (u32 j = 0; j < cnt; ++j) { const u64 pos = obase + excl + j; "
         "if (pos < cap) keys[pos] = stage[(size_t)j * " << T << " + me]; else err |= " << MAPC_ERR_CAPACITY << "u; }\n"
      << "      __syncthreads();\n"
      << "    }\n";
    if (mode == MAPC_MODE_FILTER) s << "    }\n";   // !skip_
  };
  auto fd = [](const MapcFastDiv& f) {
    std::ostringstream o;
    o << "{" << f.d << "u, " << f.m << "u, " << f.s << "u, " << f.pow2 << "u}";
    return o.str();
  };
  if (!ch.segs.empty()) {
    s << "    switch (lo) {\n";
    for (size_t i = 0; i < ch.segs.size(); ++i) {
      const MapcSeg& g = ch.segs[i];
      s << "    case " << i << ": {\n"
        << "    const Seg sg = {" << g.tuple_begin << "ull, " << g.n_tuples << "ull, " << g.tile_begin << "ull, "
        << g.key_begin << "ull, " << g.key_hi << "ull, " << g.prog_begin << "u, " << g.prog_end << "u, " << g.n_levels
        << "u, " << g.b0 << "u, " << g.lb0 << "u, " << g.n_emits << "u, " << g.dense << "u, " << g.tid_inner << "u, {";
      for (int l = 0; l < 8; ++l) s << (l ? ", " : "") << fd(g.trip_div[l]);
      s << "}, " << fd(g.tid_div) << "};\n";
      tile_body(s, g.prog_begin);
      s << "    break; }\n";
    }
    s << "    default: break;\n"        // every segment of the chunk is baked
      << "    }\n";
  } else {
    s << "    const Seg& sg = segs[lo];\n";
    tile_body(s, -1);
  }
  s << "  }\n";
  if (mode == MAPC_MODE_DIRECT)
    s << "  {\n"
      << "#pragma unroll\n"
      << "    for (int o_ = 16; o_; o_ >>= 1) cnt_all_ += __shfl_xor_sync(0xffffffffu, cnt_all_, o_);\n"
      << "    if ((threadIdx.x & 31) == 0 && cnt_all_) atomicAdd(n_ctr, cnt_all_);\n"
      << "  }\n";
  s << "  if (err) atomicOr(err_flag, err);\n"
    << "}\n";
  return s.str();
}

std::string module_source(const std::vector<JitChunk>& chunks, bool u32, uint32_t mode, uint32_t cell_bytes) {
  std::string src = prelude();
  for (size_t i = 0; i < chunks.size(); ++i) src += chunk_kernel_source(chunks[i], (int)i, u32, mode, cell_bytes);
  return src;
}

int compile_cubin(const std::string& src, std::vector<char>* cubin, std::string* log) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "mapcheck_gen.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    *log = "nvrtcCreateProgram failed";
    return 1;
  }
  const char* opts[] = {"-arch=sm_100a", "-default-device", "-std=c++17", "-lineinfo"};
  nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string l(n, '\0');
    nvrtcGetProgramLog(prog, &l[0]);
    *log = "NVRTC: " + std::string(nvrtcGetErrorString(r)) + "\n" + l.substr(0, 2000);
    nvrtcDestroyProgram(&prog);
    return 1;
  }
  size_t cubin_n = 0;
  nvrtcGetCUBINSize(prog, &cubin_n);
  cubin->resize(cubin_n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  return 0;
}

// One NVRTC program per chunk, compiled in parallel; modules cached by chunk_key.
int build_module(const std::vector<JitChunk>& chunks, bool u32, uint32_t mode, const std::vector<uint32_t>& cell_bytes,
                 const std::vector<char>& want, JitHandle* out, std::string* log) {
  const size_t nc = chunks.size();
  std::vector<std::string> keys(nc), srcs(nc);
  for (size_t i = 0; i < nc; ++i)
    if (want[i]) keys[i] = chunk_key(chunks[i], u32, mode, cell_bytes[i]);
  std::vector<int> need;                       // one chunk per distinct uncached kernel
  {
    std::lock_guard<std::mutex> g(g_mu);
    std::set<std::string> seen;
    for (size_t i = 0; i < nc; ++i)
      if (want[i] && !g_cache.count(keys[i]) && seen.insert(keys[i]).second) need.push_back((int)i);
  }
  for (int i : need) srcs[i] = prelude() + chunk_kernel_source(chunks[i], 0, u32, mode, cell_bytes[i]);
  std::vector<std::vector<char>> cubins(nc);
  std::vector<std::string> logs(nc);
  std::vector<int> rc(nc, 0);
  {
    std::atomic<size_t> next{0};
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < std::min<size_t>(hw, need.size()); ++w)
      pool.emplace_back([&]() {
        for (size_t k = next++; k < need.size(); k = next++) {
          const int i = need[k];
          rc[i] = compile_cubin(srcs[i], &cubins[i], &logs[i]);
        }
      });
    for (auto& t : pool) t.join();
  }
  std::lock_guard<std::mutex> g(g_mu);
  if (out->kernels.size() != nc) out->kernels.assign(nc, nullptr);
  for (int i : need)                           // load the new kernels first
    if (rc[i] != 0) {
      *log = logs[i];
      return 1;
    }
  for (size_t i = 0; i < nc; ++i) {
    if (!want[i]) continue;
    auto it = g_cache.find(keys[i]);
    if (it == g_cache.end()) {
      Module m;
      cudaError_t e = cudaLibraryLoadData(&m.lib, cubins[i].data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
      if (e != cudaSuccess) {
        *log = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
        return 1;
      }
      cudaKernel_t k;
      e = cudaLibraryGetKernel(&k, m.lib, "gen_0");
      if (e != cudaSuccess) {
        *log = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
        return 1;
      }
      m.kernels.push_back(k);
      it = g_cache.emplace(keys[i], std::move(m)).first;
    }
    out->kernels[i] = it->second.kernels[0];
  }
  return 0;
}

size_t distinct_kernels(const std::vector<JitChunk>& chunks, bool u32) {
  std::set<std::string> k;
  for (const JitChunk& ch : chunks) k.insert(chunk_key(ch, u32, MAPC_MODE_DIRECT, 0));
  return k.size();
}

cudaError_t launch_units(const JitHandle& h, size_t chunk, unsigned long long n_units, unsigned long long* n_ctr,
                         unsigned long long* racy, unsigned long long* racy_sf, unsigned int* err_flag,
                         uint32_t cluster, uint32_t threads, size_t smem, int n_sms, cudaStream_t s) {
  if (n_units == 0) return cudaSuccess;
  const void* fn = (const void*)h.kernels[chunk];
  void* args[] = {(void*)&n_units, (void*)&n_ctr, (void*)&racy, (void*)&racy_sf, (void*)&err_flag};
  if (cluster <= 1) {
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (int)threads, 0);
    if (occ < 1) occ = 1;
    const unsigned long long capb = (unsigned long long)n_sms * occ;
    const int grid = (int)(n_units < capb ? n_units : capb);
    return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, 0, s);
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cluster > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(cluster * n_units));
  int max_clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg);
  if (e != cudaSuccess) return e;
  if (max_clusters < 1) return cudaErrorInvalidConfiguration;
  const unsigned long long active = std::min<unsigned long long>(n_units, (unsigned long long)max_clusters);
  cfg.gridDim = dim3((unsigned)(cluster * active));
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_unit_filter(const JitHandle& h, size_t chunk, const unsigned long long* target,
                               unsigned long long* keys, unsigned long long* n_ctr, unsigned long long cap,
                               unsigned int* err_flag, unsigned long long unit_accesses, int n_sms, cudaStream_t s) {
  const void* fn = (const void*)h.kernels[chunk];
  const unsigned long long per_cta = 4ull * MAPC_GEN_THREADS;
  unsigned long long grid = (unit_accesses + per_cta - 1) / per_cta;
  grid = std::max<unsigned long long>(1, std::min<unsigned long long>(grid, (unsigned long long)n_sms));
  void* args[] = {(void*)&target, (void*)&keys, (void*)&n_ctr, (void*)&cap, (void*)&err_flag};
  return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(MAPC_GEN_THREADS), args, 0, s);
}

cudaError_t launch_chunk(const JitHandle& h, size_t chunk, const MapcSeg* segs, int n_segs,
                         unsigned long long total_tiles, unsigned long long* keys, unsigned long long* n_ctr,
                         unsigned int* err_flag, unsigned long long cap, const unsigned long long* target,
                         int n_sms, int max_ctas_per_sm, cudaStream_t s, const unsigned long long* pcomp) {
  if (total_tiles == 0) return cudaSuccess;
  const void* fn = (const void*)h.kernels[chunk];
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, MAPC_GEN_THREADS, 0);
  if (occ < 1) occ = 1;
  if (max_ctas_per_sm > 0 && occ > max_ctas_per_sm) occ = max_ctas_per_sm;
  const unsigned long long capb = (unsigned long long)n_sms * occ;
  const int grid = (int)(total_tiles < capb ? total_tiles : capb);
  void* args[] = {(void*)&segs, (void*)&n_segs, (void*)&total_tiles, (void*)&keys, (void*)&n_ctr, (void*)&err_flag,
                  (void*)&cap, (void*)&target, (void*)&pcomp};
  return cudaLaunchKernel(fn, dim3(grid), dim3(MAPC_GEN_THREADS), args, 0, s);
}

}  // namespace mapj
