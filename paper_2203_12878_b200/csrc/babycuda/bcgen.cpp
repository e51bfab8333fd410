// bcgen.cpp -- BabyCUDA -> CUDA C source for the executor (bcgen.h).
#include "bcgen.h"

#include <set>
#include <sstream>

namespace bcg {
namespace {

const char* kPrelude = R"(
typedef unsigned int u32;
typedef unsigned long long u64;
struct BcCtl { u64 n_keys, max_block, uninit, ambiguous; u32 err, pad; };   // = bcg::BcCtl
struct St {
  u64* mem; u64* cval; u32* own; u32* minw; u32* claims; unsigned char* st; u64* logb;
  u32* s_nclaim; u32* s_conf; u32* s_nkeys;
  u64* keys; u64 cap; BcCtl* ctl;
  u32 nlog, err, tid, phase;
  u64 uninit, ambig, blk;
};
// naturals, exact u64: an operation whose exact result exceeds 2^64 - 1 flags a
// range error, / and % by zero an arithmetic error (DESIGN.md R3, R4)
__device__ __forceinline__ u64 bc_add(u64 a, u64 b, u32& e) { const u64 r = a + b; if (r < a) e |= ERR_RANGE_; return r; }
__device__ __forceinline__ u64 bc_sub(u64 a, u64 b) { return a > b ? a - b : 0ull; }
__device__ __forceinline__ u64 bc_mul(u64 a, u64 b, u32& e) { if (__umul64hi(a, b)) e |= ERR_RANGE_; return a * b; }
__device__ __forceinline__ u64 bc_div(u64 a, u64 b, u32& e) { if (!b) { e |= ERR_ARITH_; return 0ull; } return a / b; }
__device__ __forceinline__ u64 bc_mod(u64 a, u64 b, u32& e) { if (!b) { e |= ERR_ARITH_; return 0ull; } return a % b; }
__device__ __forceinline__ u64 bc_shl(u64 a, u64 b, u32& e) {
  if (!a) return 0ull;
  if (b >= 64 || a > (~0ull >> b)) { e |= ERR_RANGE_; return 0ull; }
  return a << b;
}
__device__ __forceinline__ u64 bc_shr(u64 a, u64 b) { return b >= 64 ? 0ull : a >> b; }
__device__ __forceinline__ u64 bc_min(u64 a, u64 b) { return a < b ? a : b; }
__device__ __forceinline__ u64 bc_max(u64 a, u64 b) { return a > b ? a : b; }

// one access value into the block's region of the alpha buffer (S.keys = the
// region, S.cap its size; warp-aggregated slot reservation on a shared counter)
__device__ __forceinline__ void bc_emit(St& S, u64 key) {
  const u32 m = __activemask();
  const u32 lane = S.tid & 31u, lead = __ffs(m) - 1u;
  u32 b = 0;
  if (lane == lead) b = atomicAdd(S.s_nkeys, (u32)__popc(m));
  b = __shfl_sync(m, b, lead);
  const u64 p = (u64)b + __popc(m & ((1u << lane) - 1u));
  if (p < S.cap) S.keys[p] = key;
}

// rule read: lastwrite over {tid : (R, W)} :: H -- the thread's own write of this
// phase (conflict log, else the cell it claimed), else the committed value
__device__ __forceinline__ u64 bc_read(St& S, u32 c) {
  for (u32 j = 0; j < S.nlog; ++j)
    if (S.logb[2 * j] == c) return S.logb[2 * j + 1];
  if (S.own[c] == S.tid + 1u) return S.cval[c];
  const unsigned char s = S.st[c];
  if (s & 1u) {
    if (s & 2u) ++S.ambig;
    return S.mem[c];
  }
  ++S.uninit;                                     // lastwrite-undef: bottom, read as 0 (R20)
  return 0ull;
}

// rule write: W[y -> z] in the thread's own record
__device__ __forceinline__ void bc_write(St& S, u32 c, u64 z) {
  const u32 o = atomicCAS(&S.own[c], 0u, S.tid + 1u);
  if (o == 0u) {
    S.cval[c] = z;
    S.claims[atomicAdd(S.s_nclaim, 1u)] = c;
  } else if (o == S.tid + 1u) {
    S.cval[c] = z;
  } else {                                        // another thread wrote c in this phase: a race
    u32 j = 0;
    while (j < S.nlog && S.logb[2 * j] != c) ++j;
    if (j == S.nlog) {
      if (S.nlog == K_LOG_) { S.err |= ERR_LOG_; return; }
      S.logb[2 * j] = c;
      ++S.nlog;
    }
    S.logb[2 * j + 1] = z;
    atomicMin(&S.minw[c], S.tid + 1u);
    *S.s_conf = 1u;
  }
}

// sync: close the phase -- every claimed cell commits its writer's value; a cell
// written by several threads commits the smallest writer tid's value (R21)
__device__ void bc_sync(St& S) {
  __syncthreads();
  const u32 nc = *S.s_nclaim, conf = *S.s_conf;
  for (u32 i = S.tid; i < nc; i += blockDim.x) {
    const u32 c = S.claims[i];
    if (S.minw[c] == 0xFFFFFFFFu) { S.mem[c] = S.cval[c]; S.st[c] = 1; S.own[c] = 0u; }
    else atomicMin(&S.minw[c], S.own[c]);
  }
  if (conf) {
    __syncthreads();
    for (u32 i = S.tid; i < nc; i += blockDim.x) {
      const u32 c = S.claims[i];
      if (S.minw[c] != 0xFFFFFFFFu && S.minw[c] == S.own[c]) S.mem[c] = S.cval[c];
    }
    for (u32 j = 0; j < S.nlog; ++j) {
      const u32 c = (u32)S.logb[2 * j];
      if (S.minw[c] == S.tid + 1u) S.mem[c] = S.logb[2 * j + 1];
    }
    __syncthreads();
    for (u32 i = S.tid; i < nc; i += blockDim.x) {
      const u32 c = S.claims[i];
      if (S.minw[c] != 0xFFFFFFFFu) { S.st[c] = 3; S.own[c] = 0u; S.minw[c] = 0xFFFFFFFFu; }
    }
  }
  S.nlog = 0;
  __syncthreads();
  if (S.tid == 0) { *S.s_nclaim = 0u; *S.s_conf = 0u; }
  __syncthreads();
  ++S.phase;
}
)";

struct Gen {
  const bcf::Kernel& K;
  const Plan& P;
  std::set<std::string> params;
  std::ostringstream o;
  int tmp = 0;

  std::string key(int arr, const std::string& ix, int kind) const {
    const Layout& L = P.lay;
    std::ostringstream s;
    s << "((((((u64)S.phase << " << L.w_array << "u) | " << arr << "ull) << " << L.w_block << "u | S.blk) << "
      << L.w_index << "u | " << ix << ") << " << (L.w_tid + 1) << "u) | ((u64)S.tid << 1) | " << kind << "ull";
    return s.str();
  }
  std::string num(const bcf::Num* n) {
    switch (n->k) {
      case bcf::NK_NAT: return "(u64)" + std::to_string(n->v) + "ull";
      case bcf::NK_VAR: return (params.count(n->name) ? "P_" : "v_") + n->name;
      case bcf::NK_TID: return "(u64)S.tid";
      case bcf::NK_BID: return "S.blk";
      case bcf::NK_BIN: break;
    }
    const std::string a = num(n->a.get()), b = num(n->b.get());
    switch (n->op) {
      case bcf::OP_ADD: return "bc_add(" + a + ", " + b + ", S.err)";
      case bcf::OP_SUB: return "bc_sub(" + a + ", " + b + ")";
      case bcf::OP_MUL: return "bc_mul(" + a + ", " + b + ", S.err)";
      case bcf::OP_DIV: return "bc_div(" + a + ", " + b + ", S.err)";
      case bcf::OP_MOD: return "bc_mod(" + a + ", " + b + ", S.err)";
      case bcf::OP_SHL: return "bc_shl(" + a + ", " + b + ", S.err)";
      case bcf::OP_SHR: return "bc_shr(" + a + ", " + b + ")";
      case bcf::OP_MIN: return "bc_min(" + a + ", " + b + ")";
      case bcf::OP_MAX: return "bc_max(" + a + ", " + b + ")";
    }
    return "0ull";
  }
  std::string cond(const bcf::Cond* c) {
    switch (c->k) {
      case bcf::CK_TRUE: return "1";
      case bcf::CK_FALSE: return "0";
      case bcf::CK_REL: {
        static const char* r[] = {"==", "!=", "<", "<=", ">", ">="};
        return "(int)(" + num(c->a.get()) + " " + r[c->rel] + " " + num(c->b.get()) + ")";
      }
      case bcf::CK_AND: return "(" + cond(c->l.get()) + " & " + cond(c->r.get()) + ")";    // R2: both evaluated
      case bcf::CK_OR: return "(" + cond(c->l.get()) + " | " + cond(c->r.get()) + ")";
    }
    return "0";
  }
  void stmt(const bcf::Stmt* s, const std::string& ind) {
    switch (s->k) {
      case bcf::SK_SKIP: return;
      case bcf::SK_SYNC: o << ind << "bc_sync(S);\n"; return;
      case bcf::SK_WRITE: {
        const int t = tmp++;
        o << ind << "{ const u64 ix" << t << " = " << num(s->idx.get()) << "; const u64 z" << t << " = "
          << num(s->val.get()) << ";\n"
          << ind << "  if (ix" << t << " >= " << P.extents[s->arr] << "ull) S.err |= ERR_BOUNDS_;\n"
          << ind << "  else { bc_emit(S, " << key(s->arr, "ix" + std::to_string(t), 1) << "); bc_write(S, (u32)("
          << P.offsets[s->arr] << "ull + ix" << t << "), z" << t << "); } }\n";
        return;
      }
      case bcf::SK_LET: {
        const int t = tmp++;
        o << ind << "{ const u64 ix" << t << " = " << num(s->idx.get()) << "; u64 v_" << s->var << " = 0;\n"
          << ind << "  if (ix" << t << " >= " << P.extents[s->arr] << "ull) S.err |= ERR_BOUNDS_;\n"
          << ind << "  else { bc_emit(S, " << key(s->arr, "ix" + std::to_string(t), 0) << "); v_" << s->var
          << " = bc_read(S, (u32)(" << P.offsets[s->arr] << "ull + ix" << t << ")); }\n"
          << ind << "  (void)v_" << s->var << ";\n";
        stmt(s->kids[0].get(), ind + "  ");
        o << ind << "}\n";
        return;
      }
      case bcf::SK_IF:
        o << ind << "if (" << cond(s->cond.get()) << ") {\n";
        stmt(s->kids[0].get(), ind + "  ");
        o << ind << "} else {\n";
        stmt(s->kids[1].get(), ind + "  ");
        o << ind << "}\n";
        return;
      case bcf::SK_FOR: {
        // for-1 / for-2 with stride (R6); a loop without a sync stops at the
        // thread's first error, a loop around a sync has uniform, host-checked
        // bounds and must run on every thread
        const int t = tmp++;
        const std::string lo = "lo" + std::to_string(t), hi = "hi" + std::to_string(t), st = "st" + std::to_string(t);
        o << ind << "{ const u64 " << lo << " = " << num(s->lo.get()) << ", " << hi << " = " << num(s->hi.get()) << ", "
          << st << " = " << num(s->step.get()) << ";\n"
          << ind << "  if (" << st << " == 0ull) S.err |= ERR_ARITH_;\n"
          << ind << "  else for (u64 v_" << s->var << " = " << lo << "; v_" << s->var << " < " << hi
          << (s->kids[0]->has_sync ? "" : " && !S.err") << ";) {\n";
        stmt(s->kids[0].get(), ind + "    ");
        o << ind << "    if (" << hi << " - v_" << s->var << " <= " << st << ") break;\n"
          << ind << "    v_" << s->var << " += " << st << ";\n"
          << ind << "  } }\n";
        return;
      }
      case bcf::SK_SEQ:
        for (auto& k : s->kids) stmt(k.get(), ind);
        return;
    }
  }
};

uint64_t align16(uint64_t x) { return (x + 15) / 16 * 16; }

}  // namespace

uint64_t slot_bytes(const Plan& P) {
  const uint64_t n = P.n_cells;
  return align16(n * 8) * 2 + align16(n * 4) * 3 + align16(n) + align16((uint64_t)P.block_threads * P.k_log * 16);
}

std::string kernel_source(const bcf::Kernel& K, const Plan& P) {
  Gen g{K, P, std::set<std::string>(K.params.begin(), K.params.end()), {}, 0};
  std::ostringstream& o = g.o;
  o << "#define ERR_ARITH_ " << ERR_ARITH << "u\n#define ERR_RANGE_ " << ERR_RANGE << "u\n#define ERR_BOUNDS_ "
    << ERR_BOUNDS << "u\n#define ERR_LOG_ " << ERR_LOG << "u\n#define K_LOG_ " << P.k_log << "u\n"
    << kPrelude;
  const uint64_t n = P.n_cells;
  o << "extern \"C\" __global__ void __launch_bounds__(" << P.block_threads
    << ") bc_exec(u64* keys, u64 block_cap, BcCtl* ctl, unsigned char* slots, u64 slot_bytes, u64* mem_out, "
       "unsigned char* st_out) {\n"
    << "  __shared__ u32 s_nclaim, s_conf, s_nkeys;\n"
    << "  St S;\n"
    << "  unsigned char* base = slots + (u64)blockIdx.x * slot_bytes;\n"
    << "  S.mem = (u64*)base;\n"
    << "  S.cval = (u64*)(base + " << align16(n * 8) << "ull);\n"
    << "  S.own = (u32*)(base + " << 2 * align16(n * 8) << "ull);\n"
    << "  S.minw = (u32*)(base + " << 2 * align16(n * 8) + align16(n * 4) << "ull);\n"
    << "  S.claims = (u32*)(base + " << 2 * align16(n * 8) + 2 * align16(n * 4) << "ull);\n"
    << "  S.st = base + " << 2 * align16(n * 8) + 3 * align16(n * 4) << "ull;\n"
    << "  S.logb = (u64*)(base + " << 2 * align16(n * 8) + 3 * align16(n * 4) + align16(n) << "ull) + (u64)threadIdx.x * "
    << 2 * P.k_log << "ull;\n"
    << "  S.s_nclaim = &s_nclaim; S.s_conf = &s_conf; S.s_nkeys = &s_nkeys;\n"
    << "  S.cap = block_cap; S.ctl = ctl;\n"
    << "  S.nlog = 0; S.err = 0; S.tid = threadIdx.x; S.phase = 0; S.uninit = 0; S.ambig = 0;\n"
    << "  u64 keys_all = 0, keys_max = 0;      // this CTA's blocks (one atomic each at the end)\n";
  for (size_t i = 0; i < K.params.size(); ++i)
    o << "  const u64 P_" << K.params[i] << " = " << P.params[i] << "ull; (void)P_" << K.params[i] << ";\n";
  // each block's accesses go to its own region of the alpha buffer (block_cap
  // keys; unused slots keep the host's all-ones fill and sort last), counted on a
  // shared counter: no global atomic per access
  o << "  for (u64 c = threadIdx.x; c < " << n << "ull; c += blockDim.x) { S.own[c] = 0u; S.minw[c] = 0xFFFFFFFFu; }\n"
    << "  for (u64 blk = blockIdx.x; blk < " << P.n_blocks << "ull; blk += gridDim.x) {\n"
    << "    for (u64 c = threadIdx.x; c < " << n << "ull; c += blockDim.x) S.st[c] = 0;\n"
    << "    if (threadIdx.x == 0) { s_nclaim = 0u; s_conf = 0u; s_nkeys = 0u; }\n"
    << "    __syncthreads();\n"
    << "    S.blk = blk; S.phase = 0; S.keys = keys + blk * block_cap;\n"
    << "    {\n";
  g.stmt(K.body.get(), "      ");
  o << "    }\n"
    << "    bc_sync(S);                       // commit the last phase\n"
    << "    if (threadIdx.x == 0) {\n"
    << "      keys_all += s_nkeys;\n"
    << "      keys_max = s_nkeys > keys_max ? (u64)s_nkeys : keys_max;\n"
    << "    }\n"
    << "    if (mem_out)\n"
    << "      for (u64 c = threadIdx.x; c < " << n << "ull; c += blockDim.x) {\n"
    << "        mem_out[blk * " << n << "ull + c] = S.mem[c]; st_out[blk * " << n << "ull + c] = S.st[c]; }\n"
    << "    __syncthreads();\n"
    << "  }\n"
    << "  if (threadIdx.x == 0 && keys_all) { atomicAdd(&ctl->n_keys, keys_all); atomicMax(&ctl->max_block, keys_max); }\n"
    << "  if (S.uninit) atomicAdd(&ctl->uninit, S.uninit);\n"
    << "  if (S.ambig) atomicAdd(&ctl->ambiguous, S.ambig);\n"
    << "  if (S.err) atomicOr(&ctl->err, S.err);\n"
    << "}\n";
  return o.str();
}

}  // namespace bcg
