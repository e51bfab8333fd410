// compile.cpp -- phase enumeration, interval analysis and lowering of MAP
// instances to VM bytecode (product path).  See compiler.h for the pipeline.
#include <algorithm>
#include <map>
#include <set>
#include <tuple>

#include "compiler.h"

namespace mapc {

MapcFastDiv make_fastdiv(uint32_t d) {
  MapcFastDiv f{};
  f.d = d ? d : 1;
  d = f.d;
  uint32_t l = 31 - __builtin_clz(d);            // floor(log2 d)
  if ((d & (d - 1)) == 0) {
    f.pow2 = 1;
    f.s = l;
    f.m = 0;
    return f;
  }
  // m = floor(2^32 * (2^(l+1) - d) / d) + 1 ; q = (hi(m n) + ((n - hi(m n)) >> 1)) >> l
  unsigned __int128 num = ((unsigned __int128)1 << 32) * (((uint64_t)1 << (l + 1)) - d);
  f.m = (uint32_t)(num / d + 1);
  f.s = l;
  f.pow2 = 0;
  return f;
}

uint32_t fastdiv_apply(uint32_t n, const MapcFastDiv& f) {
  if (f.pow2) return n >> f.s;
  uint32_t hi = (uint32_t)(((uint64_t)f.m * n) >> 32);
  return (hi + ((n - hi) >> 1)) >> f.s;
}

namespace {

void choose_tuple_order(GroupProg* g, uint64_t n_threads);   // defined below (coalescing heuristic)

using u128 = unsigned __int128;
constexpr uint64_t kU64 = ~0ull;

[[noreturn]] void range_error(const std::string& m) { throw CompileError{4, m}; }

uint64_t checked(u128 v, const char* what) {
  if (v > (u128)kU64) range_error(std::string("a value may exceed 64 bits (") + what + ")");
  return (uint64_t)v;
}

uint64_t shl_checked(uint64_t a, uint64_t s, const char* what) {
  if (a == 0) return 0;
  if (s >= 64 || a > (kU64 >> s)) range_error(std::string("a value may exceed 64 bits (") + what + ")");
  return a << s;
}

uint64_t trip_count(uint64_t lo, uint64_t hi, uint64_t step) {
  if (hi <= lo) return 0;
  return (hi - lo - 1) / step + 1;
}

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
uint32_t log2u(uint64_t x) { return 63 - __builtin_clzll(x); }

// ----------------------------------------------------------------------------
// Exact uniform evaluation (params + forS values) for the synchronized fragment.
struct UniformEval {
  const Program& P;
  const std::vector<uint64_t>& params;
  const std::vector<uint64_t>& syncenv;   // by var id (valid for SyncLoop vars in scope)
  const std::vector<bool>& sync_set;

  bool try_eval(int e, uint64_t* out) const {   // false if it references a non-uniform var
    const Expr& x = P.exprs[e];
    if (x.kind == Expr::Nat) { *out = x.value; return true; }
    if (x.kind == Expr::Ref) {
      const Var& v = P.vars[x.var];
      if (v.kind == VarKind::Param) { *out = params[v.index]; return true; }
      if (v.kind == VarKind::SyncLoop && sync_set[x.var]) { *out = syncenv[x.var]; return true; }
      return false;
    }
    uint64_t a, b;
    if (!try_eval(x.lhs, &a) || !try_eval(x.rhs, &b)) return false;
    *out = apply(x.op, a, b, /*strict=*/true);
    return true;
  }
  // strict: errors raise CompileError (this evaluation is reached by every thread).
  static uint64_t apply(BinOp op, uint64_t a, uint64_t b, bool strict) {
    switch (op) {
      case BinOp::Add: return checked((u128)a + b, "+");
      case BinOp::Sub: return a > b ? a - b : 0;
      case BinOp::Mul: return checked((u128)a * b, "*");
      case BinOp::Div:
        if (b == 0) { if (strict) throw CompileError{5, "division by zero"}; return 0; }
        return a / b;
      case BinOp::Mod:
        if (b == 0) { if (strict) throw CompileError{5, "modulo by zero"}; return 0; }
        return a % b;
      case BinOp::Shl: return shl_checked(a, b, "<<");
      case BinOp::Shr: return b >= 64 ? 0 : a >> b;
      case BinOp::Min: return std::min(a, b);
      case BinOp::Max: return std::max(a, b);
    }
    return 0;
  }
};

// ----------------------------------------------------------------------------
// Lowering of one (instance, group) to a register program.
struct Val {
  Interval iv;
  bool is_const = false;
  uint64_t c = 0;
  uint32_t kb = 0;       // known low bits: value mod 2^kb == kv (64 for constants)
  uint64_t kv = 0;
};

inline uint64_t low_mask(uint32_t k) { return k >= 64 ? ~0ull : ((1ull << k) - 1); }
inline uint32_t ctz64(uint64_t x) { return x ? (uint32_t)__builtin_ctzll(x) : 64u; }

struct SIns {
  uint8_t code;
  int dst = -1;          // value id
  int a = -1, b = -1;    // value ids
  int auxv = -1;         // value id of the aux register operand (TRIP step, MADK k)
  uint64_t imm = 0;      // raw immediate (BAND mask)
  bool faulting = false; // side effect: may set MAPC_ERR_DIV0 under act
  uint32_t emit_aux = 0; // EMIT: array << 1 | write
};

class Lowerer {
 public:
  // unroll_depth >= 0: the forU at that depth of the nest is not a tuple
  // coordinate; its variable is the constant of iteration unroll_iter (the
  // loop's bounds and step must be uniform constants, else unroll_failed()).
  Lowerer(const Compiled& C, const std::vector<uint64_t>& syncenv, const std::vector<bool>& sync_set,
          const std::vector<int>& path, const std::set<int>& sites, bool fault_owner, const std::vector<int>& parent,
          int unroll_depth = -1, uint64_t unroll_iter = 0)
      : C_(C), P_(C.ast), syncenv_(syncenv), sync_set_(sync_set), path_(path), sites_(sites),
        fault_owner_(fault_owner), parent_(parent), unroll_depth_(unroll_depth), unroll_iter_(unroll_iter) {}

  bool unroll_failed() const { return unroll_failed_; }
  // constant trip count of the forU at `depth` (0 if its bounds are not uniform constants)
  uint64_t const_trip(int depth) const { return depth < (int)const_trip_.size() ? const_trip_[depth] : 0; }

  // Returns false if the group has an empty tuple space.
  bool run(int tmpl, GroupProg* out) {
    // fixed values: tid, bid, k_0..k_{L-1}
    tid_ = fresh({0, C_.n_threads - 1});
    bid_ = fresh({0, C_.n_blocks - 1});
    for (size_t l = 0; l < path_.size(); ++l) k_.push_back(fresh({0, 0}));   // refined on entry
    act_ = konst(1);
    vm_act_ = act_;
    xval_.assign(P_.vars.size(), -1);
    walk(tmpl, 0);
    if (empty_) return false;
    finish(out);
    return true;
  }

  uint64_t max_value() const { return max_value_; }

 private:
  const Compiled& C_;
  const Program& P_;
  const std::vector<uint64_t>& syncenv_;
  const std::vector<bool>& sync_set_;
  const std::vector<int>& path_;
  const std::set<int>& sites_;
  bool fault_owner_;
  const std::vector<int>& parent_;

  std::vector<Val> vals_;
  std::vector<SIns> ins_;
  std::map<uint64_t, int> consts_;
  std::map<std::tuple<uint8_t, int, int, int, uint64_t>, int> cse_;
  std::vector<int> k_;
  std::vector<int> xval_;
  std::map<int, std::pair<int, int>> relv_;   // cond id -> (lhs, rhs) value ids of its last evaluation
  int tid_ = -1, bid_ = -1, act_ = -1, vm_act_ = -1;
  bool empty_ = false;
  uint64_t trips_[MAPC_MAX_LEVELS] = {};
  int unroll_depth_ = -1;
  uint64_t unroll_iter_ = 0;
  bool unroll_failed_ = false;
  std::vector<uint64_t> const_trip_;    // per depth: trip count when lo, hi, step are constants
  uint64_t max_value_ = 0;
  Interval index_hull_{kU64, 0};
  uint32_t n_emits_ = 0;
  std::vector<uint32_t> emit_kb_;
  std::vector<uint64_t> emit_kv_;

  int fresh(Interval iv) {
    vals_.push_back(Val{iv, false, 0});
    return (int)vals_.size() - 1;
  }
  int konst(uint64_t c) {
    auto it = consts_.find(c);
    if (it != consts_.end()) return it->second;
    vals_.push_back(Val{{c, c}, true, c, 64u, c});
    consts_[c] = (int)vals_.size() - 1;
    return (int)vals_.size() - 1;
  }
  // known low bits of a result (a CSE hit returns a value with the same bits)
  int kbits(int d, uint32_t kb, uint64_t kv) {
    if (d >= 0 && !isc(d)) {
      vals_[d].kb = std::min<uint32_t>(kb, 64u);
      vals_[d].kv = kv & low_mask(vals_[d].kb);
    }
    return d;
  }
  // a * b mod 2^k: x_i = v_i + 2^k_i m_i, so x1 x2 = v1 v2 + 2^k1 m1 v2 + 2^k2 m2 v1 + 2^(k1+k2) m1 m2
  int kbits_mul(int d, int a, int b) {
    const uint32_t k1 = vals_[a].kb, k2 = vals_[b].kb;
    const uint64_t v1 = vals_[a].kv, v2 = vals_[b].kv;
    const uint64_t t1 = (k1 >= 64 || v2 == 0) ? 64 : (uint64_t)k1 + ctz64(v2);
    const uint64_t t2 = (k2 >= 64 || v1 == 0) ? 64 : (uint64_t)k2 + ctz64(v1);
    const uint64_t t3 = (uint64_t)k1 + k2;
    return kbits(d, (uint32_t)std::min<uint64_t>({t1, t2, t3, 64}), v1 * v2);
  }
  bool isc(int v) const { return vals_[v].is_const; }
  uint64_t cv(int v) const { return vals_[v].c; }
  const Interval& iv(int v) const { return vals_[v].iv; }

  void sync_act() {
    if (vm_act_ != act_) {
      SIns s{VM_ACT};
      s.a = act_;
      ins_.push_back(s);
      vm_act_ = act_;
    }
  }

  int emit_op(uint8_t code, int a, int b, Interval r, bool faulting, uint64_t imm = 0, int auxv = -1) {
    if (!faulting) {
      auto key = std::make_tuple(code, a, b, auxv, imm);
      auto it = cse_.find(key);
      if (it != cse_.end()) return it->second;
      int d = fresh(r);
      SIns s{code};
      s.dst = d; s.a = a; s.b = b; s.imm = imm; s.auxv = auxv;
      ins_.push_back(s);
      cse_[key] = d;
      return d;
    }
    sync_act();
    int d = fresh(r);
    SIns s{code};
    s.dst = d; s.a = a; s.b = b; s.imm = imm; s.auxv = auxv; s.faulting = true;
    ins_.push_back(s);
    return d;
  }

  // ---------------------------------------------------------------- arithmetic
  int bin(BinOp op, int a, int b) {
    const Interval A = iv(a), B = iv(b);
    bool ca = isc(a), cb = isc(b);
    switch (op) {
      case BinOp::Add:
        if (ca && cb) return konst(checked((u128)cv(a) + cv(b), "+"));
        if (ca && cv(a) == 0) return b;
        if (cb && cv(b) == 0) return a;
        return kbits(emit_op(VM_ADD, a, b, {A.lo + B.lo, checked((u128)A.hi + B.hi, "+")}, false),
                     std::min(vals_[a].kb, vals_[b].kb), vals_[a].kv + vals_[b].kv);
      case BinOp::Sub: {
        if (ca && cb) return konst(cv(a) > cv(b) ? cv(a) - cv(b) : 0);
        if (cb && cv(b) == 0) return a;
        const int d = emit_op(VM_SUB, a, b, {A.lo > B.hi ? A.lo - B.hi : 0, A.hi > B.lo ? A.hi - B.lo : 0}, false);
        // monus: exact subtraction (and its congruence) only when it never saturates
        return A.lo >= B.hi ? kbits(d, std::min(vals_[a].kb, vals_[b].kb), vals_[a].kv - vals_[b].kv) : d;
      }
      case BinOp::Mul: {
        if (ca && cb) return konst(checked((u128)cv(a) * cv(b), "*"));
        if ((ca && cv(a) == 0) || (cb && cv(b) == 0)) return konst(0);
        if (ca && cv(a) == 1) return b;
        if (cb && cv(b) == 1) return a;
        Interval r{A.lo * B.lo, checked((u128)A.hi * B.hi, "*")};
        if (cb && is_pow2(cv(b))) return kbits_mul(emit_op(VM_SHL, a, konst(log2u(cv(b))), r, false), a, b);
        if (ca && is_pow2(cv(a))) return kbits_mul(emit_op(VM_SHL, b, konst(log2u(cv(a))), r, false), a, b);
        return kbits_mul(emit_op(VM_MUL, a, b, r, false), a, b);
      }
      case BinOp::Div: {
        if (cb && cv(b) != 0) {
          uint64_t d = cv(b);
          if (ca) return konst(cv(a) / d);
          if (d == 1) return a;
          Interval r{A.lo / d, A.hi / d};
          if (is_pow2(d)) return emit_op(VM_SHR, a, konst(log2u(d)), r, false);
          return emit_op(VM_DIV, a, b, r, false);
        }
        bool may0 = B.lo == 0;
        Interval r{B.hi ? A.lo / B.hi : 0, A.hi / std::max<uint64_t>(B.lo, 1)};
        return emit_op(VM_DIV, a, b, r, may0);
      }
      case BinOp::Mod: {
        if (cb && cv(b) != 0) {
          uint64_t d = cv(b);
          if (ca) return konst(cv(a) % d);
          if (d == 1) return konst(0);
          if (A.hi < d) return a;                        // identity on [0, d)
          Interval r{0, std::min(A.hi, d - 1)};
          if (is_pow2(d))
            return kbits(emit_op(VM_BAND, a, -1, r, false, d - 1), std::min(vals_[a].kb, log2u(d)), vals_[a].kv);
          return emit_op(VM_MOD, a, b, r, false);
        }
        bool may0 = B.lo == 0;
        Interval r = (B.lo > 0 && A.hi < B.lo) ? A : Interval{0, std::min(A.hi, B.hi ? B.hi - 1 : 0)};
        return emit_op(VM_MOD, a, b, r, may0);
      }
      case BinOp::Shl: {
        if (ca && cb) return konst(shl_checked(cv(a), cv(b), "<<"));
        if (cb && cv(b) == 0) return a;
        if (ca && cv(a) == 0) return konst(0);
        uint64_t lo = (A.lo == 0) ? 0 : (B.lo >= 64 ? kU64 : shl_checked(A.lo, B.lo, "<<"));
        Interval r{lo, shl_checked(A.hi, B.hi, "<<")};
        const int d = emit_op(VM_SHL, a, b, r, false);
        if (cb && cv(b) < 64) return kbits(d, vals_[a].kb + (uint32_t)cv(b), vals_[a].kv << cv(b));
        return d;
      }
      case BinOp::Shr: {
        if (ca && cb) return konst(cv(b) >= 64 ? 0 : cv(a) >> cv(b));
        if (cb && cv(b) == 0) return a;
        Interval r{B.hi >= 64 ? 0 : A.lo >> B.hi, B.lo >= 64 ? 0 : A.hi >> B.lo};
        return emit_op(VM_SHR, a, b, r, false);
      }
      case BinOp::Min:
        if (ca && cb) return konst(std::min(cv(a), cv(b)));
        if (A.hi <= B.lo) return a;
        if (B.hi <= A.lo) return b;
        return emit_op(VM_MIN, a, b, {std::min(A.lo, B.lo), std::min(A.hi, B.hi)}, false);
      case BinOp::Max:
        if (ca && cb) return konst(std::max(cv(a), cv(b)));
        if (A.lo >= B.hi) return a;
        if (B.lo >= A.hi) return b;
        return emit_op(VM_MAX, a, b, {std::max(A.lo, B.lo), std::max(A.hi, B.hi)}, false);
    }
    return a;
  }

  int rel(RelOp r, int a, int b) {
    const Interval A = iv(a), B = iv(b);
    // decide from intervals when possible (constants are point intervals)
    int known = -1;
    switch (r) {
      case RelOp::Eq:
        if (A.lo == A.hi && B.lo == B.hi && A.lo == B.lo) known = 1;
        else if (A.hi < B.lo || B.hi < A.lo) known = 0;
        break;
      case RelOp::Ne:
        if (A.lo == A.hi && B.lo == B.hi && A.lo == B.lo) known = 0;
        else if (A.hi < B.lo || B.hi < A.lo) known = 1;
        break;
      case RelOp::Lt: if (A.hi < B.lo) known = 1; else if (A.lo >= B.hi) known = 0; break;
      case RelOp::Le: if (A.hi <= B.lo) known = 1; else if (A.lo > B.hi) known = 0; break;
      case RelOp::Gt: if (A.lo > B.hi) known = 1; else if (A.hi <= B.lo) known = 0; break;
      case RelOp::Ge: if (A.lo >= B.hi) known = 1; else if (A.hi < B.lo) known = 0; break;
    }
    if (known >= 0) return konst((uint64_t)known);
    static const uint8_t code[] = {VM_EQ, VM_NE, VM_LT, VM_LE, VM_GT, VM_GE};
    return emit_op(code[(int)r], a, b, {0, 1}, false);
  }
  int land(int a, int b) {
    if (isc(a)) return cv(a) ? b : konst(0);
    if (isc(b)) return cv(b) ? a : konst(0);
    if (a == b) return a;
    return emit_op(VM_LAND, a, b, {0, 1}, false);
  }
  int lor(int a, int b) {
    if (isc(a)) return cv(a) ? konst(1) : b;
    if (isc(b)) return cv(b) ? konst(1) : a;
    if (a == b) return a;
    return emit_op(VM_LOR, a, b, {0, 1}, false);
  }
  int lnot(int a) {
    if (isc(a)) return konst(cv(a) ? 0 : 1);
    return emit_op(VM_LNOT, a, -1, {0, 1}, false);
  }

  int expr(int e) {
    const Expr& x = P_.exprs[e];
    if (x.kind == Expr::Nat) return konst(x.value);
    if (x.kind == Expr::Ref) {
      const Var& v = P_.vars[x.var];
      switch (v.kind) {
        case VarKind::Tid: return tid_;
        case VarKind::Bid: return bid_;
        case VarKind::Param: return konst(C_.params[v.index]);
        case VarKind::SyncLoop: return konst(syncenv_[x.var]);
        case VarKind::UnsyncLoop:
          if (xval_[x.var] < 0) throw CompileError{8, "internal: unbound loop variable"};
          return xval_[x.var];
      }
    }
    int a = expr(x.lhs);
    int b = expr(x.rhs);
    return bin(x.op, a, b);
  }
  int cond(int c) {
    const Cond& x = P_.conds[c];
    switch (x.kind) {
      case Cond::True: return konst(1);
      case Cond::False: return konst(0);
      case Cond::And: { int l = cond(x.lhs); int r = cond(x.rhs); return land(l, r); }
      case Cond::Or: { int l = cond(x.lhs); int r = cond(x.rhs); return lor(l, r); }
      case Cond::Rel: {
        int a = expr(x.lhs);
        int b = expr(x.rhs);
        relv_[c] = {a, b};
        return rel(x.rel, a, b);
      }
    }
    return konst(0);
  }

  // ---- guard refinement ------------------------------------------------------
  // Inside `if (c)` every ACTIVE tuple satisfies c (inside the else branch, not
  // c), so the intervals of the values c compares can be narrowed there: the
  // index hull, the layout and the loop boxes of guarded code get tight (e.g.
  // the scans' `if (k*1024 + tid < (N >> (l+1)))`).  Values computed in the
  // branch are only used under the branch's act (EMIT and fault checks are
  // masked, nested guards are AND-ed into act), so a value an inactive tuple
  // computes outside its narrowed interval is never observed.  The narrowed
  // intervals and the CSE entries created in the branch are undone on exit.
  struct Scope {
    std::vector<std::pair<int, Interval>> undo;
    std::map<std::tuple<uint8_t, int, int, int, uint64_t>, int> cse;
    bool empty = false;
  };
  void narrow(Scope& sc, int v, uint64_t lo, uint64_t hi) {
    const Interval o = vals_[v].iv;
    const uint64_t nl = std::max(o.lo, lo), nh = std::min(o.hi, hi);
    if (nl > nh) { sc.empty = true; return; }
    if (nl == o.lo && nh == o.hi) return;
    if (isc(v)) return;                              // a constant inside its bounds
    sc.undo.push_back({v, o});
    vals_[v].iv = {nl, nh};
  }
  void refine(Scope& sc, int c, bool pos) {
    const Cond& x = P_.conds[c];
    switch (x.kind) {
      case Cond::True: case Cond::False: return;
      case Cond::And: if (pos) { refine(sc, x.lhs, true); refine(sc, x.rhs, true); } return;
      case Cond::Or: if (!pos) { refine(sc, x.lhs, false); refine(sc, x.rhs, false); } return;
      case Cond::Rel: {
        auto it = relv_.find(c);
        if (it == relv_.end()) return;
        int a = it->second.first, b = it->second.second;
        RelOp r = x.rel;
        if (!pos) {
          switch (r) {
            case RelOp::Lt: r = RelOp::Ge; break;
            case RelOp::Le: r = RelOp::Gt; break;
            case RelOp::Gt: r = RelOp::Le; break;
            case RelOp::Ge: r = RelOp::Lt; break;
            case RelOp::Eq: r = RelOp::Ne; break;
            case RelOp::Ne: r = RelOp::Eq; break;
          }
        }
        if (r == RelOp::Gt) { std::swap(a, b); r = RelOp::Lt; }
        if (r == RelOp::Ge) { std::swap(a, b); r = RelOp::Le; }
        const Interval A = iv(a), B = iv(b);
        switch (r) {
          case RelOp::Lt:                              // a < b
            if (B.hi == 0) { sc.empty = true; return; }
            narrow(sc, a, 0, B.hi - 1);
            if (A.lo == kU64) { sc.empty = true; return; }
            narrow(sc, b, A.lo + 1, kU64);
            return;
          case RelOp::Le:                              // a <= b
            narrow(sc, a, 0, B.hi);
            narrow(sc, b, A.lo, kU64);
            return;
          case RelOp::Eq:
            narrow(sc, a, B.lo, B.hi);
            narrow(sc, b, A.lo, A.hi);
            return;
          default: return;
        }
      }
    }
  }
  Scope open_scope(int c, bool pos) {
    Scope sc;
    sc.cse = cse_;
    refine(sc, c, pos);
    return sc;
  }
  void close_scope(Scope& sc) {
    for (auto it = sc.undo.rbegin(); it != sc.undo.rend(); ++it) vals_[it->first].iv = it->second;
    cse_ = std::move(sc.cse);
  }

  // ------------------------------------------------------------- fault scan
  bool expr_may_fault(int e) const {
    const Expr& x = P_.exprs[e];
    if (x.kind != Expr::Bin) return false;
    if (x.op == BinOp::Div || x.op == BinOp::Mod) {
      UniformEval U{P_, C_.params, syncenv_, sync_set_};
      uint64_t d;
      if (!U.try_eval(x.rhs, &d) || d == 0) return true;
    }
    return expr_may_fault(x.lhs) || expr_may_fault(x.rhs);
  }
  bool cond_may_fault(int c) const {
    const Cond& x = P_.conds[c];
    if (x.kind == Cond::Rel) return expr_may_fault(x.lhs) || expr_may_fault(x.rhs);
    if (x.kind == Cond::And || x.kind == Cond::Or) return cond_may_fault(x.lhs) || cond_may_fault(x.rhs);
    return false;
  }
  // Does s's subtree (not descending into forU bodies) need evaluation at the
  // group's own level: an emitted site, or a fault check we own.
  bool need_here(int s) const {
    const Stmt& st = P_.stmts[s];
    switch (st.kind) {
      case Stmt::Access: return sites_.count(s) || (fault_owner_ && expr_may_fault(st.index));
      case Stmt::Seq:
        for (int c : st.items) if (need_here(c)) return true;
        return false;
      case Stmt::If:
        return (fault_owner_ && cond_may_fault(st.cond)) || need_here(st.then_s) || need_here(st.else_s);
      case Stmt::ForU:
        return fault_owner_ && (expr_may_fault(st.lo) || expr_may_fault(st.hi) || expr_may_fault(st.step));
      default: return false;
    }
  }
  bool contains(int s, int t) const {
    for (int x = t; x >= 0; x = parent_[x]) if (x == s) return true;
    return false;
  }

  // ------------------------------------------------------------------ walk
  void walk(int s, size_t d) {
    if (empty_) return;
    if (isc(act_) && cv(act_) == 0) return;        // statically unreachable
    const Stmt& st = P_.stmts[s];
    const bool here = d == path_.size();
    switch (st.kind) {
      case Stmt::Skip:
      case Stmt::Sync:
      case Stmt::ForS:
        return;
      case Stmt::Access:
        if (here && sites_.count(s)) {
          int ix = expr(st.index);
          if (isc(act_) && cv(act_) == 0) return;
          sync_act();
          SIns e{VM_EMIT};
          e.a = ix;
          e.emit_aux = ((uint32_t)st.array << 1) | (st.write ? 1u : 0u);
          ins_.push_back(e);
          ++n_emits_;
          emit_kb_.push_back(vals_[ix].kb);
          emit_kv_.push_back(vals_[ix].kv);
          index_hull_.lo = std::min(index_hull_.lo, iv(ix).lo);
          index_hull_.hi = std::max(index_hull_.hi, iv(ix).hi);
        } else if (here && fault_owner_ && expr_may_fault(st.index)) {
          expr(st.index);
        }
        return;
      case Stmt::Seq:
        for (int c : st.items) walk(c, d);
        return;
      case Stmt::If: {
        bool rel = here ? (need_here(st.then_s) || need_here(st.else_s)) : contains(s, path_[d]);
        bool check = here && fault_owner_ && cond_may_fault(st.cond);
        if (!rel && !check) return;
        int c = cond(st.cond);
        if (!rel) return;
        int saved = act_;
        act_ = land(saved, c);
        {
          Scope sc = open_scope(st.cond, true);
          if (!sc.empty) walk(st.then_s, d);
          close_scope(sc);
        }
        act_ = land(saved, lnot(c));
        {
          Scope sc = open_scope(st.cond, false);
          if (!sc.empty) walk(st.else_s, d);
          close_scope(sc);
        }
        act_ = saved;
        return;
      }
      case Stmt::ForU:
        if (!here && path_[d] == s) {
          enter(st, d);
        } else if (here && fault_owner_ && (expr_may_fault(st.lo) || expr_may_fault(st.hi) || expr_may_fault(st.step))) {
          expr(st.lo);
          expr(st.hi);
          expr(st.step);
        }
        return;
    }
  }

  void enter(const Stmt& st, size_t d) {
    int lo = expr(st.lo), hi = expr(st.hi), sp = expr(st.step);
    const Interval L = iv(lo), H = iv(hi), S = iv(sp);
    if (S.lo == 0) range_error("a loop step may be zero");
    if (const_trip_.size() <= d) const_trip_.resize(d + 1, 0);
    if (isc(lo) && isc(hi) && isc(sp)) const_trip_[d] = trip_count(cv(lo), cv(hi), cv(sp));
    if ((int)d == unroll_depth_) {                   // one iteration, as a constant
      if (!(isc(lo) && isc(hi) && isc(sp))) { unroll_failed_ = true; empty_ = true; return; }
      if (unroll_iter_ >= const_trip_[d]) { empty_ = true; return; }
      const uint64_t xv = checked((u128)cv(lo) + (u128)unroll_iter_ * cv(sp), "loop value");
      trips_[d] = 1;
      xval_[st.var] = konst(xv);
      walk(st.body, d + 1);
      xval_[st.var] = -1;
      return;
    }
    // bounding-box trip count: trip is decreasing in lo and step, increasing in hi
    uint64_t tmax = trip_count(L.lo, H.hi, S.lo);
    uint64_t tmin = trip_count(L.hi, H.lo, S.hi);
    if (tmax == 0) { empty_ = true; return; }
    if (tmax >= (1ull << 32)) range_error("a loop has 2^32 or more iterations");
    trips_[d] = tmax;
    vals_[k_[d]].iv = {0, tmax - 1};
    int trip;
    if (isc(lo) && isc(hi) && isc(sp)) {
      trip = konst(tmax);
    } else {
      int aux;
      uint64_t step_imm = 0;
      if (isc(sp)) { aux = -1; step_imm = cv(sp); } else { aux = sp; }
      // encode constant steps in aux (< 2^31) else keep a register
      if (aux < 0 && step_imm >= (1ull << 31)) aux = materialize(sp);
      trip = emit_op(VM_TRIP, lo, hi, {tmin, tmax}, false, aux < 0 ? step_imm : 0, aux);
    }
    if (!(isc(trip) && cv(trip) == tmax)) {
      int g = rel(RelOp::Lt, k_[d], trip);
      act_ = land(act_, g);
    }
    // x = lo + k * step, exact for active tuples
    uint64_t xhi = std::min<uint64_t>(H.hi - 1, (uint64_t)std::min<u128>((u128)L.hi + (u128)(tmax - 1) * S.hi, (u128)kU64));
    int x;
    if (isc(sp) && isc(lo)) {
      int t = bin(BinOp::Mul, k_[d], sp);     // true range over the bounding box
      x = bin(BinOp::Add, t, lo);
    } else {
      x = emit_op(VM_MADK, lo, sp, {L.lo, std::max(L.lo, xhi)}, false, 0, k_[d]);
      // lo + k * step: the step's trailing zeros (k unknown) and lo's known bits
      if (isc(sp)) kbits(x, std::min<uint32_t>(vals_[lo].kb, cv(sp) ? ctz64(cv(sp)) : 64u), vals_[lo].kv);
    }
    int var = st.var;
    xval_[var] = x;
    walk(st.body, d + 1);
    xval_[var] = -1;
  }

  int materialize(int v) {   // constant -> register
    return emit_op(VM_MOVI, -1, -1, iv(v), false, cv(v));
  }

  // ------------------------------------------------------------ finishing
  void finish(GroupProg* out) {
    // liveness (reverse scan): side-effecting ops are roots
    std::vector<bool> live(vals_.size(), false);
    std::vector<bool> keep(ins_.size(), false);
    for (int i = (int)ins_.size() - 1; i >= 0; --i) {
      const SIns& s = ins_[i];
      bool root = s.code == VM_EMIT || s.code == VM_ACT || s.faulting;
      if (root || (s.dst >= 0 && live[s.dst])) {
        keep[i] = true;
        for (int v : {s.a, s.b, s.auxv})
          if (v >= 0) live[v] = true;
      }
    }
    std::vector<SIns> prog;
    for (size_t i = 0; i < ins_.size(); ++i)
      if (keep[i]) prog.push_back(ins_[i]);
    // Drop ACT ops that are never followed by an EMIT / faulting op.
    {
      std::vector<SIns> p2;
      for (size_t i = 0; i < prog.size(); ++i) {
        if (prog[i].code == VM_ACT) {
          bool used = false;
          for (size_t j = i + 1; j < prog.size(); ++j) {
            if (prog[j].code == VM_ACT) break;
            if (prog[j].code == VM_EMIT || prog[j].faulting) { used = true; break; }
          }
          if (!used) continue;
        }
        p2.push_back(prog[i]);
      }
      prog.swap(p2);
    }
    // value range for the VM width
    bool any_fault = false, any_act = false;
    for (auto& s : prog) {
      if (s.dst >= 0) max_value_ = std::max(max_value_, iv(s.dst).hi);
      for (int v : {s.a, s.b, s.auxv})
        if (v >= 0) max_value_ = std::max(max_value_, iv(v).hi);
      if (s.code == VM_BAND || s.code == VM_MOVI || (s.code == VM_TRIP && s.auxv < 0))
        max_value_ = std::max(max_value_, s.imm);
      any_fault |= s.faulting;
      any_act |= s.code == VM_ACT;
    }
    max_value_ = std::max(max_value_, C_.n_threads - 1);
    max_value_ = std::max(max_value_, C_.n_blocks - 1);

    // register allocation (linear scan over straight-line code)
    const int L = (int)path_.size();
    std::vector<int> last(vals_.size(), -1);
    for (int i = 0; i < (int)prog.size(); ++i)
      for (int v : {prog[i].a, prog[i].b, prog[i].auxv})
        if (v >= 0) last[v] = i;
    std::vector<int> reg(vals_.size(), -1);
    reg[tid_] = MAPC_REG_TID;
    reg[bid_] = MAPC_REG_BID;
    int nl = 0;                                      // tuple coordinates (the unrolled level is none)
    for (int l = 0; l < L; ++l)
      if (l != unroll_depth_) reg[k_[l]] = MAPC_REG_K0 + nl++;
    std::vector<int> freelist;
    for (int r = MAPC_NREG - 1; r >= MAPC_REG_K0 + nl; --r) freelist.push_back(r);
    auto pinned = [&](int v) { return v == tid_ || v == bid_ || std::find(k_.begin(), k_.end(), v) != k_.end(); };

    std::vector<MapcOp> ops;
    auto alloc = [&]() {
      if (freelist.empty()) range_error("group program needs more than MAPC_NREG registers");
      int r = freelist.back();
      freelist.pop_back();
      return r;
    };
    auto release_after = [&](int i, std::initializer_list<int> vs) {
      std::set<int> done;
      for (int v : vs)
        if (v >= 0 && !isc(v) && !pinned(v) && last[v] == i && reg[v] >= 0 && !done.count(v)) {
          freelist.push_back(reg[v]);
          done.insert(v);
        }
    };
    for (int i = 0; i < (int)prog.size(); ++i) {
      SIns s = prog[i];
      MapcOp op{};
      op.code = s.code;
      // two constant operands: materialise a
      if (s.a >= 0 && s.b >= 0 && isc(s.a) && isc(s.b)) {
        MapcOp mv{};
        mv.code = VM_MOVI;
        int r = alloc();
        mv.dst = (uint8_t)r;
        mv.imm = cv(s.a);
        ops.push_back(mv);
        // temporary register holds a for this op only
        op.a = (uint8_t)r;
        op.b = 0;
        op.code |= MAPC_B_IMM;
        op.imm = cv(s.b);
        freelist.push_back(r);
      } else {
        if (s.a >= 0) {
          if (isc(s.a)) { op.code |= MAPC_A_IMM; op.imm = cv(s.a); }
          else op.a = (uint8_t)reg[s.a];
        }
        if (s.b >= 0) {
          if (isc(s.b)) { op.code |= MAPC_B_IMM; op.imm = cv(s.b); }
          else op.b = (uint8_t)reg[s.b];
        }
      }
      if (s.code == VM_BAND || s.code == VM_MOVI) op.imm = s.imm;
      if (s.code == VM_TRIP) op.aux = s.auxv >= 0 ? (uint32_t)reg[s.auxv] : (MAPC_AUX_CONST | (uint32_t)s.imm);
      if (s.code == VM_MADK) op.aux = (uint32_t)reg[s.auxv];
      if (s.code == VM_EMIT) op.aux = s.emit_aux;
      if ((s.code == VM_DIV || s.code == VM_MOD) && s.faulting) op.aux = MAPC_AUX_FAULT;
      release_after(i, {s.a, s.b, s.auxv});
      if (s.dst >= 0) {
        int r = alloc();
        reg[s.dst] = r;
        op.dst = (uint8_t)r;
        if (last[s.dst] < 0) freelist.push_back(r);   // dead after def (kept for side effects)
      }
      ops.push_back(op);
    }
    out->ops = std::move(ops);
    out->n_levels = (uint32_t)nl;
    uint64_t tpb = C_.n_threads;
    for (int l = 0, j = 0; l < L; ++l) {
      if (l == unroll_depth_) continue;
      out->trips[j++] = trips_[l];
      tpb = checked((u128)tpb * trips_[l], "tuple count");
    }
    out->tuples_per_block = tpb;
    out->n_emits = n_emits_;
    out->has_emit = n_emits_ > 0;
    out->dense = out->has_emit && !any_fault && !any_act;
    out->index = n_emits_ ? index_hull_ : Interval{0, 0};
    out->site_kb = emit_kb_;
    out->site_kv = emit_kv_;
    has_fault_ = any_fault;
  }

 public:
  bool has_fault_ = false;
};

// ----------------------------------------------------------------------------
struct Builder {
  Compiled& C;
  std::vector<int> parent;
  std::vector<uint64_t> syncenv;
  std::vector<bool> sync_set;
  uint32_t phase = 0;
  uint64_t instances = 0;
  std::vector<std::pair<int, std::vector<uint64_t>>> pending;   // (tmpl, syncenv) per instance
  // choose_tuple_order per distinct group program in this compile (the phases of a
  // time loop repeat the same few programs: 5a's 16 phases have 2)
  std::map<std::string, bool> order_memo;

  explicit Builder(Compiled& c) : C(c) {}

  void parents() {
    const Program& P = C.ast;
    parent.assign(P.stmts.size(), -1);
    for (size_t s = 0; s < P.stmts.size(); ++s) {
      const Stmt& st = P.stmts[s];
      auto set = [&](int c) { if (c >= 0) parent[c] = (int)s; };
      for (int c : st.items) set(c);
      if (st.kind == Stmt::If) { set(st.then_s); set(st.else_s); }
      if (st.kind == Stmt::ForU || st.kind == Stmt::ForS) set(st.body);
    }
  }

  // Walk the synchronized fragment (phase enumeration).
  void sync_walk(int s) {
    const Program& P = C.ast;
    const Stmt& st = P.stmts[s];
    UniformEval U{P, C.params, syncenv, sync_set};
    switch (st.kind) {
      case Stmt::Sync:
        ++phase;
        if (phase > (1u << 24)) range_error("more than 2^24 barrier phases");
        return;
      case Stmt::Seq:
        for (int c : st.items) sync_walk(c);
        return;
      case Stmt::ForS: {
        uint64_t lo, hi, sp;
        if (!U.try_eval(st.lo, &lo) || !U.try_eval(st.hi, &hi) || !U.try_eval(st.step, &sp))
          throw CompileError{3, "forS bounds are not thread-uniform"};
        if (sp == 0) throw CompileError{5, "loop step is zero"};
        for (uint64_t x = lo; x < hi;) {
          syncenv[st.var] = x;
          sync_set[st.var] = true;
          sync_walk(st.body);
          if (x > kU64 - sp) break;
          x += sp;
        }
        sync_set[st.var] = false;
        return;
      }
      case Stmt::Skip:
        return;
      default:   // a u-fragment: one instance in the current phase
        if (++instances > (1u << 20)) range_error("more than 2^20 protocol instances");
        pending.emplace_back(s, syncenv);
        lower_instance(s, phase);
        return;
    }
  }

  // collect loop paths of sites / possibly-faulting expressions
  void collect(int s, std::vector<int>& path, std::map<std::vector<int>, std::vector<int>>& sites,
               std::set<std::vector<int>>& all_paths, std::vector<std::vector<int>>& order) {
    const Program& P = C.ast;
    const Stmt& st = P.stmts[s];
    auto note = [&](const std::vector<int>& p) {
      if (!all_paths.count(p)) { all_paths.insert(p); order.push_back(p); }
    };
    switch (st.kind) {
      case Stmt::Access:
        note(path);
        sites[path].push_back(s);
        return;
      case Stmt::Seq:
        for (int c : st.items) collect(c, path, sites, all_paths, order);
        return;
      case Stmt::If:
        note(path);    // conditions may fault; the lowerer decides
        collect(st.then_s, path, sites, all_paths, order);
        collect(st.else_s, path, sites, all_paths, order);
        return;
      case Stmt::ForU:
        note(path);
        if (path.size() >= MAPC_MAX_LEVELS) range_error("forU nesting deeper than 8");
        path.push_back(s);
        collect(st.body, path, sites, all_paths, order);
        path.pop_back();
        return;
      default:
        return;
    }
  }

  void lower_instance(int tmpl, uint32_t ph) {
    InstanceInfo info;
    info.tmpl = tmpl;
    info.phase = ph;
    std::vector<int> path;
    std::map<std::vector<int>, std::vector<int>> sites;
    std::set<std::vector<int>> all;
    std::vector<std::vector<int>> order;
    collect(tmpl, path, sites, all, order);
    for (const auto& p : order) {
      std::vector<int> ss = sites.count(p) ? sites[p] : std::vector<int>{};
      size_t nsub = ss.empty() ? 1 : (ss.size() + MAPC_MAX_EMITS - 1) / MAPC_MAX_EMITS;
      for (size_t k = 0; k < nsub; ++k) {
        std::set<int> filt;
        for (size_t j = k * MAPC_MAX_EMITS; j < std::min(ss.size(), (k + 1) * MAPC_MAX_EMITS); ++j) filt.insert(ss[j]);
        Lowerer Lw(C, syncenv, sync_set, p, filt, /*fault_owner=*/k == 0, parent);
        GroupProg g;
        if (!Lw.run(tmpl, &g)) continue;
        if (!g.has_emit && !Lw.has_fault_) continue;
        std::vector<GroupProg> parts;
        std::vector<uint64_t> part_max;
        // A sparse group -- its index hull far wider than its accesses, e.g. a
        // loop variable in both factors of a product, which intervals cannot
        // correlate (Blelloch down-sweep with forU levels) -- is split into one
        // group per iteration of its outermost constant-bounds loop of <= 64
        // iterations: each part's hull is exact for that value.
        const unsigned __int128 acc = (unsigned __int128)g.tuples_per_block * std::max<uint32_t>(g.n_emits, 1);
        const uint64_t span = g.has_emit && g.index.hi >= g.index.lo ? g.index.hi - g.index.lo : 0;
        if (g.has_emit && (unsigned __int128)span > 64 * acc) {
          for (size_t d = 0; d < p.size(); ++d) {
            const uint64_t T = Lw.const_trip(d);
            if (T == 0 || T > 64) continue;
            std::vector<GroupProg> ps;
            std::vector<uint64_t> pm;
            uint64_t lo = ~0ull, hi = 0;
            bool ok = true;
            for (uint64_t u = 0; u < T && ok; ++u) {
              Lowerer Lu(C, syncenv, sync_set, p, filt, k == 0, parent, (int)d, u);
              GroupProg gu;
              const bool nonempty = Lu.run(tmpl, &gu);
              if (Lu.unroll_failed()) { ok = false; break; }
              if (!nonempty || (!gu.has_emit && !Lu.has_fault_)) continue;
              if (gu.has_emit) { lo = std::min(lo, gu.index.lo); hi = std::max(hi, gu.index.hi); }
              pm.push_back(Lu.max_value());
              ps.push_back(std::move(gu));
            }
            if (ok && !ps.empty() && hi >= lo && (hi - lo) < span / 4) {
              parts = std::move(ps);
              part_max = std::move(pm);
            }
            break;
          }
        }
        if (parts.empty()) {
          parts.push_back(std::move(g));
          part_max.push_back(Lw.max_value());
        }
        for (size_t q = 0; q < parts.size(); ++q) {
          GroupProg& gq = parts[q];
          if (part_max[q] >= (1ull << 32)) C.u32_mode = false;
          {
            std::string key(reinterpret_cast<const char*>(gq.ops.data()), gq.ops.size() * sizeof(MapcOp));
            key.append(reinterpret_cast<const char*>(gq.trips), sizeof(gq.trips));
            key.append(reinterpret_cast<const char*>(&gq.n_levels), sizeof(gq.n_levels));
            key.append(reinterpret_cast<const char*>(&gq.n_emits), sizeof(gq.n_emits));
            key.append(reinterpret_cast<const char*>(&gq.tuples_per_block), sizeof(gq.tuples_per_block));
            auto it = order_memo.find(key);
            if (it != order_memo.end()) {
              gq.tid_inner = it->second;
            } else {
              choose_tuple_order(&gq, C.n_threads);
              order_memo.emplace(std::move(key), gq.tid_inner);
            }
          }
          info.bound_per_block = checked((u128)info.bound_per_block +
                                             (u128)gq.tuples_per_block * std::max<uint32_t>(gq.n_emits, 0),
                                         "access bound");
          C.total_ops += (uint32_t)gq.ops.size();
          ++C.n_groups;
          info.groups.push_back(std::move(gq));
        }
      }
    }
    if (!info.groups.empty()) C.inst.push_back(std::move(info));
  }
};

// ---- tuple order (coalescing) ------------------------------------------------
// Concrete evaluation of a group program for one tuple on the host (64-bit
// naturals; the interval analysis already proved the device's width exact).
// Records the index of every EMIT whose guard holds, in site order (-1 = no emit).
void eval_sites(const GroupProg& g, uint64_t tid, uint64_t bid, const uint64_t* k, std::vector<int64_t>* out) {
  uint64_t r[MAPC_NREG] = {};
  r[MAPC_REG_TID] = tid;
  r[MAPC_REG_BID] = bid;
  for (uint32_t l = 0; l < g.n_levels; ++l) r[MAPC_REG_K0 + l] = k[l];
  bool act = true;
  out->clear();
  for (const MapcOp& op : g.ops) {
    const uint32_t c = op.code & MAPC_CODE_MASK;
    const uint64_t A = (op.code & MAPC_A_IMM) ? op.imm : r[op.a];
    const uint64_t B = (op.code & MAPC_B_IMM) ? op.imm : r[op.b];
    uint64_t v = 0;
    switch (c) {
      case VM_ADD: v = A + B; break;
      case VM_SUB: v = A > B ? A - B : 0; break;
      case VM_MUL: v = A * B; break;
      case VM_DIV: v = B ? A / B : 0; break;
      case VM_MOD: v = B ? A % B : 0; break;
      case VM_SHL: v = B >= 64 ? 0 : A << B; break;
      case VM_SHR: v = B >= 64 ? 0 : A >> B; break;
      case VM_MIN: v = std::min(A, B); break;
      case VM_MAX: v = std::max(A, B); break;
      case VM_BAND: v = A & op.imm; break;
      case VM_EQ: v = A == B; break;
      case VM_NE: v = A != B; break;
      case VM_LT: v = A < B; break;
      case VM_LE: v = A <= B; break;
      case VM_GT: v = A > B; break;
      case VM_GE: v = A >= B; break;
      case VM_LAND: v = (A != 0) && (B != 0); break;
      case VM_LOR: v = (A != 0) || (B != 0); break;
      case VM_LNOT: v = A == 0; break;
      case VM_TRIP: {
        const uint64_t st = (op.aux & MAPC_AUX_CONST) ? (op.aux & ~MAPC_AUX_CONST) : r[op.aux];
        const uint64_t sp = B > A ? B - A : 0;
        v = sp == 0 ? 0 : (st <= 1 ? sp : (sp - 1) / st + 1);
        break;
      }
      case VM_MADK: v = A + r[op.aux] * B; break;
      case VM_MOVI: v = op.imm; break;
      case VM_ACT: act = A != 0; continue;
      case VM_EMIT: out->push_back(act ? (int64_t)A : -1); continue;
      default: continue;
    }
    r[op.dst] = v;
  }
}

// Sectors (32 B of u32 cells) touched by one warp of 32 consecutive tuples at a
// few positions of block 0's tuple space, per site, summed.
uint64_t warp_sectors(const GroupProg& g, uint64_t n_threads, bool tid_inner) {
  const uint64_t n = g.tuples_per_block;
  uint64_t total = 0;
  std::vector<int64_t> idx;
  for (int pos = 1; pos <= 3; ++pos) {
    const uint64_t t0 = (n * pos / 4) / 32 * 32;
    std::vector<std::vector<int64_t>> sec(g.n_emits);
    for (auto& v : sec) v.reserve(32);
    for (uint64_t t = t0; t < std::min(n, t0 + 32); ++t) {
      uint64_t rem = t, tid, k[MAPC_MAX_LEVELS] = {};
      if (tid_inner) { tid = rem % n_threads; rem /= n_threads; }
      for (int l = (int)g.n_levels - 1; l >= 0; --l) { k[l] = rem % g.trips[l]; rem /= g.trips[l]; }
      if (!tid_inner) tid = rem % n_threads;
      eval_sites(g, tid, 0, k, &idx);
      for (size_t e = 0; e < idx.size() && e < sec.size(); ++e)
        if (idx[e] >= 0) sec[e].push_back(idx[e] >> 3);
    }
    for (auto& v : sec) {
      std::sort(v.begin(), v.end());
      total += std::unique(v.begin(), v.end()) - v.begin();
    }
  }
  return total;
}

void choose_tuple_order(GroupProg* g, uint64_t n_threads) {
  g->tid_inner = false;
  if (g->n_levels == 0 || n_threads == 1 || !g->has_emit) return;
  g->tid_inner = warp_sectors(*g, n_threads, true) < warp_sectors(*g, n_threads, false);
}

}  // namespace

void eval_ops_sites(const std::vector<MapcOp>& ops, uint32_t n_levels, uint64_t tid, uint64_t bid, const uint64_t* k,
                    std::vector<int64_t>* out) {
  GroupProg g;
  g.ops = ops;
  g.n_levels = n_levels;
  eval_sites(g, tid, bid, k, out);
}

Compiled compile_map(const std::string& text, const uint32_t grid[3], const uint32_t block[3],
                     const std::vector<std::string>& names, const std::vector<uint64_t>& values) {
  Compiled C;
  C.ast = parse_map(text);
  C.n_threads = (uint64_t)block[0] * block[1] * block[2];
  C.n_blocks = (uint64_t)grid[0] * grid[1] * grid[2];
  if (C.n_threads == 0 || C.n_blocks == 0) throw CompileError{8, "empty grid or block"};
  if (C.n_threads > (1ull << 20)) throw CompileError{4, "blockDim exceeds 2^20 threads"};
  if (C.n_blocks > (1ull << 31)) throw CompileError{4, "gridDim exceeds 2^31 blocks"};
  C.w_tid = bits_for(C.n_threads - 1);
  C.params.assign(C.ast.params.size(), 0);
  std::vector<bool> given(C.ast.params.size(), false);
  for (size_t i = 0; i < names.size(); ++i) {
    auto it = std::find(C.ast.params.begin(), C.ast.params.end(), names[i]);
    if (it == C.ast.params.end()) throw CompileError{8, "unknown parameter '" + names[i] + "'"};
    size_t k = it - C.ast.params.begin();
    C.params[k] = values[i];
    given[k] = true;
  }
  for (size_t k = 0; k < given.size(); ++k)
    if (!given[k]) throw CompileError{8, "parameter '" + C.ast.params[k] + "' has no value"};

  Builder B(C);
  B.parents();
  B.syncenv.assign(C.ast.vars.size(), 0);
  B.sync_set.assign(C.ast.vars.size(), false);
  B.sync_walk(C.ast.root);
  C.n_phases = B.phase + 1;

  // bounds per phase
  std::map<uint32_t, uint64_t> per_phase;
  for (auto& in : C.inst) {
    per_phase[in.phase] = checked((u128)per_phase[in.phase] + in.bound_per_block, "bound");
    C.max_accesses = checked((u128)C.max_accesses + (u128)in.bound_per_block * C.n_blocks, "bound");
  }
  for (auto& kv : per_phase) C.max_unit = std::max(C.max_unit, kv.second);
  return C;
}

}  // namespace mapc
