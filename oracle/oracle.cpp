// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY (not part of the product path).
//
// A plain, slow, obviously-correct CPU definition of what the hot path computes:
// the concrete, exhaustive data-race check of a memory access protocol (MAP)
// instantiated at fixed grid/block dimensions and parameter values.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  It shares no code, header,
// table or helper with paper_2203_12878_b200/ (the CUDA path); the two agree
// only through the MAP text grammar written down in DESIGN.md §3.
//
// What it computes, step by step:
//   1. parse the MAP text with its own recursive-descent parser and resolve
//      names (an unbound identifier is an error);
//   2. for every block b and every thread i in T = {0..blockDim-1} walk the
//      protocol with env {tid -> i, bid -> b, params}: this is the per-thread
//      big-step evaluation of PAPER.md:479-558 with the data erased (seq,
//      if-t/if-f, for-1/for-2 -- rules at PAPER.md:506-551), unioned over
//      threads as in rule par.  Each access o[n] emits the
//      access value alpha = i : o[y] tagged with the
//      barrier phase (number of syncs executed before it),
//      the array and the block;
//   3. Lambda per (phase, array, block) is the SET of access values
//      (PAPER.md:894); n_accesses counts the multiset (the throughput unit);
//   4. a data race is two accesses to the same index by two distinct threads,
//      at least one a write, within one phase (
//      SPEC.md:423-426, 490, 502).  The oracle buckets the access values by
//      (phase, array, block, index) and tests EVERY pair of distinct access
//      values in the bucket naively;
//   5. the witness is the lexicographic minimum of
//      (phase, array, block, index, t_lo, t_hi, k_lo, k_hi), t_lo < t_hi,
//      rd = 0 < wr = 1 (reading R14).
//
// Arithmetic is exact on naturals computed in uint64;
// an actual overflow is an error (status 4), so is div/mod by zero (status 5).
// Subtraction is monus.
//
// Status codes (same numbers as DESIGN.md §4 by specification, not by shared
// header): 0 ok, 1 parse, 2 scope, 3 barrier, 4 range/overflow, 5 arith,
// 8 bad argument.

#include <algorithm>
#include <array>
#include <atomic>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#include <parallel/algorithm>
#endif

namespace {

enum Status { OK = 0, E_PARSE = 1, E_SCOPE = 2, E_BARRIER = 3, E_RANGE = 4, E_ARITH = 5, E_ARG = 8 };

struct Error {
  int status;
  std::string msg;
};

// ------------------------------------------------------------------ lexer --
enum Tok { T_EOF, T_NAT, T_ID, T_PUNCT };

struct Token {
  Tok kind;
  std::string text;
  uint64_t value = 0;
  int line = 1, col = 1;
};

std::vector<Token> lex(const std::string& s) {
  std::vector<Token> out;
  int line = 1, col = 1;
  size_t i = 0;
  auto adv = [&](size_t n) {
    for (size_t k = 0; k < n; ++k) {
      if (s[i] == '\n') { ++line; col = 1; } else { ++col; }
      ++i;
    }
  };
  while (i < s.size()) {
    char c = s[i];
    if (isspace((unsigned char)c)) { adv(1); continue; }
    if (c == '/' && i + 1 < s.size() && s[i + 1] == '/') {
      while (i < s.size() && s[i] != '\n') adv(1);
      continue;
    }
    Token t;
    t.line = line; t.col = col;
    if (isdigit((unsigned char)c)) {
      size_t j = i;
      uint64_t v = 0;
      bool big = false;
      while (j < s.size() && isdigit((unsigned char)s[j])) {
        uint64_t d = (uint64_t)(s[j] - '0');
        if (v > (UINT64_MAX - d) / 10) big = true;
        v = v * 10 + d;
        ++j;
      }
      if (big) throw Error{E_RANGE, std::to_string(line) + ":" + std::to_string(col) + ": literal too large"};
      t.kind = T_NAT; t.value = v; t.text = s.substr(i, j - i);
      adv(j - i);
    } else if (isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < s.size() && (isalnum((unsigned char)s[j]) || s[j] == '_')) ++j;
      t.kind = T_ID; t.text = s.substr(i, j - i);
      adv(j - i);
    } else {
      static const char* two[] = {"..", "<<", ">>", "<=", ">=", "!="};
      std::string p;
      for (const char* tw : two)
        if (s.compare(i, 2, tw) == 0) { p = tw; break; }
      if (p.empty()) {
        if (std::strchr(";,(){}[]+-*/%=<>", c) == nullptr)
          throw Error{E_PARSE, std::to_string(line) + ":" + std::to_string(col) + ": unexpected character"};
        p = std::string(1, c);
      }
      t.kind = T_PUNCT; t.text = p;
      adv(p.size());
    }
    out.push_back(t);
  }
  Token e; e.kind = T_EOF; e.line = line; e.col = col;
  out.push_back(e);
  return out;
}

// -------------------------------------------------------------------- AST --
// Variables are resolved to slots of a per-thread environment vector.
enum NKind { N_NAT, N_SLOT, N_BIN };
struct Num {
  NKind k;
  uint64_t v = 0;      // N_NAT literal
  int slot = -1;       // N_SLOT
  std::string op;      // N_BIN: + - * / % << >> min max
  std::unique_ptr<Num> a, b;
};

enum CKind { C_TRUE, C_FALSE, C_REL, C_AND, C_OR };
struct Cond {
  CKind k;
  std::string rel;     // = != < <= > >=
  std::unique_ptr<Num> a, b;
  std::unique_ptr<Cond> l, r;
};

enum SKind { S_SKIP, S_SYNC, S_ACC, S_SEQ, S_IF, S_FORU, S_FORS };
struct Stmt {
  SKind k;
  int wr = 0, array = 0;                    // S_ACC
  std::unique_ptr<Num> idx;                 // S_ACC
  std::vector<std::unique_ptr<Stmt>> seq;   // S_SEQ
  std::unique_ptr<Cond> cond;               // S_IF
  std::unique_ptr<Stmt> thn, els;           // S_IF
  int slot = -1;                            // loops: the loop variable's slot
  std::unique_ptr<Num> lo, hi, step;        // loops
  std::unique_ptr<Stmt> body;               // loops
};

// Slot 0 = tid, slot 1 = bid, then params, then one slot per loop binder.
constexpr int SLOT_TID = 0, SLOT_BID = 1;

struct Program {
  std::vector<std::string> params;
  std::vector<std::string> arrays;
  int n_slots = 2;
  std::unique_ptr<Stmt> body;
};

// ----------------------------------------------------------------- parser --
struct Parser {
  std::vector<Token> t;
  size_t p = 0;
  Program prog;
  std::vector<std::pair<std::string, int>> scope;  // visible names -> slot

  [[noreturn]] void fail(int st, const Token& at, const std::string& m) {
    throw Error{st, std::to_string(at.line) + ":" + std::to_string(at.col) + ": " + m};
  }
  const Token& cur() { return t[p]; }
  bool is(const char* s) { return (t[p].kind == T_PUNCT || t[p].kind == T_ID) && t[p].text == s; }
  void expect(const char* s) {
    if (!is(s)) fail(E_PARSE, cur(), std::string("expected '") + s + "'");
    ++p;
  }
  static bool reserved(const std::string& s) {
    static const char* kw[] = {"skip", "sync", "rd", "wr", "if", "else", "forU", "forS", "in", "step",
                               "true", "false", "and", "or", "tid", "bid", "params", "shared", "min", "max"};
    for (const char* k : kw) if (s == k) return true;
    return false;
  }
  int lookup(const std::string& name) {
    for (auto it = scope.rbegin(); it != scope.rend(); ++it)
      if (it->first == name) return it->second;
    return -1;
  }
  std::string ident() {
    if (cur().kind != T_ID || reserved(cur().text)) fail(E_PARSE, cur(), "expected identifier");
    return t[p++].text;
  }

  // n: shift-level (lowest) < additive < multiplicative < atom
  std::unique_ptr<Num> num() {
    auto a = additive();
    while (is("<<") || is(">>")) {
      std::string op = t[p++].text;
      auto n = std::make_unique<Num>();
      n->k = N_BIN; n->op = op; n->a = std::move(a); n->b = additive();
      a = std::move(n);
    }
    return a;
  }
  std::unique_ptr<Num> additive() {
    auto a = mult();
    while (is("+") || is("-")) {
      std::string op = t[p++].text;
      auto n = std::make_unique<Num>();
      n->k = N_BIN; n->op = op; n->a = std::move(a); n->b = mult();
      a = std::move(n);
    }
    return a;
  }
  std::unique_ptr<Num> mult() {
    auto a = atom();
    while (is("*") || is("/") || is("%")) {
      std::string op = t[p++].text;
      auto n = std::make_unique<Num>();
      n->k = N_BIN; n->op = op; n->a = std::move(a); n->b = atom();
      a = std::move(n);
    }
    return a;
  }
  std::unique_ptr<Num> atom() {
    auto n = std::make_unique<Num>();
    const Token& c = cur();
    if (c.kind == T_NAT) { n->k = N_NAT; n->v = c.value; ++p; return n; }
    if (is("(")) { ++p; auto e = num(); expect(")"); return e; }
    if (is("min") || is("max")) {
      n->k = N_BIN; n->op = t[p++].text;
      expect("("); n->a = num(); expect(","); n->b = num(); expect(")");
      return n;
    }
    if (is("tid")) { ++p; n->k = N_SLOT; n->slot = SLOT_TID; return n; }
    if (is("bid")) { ++p; n->k = N_SLOT; n->slot = SLOT_BID; return n; }
    if (c.kind == T_ID && !reserved(c.text)) {
      int s = lookup(c.text);
      if (s < 0) fail(E_SCOPE, c, "unbound identifier '" + c.text + "'");
      ++p; n->k = N_SLOT; n->slot = s; return n;
    }
    fail(E_PARSE, c, "expected an arithmetic expression");
  }

  static bool is_rel(const Token& k) {
    if (k.kind != T_PUNCT) return false;
    return k.text == "=" || k.text == "!=" || k.text == "<" || k.text == "<=" || k.text == ">" || k.text == ">=";
  }
  // c: or-level < and-level < atom
  std::unique_ptr<Cond> cond() {
    auto a = cand();
    while (is("or")) {
      ++p;
      auto c = std::make_unique<Cond>();
      c->k = C_OR; c->l = std::move(a); c->r = cand();
      a = std::move(c);
    }
    return a;
  }
  std::unique_ptr<Cond> cand() {
    auto a = catom();
    while (is("and")) {
      ++p;
      auto c = std::make_unique<Cond>();
      c->k = C_AND; c->l = std::move(a); c->r = catom();
      a = std::move(c);
    }
    return a;
  }
  std::unique_ptr<Cond> catom() {
    auto c = std::make_unique<Cond>();
    if (is("true")) { ++p; c->k = C_TRUE; return c; }
    if (is("false")) { ++p; c->k = C_FALSE; return c; }
    if (is("(")) {
      // Either a parenthesised condition or a parenthesised arithmetic operand
      // of a comparison: try the condition first, backtrack if it does not fit.
      size_t save = p;
      try {
        ++p;
        auto inner = cond();
        expect(")");
        if (!is_rel(cur())) return inner;
      } catch (const Error& e) {
        if (e.status == E_SCOPE) throw;
      }
      p = save;
    }
    c->k = C_REL;
    c->a = num();
    if (!is_rel(cur())) fail(E_PARSE, cur(), "expected a comparison operator");
    c->rel = t[p++].text;
    c->b = num();
    return c;
  }

  // proto := stmt (";" stmt)* [";"]
  std::unique_ptr<Stmt> proto(const char* closer) {
    auto s = std::make_unique<Stmt>();
    s->k = S_SEQ;
    s->seq.push_back(stmt());
    while (is(";")) {
      ++p;
      if ((closer && is(closer)) || cur().kind == T_EOF) break;
      s->seq.push_back(stmt());
    }
    return s;
  }
  std::unique_ptr<Stmt> block() {
    expect("{");
    auto b = proto("}");
    expect("}");
    return b;
  }
  std::unique_ptr<Stmt> stmt() {
    auto s = std::make_unique<Stmt>();
    const Token& c = cur();
    if (is("skip")) { ++p; s->k = S_SKIP; return s; }
    if (is("sync")) { ++p; s->k = S_SYNC; return s; }
    if (is("rd") || is("wr")) {
      s->k = S_ACC; s->wr = is("wr") ? 1 : 0; ++p;
      s->array = 0;
      if (!is("[")) {
        const Token& an = cur();
        std::string a = ident();
        auto it = std::find(prog.arrays.begin(), prog.arrays.end(), a);
        if (it == prog.arrays.end()) fail(E_SCOPE, an, "undeclared array '" + a + "'");
        s->array = (int)(it - prog.arrays.begin());
      }
      expect("["); s->idx = num(); expect("]");
      return s;
    }
    if (is("if")) {
      ++p; s->k = S_IF;
      expect("("); s->cond = cond(); expect(")");
      s->thn = block();
      if (is("else")) { ++p; s->els = block(); }
      else { s->els = std::make_unique<Stmt>(); s->els->k = S_SKIP; }
      return s;
    }
    if (is("forU") || is("forS")) {
      s->k = is("forU") ? S_FORU : S_FORS; ++p;
      const Token& vt = cur();
      std::string v = ident();
      if (lookup(v) >= 0) fail(E_SCOPE, vt, "binder '" + v + "' shadows a visible name");
      expect("in");
      s->lo = num(); expect(".."); s->hi = num();
      if (is("step")) { ++p; s->step = num(); }
      else { s->step = std::make_unique<Num>(); s->step->k = N_NAT; s->step->v = 1; }
      s->slot = prog.n_slots++;
      scope.push_back({v, s->slot});
      s->body = block();
      scope.pop_back();
      return s;
    }
    fail(E_PARSE, c, "expected a statement");
  }

  void parse() {
    scope.push_back({"tid", SLOT_TID});
    scope.push_back({"bid", SLOT_BID});
    while (is("params") || is("shared")) {
      bool params = is("params");
      ++p;
      for (;;) {
        const Token& nt = cur();
        std::string n = ident();
        if (lookup(n) >= 0 || std::find(prog.arrays.begin(), prog.arrays.end(), n) != prog.arrays.end())
          fail(E_SCOPE, nt, "duplicate declaration of '" + n + "'");
        if (params) {
          prog.params.push_back(n);
          scope.push_back({n, prog.n_slots++});
        } else {
          prog.arrays.push_back(n);
        }
        if (is(",")) { ++p; continue; }
        break;
      }
      expect(";");
    }
    if (prog.arrays.empty()) prog.arrays.push_back("A");  // the single array of PAPER.md:335-337
    prog.body = proto(nullptr);
    if (cur().kind != T_EOF) fail(E_PARSE, cur(), "trailing input");
  }
};

// Barrier placement (readings R7/R8): sync and forS belong to the
// synchronized fragment p; they may not occur under if or
// forU (the unsynchronized fragment u), and forS bounds must
// be thread-uniform (no tid, no bid).
bool mentions_thread(const Num* n) {
  if (!n) return false;
  if (n->k == N_SLOT) return n->slot == SLOT_TID || n->slot == SLOT_BID;
  if (n->k == N_BIN) return mentions_thread(n->a.get()) || mentions_thread(n->b.get());
  return false;
}
void check_barriers(const Stmt* s, bool in_u) {
  switch (s->k) {
    case S_SYNC:
      if (in_u) throw Error{E_BARRIER, "sync inside if/forU"};
      break;
    case S_SEQ:
      for (auto& c : s->seq) check_barriers(c.get(), in_u);
      break;
    case S_IF:
      check_barriers(s->thn.get(), true);
      check_barriers(s->els.get(), true);
      break;
    case S_FORU:
      check_barriers(s->body.get(), true);
      break;
    case S_FORS:
      if (in_u) throw Error{E_BARRIER, "forS inside if/forU"};
      if (mentions_thread(s->lo.get()) || mentions_thread(s->hi.get()) || mentions_thread(s->step.get()))
        throw Error{E_BARRIER, "forS bounds depend on tid/bid"};
      check_barriers(s->body.get(), false);
      break;
    default:
      break;
  }
}

// -------------------------------------------------------------- evaluator --
struct Record {          // one emitted access value, tagged
  uint32_t phase, array, block, tid;
  uint64_t index;
  uint32_t wr;
};

struct Walker {
  const Program& prog;
  std::vector<uint64_t> env;
  uint32_t phase = 0;
  uint32_t block = 0;
  std::vector<Record>* out;

  uint64_t eval(const Num* n) {
    if (n->k == N_NAT) return n->v;
    if (n->k == N_SLOT) return env[n->slot];
    uint64_t a = eval(n->a.get()), b = eval(n->b.get());
    const std::string& op = n->op;
    if (op == "+") {
      if (a > UINT64_MAX - b) throw Error{E_RANGE, "overflow in +"};
      return a + b;
    }
    if (op == "-") return a > b ? a - b : 0;                 // monus
    if (op == "*") {
      if (a != 0 && b > UINT64_MAX / a) throw Error{E_RANGE, "overflow in *"};
      return a * b;
    }
    if (op == "/") { if (b == 0) throw Error{E_ARITH, "division by zero"}; return a / b; }
    if (op == "%") { if (b == 0) throw Error{E_ARITH, "modulo by zero"}; return a % b; }
    if (op == "<<") {
      if (a == 0) return 0;
      if (b >= 64 || a > (UINT64_MAX >> b)) throw Error{E_RANGE, "overflow in <<"};
      return a << b;
    }
    if (op == ">>") return b >= 64 ? 0 : a >> b;
    if (op == "min") return a < b ? a : b;
    return a > b ? a : b;                                     // max
  }
  bool test(const Cond* c) {
    switch (c->k) {
      case C_TRUE: return true;
      case C_FALSE: return false;
      case C_AND: { bool l = test(c->l.get()); bool r = test(c->r.get()); return l && r; }
      case C_OR: { bool l = test(c->l.get()); bool r = test(c->r.get()); return l || r; }
      default: break;
    }
    uint64_t a = eval(c->a.get()), b = eval(c->b.get());
    const std::string& r = c->rel;
    if (r == "=") return a == b;
    if (r == "!=") return a != b;
    if (r == "<") return a < b;
    if (r == "<=") return a <= b;
    if (r == ">") return a > b;
    return a >= b;
  }
  void run(const Stmt* s) {
    switch (s->k) {
      case S_SKIP: return;                                   // rule skip
      case S_SYNC: ++phase; return;                          // barrier: next phase
      case S_ACC:                                            // o[n]: emit alpha
        out->push_back(Record{phase, (uint32_t)s->array, block, (uint32_t)env[SLOT_TID], eval(s->idx.get()),
                              (uint32_t)s->wr});
        return;
      case S_SEQ:                                            // rule seq
        for (auto& c : s->seq) run(c.get());
        return;
      case S_IF:                                             // rules if-t / if-f
        if (test(s->cond.get())) run(s->thn.get()); else run(s->els.get());
        return;
      case S_FORU:
      case S_FORS: {                                         // rules for-1 / for-2
        uint64_t lo = eval(s->lo.get()), hi = eval(s->hi.get()), st = eval(s->step.get());
        if (st == 0) throw Error{E_ARITH, "loop step is zero"};
        for (uint64_t x = lo; x < hi;) {
          env[s->slot] = x;
          run(s->body.get());
          if (x > UINT64_MAX - st) break;
          x += st;
        }
        return;
      }
    }
  }
};

struct Result {
  int32_t status = 0;
  int32_t verdict = 0;                 // 0 DRF, 1 racy
  uint64_t n_accesses = 0;
  uint64_t n_racy_segments = 0;
  uint32_t phase = 0, array = 0, block = 0;
  uint64_t index = 0;
  uint32_t tid_lo = 0, tid_hi = 0;
  uint32_t kind_lo = 0, kind_hi = 0;
  uint32_t n_phases = 0;
};

struct Setup {
  Program prog;
  uint64_t n_blocks = 1, n_threads = 1;
  std::vector<uint64_t> env0;
};

int setup(const char* src, const uint32_t grid[3], const uint32_t blk[3], uint32_t n_params,
          const char* const* names, const uint64_t* values, Setup& S, std::string& diag) {
  try {
    Parser P;
    P.t = lex(src ? std::string(src) : std::string());
    P.parse();
    check_barriers(P.prog.body.get(), false);
    S.prog = std::move(P.prog);
  } catch (const Error& e) {
    diag = e.msg;
    return e.status;
  }
  S.n_blocks = (uint64_t)grid[0] * grid[1] * grid[2];
  S.n_threads = (uint64_t)blk[0] * blk[1] * blk[2];
  if (S.n_blocks == 0 || S.n_threads == 0) { diag = "empty grid or block"; return E_ARG; }
  S.env0.assign(S.prog.n_slots, 0);
  std::vector<bool> given(S.prog.params.size(), false);
  for (uint32_t i = 0; i < n_params; ++i) {
    auto it = std::find(S.prog.params.begin(), S.prog.params.end(), std::string(names[i]));
    if (it == S.prog.params.end()) { diag = std::string("unknown parameter '") + names[i] + "'"; return E_ARG; }
    size_t k = it - S.prog.params.begin();
    S.env0[2 + k] = values[i];
    given[k] = true;
  }
  for (size_t k = 0; k < given.size(); ++k)
    if (!given[k]) { diag = "parameter '" + S.prog.params[k] + "' has no value"; return E_ARG; }
  return OK;
}

// Step 2: walk every (block, thread); records of all threads, unsorted.
int enumerate(const Setup& S, int n_threads_omp, std::vector<Record>& all, std::string& diag) {
  const uint64_t units = S.n_blocks * S.n_threads;
  std::atomic<int> status{0};
  std::mutex mu;
  uint64_t err_unit = UINT64_MAX;
  std::string err_msg;
  int nt = n_threads_omp > 0 ? n_threads_omp : 1;
  std::vector<std::vector<Record>> part(nt);
#pragma omp parallel num_threads(nt)
  {
    int me = 0;
#ifdef _OPENMP
    me = omp_get_thread_num();
#endif
    Walker w{S.prog, S.env0, 0, 0, &part[me]};
#pragma omp for schedule(dynamic, 1)
    for (int64_t u = 0; u < (int64_t)units; ++u) {
      w.env = S.env0;
      w.block = (uint32_t)(u / S.n_threads);
      w.env[SLOT_TID] = (uint64_t)u % S.n_threads;
      w.env[SLOT_BID] = w.block;
      w.phase = 0;
      try {
        w.run(S.prog.body.get());
      } catch (const Error& e) {
        std::lock_guard<std::mutex> g(mu);
        if ((uint64_t)u < err_unit) { err_unit = u; err_msg = e.msg; status = e.status; }
      }
    }
  }
  if (status.load() != 0) { diag = err_msg; return status.load(); }
  size_t total = 0;
  for (auto& p : part) total += p.size();
  all.clear();
  all.reserve(total);
  for (auto& p : part) { all.insert(all.end(), p.begin(), p.end()); std::vector<Record>().swap(p); }
  return OK;
}

bool rec_less(const Record& x, const Record& y) {
  if (x.phase != y.phase) return x.phase < y.phase;
  if (x.array != y.array) return x.array < y.array;
  if (x.block != y.block) return x.block < y.block;
  if (x.index != y.index) return x.index < y.index;
  if (x.tid != y.tid) return x.tid < y.tid;
  return x.wr < y.wr;
}
bool rec_eq(const Record& x, const Record& y) {
  return x.phase == y.phase && x.array == y.array && x.block == y.block && x.index == y.index &&
         x.tid == y.tid && x.wr == y.wr;
}

// Steps 3-5.  `list` (optional): every racy bucket's minimal pair, in bucket
// order -- the per-segment form of SPEC.md:434-437 races_of.
void races(std::vector<Record>& recs, int nt, Result& r, std::vector<std::array<uint64_t, 8>>* list = nullptr) {
  r.n_accesses = recs.size();
  uint32_t maxphase = 0;
  for (auto& x : recs) maxphase = std::max(maxphase, x.phase);
  r.n_phases = recs.empty() ? 0 : maxphase + 1;
  // Lambda is a set: sort and drop duplicate access values.
#ifdef _OPENMP
  if (nt > 1) __gnu_parallel::sort(recs.begin(), recs.end(), rec_less);
  else std::sort(recs.begin(), recs.end(), rec_less);
#else
  (void)nt;
  std::sort(recs.begin(), recs.end(), rec_less);
#endif
  recs.erase(std::unique(recs.begin(), recs.end(), rec_eq), recs.end());
  bool have = false;
  size_t i = 0;
  while (i < recs.size()) {
    size_t j = i;
    while (j < recs.size() && recs[j].phase == recs[i].phase && recs[j].array == recs[i].array &&
           recs[j].block == recs[i].block && recs[j].index == recs[i].index)
      ++j;
    // Bucket [i, j): every pair of distinct access values, naively.
    bool racy = false;
    uint32_t best[4] = {0, 0, 0, 0};   // t_lo, t_hi, k_lo, k_hi
    for (size_t a = i; a < j; ++a)
      for (size_t b = a + 1; b < j; ++b) {
        const Record& x = recs[a];
        const Record& y = recs[b];
        if (x.tid == y.tid) continue;            // same thread never races
        if (!x.wr && !y.wr) continue;            // at least one write
        const Record& lo = x.tid < y.tid ? x : y;
        const Record& hi = x.tid < y.tid ? y : x;
        uint32_t cand[4] = {lo.tid, hi.tid, lo.wr, hi.wr};
        if (!racy || std::lexicographical_compare(cand, cand + 4, best, best + 4)) {
          std::copy(cand, cand + 4, best);
        }
        racy = true;
      }
    if (racy) {
      ++r.n_racy_segments;
      if (list)
        list->push_back({recs[i].phase, recs[i].array, recs[i].block, recs[i].index, best[0], best[1], best[2],
                         best[3]});
      if (!have) {     // buckets are visited in lexicographic order: first is min
        have = true;
        r.phase = recs[i].phase; r.array = recs[i].array; r.block = recs[i].block; r.index = recs[i].index;
        r.tid_lo = best[0]; r.tid_hi = best[1]; r.kind_lo = best[2]; r.kind_hi = best[3];
      }
    }
    i = j;
  }
  r.verdict = have ? 1 : 0;
}

void put_diag(const std::string& d, char* diag, size_t cap) {
  if (!diag || cap == 0) return;
  size_t n = std::min(cap - 1, d.size());
  std::memcpy(diag, d.data(), n);
  diag[n] = 0;
}

}  // namespace

extern "C" {

// Result record exported to Python (ctypes mirror in oracle/__init__.py).
typedef struct {
  int32_t status;
  int32_t verdict;
  uint64_t n_accesses;
  uint64_t n_racy_segments;
  uint32_t phase, array, block, pad0;
  uint64_t index;
  uint32_t tid_lo, tid_hi;
  uint32_t kind_lo, kind_hi;
  uint32_t n_phases, pad1;
} oracle_result;

int oracle_check(const char* src, const uint32_t grid[3], const uint32_t blk[3], uint32_t n_params,
                 const char* const* names, const uint64_t* values, int n_threads, oracle_result* out,
                 char* diag, size_t diag_cap) {
  std::memset(out, 0, sizeof(*out));
  Setup S;
  std::string d;
  int st = setup(src, grid, blk, n_params, names, values, S, d);
  if (st == OK) {
    std::vector<Record> recs;
    st = enumerate(S, n_threads, recs, d);
    if (st == OK) {
      Result r;
      races(recs, n_threads, r);
      out->verdict = r.verdict;
      out->n_accesses = r.n_accesses;
      out->n_racy_segments = r.n_racy_segments;
      out->phase = r.phase; out->array = r.array; out->block = r.block; out->index = r.index;
      out->tid_lo = r.tid_lo; out->tid_hi = r.tid_hi; out->kind_lo = r.kind_lo; out->kind_hi = r.kind_hi;
      out->n_phases = r.n_phases;
    }
  }
  out->status = st;
  put_diag(d, diag, diag_cap);
  return st;
}

// All emitted access records (multiset, thread walk order), 6 x u64 each:
// (phase, array, block, index, tid, kind).  Returns the record count, or
// -status on error; writes at most `cap` records.
int64_t oracle_enumerate(const char* src, const uint32_t grid[3], const uint32_t blk[3], uint32_t n_params,
                         const char* const* names, const uint64_t* values, int n_threads, uint64_t* rec_out,
                         uint64_t cap, char* diag, size_t diag_cap) {
  Setup S;
  std::string d;
  int st = setup(src, grid, blk, n_params, names, values, S, d);
  std::vector<Record> recs;
  if (st == OK) st = enumerate(S, n_threads, recs, d);
  put_diag(d, diag, diag_cap);
  if (st != OK) return -(int64_t)st;
  for (uint64_t i = 0; i < recs.size() && i < cap; ++i) {
    const Record& x = recs[i];
    uint64_t* o = rec_out + 6 * i;
    o[0] = x.phase; o[1] = x.array; o[2] = x.block; o[3] = x.index; o[4] = x.tid; o[5] = x.wr;
  }
  return (int64_t)recs.size();
}

// Every racy segment's minimal pair (phase, array, block, index, t_lo, t_hi,
// k_lo, k_hi) as 8 x u64, in canonical order; returns the number of racy
// segments (or -status), writes at most `cap` of them.
int64_t oracle_list_races(const char* src, const uint32_t grid[3], const uint32_t blk[3], uint32_t n_params,
                          const char* const* names, const uint64_t* values, int n_threads, uint64_t* out,
                          uint64_t cap, char* diag, size_t diag_cap) {
  Setup S;
  std::string d;
  int st = setup(src, grid, blk, n_params, names, values, S, d);
  std::vector<Record> recs;
  if (st == OK) st = enumerate(S, n_threads, recs, d);
  put_diag(d, diag, diag_cap);
  if (st != OK) return -(int64_t)st;
  Result r;
  std::vector<std::array<uint64_t, 8>> list;
  races(recs, n_threads, r, &list);
  for (uint64_t i = 0; i < list.size() && i < cap; ++i)
    for (int f = 0; f < 8; ++f) out[8 * i + f] = list[i][f];
  return (int64_t)list.size();
}

// Array names in declaration order (array ids); returns count.
int oracle_arrays(const char* src, char* buf, size_t cap) {
  try {
    Parser P;
    P.t = lex(src ? std::string(src) : std::string());
    P.parse();
    std::string s;
    for (auto& a : P.prog.arrays) { s += a; s += '\n'; }
    put_diag(s, buf, cap);
    return (int)P.prog.arrays.size();
  } catch (const Error& e) {
    put_diag(e.msg, buf, cap);
    return -e.status;
  }
}

}  // extern "C"
