// bcfront.cpp -- BabyCUDA parser, checks, Fig. 6 typing and MAP printing
// (bcfront.h).  Expressions by precedence climbing; the "(" of a condition is
// told from a parenthesised number by scanning to the matching ")" for a
// relation or and/or at its own nesting depth.
#include "bcfront.h"

#include <cctype>
#include <functional>
#include <set>
#include <sstream>

namespace bcf {
namespace {

enum class T { Num, Ident, Kw, Sym, End };

struct Tok {
  T t = T::End;
  std::string s;
  uint64_t v = 0;
  int line = 1, col = 1;
};

const char* kKeywords[] = {"params", "shared", "skip", "sync", "let", "in", "if", "else", "for", "step",
                           "true",   "false",  "and",  "or",   "min", "max", "tid", "bid"};

std::string at(int line, int col) { return std::to_string(line) + ":" + std::to_string(col) + ": "; }

std::vector<Tok> lex(const std::string& src) {
  std::vector<Tok> out;
  int line = 1, col = 1;
  size_t i = 0;
  const size_t n = src.size();
  while (i < n) {
    const char c = src[i];
    if (c == '\n') { ++i; ++line; col = 1; continue; }
    if (c == ' ' || c == '\t' || c == '\r') { ++i; ++col; continue; }
    if (c == '/' && i + 1 < n && src[i + 1] == '/') {
      while (i < n && src[i] != '\n') ++i;
      continue;
    }
    Tok tk;
    tk.line = line;
    tk.col = col;
    size_t j = i;
    if (std::isdigit((unsigned char)c)) {
      unsigned __int128 v = 0;
      while (j < n && std::isdigit((unsigned char)src[j])) {
        v = v * 10 + (unsigned)(src[j] - '0');
        if (v > (unsigned __int128)UINT64_MAX) throw Error{4, at(line, col) + "integer literal exceeds 64 bits"};
        ++j;
      }
      tk.t = T::Num;
      tk.v = (uint64_t)v;
    } else if (std::isalpha((unsigned char)c) || c == '_') {
      while (j < n && (std::isalnum((unsigned char)src[j]) || src[j] == '_')) ++j;
      tk.s = src.substr(i, j - i);
      tk.t = T::Ident;
      for (const char* k : kKeywords)
        if (tk.s == k) tk.t = T::Kw;
    } else {
      static const char* two[] = {":=", "..", "<=", ">=", "!=", "<<", ">>"};
      tk.t = T::Sym;
      for (const char* t2 : two)
        if (src.compare(i, 2, t2) == 0) { tk.s = t2; j = i + 2; }
      if (tk.s.empty()) {
        if (std::string("+-*/%<>=(){}[];,").find(c) == std::string::npos)
          throw Error{1, at(line, col) + "unexpected character '" + std::string(1, c) + "'"};
        tk.s = std::string(1, c);
        j = i + 1;
      }
    }
    col += (int)(j - i);
    i = j;
    out.push_back(std::move(tk));
  }
  Tok end;
  end.line = line;
  end.col = col;
  out.push_back(end);
  return out;
}

struct Parser {
  std::vector<Tok> tk;
  size_t p = 0;
  Kernel* K = nullptr;

  const Tok& cur() const { return tk[p]; }
  bool sym(const char* s) const { return (cur().t == T::Sym || cur().t == T::Kw) && cur().s == s; }
  [[noreturn]] void fail(const std::string& what) const {
    throw Error{1, at(cur().line, cur().col) + "expected " + what +
                       (cur().t == T::End ? std::string(", got end of input") : ", got '" + cur().s + "'")};
  }
  void expect(const char* s) {
    if (!sym(s)) fail(std::string("'") + s + "'");
    ++p;
  }
  std::string ident() {
    if (cur().t != T::Ident) fail("an identifier");
    return tk[p++].s;
  }

  // ---- numbers: precedence climbing over  << >>  <  + -  <  * / %
  static int prec(const std::string& s) {
    if (s == "<<" || s == ">>") return 1;
    if (s == "+" || s == "-") return 2;
    if (s == "*" || s == "/" || s == "%") return 3;
    return 0;
  }
  static BinOp opcode(const std::string& s) {
    if (s == "+") return OP_ADD;
    if (s == "-") return OP_SUB;
    if (s == "*") return OP_MUL;
    if (s == "/") return OP_DIV;
    if (s == "%") return OP_MOD;
    if (s == "<<") return OP_SHL;
    return OP_SHR;
  }
  std::unique_ptr<Num> num(int min_prec = 1) {
    std::unique_ptr<Num> lhs = primary();
    while (cur().t == T::Sym && prec(cur().s) >= min_prec) {
      const int pr = prec(cur().s);
      auto node = std::make_unique<Num>();
      node->k = NK_BIN;
      node->op = opcode(cur().s);
      node->line = cur().line;
      node->col = cur().col;
      ++p;
      node->a = std::move(lhs);
      node->b = num(pr + 1);
      lhs = std::move(node);
    }
    return lhs;
  }
  std::unique_ptr<Num> primary() {
    auto n = std::make_unique<Num>();
    n->line = cur().line;
    n->col = cur().col;
    if (cur().t == T::Num) { n->k = NK_NAT; n->v = tk[p++].v; return n; }
    if (cur().t == T::Ident) { n->k = NK_VAR; n->name = tk[p++].s; return n; }
    if (sym("tid")) { ++p; n->k = NK_TID; return n; }
    if (sym("bid")) { ++p; n->k = NK_BID; return n; }
    if (sym("min") || sym("max")) {
      n->k = NK_BIN;
      n->op = cur().s == "min" ? OP_MIN : OP_MAX;
      ++p;
      expect("(");
      n->a = num();
      expect(",");
      n->b = num();
      expect(")");
      return n;
    }
    if (sym("(")) {
      ++p;
      auto e = num();
      expect(")");
      return e;
    }
    fail("an expression");
  }

  // ---- conditions
  bool paren_is_cond() const {       // at "(": a relation / and / or directly inside?
    int depth = 0;
    for (size_t q = p; q < tk.size() && tk[q].t != T::End; ++q) {
      const Tok& t = tk[q];
      if (t.t == T::Sym && t.s == "(") { ++depth; continue; }
      if (t.t == T::Sym && t.s == ")") { if (--depth == 0) return false; continue; }
      if (depth == 1) {
        if (t.t == T::Kw && (t.s == "and" || t.s == "or" || t.s == "true" || t.s == "false")) return true;
        if (t.t == T::Sym && (t.s == "=" || t.s == "!=" || t.s == "<" || t.s == "<=" || t.s == ">" || t.s == ">="))
          return true;
      }
    }
    return false;
  }
  std::unique_ptr<Cond> cond() {
    auto l = cand();
    while (sym("or")) {
      auto c = std::make_unique<Cond>();
      c->k = CK_OR;
      c->line = cur().line;
      c->col = cur().col;
      ++p;
      c->l = std::move(l);
      c->r = cand();
      l = std::move(c);
    }
    return l;
  }
  std::unique_ptr<Cond> cand() {
    auto l = catom();
    while (sym("and")) {
      auto c = std::make_unique<Cond>();
      c->k = CK_AND;
      c->line = cur().line;
      c->col = cur().col;
      ++p;
      c->l = std::move(l);
      c->r = catom();
      l = std::move(c);
    }
    return l;
  }
  std::unique_ptr<Cond> catom() {
    auto c = std::make_unique<Cond>();
    c->line = cur().line;
    c->col = cur().col;
    if (sym("true")) { ++p; c->k = CK_TRUE; return c; }
    if (sym("false")) { ++p; c->k = CK_FALSE; return c; }
    if (sym("(") && paren_is_cond()) {
      ++p;
      auto in = cond();
      expect(")");
      return in;
    }
    c->k = CK_REL;
    c->a = num();
    static const std::pair<const char*, RelOp> rels[] = {{"=", R_EQ},  {"!=", R_NE}, {"<", R_LT},
                                                         {"<=", R_LE}, {">", R_GT},  {">=", R_GE}};
    for (auto& r : rels)
      if (sym(r.first)) {
        ++p;
        c->rel = r.second;
        c->b = num();
        return c;
      }
    fail("a comparison");
  }

  // ---- statements; `let ... in` takes the rest of the enclosing block
  std::unique_ptr<Stmt> block() {
    auto seq = std::make_unique<Stmt>();
    seq->k = SK_SEQ;
    seq->line = cur().line;
    seq->col = cur().col;
    while (true) {
      if (sym("let")) {
        seq->kids.push_back(let_stmt());
        break;
      }
      seq->kids.push_back(stmt());
      if (!sym(";")) break;
      ++p;
      if (cur().t == T::End || sym("}")) break;
    }
    if (seq->kids.size() == 1) return std::move(seq->kids[0]);
    return seq;
  }
  std::unique_ptr<Stmt> let_stmt() {
    auto s = std::make_unique<Stmt>();
    s->k = SK_LET;
    s->line = cur().line;
    s->col = cur().col;
    expect("let");
    s->var = ident();
    expect("=");
    s->arr_name = ident();
    expect("[");
    s->idx = num();
    expect("]");
    expect("in");
    s->kids.push_back(block());
    return s;
  }
  std::unique_ptr<Stmt> stmt() {
    auto s = std::make_unique<Stmt>();
    s->line = cur().line;
    s->col = cur().col;
    if (sym("skip")) { ++p; s->k = SK_SKIP; return s; }
    if (sym("sync")) { ++p; s->k = SK_SYNC; return s; }
    if (sym("if")) {
      ++p;
      s->k = SK_IF;
      expect("(");
      s->cond = cond();
      expect(")");
      expect("{");
      s->kids.push_back(block());
      expect("}");
      expect("else");                 // always an else branch
      expect("{");
      s->kids.push_back(block());
      expect("}");
      return s;
    }
    if (sym("for")) {
      ++p;
      s->k = SK_FOR;
      s->var = ident();
      expect("in");
      s->lo = num();
      expect("..");
      s->hi = num();
      if (sym("step")) {
        ++p;
        s->step = num();
      } else {
        s->step = std::make_unique<Num>();
        s->step->v = 1;
        s->step->line = s->line;
        s->step->col = s->col;
      }
      expect("{");
      s->kids.push_back(block());
      expect("}");
      return s;
    }
    if (cur().t == T::Ident) {
      s->k = SK_WRITE;
      s->arr_name = ident();
      expect("[");
      s->idx = num();
      expect("]");
      expect(":=");
      s->val = num();
      return s;
    }
    fail("a statement");
  }
};

// names in scope: the binders must be distinct from every visible name
void resolve_num(const Num* n, const std::set<std::string>& scope) {
  if (!n) return;
  if (n->k == NK_VAR && !scope.count(n->name))
    throw Error{2, at(n->line, n->col) + "unbound variable '" + n->name + "'"};
  resolve_num(n->a.get(), scope);
  resolve_num(n->b.get(), scope);
}
void resolve_cond(const Cond* c, const std::set<std::string>& scope) {
  if (!c) return;
  resolve_num(c->a.get(), scope);
  resolve_num(c->b.get(), scope);
  resolve_cond(c->l.get(), scope);
  resolve_cond(c->r.get(), scope);
}
bool resolve(Stmt* s, const Kernel& K, std::set<std::string> scope) {
  bool sync = false;
  if (s->k == SK_WRITE || s->k == SK_LET) {
    for (size_t i = 0; i < K.arrays.size(); ++i)
      if (K.arrays[i] == s->arr_name) s->arr = (int)i;
    if (s->arr < 0) throw Error{2, at(s->line, s->col) + "unknown array '" + s->arr_name + "'"};
  }
  auto bind = [&](const std::string& x) {
    bool clash = scope.count(x) > 0;
    for (const auto& a : K.arrays) clash = clash || a == x;
    if (clash) throw Error{2, at(s->line, s->col) + "binder '" + x + "' shadows a name in scope"};
    scope.insert(x);
  };
  switch (s->k) {
    case SK_SYNC: sync = true; break;
    case SK_WRITE:
      resolve_num(s->idx.get(), scope);
      resolve_num(s->val.get(), scope);
      break;
    case SK_LET:
      resolve_num(s->idx.get(), scope);
      bind(s->var);
      sync = resolve(s->kids[0].get(), K, scope);
      break;
    case SK_IF:
      resolve_cond(s->cond.get(), scope);
      sync = resolve(s->kids[0].get(), K, scope);
      sync = resolve(s->kids[1].get(), K, scope) || sync;
      break;
    case SK_FOR:
      resolve_num(s->lo.get(), scope);
      resolve_num(s->hi.get(), scope);
      resolve_num(s->step.get(), scope);
      bind(s->var);
      sync = resolve(s->kids[0].get(), K, scope);
      break;
    case SK_SEQ:
      for (auto& k : s->kids) sync = resolve(k.get(), K, scope) || sync;
      break;
    default: break;
  }
  s->has_sync = sync;
  return sync;
}

// free variables (incl. tid/bid) of an expression, left to right
void fv(const Num* n, std::vector<const Num*>* out) {
  if (!n) return;
  if (n->k == NK_VAR || n->k == NK_TID || n->k == NK_BID) out->push_back(n);
  fv(n->a.get(), out);
  fv(n->b.get(), out);
}
void fv(const Cond* c, std::vector<const Num*>* out) {
  if (!c) return;
  fv(c->a.get(), out);
  fv(c->b.get(), out);
  fv(c->l.get(), out);
  fv(c->r.get(), out);
}

// R8 for kernels: no sync under if; a loop around a sync has thread-uniform,
// data-free bounds
void check_barriers(const Stmt* s, bool under_if, std::set<std::string> data) {
  switch (s->k) {
    case SK_SYNC:
      if (under_if) throw Error{3, at(s->line, s->col) + "sync under a conditional"};
      break;
    case SK_LET:
      data.insert(s->var);
      check_barriers(s->kids[0].get(), under_if, data);
      break;
    case SK_IF:
      check_barriers(s->kids[0].get(), true, data);
      check_barriers(s->kids[1].get(), true, data);
      break;
    case SK_FOR:
      if (s->kids[0]->has_sync) {
        std::vector<const Num*> vs;
        fv(s->lo.get(), &vs);
        fv(s->hi.get(), &vs);
        fv(s->step.get(), &vs);
        for (const Num* v : vs)
          if (v->k != NK_VAR || data.count(v->name))
            throw Error{3, at(v->line, v->col) + "loop around a sync depends on " +
                               (v->k == NK_TID ? std::string("tid") : v->k == NK_BID ? "bid" : v->name)};
      }
      check_barriers(s->kids[0].get(), under_if, data);
      break;
    case SK_SEQ:
      for (auto& k : s->kids) check_barriers(k.get(), under_if, data);
      break;
    default: break;
  }
}

// ---- typing (Fig. 6) ----------------------------------------------------
struct IllTyped {
  TypeKind kind;
  const Num* at;
};

void t_expr(const std::set<std::string>& V, const Num* n, TypeKind kind) {    // t-n
  std::vector<const Num*> vs;
  fv(n, &vs);
  for (const Num* v : vs)
    if (v->k == NK_VAR && !V.count(v->name)) throw IllTyped{kind, v};
}
void t_cond(const std::set<std::string>& V, const Cond* c) {                    // t-b
  std::vector<const Num*> vs;
  fv(c, &vs);
  for (const Num* v : vs)
    if (v->k == NK_VAR && !V.count(v->name)) throw IllTyped{TY_DATA_CONTROL, v};
}
void t_stmt(std::set<std::string> V, const Stmt* s) {
  switch (s->k) {
    case SK_SKIP:                                           // t-skip
    case SK_SYNC: break;                                    // (synchronized extension)
    case SK_WRITE: t_expr(V, s->idx.get(), TY_DATA_INDEX); break;          // t-write (payload erased)
    case SK_LET:                                            // t-read: V |- n; y not in V; V |- b => u
      t_expr(V, s->idx.get(), TY_DATA_INDEX);
      t_stmt(V, s->kids[0].get());                          // y is NOT added to V
      break;
    case SK_IF:                                             // t-if
      t_cond(V, s->cond.get());
      t_stmt(V, s->kids[0].get());
      t_stmt(V, s->kids[1].get());
      break;
    case SK_FOR:                                            // t-for: V |- n, V |- m, V u {x} |- b
      t_expr(V, s->lo.get(), TY_DATA_CONTROL);
      t_expr(V, s->hi.get(), TY_DATA_CONTROL);
      t_expr(V, s->step.get(), TY_DATA_CONTROL);
      V.insert(s->var);
      t_stmt(V, s->kids[0].get());
      break;
    case SK_SEQ:                                            // t-seq
      for (auto& k : s->kids) t_stmt(V, k.get());
      break;
  }
}

// ---- printing -------------------------------------------------------------
void put_num(std::ostringstream& o, const Num* n) {
  switch (n->k) {
    case NK_NAT: o << n->v; return;
    case NK_VAR: o << n->name; return;
    case NK_TID: o << "tid"; return;
    case NK_BID: o << "bid"; return;
    case NK_BIN: break;
  }
  if (n->op == OP_MIN || n->op == OP_MAX) {
    o << (n->op == OP_MIN ? "min(" : "max(");
    put_num(o, n->a.get());
    o << ", ";
    put_num(o, n->b.get());
    o << ")";
    return;
  }
  static const char* sy[] = {"+", "-", "*", "/", "%", "<<", ">>"};
  o << "(";
  put_num(o, n->a.get());
  o << " " << sy[n->op] << " ";
  put_num(o, n->b.get());
  o << ")";
}
void put_cond(std::ostringstream& o, const Cond* c) {
  switch (c->k) {
    case CK_TRUE: o << "true"; return;
    case CK_FALSE: o << "false"; return;
    case CK_REL: {
      static const char* rs[] = {"=", "!=", "<", "<=", ">", ">="};
      put_num(o, c->a.get());
      o << " " << rs[c->rel] << " ";
      put_num(o, c->b.get());
      return;
    }
    default:
      o << "(";
      put_cond(o, c->l.get());
      o << (c->k == CK_AND ? " and " : " or ");
      put_cond(o, c->r.get());
      o << ")";
  }
}

// does data variable y reach a typed position (index, condition, loop bound) in s?
bool reaches_typed(const Stmt* s, const std::string& y) {
  auto in = [&](const Num* n) {
    std::vector<const Num*> vs;
    fv(n, &vs);
    for (const Num* v : vs)
      if (v->k == NK_VAR && v->name == y) return true;
    return false;
  };
  switch (s->k) {
    case SK_WRITE: return in(s->idx.get());
    case SK_LET: return in(s->idx.get()) || reaches_typed(s->kids[0].get(), y);
    case SK_IF: {
      std::vector<const Num*> vs;
      fv(s->cond.get(), &vs);
      for (const Num* v : vs)
        if (v->k == NK_VAR && v->name == y) return true;
      return reaches_typed(s->kids[0].get(), y) || reaches_typed(s->kids[1].get(), y);
    }
    case SK_FOR:
      return in(s->lo.get()) || in(s->hi.get()) || in(s->step.get()) || reaches_typed(s->kids[0].get(), y);
    case SK_SEQ:
      for (auto& k : s->kids)
        if (reaches_typed(k.get(), y)) return true;
      return false;
    default: return false;
  }
}

void put_stmt(std::ostringstream& o, const Kernel& K, const Stmt* s, uint64_t domain) {
  switch (s->k) {
    case SK_SKIP: o << "skip"; return;
    case SK_SYNC: o << "sync"; return;
    case SK_WRITE:                                          // t-write: wr[n]
      o << "wr " << K.arrays[s->arr] << "[";
      put_num(o, s->idx.get());
      o << "]";
      return;
    case SK_LET:                                            // t-read: rd[n]; u
      o << "rd " << K.arrays[s->arr] << "[";
      put_num(o, s->idx.get());
      o << "]; ";
      if (domain > 0 && reaches_typed(s->kids[0].get(), s->var)) {
        o << "forU " << s->var << " in 0.." << domain << " { ";
        put_stmt(o, K, s->kids[0].get(), domain);
        o << " }";
      } else {
        put_stmt(o, K, s->kids[0].get(), domain);
      }
      return;
    case SK_IF:
      o << "if (";
      put_cond(o, s->cond.get());
      o << ") { ";
      put_stmt(o, K, s->kids[0].get(), domain);
      o << " } else { ";
      put_stmt(o, K, s->kids[1].get(), domain);
      o << " }";
      return;
    case SK_FOR:                                            // t-for (forS around a sync)
      o << (s->kids[0]->has_sync ? "forS " : "forU ") << s->var << " in ";
      put_num(o, s->lo.get());
      o << "..";
      put_num(o, s->hi.get());
      if (!(s->step->k == NK_NAT && s->step->v == 1)) {
        o << " step ";
        put_num(o, s->step.get());
      }
      o << " { ";
      put_stmt(o, K, s->kids[0].get(), domain);
      o << " }";
      return;
    case SK_SEQ:
      for (size_t i = 0; i < s->kids.size(); ++i) {
        if (i) o << "; ";
        put_stmt(o, K, s->kids[i].get(), domain);
      }
      return;
  }
}

// ---- phase counting (host evaluation of sync-loop bounds) -----------------
struct PhaseCounter {
  const Kernel& K;
  std::vector<std::pair<std::string, uint64_t>> env;
  uint64_t syncs = 0;

  uint64_t eval(const Num* n) {
    switch (n->k) {
      case NK_NAT: return n->v;
      case NK_VAR:
        for (auto it = env.rbegin(); it != env.rend(); ++it)
          if (it->first == n->name) return it->second;
        throw Error{3, at(n->line, n->col) + "'" + n->name + "' is not thread-uniform here"};
      case NK_TID:
      case NK_BID: throw Error{3, at(n->line, n->col) + "thread-dependent bound of a loop around a sync"};
      case NK_BIN: break;
    }
    const uint64_t a = eval(n->a.get()), b = eval(n->b.get());
    switch (n->op) {
      case OP_ADD:
        if (a > UINT64_MAX - b) throw Error{4, at(n->line, n->col) + "value exceeds 64 bits"};
        return a + b;
      case OP_SUB: return a > b ? a - b : 0;
      case OP_MUL:
        if (a && b > UINT64_MAX / a) throw Error{4, at(n->line, n->col) + "value exceeds 64 bits"};
        return a * b;
      case OP_DIV:
      case OP_MOD:
        if (!b) throw Error{5, at(n->line, n->col) + "division by zero"};
        return n->op == OP_DIV ? a / b : a % b;
      case OP_SHL:
        if (!a) return 0;
        if (b >= 64 || a > (UINT64_MAX >> b)) throw Error{4, at(n->line, n->col) + "value exceeds 64 bits"};
        return a << b;
      case OP_SHR: return b >= 64 ? 0 : a >> b;
      case OP_MIN: return a < b ? a : b;
      case OP_MAX: return a > b ? a : b;
    }
    return 0;
  }
  void walk(const Stmt* s) {
    if (!s->has_sync) return;
    switch (s->k) {
      case SK_SYNC:
        if (++syncs >= (1u << 24)) throw Error{4, at(s->line, s->col) + "too many barrier phases"};
        break;
      case SK_LET: walk(s->kids[0].get()); break;
      case SK_SEQ:
        for (auto& k : s->kids) walk(k.get());
        break;
      case SK_FOR: {
        const uint64_t lo = eval(s->lo.get()), hi = eval(s->hi.get()), st = eval(s->step.get());
        if (st == 0) throw Error{5, at(s->line, s->col) + "loop step is zero"};
        for (uint64_t x = lo; x < hi;) {
          env.emplace_back(s->var, x);
          walk(s->kids[0].get());
          env.pop_back();
          if (hi - x <= st) break;
          x += st;
        }
        break;
      }
      default: break;
    }
  }
};

}  // namespace

Kernel parse(const std::string& src) {
  Kernel K;
  Parser P;
  P.tk = lex(src);
  P.K = &K;
  while (P.sym("params") || P.sym("shared")) {
    if (P.sym("params")) {
      ++P.p;
      K.params.push_back(P.ident());
      while (P.sym(",")) { ++P.p; K.params.push_back(P.ident()); }
    } else {
      ++P.p;
      while (true) {
        K.arrays.push_back(P.ident());
        int64_t ext = -1;
        if (P.sym("[")) {
          ++P.p;
          if (P.cur().t != T::Num) P.fail("an array extent");
          ext = (int64_t)std::min<uint64_t>(P.tk[P.p++].v, (uint64_t)INT64_MAX);
          P.expect("]");
        }
        K.extents.push_back(ext);
        if (!P.sym(",")) break;
        ++P.p;
      }
    }
    P.expect(";");
  }
  if (K.arrays.empty()) {                         // the paper's single array A
    K.arrays.push_back("A");
    K.extents.push_back(-1);
  }
  {
    std::set<std::string> names;
    for (auto& x : K.params) names.insert(x);
    for (auto& x : K.arrays) names.insert(x);
    if (names.size() != K.params.size() + K.arrays.size()) throw Error{2, "1:1: duplicate parameter or array name"};
  }
  K.body = P.block();
  if (P.cur().t != T::End) throw Error{1, at(P.cur().line, P.cur().col) + "unexpected '" + P.cur().s + "'"};
  resolve(K.body.get(), K, std::set<std::string>(K.params.begin(), K.params.end()));
  check_barriers(K.body.get(), false, {});
  return K;
}

Typing type_check(const Kernel& k) {
  std::set<std::string> V(k.params.begin(), k.params.end());   // tid, bid are NK_TID / NK_BID
  Typing ty;
  try {
    t_stmt(V, k.body.get());
  } catch (const IllTyped& e) {
    ty.typable = false;
    ty.kind = e.kind;
    ty.var = e.at->name;
    ty.line = e.at->line;
    ty.col = e.at->col;
  }
  return ty;
}

std::string map_text(const Kernel& k, uint64_t domain) {
  std::ostringstream o;
  if (!k.params.empty()) {
    o << "params ";
    for (size_t i = 0; i < k.params.size(); ++i) o << (i ? ", " : "") << k.params[i];
    o << "; ";
  }
  o << "shared ";
  for (size_t i = 0; i < k.arrays.size(); ++i) o << (i ? ", " : "") << k.arrays[i];
  o << "; ";
  put_stmt(o, k, k.body.get(), domain);
  return o.str();
}

uint32_t count_phases(const Kernel& k, const std::vector<uint64_t>& param_values) {
  PhaseCounter pc{k, {}, 0};
  for (size_t i = 0; i < k.params.size() && i < param_values.size(); ++i) pc.env.emplace_back(k.params[i], param_values[i]);
  pc.walk(k.body.get());
  return (uint32_t)(pc.syncs + 1);
}

}  // namespace bcf
