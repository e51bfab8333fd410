// front.cpp -- lexer, parser and name resolution for MAP text (product path).
//
// Grammar:
//   program := decl* proto
//   decl    := "params" id {"," id} ";" | "shared" id {"," id} ";"
//   proto   := stmt {";" stmt} [";"]
//   stmt    := "skip" | "sync" | ("rd"|"wr") [id] "[" n "]"
//            | "if" "(" c ")" "{" proto "}" ["else" "{" proto "}"]
//            | ("forU"|"forS") id "in" n ".." n ["step" n] "{" proto "}"
//   n       := precedence levels  << >>  <  + -  <  * / %  < atom
//   atom    := nat | id | tid | bid | "(" n ")" | ("min"|"max") "(" n "," n ")"
//   c       := c "or" c | c "and" c | "true" | "false" | n rel n | "(" c ")"
// `-` is monus; `..` is half-open (for-1/for-2).
#include "front.h"

#include <cctype>
#include <cstring>

namespace mapc {
namespace {

enum class T : uint8_t { End, Num, Ident, Sym };

struct Tok {
  T t;
  std::string s;
  uint64_t v = 0;
  int line = 0, col = 0;
};

const char* kKeywords[] = {"skip", "sync", "rd",   "wr",  "if",    "else",   "forU", "forS", "in",  "step",
                           "true", "false", "and", "or",  "tid",   "bid",    "params", "shared", "min", "max"};

bool is_keyword(const std::string& s) {
  for (const char* k : kKeywords)
    if (s == k) return true;
  return false;
}

std::string where(int line, int col) { return std::to_string(line) + ":" + std::to_string(col) + ": "; }

std::vector<Tok> tokenize(const std::string& src) {
  std::vector<Tok> toks;
  int line = 1, col = 1;
  size_t i = 0, n = src.size();
  auto step = [&](size_t k) {
    while (k--) {
      if (src[i] == '\n') { ++line; col = 1; } else { ++col; }
      ++i;
    }
  };
  while (i < n) {
    unsigned char c = (unsigned char)src[i];
    if (std::isspace(c)) { step(1); continue; }
    if (c == '/' && i + 1 < n && src[i + 1] == '/') {
      while (i < n && src[i] != '\n') step(1);
      continue;
    }
    Tok tk;
    tk.line = line;
    tk.col = col;
    if (std::isdigit(c)) {
      size_t j = i;
      unsigned __int128 v = 0;
      while (j < n && std::isdigit((unsigned char)src[j])) {
        v = v * 10 + (unsigned)(src[j] - '0');
        if (v > (unsigned __int128)UINT64_MAX)
          throw CompileError{4, where(line, col) + "integer literal exceeds 64 bits"};
        ++j;
      }
      tk.t = T::Num;
      tk.v = (uint64_t)v;
      step(j - i);
    } else if (std::isalpha(c) || c == '_') {
      size_t j = i;
      while (j < n && (std::isalnum((unsigned char)src[j]) || src[j] == '_')) ++j;
      tk.t = T::Ident;
      tk.s = src.substr(i, j - i);
      step(j - i);
    } else {
      static const char* kTwo[] = {"..", "<<", ">>", "<=", ">=", "!="};
      tk.t = T::Sym;
      for (const char* s2 : kTwo)
        if (i + 1 < n && src[i] == s2[0] && src[i + 1] == s2[1]) tk.s = s2;
      if (tk.s.empty()) {
        if (!std::strchr("=<>+-*/%()[]{};,", (int)c))
          throw CompileError{1, where(line, col) + "unexpected character '" + std::string(1, (char)c) + "'"};
        tk.s = std::string(1, (char)c);
      }
      step(tk.s.size());
    }
    toks.push_back(std::move(tk));
  }
  Tok end;
  end.t = T::End;
  end.line = line;
  end.col = col;
  toks.push_back(end);
  return toks;
}

class Parser {
 public:
  explicit Parser(const std::string& src) : toks_(tokenize(src)) {}

  Program run() {
    prog_.vars.push_back({"tid", VarKind::Tid, 0});
    prog_.vars.push_back({"bid", VarKind::Bid, 0});
    visible_ = {0, 1};
    while (peek_word("params") || peek_word("shared")) decl();
    if (prog_.arrays.empty()) prog_.arrays.push_back("A");
    prog_.root = proto(/*closing=*/nullptr);
    if (cur().t != T::End) fail(1, "unexpected trailing input");
    return std::move(prog_);
  }

 private:
  std::vector<Tok> toks_;
  size_t pos_ = 0;
  Program prog_;
  std::vector<int> visible_;   // var ids in scope, innermost last

  const Tok& cur() const { return toks_[pos_]; }
  const Tok& at(size_t k) const { return toks_[std::min(pos_ + k, toks_.size() - 1)]; }
  [[noreturn]] void fail(int st, const std::string& m) { throw CompileError{st, where(cur().line, cur().col) + m}; }
  bool peek_sym(const char* s) const { return cur().t == T::Sym && cur().s == s; }
  bool peek_word(const char* s) const { return cur().t == T::Ident && cur().s == s; }
  void need_sym(const char* s) {
    if (!peek_sym(s)) fail(1, std::string("expected '") + s + "'");
    ++pos_;
  }
  void need_word(const char* s) {
    if (!peek_word(s)) fail(1, std::string("expected '") + s + "'");
    ++pos_;
  }
  std::string name() {
    if (cur().t != T::Ident || is_keyword(cur().s)) fail(1, "expected an identifier");
    return toks_[pos_++].s;
  }
  int find_visible(const std::string& s) const {
    for (auto it = visible_.rbegin(); it != visible_.rend(); ++it)
      if (prog_.vars[*it].name == s) return *it;
    return -1;
  }

  void decl() {
    bool is_params = peek_word("params");
    ++pos_;
    do {
      int line = cur().line, col = cur().col;
      std::string nm = name();
      bool dup = find_visible(nm) >= 0;
      for (auto& a : prog_.arrays) dup |= (a == nm);
      if (dup) throw CompileError{2, where(line, col) + "'" + nm + "' is declared twice"};
      if (is_params) {
        prog_.vars.push_back({nm, VarKind::Param, (int)prog_.params.size()});
        prog_.params.push_back(nm);
        visible_.push_back((int)prog_.vars.size() - 1);
      } else {
        prog_.arrays.push_back(nm);
      }
    } while (peek_sym(",") && (++pos_, true));
    need_sym(";");
  }

  // ---- arithmetic: precedence climbing over three binary levels ----
  static int level_of(const Tok& t, BinOp* op) {
    if (t.t != T::Sym) return -1;
    const std::string& s = t.s;
    if (s == "<<") { *op = BinOp::Shl; return 0; }
    if (s == ">>") { *op = BinOp::Shr; return 0; }
    if (s == "+") { *op = BinOp::Add; return 1; }
    if (s == "-") { *op = BinOp::Sub; return 1; }
    if (s == "*") { *op = BinOp::Mul; return 2; }
    if (s == "/") { *op = BinOp::Div; return 2; }
    if (s == "%") { *op = BinOp::Mod; return 2; }
    return -1;
  }
  int mk(Expr e) {
    prog_.exprs.push_back(e);
    return (int)prog_.exprs.size() - 1;
  }
  int expr(int min_level = 0) {
    int lhs = primary();
    for (;;) {
      BinOp op;
      int lv = level_of(cur(), &op);
      if (lv < min_level) return lhs;   // also handles lv == -1
      Expr e{Expr::Bin};
      e.op = op;
      e.line = cur().line;
      e.col = cur().col;
      ++pos_;
      e.lhs = lhs;
      e.rhs = expr(lv + 1);             // left associative
      lhs = mk(e);
    }
  }
  int primary() {
    const Tok& t = cur();
    Expr e{Expr::Nat};
    e.line = t.line;
    e.col = t.col;
    if (t.t == T::Num) {
      e.value = t.v;
      ++pos_;
      return mk(e);
    }
    if (peek_sym("(")) {
      ++pos_;
      int inner = expr();
      need_sym(")");
      return inner;
    }
    if (peek_word("min") || peek_word("max")) {
      e.kind = Expr::Bin;
      e.op = peek_word("min") ? BinOp::Min : BinOp::Max;
      ++pos_;
      need_sym("(");
      e.lhs = expr();
      need_sym(",");
      e.rhs = expr();
      need_sym(")");
      return mk(e);
    }
    if (t.t == T::Ident && (t.s == "tid" || t.s == "bid")) {
      e.kind = Expr::Ref;
      e.var = t.s == "tid" ? 0 : 1;
      ++pos_;
      return mk(e);
    }
    if (t.t == T::Ident && !is_keyword(t.s)) {
      int v = find_visible(t.s);
      if (v < 0) fail(2, "unbound identifier '" + t.s + "'");
      e.kind = Expr::Ref;
      e.var = v;
      ++pos_;
      return mk(e);
    }
    fail(1, "expected an arithmetic expression");
  }

  // ---- conditions ----
  static bool rel_of(const Tok& t, RelOp* r) {
    if (t.t != T::Sym) return false;
    const std::string& s = t.s;
    if (s == "=") *r = RelOp::Eq;
    else if (s == "!=") *r = RelOp::Ne;
    else if (s == "<") *r = RelOp::Lt;
    else if (s == "<=") *r = RelOp::Le;
    else if (s == ">") *r = RelOp::Gt;
    else if (s == ">=") *r = RelOp::Ge;
    else return false;
    return true;
  }
  int mkc(Cond c) {
    prog_.conds.push_back(c);
    return (int)prog_.conds.size() - 1;
  }
  int cond_or() {
    int l = cond_and();
    while (peek_word("or")) {
      ++pos_;
      Cond c{Cond::Or};
      c.lhs = l;
      c.rhs = cond_and();
      l = mkc(c);
    }
    return l;
  }
  int cond_and() {
    int l = cond_atom();
    while (peek_word("and")) {
      ++pos_;
      Cond c{Cond::And};
      c.lhs = l;
      c.rhs = cond_atom();
      l = mkc(c);
    }
    return l;
  }
  // "(" starts a parenthesised condition unless the token after its matching
  // ")" continues an arithmetic expression or a comparison.
  bool paren_is_arith() const {
    int depth = 0;
    for (size_t k = pos_; k < toks_.size(); ++k) {
      const Tok& t = toks_[k];
      if (t.t == T::End) return false;
      if (t.t == T::Sym && t.s == "(") ++depth;
      if (t.t == T::Sym && t.s == ")" && --depth == 0) {
        const Tok& nx = toks_[std::min(k + 1, toks_.size() - 1)];
        BinOp op;
        RelOp r;
        return level_of(nx, &op) >= 0 || rel_of(nx, &r);
      }
    }
    return false;
  }
  int cond_atom() {
    if (peek_word("true")) { ++pos_; return mkc(Cond{Cond::True}); }
    if (peek_word("false")) { ++pos_; return mkc(Cond{Cond::False}); }
    if (peek_sym("(") && !paren_is_arith()) {
      ++pos_;
      int c = cond_or();
      need_sym(")");
      return c;
    }
    Cond c{Cond::Rel};
    c.lhs = expr();
    if (!rel_of(cur(), &c.rel)) fail(1, "expected a comparison operator");
    ++pos_;
    c.rhs = expr();
    return mkc(c);
  }

  // ---- statements ----
  int mks(Stmt s) {
    prog_.stmts.push_back(std::move(s));
    return (int)prog_.stmts.size() - 1;
  }
  int proto(const char* closing) {
    Stmt seq;
    seq.kind = Stmt::Seq;
    seq.line = cur().line;
    seq.col = cur().col;
    seq.items.push_back(stmt());
    while (peek_sym(";")) {
      ++pos_;
      if (cur().t == T::End || (closing && peek_sym(closing))) break;
      seq.items.push_back(stmt());
    }
    if (seq.items.size() == 1) return seq.items[0];
    return mks(std::move(seq));
  }
  int braced() {
    need_sym("{");
    int b = proto("}");
    need_sym("}");
    return b;
  }
  int stmt() {
    Stmt s;
    s.line = cur().line;
    s.col = cur().col;
    if (peek_word("skip")) { ++pos_; s.kind = Stmt::Skip; return mks(std::move(s)); }
    if (peek_word("sync")) { ++pos_; s.kind = Stmt::Sync; return mks(std::move(s)); }
    if (peek_word("rd") || peek_word("wr")) {
      s.kind = Stmt::Access;
      s.write = peek_word("wr");
      ++pos_;
      s.array = 0;
      if (!peek_sym("[")) {
        int line = cur().line, col = cur().col;
        std::string a = name();
        s.array = -1;
        for (size_t k = 0; k < prog_.arrays.size(); ++k)
          if (prog_.arrays[k] == a) s.array = (int)k;
        if (s.array < 0) throw CompileError{2, where(line, col) + "undeclared array '" + a + "'"};
      }
      need_sym("[");
      s.index = expr();
      need_sym("]");
      return mks(std::move(s));
    }
    if (peek_word("if")) {
      ++pos_;
      s.kind = Stmt::If;
      need_sym("(");
      s.cond = cond_or();
      need_sym(")");
      s.then_s = braced();
      if (peek_word("else")) {
        ++pos_;
        s.else_s = braced();
      } else {
        Stmt sk;
        sk.kind = Stmt::Skip;
        s.else_s = mks(std::move(sk));
      }
      return mks(std::move(s));
    }
    if (peek_word("forU") || peek_word("forS")) {
      s.kind = peek_word("forU") ? Stmt::ForU : Stmt::ForS;
      ++pos_;
      int line = cur().line, col = cur().col;
      std::string v = name();
      if (find_visible(v) >= 0) throw CompileError{2, where(line, col) + "binder '" + v + "' shadows a visible name"};
      need_word("in");
      s.lo = expr();
      need_sym("..");
      s.hi = expr();
      if (peek_word("step")) {
        ++pos_;
        s.step = expr();
      } else {
        Expr one{Expr::Nat};
        one.value = 1;
        s.step = mk(one);
      }
      // The binder id is the statement id the loop will get; fix up below.
      prog_.vars.push_back({v, s.kind == Stmt::ForU ? VarKind::UnsyncLoop : VarKind::SyncLoop, -1});
      s.var = (int)prog_.vars.size() - 1;
      visible_.push_back(s.var);
      s.body = braced();
      visible_.pop_back();
      int id = mks(std::move(s));
      prog_.vars[prog_.stmts[id].var].index = id;
      return id;
    }
    fail(1, "expected a statement");
  }
};

bool expr_mentions_thread(const Program& p, int e) {
  const Expr& x = p.exprs[e];
  if (x.kind == Expr::Ref) return p.vars[x.var].kind == VarKind::Tid || p.vars[x.var].kind == VarKind::Bid;
  if (x.kind == Expr::Bin) return expr_mentions_thread(p, x.lhs) || expr_mentions_thread(p, x.rhs);
  return false;
}

// sync / forS form the synchronized fragment p: they never
// occur under if/forU (the u fragment); forS bounds must be
// thread-uniform (R8).
void check_fragments(const Program& p, int s, bool in_u) {
  const Stmt& st = p.stmts[s];
  auto bad = [&](const char* m) {
    throw CompileError{3, where(st.line, st.col) + m};
  };
  switch (st.kind) {
    case Stmt::Sync:
      if (in_u) bad("sync inside if/forU (barrier under divergent control)");
      return;
    case Stmt::Seq:
      for (int c : st.items) check_fragments(p, c, in_u);
      return;
    case Stmt::If:
      check_fragments(p, st.then_s, true);
      check_fragments(p, st.else_s, true);
      return;
    case Stmt::ForU:
      check_fragments(p, st.body, true);
      return;
    case Stmt::ForS:
      if (in_u) bad("forS inside if/forU");
      if (expr_mentions_thread(p, st.lo) || expr_mentions_thread(p, st.hi) || expr_mentions_thread(p, st.step))
        bad("forS bounds depend on tid/bid");
      check_fragments(p, st.body, false);
      return;
    default:
      return;
  }
}

}  // namespace

Program parse_map(const std::string& text) {
  Parser ps(text);
  Program p = ps.run();
  check_fragments(p, p.root, false);
  return p;
}

}  // namespace mapc
