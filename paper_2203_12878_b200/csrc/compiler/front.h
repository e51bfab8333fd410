// front.h -- MAP text front end of the product path: tokens, AST, parser.
//
// Grammar: DESIGN.md §3, extending SPEC.md:179.  The AST is
// the MAP syntax of PAPER.md:191-219 (Fig. 2): arithmetic n (x | i | n op n),
// conditions c (true | false | n rel n | c and/or c), unsynchronized protocols
// u (skip | o[n] | u;u | if | forU) and synchronized protocols p (sync | p;p |
// forS), with the reading p ::= u | sync | p;p | forS (R7).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace mapc {

struct CompileError {
  int status;          // map_status
  std::string msg;     // "line:col: message"
};

enum class BinOp : uint8_t { Add, Sub, Mul, Div, Mod, Shl, Shr, Min, Max };
enum class RelOp : uint8_t { Eq, Ne, Lt, Le, Gt, Ge };

// Variable classes after resolution.
enum class VarKind : uint8_t { Tid, Bid, Param, SyncLoop, UnsyncLoop };

struct Var {
  std::string name;
  VarKind kind;
  int index;           // param index / loop statement id
};

struct Expr {          // arithmetic expression node (pool-allocated)
  enum Kind : uint8_t { Nat, Ref, Bin } kind;
  BinOp op = BinOp::Add;
  uint64_t value = 0;  // Nat
  int var = -1;        // Ref: index into Program::vars
  int lhs = -1, rhs = -1;
  int line = 0, col = 0;
};

struct Cond {
  enum Kind : uint8_t { True, False, Rel, And, Or } kind;
  RelOp rel = RelOp::Eq;
  int lhs = -1, rhs = -1;          // Rel: expr ids;  And/Or: cond ids
};

struct Stmt {
  enum Kind : uint8_t { Skip, Sync, Access, Seq, If, ForU, ForS } kind;
  // Access
  bool write = false;
  int array = 0;
  int index = -1;                  // expr id
  // Seq
  std::vector<int> items;          // stmt ids
  // If
  int cond = -1, then_s = -1, else_s = -1;
  // loops
  int var = -1;                    // var id of the binder
  int lo = -1, hi = -1, step = -1; // expr ids
  int body = -1;
  int line = 0, col = 0;
};

struct Program {
  std::vector<Expr> exprs;
  std::vector<Cond> conds;
  std::vector<Stmt> stmts;
  std::vector<Var> vars;           // 0 = tid, 1 = bid, then params, then binders
  std::vector<std::string> params; // declared parameter names
  std::vector<std::string> arrays; // declared arrays (default: the single "A")
  int root = -1;
};

// Parse + resolve names + check barrier placement.  Throws CompileError.
Program parse_map(const std::string& text);

}  // namespace mapc
