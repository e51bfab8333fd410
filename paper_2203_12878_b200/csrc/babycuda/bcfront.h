// bcfront.h -- BabyCUDA front end (product path, host side): parser, scope and
// barrier checks, the behavioural type system of Fig. 6 that
// infers a kernel's MAP, and the data abstraction of ill-typed kernels.
//
// BabyCUDA (Fig. 5) is the data-carrying source language:
//   A[n] := m                 write the value of m to A[n]          (rule write)
//   let y = A[n] in b         read A[n] into y for b                (rule read)
//   if (c) { b } else { b }   for x in n..m [step s] { b }   skip   b ; b
// plus `sync` (the synchronized fragment; R18).
// Grammar: DESIGN.md §3b.  Independent of oracle/babycuda.py (shared by
// specification only).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace bcf {

struct Error {
  int status;        // map_status (1 parse, 2 scope, 3 barrier, 4 range, 8 arg)
  std::string msg;   // "line:col: message"
};

enum NumKind { NK_NAT, NK_VAR, NK_TID, NK_BID, NK_BIN };
enum BinOp { OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MOD, OP_SHL, OP_SHR, OP_MIN, OP_MAX };

struct Num {
  NumKind k = NK_NAT;
  uint64_t v = 0;
  std::string name;          // NK_VAR
  BinOp op = OP_ADD;         // NK_BIN
  std::unique_ptr<Num> a, b;
  int line = 0, col = 0;
};

enum CondKind { CK_TRUE, CK_FALSE, CK_REL, CK_AND, CK_OR };
enum RelOp { R_EQ, R_NE, R_LT, R_LE, R_GT, R_GE };

struct Cond {
  CondKind k = CK_TRUE;
  RelOp rel = R_EQ;
  std::unique_ptr<Num> a, b;      // CK_REL
  std::unique_ptr<Cond> l, r;     // CK_AND / CK_OR
  int line = 0, col = 0;
};

enum StmtKind { SK_SKIP, SK_SYNC, SK_WRITE, SK_LET, SK_IF, SK_FOR, SK_SEQ };

struct Stmt {
  StmtKind k = SK_SKIP;
  std::string var;                // SK_LET binder / SK_FOR loop variable
  int arr = -1;                   // SK_WRITE / SK_LET array id (declaration order)
  std::string arr_name;           // as written (resolved to arr after parsing)
  std::unique_ptr<Num> idx, val;  // index; SK_WRITE payload
  std::unique_ptr<Num> lo, hi, step;
  std::unique_ptr<Cond> cond;
  std::vector<std::unique_ptr<Stmt>> kids;   // SK_LET: [body]; SK_IF: [then, else]; SK_FOR: [body]; SK_SEQ
  bool has_sync = false;          // a sync is reachable inside (set by parse)
  int line = 0, col = 0;
};

struct Kernel {
  std::vector<std::string> params;
  std::vector<std::string> arrays;
  std::vector<int64_t> extents;   // declared extent per array, -1 = not declared
  std::unique_ptr<Stmt> body;
};

// Parse + resolve names + barrier placement check.  Throws Error.
Kernel parse(const std::string& src);

enum TypeKind { TY_OK = 0, TY_DATA_INDEX = 1, TY_DATA_CONTROL = 2 };
struct Typing {
  bool typable = true;
  TypeKind kind = TY_OK;
  std::string var;                // the first data variable in a typed position
  int line = 0, col = 0;          // of that use
};

// V |- b => u (Fig. 6) with V = {tid, bid} u params: reports the first failing
// premise in rule order (left to right, outer to inner).
Typing type_check(const Kernel& k);

// The MAP text (DESIGN.md §3 grammar) of the kernel: the t-rules' image when
// typable; with domain > 0, every read whose value reaches an index, a
// condition or a loop bound becomes `rd A[n]; forU y in 0..domain { u }`.
std::string map_text(const Kernel& k, uint64_t domain);

// Number of barrier phases (syncs executed + 1), evaluating the bounds of loops
// that contain a sync with the parameter values (thread-uniform by the barrier
// check).  Throws Error (range / arith) on a bad bound.
uint32_t count_phases(const Kernel& k, const std::vector<uint64_t>& param_values);

}  // namespace bcf
