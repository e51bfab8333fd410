// compiler.h -- MAP -> per-(instance, group) bytecode (product path, host side).
//
// Pipeline:
//  1. parse + resolve + fragment check              (front.cpp)
//  2. phase enumeration: walk the synchronized fragment with concrete forS
//     values; every u-fragment met becomes an INSTANCE (template, forS values,
//     phase = number of syncs executed before it).  Phases are
//     thread-uniform by construction (R8), so this runs on the host.
//  3. per instance, access sites are grouped by their enclosing forU nest
//     (the GROUP); each group is lowered to one straight-line register program
//     whose tuple space is the bounding box (block, tid, k_0..k_{L-1}) of its
//     loops, computed by interval analysis with the concrete parameters.
//     Non-rectangular loops get an in-program guard k < trip(lo, hi, step).
//  4. interval analysis proves every reachable value fits 64 bits (else
//     MAP_E_RANGE) and selects the u32 VM when everything fits 32 bits.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../devabi.h"
#include "front.h"

namespace mapc {

struct Interval {
  uint64_t lo = 0, hi = 0;
};

struct GroupProg {
  std::vector<MapcOp> ops;
  uint32_t n_levels = 0;
  uint64_t trips[MAPC_MAX_LEVELS] = {};   // bounding-box trip counts, outermost first
  uint32_t n_emits = 0;
  bool dense = false;                     // no guard and no fault check: every tuple emits n_emits keys
  bool has_emit = false;
  Interval index;                         // hull of emitted index values
  uint64_t tuples_per_block = 0;          // blockDim * prod(trips)
  // Tuple order within a block: false = innermost loop fastest (tid above the
  // loops), true = tid fastest (loops above tid).  Chosen so that 32
  // consecutive tuples (a warp) touch the fewest 32-byte sectors of cells
  // (choose_tuple_order); any order enumerates the same accesses.
  bool tid_inner = false;
  // Per access site (EMIT order): the index's known low bits -- index mod 2^site_kb
  // == site_kv for every tuple (a congruence proved during lowering; 0 = nothing
  // known).  The direct table of a phase whose sites share a residue modulo 2^k is
  // compressed by 2^k.
  std::vector<uint32_t> site_kb;
  std::vector<uint64_t> site_kv;
};

struct InstanceInfo {
  int tmpl = -1;                          // u-statement id
  uint32_t phase = 0;
  std::vector<GroupProg> groups;
  uint64_t bound_per_block = 0;           // sum over groups of tuples_per_block * n_emits
};

struct Compiled {
  Program ast;
  uint64_t n_threads = 1, n_blocks = 1;   // prod(block), prod(grid)
  uint32_t w_tid = 0;
  std::vector<uint64_t> params;           // values by param index
  std::vector<InstanceInfo> inst;         // in phase order
  uint32_t n_phases = 1;
  bool u32_mode = true;
  uint64_t max_accesses = 0;              // sum of bounds
  uint64_t max_unit = 0;                  // largest (phase, block) bound
  uint32_t total_ops = 0;
  uint32_t n_groups = 0;
};

// Throws CompileError.
Compiled compile_map(const std::string& text, const uint32_t grid[3], const uint32_t block[3],
                     const std::vector<std::string>& names, const std::vector<uint64_t>& values);

// Host copy of the u32 invariant-divisor parameters (also used by tests).
MapcFastDiv make_fastdiv(uint32_t d);
uint32_t fastdiv_apply(uint32_t n, const MapcFastDiv& f);

inline uint32_t bits_for(uint64_t max_value) {   // bits to hold 0..max_value
  uint32_t b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

// Host evaluation of a group program's access sites for one tuple (the VM's
// semantics): the index of every EMIT whose guard holds, in site order, -1 where
// it does not (the JIT's row-jam samples it to find sites one row apart).
void eval_ops_sites(const std::vector<MapcOp>& ops, uint32_t n_levels, uint64_t tid, uint64_t bid, const uint64_t* k,
                    std::vector<int64_t>* out);

}  // namespace mapc
