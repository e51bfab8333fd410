// bcgen.h -- BabyCUDA -> CUDA C for the data-carrying executor (NEXT-2).
//
// One CTA executes one BabyCUDA block (blockDim <= 1024, CUDA's own limit): CUDA
// thread t runs BabyCUDA thread t straight through its statements with its
// values in registers; `sync` is a __syncthreads()-delimited phase commit
// (DESIGN.md §5.12).  The per-block arrays live in the CTA's slot of the scratch
// buffer (grid-stride over blocks, one slot per resident CTA):
//   mem[c]   committed value of cell c = lastwrite over the closed phases
//   st[c]    bit 0: defined (else bottom, rule lastwrite-undef), bit 1: the
//            committing phase had several writers (the read is ambiguous, R21)
//   own[c]   tid+1 of the thread that claimed c in the current phase (0: none)
//   cval[c]  that thread's current value of c (its own record W, rule write)
//   minw[c]  smallest tid+1 of a second writer of c in the phase (~0: none)
//   claims[] cells claimed in the phase (for the commit)
//   log      per thread: (cell, value) of its writes to cells another thread
//            claimed first (only in racy phases; K_LOG entries)
// A read (rule read) returns the thread's own current value (log, then cval when
// it owns the cell), else the committed one: lastwrite over {i : (R, W)} :: H.
// Every executed access appends its key phase|array|block|index|tid|kind to the
// alpha buffer (warp-aggregated slot reservation).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "bcfront.h"

namespace bcg {

struct Layout {                 // the global access key, MSB -> LSB
  uint32_t w_phase = 0, w_array = 0, w_block = 0, w_index = 0, w_tid = 0;
  uint32_t bits() const { return w_phase + w_array + w_block + w_index + w_tid + 1; }
};

struct Plan {
  uint64_t n_blocks = 1;
  uint32_t block_threads = 1;
  std::vector<uint64_t> params;          // values, by kernel parameter order
  std::vector<uint64_t> extents;         // per array
  std::vector<uint64_t> offsets;         // first cell of each array in a block's slot
  uint64_t n_cells = 0;
  uint32_t k_log = 16;                   // conflict-log entries per thread
  uint64_t block_bound = 0;              // accesses per block, bounded by the inferred MAP (0 = unknown)
  Layout lay;
};

// Device error bits of the executor (BcCtl.err).
constexpr uint32_t ERR_ARITH = 1u;      // division / modulo by zero, loop step zero
constexpr uint32_t ERR_RANGE = 2u;      // a value exceeds 64 bits
constexpr uint32_t ERR_BOUNDS = 4u;     // an index at or beyond the array's extent
constexpr uint32_t ERR_LOG = 8u;        // a thread's conflict log overflowed

// The executor's control block (device).
struct BcCtl {
  unsigned long long n_keys;            // accesses executed (alpha keys emitted, incl. beyond capacity)
  unsigned long long max_block;         // most accesses of one block (its region of the alpha buffer)
  unsigned long long uninit;            // reads of bottom
  unsigned long long ambiguous;         // reads of a value committed by a multi-writer phase
  unsigned int err;
  unsigned int pad;
};

// Byte size of one CTA slot, and the offsets of its regions.
uint64_t slot_bytes(const Plan& P);

// CUDA C source of `extern "C" __global__ void bc_exec(...)`.
std::string kernel_source(const bcf::Kernel& K, const Plan& P);

}  // namespace bcg
