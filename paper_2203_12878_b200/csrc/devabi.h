// devabi.h -- data shared between the host compiler/runtime and the sm_100a
// kernels of the product path (NOT shared with oracle/).
//
// Bytecode: one straight-line register program per
// (instance, loop-nest group).  It evaluates, for one tuple
// (block, tid, k_0..k_{L-1}) of the group's bounding box, the guards and index
// expressions of every access site in the group: the data-free image of the
// per-thread rules seq / if-t / if-f / for-1 / for-2,
// flattened so that loop iterations become tuple coordinates.  The programs of
// a chunk live in __constant__ memory (uniform fetch across a warp).
#pragma once
#include <stdint.h>

#define MAPC_MAX_LEVELS 8        // forU nesting depth per group
#define MAPC_MAX_EMITS 8         // access sites per group program (larger groups are split)
#define MAPC_NREG 32             // per-thread VM registers
#define MAPC_MAX_OPS 4000        // ops per chunk (16 B each; 64 KB of __constant__ minus headroom)
#define MAPC_MAX_PASSES 8        // 64-bit keys / 8-bit digits
#define MAPC_RADIX_BITS 8
#define MAPC_RADIX 256
#define MAPC_MAX_RANGES 768          // static key ranges per radix pass (>= 2 x SM count)

// Fixed registers: r0 = tid, r1 = bid (global block id), r2.. = k_0..k_{L-1}.
#define MAPC_REG_TID 0
#define MAPC_REG_BID 1
#define MAPC_REG_K0 2
#define MAPC_GEN_THREADS 128
#define MAPC_GEN_V 4                 // tuples per thread per VM pass
#define MAPC_GEN_TILE (MAPC_GEN_THREADS * MAPC_GEN_V)

// Direct-address detect cell codes (direct.cu).  16-bit cells (blockDim <=
// 1024): tid = (hi, lo) 5-bit digits, each encoded as one of the 32 smallest
// 7-bit words with exactly three ones (a constant-weight code: the OR of two
// DISTINCT codewords has more than three ones), kind at bit 14:
//   code16(t, k) = CW7[t & 31] | CW7[(t >> 5) & 31] << 7 | k << 14
// racy16(c) <=> bit 14 and (popc(c & 0x7F) > 3 or popc((c >> 7) & 0x7F) > 3).
// The 32 codewords, 8 per 56-bit word, 7 bits each (low codeword first):
#define MAPC_CW7_W0 0x3258a931c34587ull
#define MAPC_CW7_W1 0x58a94a64a8ce1aull
#define MAPC_CW7_W2 0x931a2c370d1931ull
#define MAPC_CW7_W3 0xc586c54a54664aull
#define MAPC_CW16_MAX_WT 10

// Generate modes (generate.cu, capi/jit.cpp).
#define MAPC_MODE_KEYS 0u      // write every access as a packed u64 key (sort / table detect)
#define MAPC_MODE_DIRECT 1u    // fold every access into its cell of the direct-address table (direct.cu)
#define MAPC_MODE_FILTER 2u    // re-emit only the keys whose sort field is ctrl->racy_sf (witness cell)
#define MAPC_MODE_UNIT 3u      // per (phase, block) unit: fold its accesses into a shared-memory table and scan it (JIT only)
#define MAPC_MODE_UNITF 4u     // unit mode's filter: re-emit the witness cell's keys from its unit's tuples only
#define MAPC_UNIT_MAX_BYTES 32768u  // table bytes of one unit (static shared memory)
#define MAPC_UNIT_MAX_SEGS 64u      // segments of a unit-mode chunk (baked as literals)
#define MAPC_CLUSTER_MAX 16u         // CTAs per cluster unit (non-portable cluster size)
#define MAPC_CLUSTER_CTA_BYTES 196608u  // unit-table bytes per CTA of a cluster unit
#define MAPC_CLUSTER_THREADS 512u    // threads per CTA of a cluster unit
#define MAPC_JIT_BAKE_SEGS 16u      // segments of a chunk baked as literals into its specialised kernels

enum MapcOpcode : uint8_t {
  VM_ADD = 0, VM_SUB,   /* monus */
  VM_MUL, VM_DIV, VM_MOD, VM_SHL, VM_SHR, VM_MIN, VM_MAX,
  VM_DIVM, VM_MODM,     /* by constant d (not a power of two): imm = d << 32 | magic, aux = shift (u32 mode) */
  VM_BAND,              /* a & imm (mod by power of two) */
  VM_EQ, VM_NE, VM_LT, VM_LE, VM_GT, VM_GE,
  VM_LAND, VM_LOR, VM_LNOT,
  VM_TRIP,              /* dst = ceil((b monus a) / step), step = operand in aux (see MAPC_AUX_*) */
  VM_MADK,              /* dst = a + k * b, k = register aux */
  VM_ACT,               /* act = a (0/1) */
  VM_EMIT,              /* if act: emit key for index a; aux = array << 1 | is_write */
  VM_MOVI,              /* dst = imm */
  VM_NOP
};

// Operand encoding: a/b are register numbers unless the opcode byte carries
// MAPC_A_IMM / MAPC_B_IMM, in which case that operand is `imm` (at most one
// immediate operand per op; the compiler materialises others with VM_MOVI).
#define MAPC_CODE_MASK 0x3F
#define MAPC_A_IMM 0x40
#define MAPC_B_IMM 0x80
// VM_TRIP step operand in aux: register number, or a constant when bit 31 is set.
#define MAPC_AUX_CONST 0x80000000u
// VM_DIV / VM_MOD: the op may divide by zero on a reached path -> check under act.
#define MAPC_AUX_FAULT 0x80000000u

struct MapcOp {
  uint8_t code;     // opcode | MAPC_A_IMM | MAPC_B_IMM
  uint8_t dst;
  uint8_t a;
  uint8_t b;
  uint32_t aux;
  uint64_t imm;
};  // 16 bytes

// u32 division by an invariant d via the round-up "branchfree" multiplier
// (Granlund & Montgomery 1994): q = (hi(m*n) + ((n - hi(m*n)) >> 1)) >> s.
struct MapcFastDiv {
  uint32_t d;       // divisor (>= 1)
  uint32_t m;       // multiplier (0 when d is a power of two)
  uint32_t s;       // shift
  uint32_t pow2;    // 1 if d is a power of two (q = n >> s)
};

// One generate segment: (instance, group, block range) of a chunk.
struct MapcSeg {
  uint64_t tuple_begin;               // exclusive prefix of tuples within the chunk
  uint64_t n_tuples;                  // (#blocks) * blockDim * prod(trips)
  uint64_t tile_begin;                // exclusive prefix of generate tiles (MAPC_GEN_TILE tuples each)
  uint64_t key_begin;                 // dense segments: first output slot (site-major layout)
  uint64_t key_hi;                    // local-phase field, already shifted to its place in the sort field
  uint32_t prog_begin, prog_end;      // op range in the chunk's constant program
  uint32_t n_levels;
  uint32_t b0;                        // first global block id of the range
  uint32_t lb0;                       // local block index of b0 in the chunk layout
  uint32_t n_emits;                   // EMIT ops in the program (max keys per tuple)
  uint32_t dense;                     // 1: every tuple emits exactly n_emits keys
  uint32_t tid_inner;                 // tuple order: 1 = tid fastest, 0 = innermost loop fastest
  MapcFastDiv trip_div[MAPC_MAX_LEVELS];  // innermost level last
  MapcFastDiv tid_div;                // blockDim
};

// Chunk key layout.  key (u64, MSB..LSB):
//   [ sort field: lphase | array | lblock | index-idx_lo ][ tid ][ kind ]
struct MapcLayout {
  uint32_t w_index, w_block, w_array, w_phase;
  uint32_t w_tid;        // bits of tid
  uint32_t pay_bits;     // w_tid + 1
  uint32_t sort_bits;    // S = w_phase + w_array + w_block + w_index
  uint32_t n_passes;     // radix passes: ceil((S - tb) / 8)
  uint64_t idx_lo;
  uint64_t cap;          // key buffer capacity (keys)
  uint32_t tb;           // bucket-table detect: low sf bits resolved in a table (0 = full sort)
  uint32_t sort_lo;      // lowest key bit the radix passes sort on: pay_bits + tb
};

// Bucket-table detect (table.cu): partial tables of buckets crossing ranges.
#define MAPC_TABLE_BITS_MAX 13
#define MAPC_TABLE_WORDS (2 * (1 << MAPC_TABLE_BITS_MAX) + (1 << MAPC_TABLE_BITS_MAX) / 4)
#define MAPC_TABLE_MAX_CTAS 448
struct MapcTablePart {
  unsigned long long bucket;
  uint32_t ends;         // the bucket ends inside this range (head partials)
  uint32_t valid;
};

// Per-chunk device control block (reset by the init kernel).
struct MapcCtrl {
  unsigned long long n;            // keys generated
  unsigned long long witness;      // packed canonical witness (UINT64_MAX = DRF)
  unsigned long long racy;         // racy segments
  unsigned long long racy_sf;      // smallest sort field of a racy segment (UINT64_MAX = none)
  unsigned int err;                // MAPC_ERR_* bits
  unsigned int n_sort_tiles;
  unsigned int tickets[MAPC_MAX_PASSES + 4];
  unsigned int active[MAPC_MAX_PASSES];
  unsigned int sel[MAPC_MAX_PASSES + 1];   // buffer holding the keys before pass p (0 = A, 1 = B)
  unsigned int hist[MAPC_MAX_PASSES][MAPC_RADIX];
  unsigned long long offs[MAPC_MAX_PASSES][MAPC_RADIX];
  // static-range radix passes (k_rsweep): CTA c owns keys [c*rng_L, (c+1)*rng_L)
  unsigned int rng_L;
  unsigned int first_active;                // first active pass (MAPC_MAX_PASSES if none)
  unsigned int next_active[MAPC_MAX_PASSES];// next active pass after p (MAPC_MAX_PASSES if none)
  unsigned int rt_done[MAPC_MAX_PASSES];    // pass p's range table accumulated by the previous scatter
  unsigned int rt_bad[MAPC_MAX_PASSES];     // ... but abandoned (digits not warp-uniform): recompute
  MapcFastDiv rng_div;                      // divides a key position by rng_L
  unsigned long long nf;                    // direct detect: keys of the witness cell re-emitted (filter mode)
  unsigned long long wit_sf;                // direct detect: cell whose witness is folded (UINT64_MAX = none)
};

// Per-chunk result copied out by the last kernel of the chunk.
struct MapcChunkResult {
  unsigned long long n;
  unsigned long long witness;
  unsigned long long racy;
  unsigned int err;
  unsigned int active_passes;      // radix passes that were not skipped
  unsigned int table_reads;        // range-table reads of the keys (k_hist_ranges + k_range_hist that ran)
  unsigned int active_mask;        // bit p: radix pass p ran
};

#define MAPC_ERR_DIV0 1u        // division/modulo by zero on a reached path
#define MAPC_ERR_CAPACITY 2u    // more keys than the chunk bound (library bug guard)
#define MAPC_ERR_LAYOUT 4u      // index outside the chunk layout (library bug guard)
#define MAPC_ERR_WATCHDOG 8u    // look-back spin exceeded its bound (library bug guard)

// Per-tile fragment state of the detect kernel: the racy test
// of a segment only needs (has a write, min tid, max tid).
#define MAPC_DETECT_MAX_UNITS 8192   /* fragment records: max(tiles, warp ranges) */
struct MapcSegState {
  uint32_t first_tid, last_tid;  // tids of the fragment's first and last key
  uint8_t wr;                    // fragment holds a write
  uint8_t diff;                  // two adjacent keys of the fragment have different tids
  uint8_t valid, ends;           // fragment present; fragment ends inside this chunk
  unsigned long long sf;         // sort field of the fragment's segment
};
