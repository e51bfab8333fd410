/*
 * mapcheck.h -- C ABI of the B200-native concrete MAP data-race checker.
 *
 * What it computes (arxiv 2203.12878, "BabyCUDA"): a memory access protocol
 * (MAP; Fig. 2) is instantiated at fixed grid/block
 * dimensions and parameter values; every access value alpha = i : o[y]
 * of every thread i in T = {0..blockDim-1} (rule par,
 * PAPER.md:579-589) is enumerated on the GPU, tagged with its barrier phase
 * (PAPER.md:179-182), array and block, and the library decides whether two
 * DISTINCT threads touch the same index of the same array in the same phase of
 * the same block with at least one write (the data-race definition of
 * PAPER.md:111-113).  By Theorem 1 the verdict is the
 * ground truth for a typable kernel at this instantiation.  The reported
 * witness is canonical: the lexicographic minimum of
 *   (phase, array, block, index, tid_lo, tid_hi, kind_lo, kind_hi),
 * tid_lo < tid_hi, rd = 0 < wr = 1 -- independent of launch order and of the
 * number of GPUs (reading R14).
 *
 * MAP text grammar: DESIGN.md §3 (extends SPEC.md:179 with sync/forS, named
 * arrays, params, `step`, bid, shifts and min/max).
 *
 * Conventions
 *  - Every entry point returns a map_status; out-parameters are written only
 *    on MAP_OK.  No C++ exception crosses the ABI.
 *  - map_program is opaque and library-owned (free with map_program_free).
 *    Distinct programs may be used concurrently from different host threads;
 *    one program is not re-entrant.
 *  - Device memory is BORROWED: the caller passes a device scratch buffer of
 *    at least map_scratch_bytes() bytes (PyTorch allocates it) and a CUDA
 *    stream; the library never cudaMallocs on the hot path.  All work is
 *    enqueued on that stream; map_check_races synchronizes it once at the end.
 *    The overlapped direct-address pipeline additionally runs the table scans
 *    on one library-owned side stream per program (created at first use,
 *    destroyed by map_program_free), ordered by events and joined back into
 *    the caller's stream before the run ends.  Without per-kernel timing
 *    (map_exec.stats == NULL), the second identical call on a program (same
 *    plan, flags, scratch, stream, shard) captures the run into a CUDA graph
 *    on a library-owned capture stream and later identical calls replay it
 *    on the caller's stream; results are the same either way.
 *  - There is no CPU fallback: without a usable CUDA device the run entry
 *    points return MAP_E_CUDA.
 */
#ifndef MAPCHECK_H
#define MAPCHECK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MAP_OK = 0,
  MAP_E_PARSE = 1,   /* syntax error in the MAP text (diag: "line:col: msg")            */
  MAP_E_SCOPE = 2,   /* unbound / duplicate / shadowing identifier          */
  MAP_E_BARRIER = 3, /* sync/forS under if or forU, or forS bounds mention tid/bid       */
  MAP_E_RANGE = 4,   /* a value may exceed 64 bits, key/witness fields do not fit 64
                        bits, a loop step may be 0, or too many phases/instances        */
  MAP_E_ARITH = 5,   /* division or modulo by zero reached at run time                  */
  MAP_E_CUDA = 6,    /* CUDA error or no device                                          */
  MAP_E_COMM = 7,    /* reserved for the multi-GPU orchestration (NCCL lives in Python)  */
  MAP_E_ARG = 8,     /* bad argument: null pointer, missing/unknown parameter, ...       */
  MAP_E_NOMEM = 9,   /* scratch too small for one (phase, block) unit                    */
  MAP_E_TYPE = 10    /* BabyCUDA kernel is not typable (Fig. 6) and no MAP was requested */
} map_status;

typedef struct map_program map_program;

/* Instantiation (PAPER.md:431 T subset of N; here T = {0..prod(block)-1}).
 * 3-D dims are flattened: tid = tz*bx*by + ty*bx + tx, same for bid. */
typedef struct {
  uint32_t grid[3];
  uint32_t block[3];
  uint32_t n_params;
  const char *const *param_names;   /* n_params NUL-terminated names        */
  const uint64_t *param_values;     /* n_params naturals     */
} map_instance;

/* Per-kernel-class device timings of one map_check_races call, measured with
 * CUDA events recorded on the caller's stream around every launch (optional:
 * map_exec.stats == NULL disables them).  bytes = ALGORITHMIC bytes the
 * launches had to move: generate writes 8 B per key, the
 * histogram reads 8 B per key, an active radix pass reads + writes 8 B per
 * key, detect reads 8 B per key.  Direct-address detect (table of 2^S cells
 * of 4 or 8 B, larger than L2 at the bench sizes): the fused generate
 * (MAP_K_DIRECT) reads and writes every cell once (its per-access reductions
 * are served by L2), the clear (MAP_K_CLEAR) writes and the scan
 * (MAP_K_DETECT) reads every cell once. */
enum {
  MAP_K_GENERATE = 0,
  MAP_K_HIST = 1,
  MAP_K_SCAN = 2,
  MAP_K_ONESWEEP = 3,
  MAP_K_DETECT = 4,
  MAP_K_OTHER = 5,
  MAP_K_SORT_NEXT = 6,      /* radix passes that also build the next pass's range table */
  MAP_K_DIRECT = 7,         /* generate fused with the direct-address table reductions  */
  MAP_K_CLEAR = 8,          /* direct-address table clear                               */
  MAP_K_UNIT = 9,           /* on-chip per-(phase, block) tables: generate + fold + scan */
  MAP_K_COUNT = 10
};
typedef struct {
  float ms[MAP_K_COUNT];            /* summed over the timed launches                      */
  uint32_t launches[MAP_K_COUNT];   /* every launch of the class                           */
  uint64_t bytes[MAP_K_COUNT];      /* algorithmic bytes of every launch                   */
  uint32_t timed[MAP_K_COUNT];      /* launches that carried timing events (ms / timed =   */
                                    /* the average launch duration)                        */
} map_kernel_stats;

/* Execution resources borrowed from the caller. */
typedef struct {
  int device;                 /* CUDA device ordinal                                  */
  void *stream;               /* cudaStream_t (0 = legacy default stream)             */
  void *scratch;              /* device buffer, >= map_scratch_bytes(p, chunk)        */
  size_t scratch_bytes;
  uint64_t chunk_max_accesses;/* accesses per chunk (0 = library default)            */
  uint32_t rank, world;       /* shard: process rank `rank`'s chunks of `world`
                                 (map_rank_chunks: a contiguous, bound-balanced range;
                                 world 0 or 1 = all chunks; multi-GPU) */
  map_kernel_stats *stats;    /* optional per-kernel timings (NULL = off)            */
  uint32_t flags;             /* MAP_GEN_* (generate path); 0 = automatic            */
} map_exec;

/* Generate path (map_exec.flags): the bytecode VM, or kernels specialised from
 * the same bytecode with NVRTC at first use (cached per process).  AUTO picks
 * the specialised kernels for plans of >= 2^23 accesses whose chunks need <= 64
 * distinct kernels (chunks differing only in data the kernel does not bake,
 * e.g. the phases of a time loop, share one). */
#define MAP_GEN_AUTO 0u
#define MAP_GEN_VM 1u
#define MAP_GEN_JIT 2u

/* Detect path (map_exec.flags, OR-ed with MAP_GEN_*).
 *   MAP_DETECT_SORT:  full LSD radix sort on all S sort-field bits, then the
 *                     segmented scan over equal sort fields.
 *   MAP_DETECT_TABLE: LSD passes only on the bits above the low tb <= 13 bits
 *                     ("buckets"), then each bucket is folded into a 2^tb-cell
 *                     direct-address table in shared memory (min tid, max tid,
 *                     write bit per cell).  Same verdict,
 *                     witness, access count and racy-segment count.
 *   MAP_DETECT_DIRECT: no keys and no sort: every access is folded into its
 *                     cell of a 2^S-cell direct-address table in device
 *                     memory with one atomic OR of tid | ~tid << wt |
 *                     kind << 2wt (racy <=> write bit and two distinct tids
 *                     <=> (OR tid) & (OR ~tid) != 0), the table is scanned
 *                     once, and the witness cell's keys are re-generated and
 *                     folded (sort-free).  Used for a
 *                     chunk when its estimated time (fixed cost + clear and
 *                     scan of the table + per-access generate) beats the keys
 *                     pipelines' estimate and the table fits the scratch plan
 *                     (DESIGN.md §5.6); other chunks take the AUTO choice below.
 *   MAP_DETECT_AUTO:  DIRECT where it qualifies; otherwise TABLE when the
 *                     chunk holds >= 2^16 keys and at least 2^(S-1) of them
 *                     (dense sort-field space), else SORT.
 * All paths give the same verdict, witness, access count and racy-segment
 * count. */
#define MAP_DETECT_AUTO 0u
#define MAP_DETECT_SORT 0x10u
#define MAP_DETECT_TABLE 0x20u
#define MAP_DETECT_DIRECT 0x40u
/*   MAP_DETECT_UNIT:  per (phase, block) unit, entirely on chip: one CTA folds
 *                     the unit's accesses into a shared-memory table of its
 *                     (array, index) cells (same cell code as DIRECT) and scans
 *                     it; no table in HBM (SURVEY.md §8f NEXT-3 on chip).  For
 *                     chunks whose unit table fits MAPC_UNIT_MAX_BYTES and that
 *                     have enough units (or few accesses), with the specialised
 *                     generate; AUTO takes it where it applies, other chunks
 *                     fall back as AUTO. */
#define MAP_DETECT_UNIT 0x80u
#define MAP_DETECT_MASK 0xF0u

/* MAP_EXEC_SEQUENTIAL (map_exec.flags): run the direct path's chunks one after
 * another on the caller's stream only (no side stream: each chunk's clear,
 * generate and scan in turn) -- for measuring the kernels alone; same results. */
#define MAP_EXEC_SEQUENTIAL 0x100u
/* MAP_EXEC_PROFILE_GENERATE (map_exec.flags, with map_exec.stats): time only the
 * generate launches (MAP_K_GENERATE, MAP_K_DIRECT, MAP_K_UNIT) with CUDA events;
 * the other classes are counted (launches, bytes) but not timed (ms = 0), so
 * the timing events perturb the run less (one event pair per chunk). */
#define MAP_EXEC_PROFILE_GENERATE 0x200u
/* MAP_EXEC_PROFILE_SAMPLED (with MAP_EXEC_PROFILE_GENERATE): time only the generate
 * launches of every fourth chunk of the run (positions 2, 6, 10, ...: past the
 * pipeline's fill), so the timing perturbs the run least; `timed` counts them. */
#define MAP_EXEC_PROFILE_SAMPLED 0x400u

typedef struct {
  int32_t verdict;            /* 0 = DRF, 1 = RACY (over the chunks this call ran)   */
  int32_t n_chunks;           /* chunks this call processed                          */
  uint64_t n_accesses;        /* accesses enumerated, counted with multiplicity      */
  uint64_t racy_segments;     /* (phase, array, block, index) cells holding a race   */
  float device_ms;            /* device time of the whole run (CUDA events)          */
  uint32_t gpu_launches;      /* kernels launched by this call                       */
  uint64_t h2d_bytes;         /* host->device bytes copied (bytecode, segment tables)*/
  uint64_t d2h_bytes;         /* device->host bytes copied (per-chunk results)       */
} map_result;

typedef struct {
  uint32_t phase, array, block;
  uint64_t index;
  uint32_t tid_lo, tid_hi;
  uint8_t kind_lo, kind_hi;   /* 0 = rd, 1 = wr                                       */
  const char *array_name;     /* valid until map_program_free                        */
} map_witness;

/* Static facts of a compiled program (for sizing and reporting). */
typedef struct {
  uint32_t n_phases;          /* barrier phases (syncs executed + 1)                  */
  uint32_t n_arrays;
  uint32_t n_instances;       /* (u-fragment, forS iteration) instances              */
  uint32_t n_groups;          /* (instance, loop nest) groups = generate segments    */
  uint64_t max_accesses;      /* upper bound on accesses (bounding boxes)            */
  uint64_t max_unit_accesses; /* largest (phase, block) unit bound                   */
  uint32_t u32_mode;          /* 1 if every value provably fits 32 bits              */
  uint32_t bytecode_ops;
} map_info;

/* Parse, resolve, interval-analyse and lower the MAP `src` (len bytes, need not
 * be NUL-terminated) at the instantiation `inst`.  On error a diagnostic
 * "line:col: message" is written to diag (if non-null). */
map_status map_compile(const char *src, size_t len, const map_instance *inst, map_program **out,
                       char *diag, size_t diag_cap);

map_status map_info_get(const map_program *p, map_info *out);

/* Device scratch needed to process chunks of up to chunk_max_accesses
 * accesses (0 = the largest (phase, block) unit of this program). */
size_t map_scratch_bytes(const map_program *p, uint64_t chunk_max_accesses);

/* Run the whole pipeline on one GPU; blocking.  Per chunk: generate, then the
 * detect path map_exec.flags selects -- by default the sort-free direct-address
 * table for dense chunks (MAP_DETECT_DIRECT below), else partial sort + bucket
 * tables or full radix sort + segmented scan.  Writes verdict, counts and
 * timing to *out.  With chunk_max_accesses == 0 and world > 1 the plan uses
 * map_default_chunk(p, world) (size the scratch with that value). */
map_status map_check_races(map_program *p, const map_exec *ex, map_result *out);

/* Canonical witness of the last racy map_check_races; MAP_E_ARG if it was DRF. */
map_status map_witness_get(const map_program *p, map_witness *out);

/* Full race listing (SPEC.md:434-437 races_of, one entry
 * per racy (phase, array, block, index) segment): the canonical witness of
 * every racy segment, in canonical (lexicographic) order.  Runs the whole
 * pipeline with the full sort on every chunk of the plan (ex->rank/world and
 * the MAP_DETECT_* flags are ignored).  out[cap] (HOST, caller-owned) receives
 * the min(cap, *n_total) smallest; *n_total = the number of racy segments (the
 * racy_segments of map_check_races).  array_name pointers stay valid until
 * map_program_free.  Errors as map_check_races. */
map_status map_list_races(map_program *p, const map_exec *ex, map_witness *out, uint64_t cap, uint64_t *n_total);

/* Name of array `idx` (declaration order; NULL if out of range). */
const char *map_array_name(const map_program *p, uint32_t idx);

void map_program_free(map_program *p);
const char *map_status_str(map_status s);

/* ---- optional scratch allocator ----
 * The library never allocates its device scratch; a caller may take it from
 * here to get *compressible* device memory (flags MAP_ALLOC_COMPRESSIBLE:
 * cuMemCreate with generic compression when the device supports it, else plain
 * cudaMalloc).  The direct path (MAP_DETECT_DIRECT) clears its tables to zero
 * before each chunk and its atomic ORs then fill those lines from DRAM; all-zero
 * lines compress, so the clear and the fills move fewer DRAM bytes (DESIGN.md
 * §6.1, 5a: 1262 -> 1391 G acc/s).  Results are identical in either memory.
 * map_scratch_alloc: `bytes` (> 0) of device memory on `device` (made current);
 * *ptr receives the address (caller-owned until map_scratch_free), *size (may be
 * NULL) the rounded-up size, *compressed (may be NULL) 1 if the driver granted
 * compression.  Errors: MAP_E_ARG (null ptr, bytes 0, unknown flag), MAP_E_CUDA
 * (no device / driver), MAP_E_NOMEM (out of device memory).
 * map_scratch_free: release a map_scratch_alloc block (synchronises the device
 * first); NULL is a no-op; MAP_E_ARG for a pointer this helper did not return. */
#define MAP_ALLOC_COMPRESSIBLE 1u
map_status map_scratch_alloc(int device, uint64_t bytes, uint32_t flags, void **ptr, uint64_t *size,
                             uint32_t *compressed);
map_status map_scratch_free(void *ptr);

/* ---- stage API (multi-GPU key exchange; NCCL via torch) ----
 * The hot path split at the exchange point, for a (phase, block) unit too
 * large for one GPU: every rank generates a slice of a chunk's tuples, the keys
 * are routed to the rank that owns their sort field (hash), and every rank
 * sorts + detects what it received; a segment never straddles ranks, so the
 * racy counts add up and the global witness is the minimum of the ranks'.
 *
 * map_chunk_count / map_chunk_info: the plan's chunks (same plan as
 * map_check_races for the same chunk_max_accesses; 0 = library default). */
map_status map_chunk_count(const map_program *p, uint64_t chunk_max_accesses, uint32_t *n_chunks);
/* Default chunk capacity (accesses) for a job sharded over `world` ranks: the
 * single-GPU default (world <= 1), or smaller so that the plan has at least two
 * chunks per rank where its (phase, block) units allow (PAPER.md:179-182:
 * phases and blocks are independent units).  0 if p is NULL. */
uint64_t map_default_chunk(const map_program *p, uint32_t world);
/* The chunk indices rank `rank` of `world` processes in map_check_races (a
 * contiguous range balanced by chunk bound): out[cap] (HOST) receives the first
 * min(cap, *n) of them, *n their number.  chunk_max_accesses 0 = the default
 * for that world.  Errors: MAP_E_ARG, plan errors as map_check_races. */
map_status map_rank_chunks(const map_program *p, uint64_t chunk_max_accesses, uint32_t rank, uint32_t world,
                           uint32_t *out, uint32_t cap, uint32_t *n);
typedef struct {
  uint32_t phase_lo, phase_hi;   /* inclusive range of barrier phases                 */
  uint32_t block_lo, block_hi;   /* [block_lo, block_hi)                              */
  uint64_t bound;                /* upper bound on the chunk's keys (key buffer size)  */
  uint32_t sort_bits, n_passes;  /* sort-field width and radix passes                  */
} map_chunk_desc;
map_status map_chunk_info(const map_program *p, uint64_t chunk_max_accesses, uint32_t chunk, map_chunk_desc *out);
/* map_generate_bucketed: rank `rank` of `world` (world <= 64) generates the
 * generate tiles [T*rank/world, T*(rank+1)/world) of chunk `chunk` (T = the
 * chunk's tile count; every key compacted, bytecode VM) and writes them to
 * keys_out (DEVICE, u64[>= map_chunk_desc.bound], caller-owned) grouped by
 * destination d = hi64(splitmix64(sort field) * world), in order of d;
 * counts_out[world] (HOST) receives the per-destination counts.  Uses ex's
 * scratch and stream and synchronises the stream.  Errors: MAP_E_ARG (bad
 * rank/world/chunk/pointers), MAP_E_NOMEM (scratch), MAP_E_ARITH (division by
 * zero reached), MAP_E_CUDA. */
map_status map_generate_bucketed(map_program *p, const map_exec *ex, uint32_t rank, uint32_t world,
                                 uint32_t chunk, void *keys_out, uint64_t *counts_out);
/* map_sort_detect: sort + detect n DEVICE-resident keys of chunk `chunk` (e.g.
 * the keys a rank received; n <= the plan's capacity, keys not modified, copied
 * into scratch); the detect path follows ex->flags (MAP_DETECT_*).  The
 * chunk's packed canonical witness (UINT64_MAX = DRF; decode with
 * map_unpack_witness) and racy-segment count are written to the HOST.  Errors:
 * MAP_E_ARG, MAP_E_NOMEM (n too large / scratch), MAP_E_CUDA. */
map_status map_sort_detect(map_program *p, const map_exec *ex, uint32_t chunk, void *keys, uint64_t n,
                           uint64_t *packed_witness, uint64_t *racy_segments);
map_status map_unpack_witness(const map_program *p, uint32_t chunk, uint64_t packed, map_witness *out);

/* ---- BabyCUDA front end ------------------------------
 * BabyCUDA (Fig. 5) is the data-carrying kernel language the
 * paper types into MAPs: `A[n] := m` (write), `let y = A[n] in b` (read into y
 * for the rest of the block), if/else, `for x in n..m [step s]`, skip, `;`, plus
 * `sync` (the synchronized fragment) and the declarations
 * `params P, ...;` and `shared A[extent], B, ...;` (grammar: DESIGN.md §3b).
 *
 * map_infer: parse `src` (len bytes) and type it with the behavioural type system
 * of Fig. 6 (t-n, t-b, t-write, t-read, t-seq, t-if, t-for,
 * t-skip) under V = {tid, bid} u params.  A kernel is typable iff no value read
 * from an array reaches an array index, a condition or a loop bound (Eq. 1,
 * PAPER.md:887-891); by Theorem 1 every race reported on a
 * typable kernel's MAP is then a TRUE alarm.  *ty (HOST, caller-owned) receives
 * typable, the kind of the first failing premise (MAP_TYPE_DATA_INDEX: a read
 * value indexes an array; MAP_TYPE_DATA_CONTROL: it decides a condition or a loop
 * bound), the offending variable and its line:col.
 * Output: the MAP text (DESIGN.md §3 grammar, input to map_compile) into
 * map_out[map_cap] (HOST, NUL-terminated, truncated to map_cap - 1; *map_len =
 * the full length): the t-rules' image of a typable kernel; for an ill-typed
 * one, when data_domain > 0, the DATA-ABSTRACTED MAP in which a read whose value
 * reaches a typed position becomes `rd A[n]; forU y in 0..data_domain { u }` (the
 * value may be anything in [0, data_domain): Faial's view of array data,
 * PAPER.md:880-885; its races may be false alarms).
 * Returns MAP_OK, MAP_E_TYPE (ill-typed and data_domain == 0; *ty filled, no
 * text), MAP_E_PARSE / MAP_E_SCOPE (unbound or shadowing name) / MAP_E_BARRIER
 * (sync under if, or a loop around a sync whose bounds depend on tid, bid or a
 * read value) / MAP_E_RANGE (literal >= 2^64) with "line:col: message" in diag,
 * MAP_E_ARG (null pointers). */
#define MAP_TYPE_OK 0
#define MAP_TYPE_DATA_INDEX 1
#define MAP_TYPE_DATA_CONTROL 2
typedef struct {
  int32_t typable;
  int32_t kind;              /* MAP_TYPE_*                                      */
  uint32_t line, col;        /* first offending use (1-based)                   */
  char var[64];              /* its variable (NUL-terminated, truncated)        */
} map_typing;
map_status map_infer(const char *src, size_t len, uint64_t data_domain, char *map_out, size_t map_cap,
                     size_t *map_len, map_typing *ty, char *diag, size_t diag_cap);

/* ---- BabyCUDA executor and the Theorem-1 differential check (NEXT-2) ---------
 * map_kernel_compile: parse + type a BabyCUDA kernel (as map_infer) and plan its
 * execution at the instantiation `inst` (parameters as map_compile; blockDim
 * <= 1024, CUDA's own limit).  Array extents: as declared (`shared A[n]`), else,
 * for a typable kernel, the index hull of its inferred MAP; an ill-typed kernel
 * must declare them (MAP_E_ARG).  The executor kernel is generated as CUDA C and
 * compiled with NVRTC for sm_100a at the first map_execute.  Errors: as
 * map_infer, MAP_E_ARG (blockDim > 1024, missing parameter or extent), MAP_E_RANGE
 * (the access key phase|array|block|index|tid|kind exceeds 64 bits).
 *
 * map_execute: run the kernel WITH DATA on the GPU under the semantics of Fig. 5
 * (PAPER.md:443-589): one CTA per block, CUDA thread t = BabyCUDA thread t; a
 * read returns lastwrite over the thread's own current record consed onto the
 * closed phases (own writes of the phase visible, other threads' not,
 * PAPER.md:482-495), arrays start undefined (bottom reads as 0 and is counted,
 * DESIGN.md R20), `sync` closes the phase (a cell written by several threads
 * keeps the smallest writer tid's value, R21).  Every executed access value
 * (alpha in^ P) is recorded and race-checked exactly as
 * map_check_races checks a MAP: verdict, canonical witness (map_kernel_witness),
 * racy cells.  ex->scratch must hold map_kernel_scratch_bytes(k, max_events,
 * 0, ex->flags) bytes; max_events bounds the executed accesses (typable kernels:
 * map_kernel_info.max_events is exact).  MAP_EXEC_KEEP_MEMORY (ex->flags) keeps
 * every block's final array contents for map_kernel_memory.  Errors:
 * MAP_E_ARITH (division / modulo by zero, loop step zero), MAP_E_RANGE (a value
 * exceeds 64 bits, or an index reaches its array's extent), MAP_E_NOMEM (more
 * than max_events accesses -- *out->n_events says how many -- or a thread's
 * conflict log overflowed), MAP_E_CUDA. */
typedef struct map_kernel map_kernel;
map_status map_kernel_compile(const char *src, size_t len, const map_instance *inst, map_kernel **out, char *diag,
                              size_t diag_cap);
typedef struct {
  int32_t typable;           /* Fig. 6 derivation exists                          */
  uint32_t n_phases, n_arrays, block_threads;
  uint64_t n_blocks;
  uint64_t cells_per_block;  /* sum of the array extents                          */
  uint32_t key_bits;         /* width of the access key                           */
  uint64_t max_events;       /* accesses of the inferred MAP (typable), else 0     */
} map_kernel_info;
map_status map_kernel_info_get(const map_kernel *k, map_kernel_info *out);
/* Extent (cells) of array `array` as planned (0 if out of range). */
uint64_t map_kernel_extent(const map_kernel *k, uint32_t array);
#define MAP_EXEC_KEEP_MEMORY 0x200u
size_t map_kernel_scratch_bytes(const map_kernel *k, uint64_t max_events, uint64_t lambda_cap, uint32_t flags);
typedef struct {
  int32_t verdict;           /* races among the executed accesses                 */
  int32_t typable;           /* 1: every alarm is a true alarm (Theorem 1)        */
  uint64_t n_events;         /* accesses executed (multiset)                      */
  uint64_t n_alpha;          /* distinct access values                            */
  uint64_t racy_segments;    /* racy (phase, array, block, index) cells           */
  uint64_t uninit_reads;     /* reads of bottom (lastwrite-undef)                 */
  uint64_t ambiguous_reads;  /* reads of a cell last written by several threads   */
  float device_ms;
  uint32_t gpu_launches;
} map_exec_result;
map_status map_execute(map_kernel *k, const map_exec *ex, uint64_t max_events, map_exec_result *out);
map_status map_kernel_witness(const map_kernel *k, map_witness *out);
/* Final contents of array `array` of block `block` after the last map_execute
 * with MAP_EXEC_KEEP_MEMORY on the same scratch: values[i] and defined[i] (HOST,
 * n <= the array's extent) for indices 0..n-1 (defined 0 = never written). */
map_status map_kernel_memory(const map_kernel *k, const map_exec *ex, uint32_t block, uint32_t array, uint64_t *values,
                             uint8_t *defined, uint64_t n);
/* Theorem 1, checked: execute the kernel (as map_execute) and
 * compare the SET of executed access values with the set Lambda the MAP program
 * `lambda` enumerates (compiled from map_infer's text at the same instantiation;
 * ex_lambda = its own scratch, same device and stream), both sorted on the GPU.
 * For a typable kernel and its inferred MAP the sets are equal; for an ill-typed
 * kernel and its data-abstracted MAP, alpha is a subset (the MAP's extra values
 * are the source of false alarms).  lambda_cap bounds Lambda's keys. */
typedef struct {
  uint32_t phase, array, block;
  uint64_t index;
  uint32_t tid;
  uint8_t kind;
} map_access;
typedef struct {
  int32_t equal;                       /* alpha set == Lambda set                       */
  uint64_t n_alpha, n_lambda;          /* distinct values on each side                  */
  uint64_t only_alpha, only_lambda;    /* values missing on the other side              */
  int32_t has_first_alpha, has_first_lambda;
  map_access first_alpha, first_lambda;/* the smallest such value of each side          */
  map_exec_result exec;                /* the execution's own result                    */
} map_diff;
map_status map_theorem1_diff(map_kernel *k, map_program *lambda, const map_exec *ex, const map_exec *ex_lambda,
                             uint64_t max_events, uint64_t lambda_cap, map_diff *out);
void map_kernel_free(map_kernel *k);

#ifdef __cplusplus
}
#endif
#endif /* MAPCHECK_H */
