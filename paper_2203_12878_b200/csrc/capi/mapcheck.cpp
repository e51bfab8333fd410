// mapcheck.cpp -- C ABI (include/mapcheck.h): compile, plan, launch, decode.
//
// Host orchestration of the hot path on one GPU:
//   per chunk (a range of barrier phases, or of blocks of one phase):
//     upload bytecode (__constant__) + segment table
//     k_chunk_init -> k_generate -> k_hist -> k_digit_scan -> k_onesweep x P
//     -> k_detect -> k_detect_fixup -> k_chunk_finish
//   all on the caller's stream; one synchronisation at the very end.
// Chunks are exact units because races are intra-(phase, block)
// (R10): the canonical witness is the
// lexicographic minimum of the per-chunk witnesses, taken on the host.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../../include/mapcheck.h"
#include "../compiler/compiler.h"
#include "../devabi.h"
#include "jit.h"

extern "C" {
cudaError_t mapc_upload_ops(const MapcOp* host_ops, size_t n_ops, cudaStream_t s);
cudaError_t mapc_launch_generate(const MapcSeg* segs, int n_segs, unsigned long long tile_lo,
                                 unsigned long long tile_hi, const MapcLayout* lay, int u32_mode,
                                 unsigned long long* keys, MapcCtrl* ctrl, int n_sms, uint32_t nreg,
                                 uint32_t max_emits, uint32_t force_compact, uint32_t mode, void* tab,
                                 uint32_t cell_bytes, cudaStream_t s);
cudaError_t mapc_launch_table_clear(void* tab, unsigned long long bytes, int n_sms, int ctas_per_sm, cudaStream_t s);
cudaError_t mapc_launch_direct_scan(const void* tab, unsigned long long cells, uint32_t cell_bytes, uint32_t w_tid,
                                    MapcCtrl* ctrl, int n_sms, int ctas_per_sm, cudaStream_t s, int unroll);
cudaError_t mapc_launch_witness_gate(MapcCtrl* ctrl, uint32_t* gate, uint32_t ph_lo, uint32_t ph_hi, cudaStream_t s,
                                     const unsigned long long* pcomp, uint32_t nph, uint32_t wa, uint32_t wb, uint32_t wi);
cudaError_t mapc_launch_witness_flat(const unsigned long long* keys, MapcCtrl* ctrl, uint32_t pay_bits, uint32_t w_tid,
                                     unsigned long long cap, cudaStream_t s, MapcChunkResult* out);
int mapc_bucket_max_world();
cudaError_t mapc_launch_bucket_count(const unsigned long long* keys, const MapcCtrl* ctrl, uint32_t pay_bits,
                                     uint32_t world, unsigned long long* counts, int n_sms, cudaStream_t s);
cudaError_t mapc_launch_bucket_scatter(const unsigned long long* keys, const MapcCtrl* ctrl, uint32_t pay_bits,
                                       uint32_t world, unsigned long long* cursors, unsigned long long* out,
                                       int n_sms, cudaStream_t s);
cudaError_t mapc_launch_hist(const unsigned long long* keys, MapcCtrl* ctrl, uint32_t pay_bits, uint32_t n_passes,
                             unsigned long long max_keys, int n_sms, cudaStream_t s);
cudaError_t mapc_launch_digit_scan(MapcCtrl* ctrl, uint32_t n_passes, cudaStream_t s);
unsigned long long mapc_sort_tile();
cudaError_t mapc_launch_onesweep(unsigned long long* bufA, unsigned long long* bufB, MapcCtrl* ctrl,
                                 unsigned long long* lookback, uint32_t pass, uint32_t shift,
                                 unsigned long long epoch, unsigned long long max_keys, int n_sms, cudaStream_t s);
unsigned long long mapc_detect_tile();
cudaError_t mapc_launch_chunk_init(MapcCtrl* ctrl, unsigned long long n0, cudaStream_t s);
cudaError_t mapc_launch_detect(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                               uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid, MapcSegState* first_frag,
                               MapcSegState* last_frag, unsigned long long max_keys, int n_sms, cudaStream_t s);
cudaError_t mapc_launch_chunk_finish(const MapcCtrl* ctrl, uint32_t n_passes, MapcChunkResult* out, cudaStream_t s);
unsigned long long mapc_rsweep_tile();
int mapc_rsweep_ranges(int n_sms);
cudaError_t mapc_launch_hist_ranges(const unsigned long long* keys, MapcCtrl* ctrl, unsigned int* rhist,
                                    uint32_t pay_bits, uint32_t n_passes, int G, cudaStream_t s);
cudaError_t mapc_launch_range_hist(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                                   unsigned int* rhist, uint32_t pass, uint32_t pay_bits, int G, cudaStream_t s);
int mapc_rsweep_fused();
int mapc_table_ctas(int n_sms);
unsigned long long mapc_table_tile();
cudaError_t mapc_launch_list_racy(const unsigned long long* bufA, const unsigned long long* bufB, const MapcCtrl* ctrl,
                                  uint32_t n_passes, uint32_t pay_bits, uint32_t w_tid, unsigned long long* counts,
                                  unsigned int max_warps, unsigned long long* out, unsigned long long cap,
                                  unsigned long long* total, unsigned long long max_keys, int n_sms, cudaStream_t s);
cudaError_t mapc_launch_detect_table(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                                     uint32_t n_passes, uint32_t pay_bits, uint32_t tb, uint32_t w_tid,
                                     MapcTablePart* parts, uint32_t* store, unsigned long long max_keys, int n_sms,
                                     cudaStream_t s);
cudaError_t mapc_launch_witness(const unsigned long long* bufA, const unsigned long long* bufB, MapcCtrl* ctrl,
                                uint32_t n_passes, uint32_t pay_bits, uint32_t tb, uint32_t w_tid, cudaStream_t s);
cudaError_t mapc_launch_rsweep(unsigned long long* bufA, unsigned long long* bufB, MapcCtrl* ctrl,
                               unsigned int* rhist, uint32_t pass, uint32_t pay_bits, int G, int red_next,
                               cudaStream_t s);
}

namespace {

using mapc::bits_for;

struct Chunk {
  uint32_t phase_lo = 0, phase_hi = 0;      // inclusive range of phases covered
  uint64_t b_lo = 0, b_hi = 0;              // [b_lo, b_hi)
  MapcLayout lay{};
  std::vector<MapcSeg> segs;
  std::vector<MapcOp> ops;
  uint64_t bound = 0;
  uint64_t total_tuples = 0;
  uint64_t total_tiles = 0;                 // generate tiles (segment-aligned)
  uint64_t dense_total = 0;                 // keys of dense segments (placed directly)
  uint32_t nreg = MAPC_REG_K0;              // VM registers used by the chunk's programs
  uint32_t max_emits = 0;                   // largest n_emits of a non-dense segment
  size_t stage_ops = 0, stage_segs = 0;     // offsets in the pinned staging buffer
  mapj::JitChunk jit;                       // straight-line programs for the specialised generate
  // sort-free direct-address detect (direct.cu): one cell per sort-field value
  uint64_t cells = 0;                       // 2^S
  uint32_t cell_bytes = 4;                  // 2 if w_tid <= 10 (devabi.h code16), 4 if 2 w_tid + 1 <= 32, else 8
  bool direct_ok = false;                   // the table is cheap enough and fits the scratch plan
  bool unit_ok = false;                     // per-(phase, block) tables fit shared memory (MAPC_MODE_UNIT)
  size_t unit_smem = 0;                     // dynamic shared bytes per CTA of a cluster unit
  size_t dev_segs = 0;                      // offset of this chunk's segment table in the all-chunks region
  // stride-compressed direct table (JIT direct mode, 16-bit cells): every site of local
  // phase q has index - idx_lo == res[q] (mod 2^sh[q]), so the phase's block keeps one
  // cell per 2^sh[q] indices; pcomp = per q {base, sh | res << 8} (device copy follows
  // the segment table); comp_cells = the compressed table's cells
  bool comp_ok = false;
  uint64_t comp_cells = 0;
  std::vector<unsigned long long> pcomp;
};

struct Plan {
  uint64_t cap = 0;                         // max keys of any chunk
  std::vector<Chunk> chunks;
  mapj::JitHandle jit[5];                    // per generate mode (MAPC_MODE_*); null = not built yet
  size_t jit_distinct = 0;                  // distinct specialised kernels of the chunks (0 = not counted)
  size_t off_dtab = 0, dtab_bytes = 0;      // direct-address table (overlays key buffer B when it fits)
  size_t off_gate = 0;                      // witness gate word (direct.cu k_witness_gate)
  size_t off_ctrl2 = 0;                     // second control block (overlapped direct pipeline)
  size_t off_allsegs = 0;                   // every chunk's segment table (overlapped direct pipeline)
  size_t max_segs = 0;
  // scratch offsets
  size_t off_a = 0, off_b = 0, off_lb = 0, off_ff = 0, off_lf = 0, off_segs = 0, off_ctrl = 0, off_res = 0, off_rh = 0;
  size_t rh_bytes = 0, off_xch = 0;
  size_t off_tparts = 0, off_tstore = 0;    // bucket-table detect: partial tables
  uint32_t table_ctas = 0;
  size_t lb_bytes = 0, total = 0, stage_bytes = 0;
};

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// a chunk's segment table, then its stride-compression table (Chunk::pcomp): staged
// and uploaded together
size_t pcomp_off(const Chunk& ch) { return align_up(std::max<size_t>(1, ch.segs.size()) * sizeof(MapcSeg), 64); }
size_t seg_blob(const Chunk& ch) { return pcomp_off(ch) + ch.pcomp.size() * sizeof(unsigned long long); }
// the direct table of a chunk: stride-compressed with the specialised generate
bool comp_on(const Chunk& ch, int gen_mode) { return ch.comp_ok && ch.cell_bytes == 2 && gen_mode == 1; }
uint64_t dcells(const Chunk& ch, int gen_mode) { return comp_on(ch, gen_mode) ? ch.comp_cells : ch.cells; }

// NVTX range for the host-side stages (visible in nsys / ncu timelines)
struct NvtxRange {
  explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Host-side CUDA resources recycled across programs: a caller that compiles a
// fresh program per call (the e2e path: MAP text in, verdict out) would otherwise
// pay cudaMallocHost, stream and event creation (and their destruction) on every
// call.  Never freed: the process's exit releases them (no CUDA calls from static
// destructors).
struct ResourcePool {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> pinned;
  std::vector<std::pair<int, cudaStream_t>> streams;       // (device, non-blocking stream)
  std::vector<std::pair<int, cudaEvent_t>> timing, sync;   // (device, event)
};
ResourcePool& pool() {
  static ResourcePool* p = new ResourcePool();
  return *p;
}
void* pool_pinned(size_t bytes, size_t* got) {
  {
    ResourcePool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    size_t best = P.pinned.size();
    for (size_t i = 0; i < P.pinned.size(); ++i)
      if (P.pinned[i].second >= bytes && (best == P.pinned.size() || P.pinned[i].second < P.pinned[best].second))
        best = i;
    if (best < P.pinned.size()) {
      void* r = P.pinned[best].first;
      *got = P.pinned[best].second;
      P.pinned.erase(P.pinned.begin() + best);
      return r;
    }
  }
  void* r = nullptr;
  if (cudaMallocHost(&r, bytes) != cudaSuccess) return nullptr;
  *got = bytes;
  return r;
}
void pool_release_pinned(void* ptr, size_t bytes) {
  if (!ptr) return;
  ResourcePool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  P.pinned.emplace_back(ptr, bytes);
}
cudaError_t pool_stream(int dev, cudaStream_t* out) {
  {
    ResourcePool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    for (size_t i = 0; i < P.streams.size(); ++i)
      if (P.streams[i].first == dev) {
        *out = P.streams[i].second;
        P.streams.erase(P.streams.begin() + i);
        return cudaSuccess;
      }
  }
  return cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
}
cudaError_t pool_event(int dev, bool timing, cudaEvent_t* out) {
  {
    ResourcePool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    auto& v = timing ? P.timing : P.sync;
    for (size_t i = v.size(); i-- > 0;)
      if (v[i].first == dev) {
        *out = v[i].second;
        v.erase(v.begin() + i);
        return cudaSuccess;
      }
  }
  return timing ? cudaEventCreate(out) : cudaEventCreateWithFlags(out, cudaEventDisableTiming);
}

}  // namespace

struct map_program {
  mapc::Compiled C;
  uint64_t plan_for = ~0ull;
  Plan plan;
  bool have_witness = false;
  map_witness wit{};
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* last_lookback = nullptr;
  uint64_t epoch = 0;
  int device = -1;
  std::string last_error;
  std::vector<cudaEvent_t> events;   // pool for per-kernel timing
  int events_dev = -1;               // device of events and sync_events
  // overlapped direct pipeline: a library-owned side stream (scan, clear and
  // witness of chunk k run there while chunk k+1's generate runs on the caller's
  // stream) and its ordering events
  cudaStream_t side = nullptr;
  int side_dev = -1;
  cudaStream_t side2 = nullptr;      // the table clears when three tables rotate (MAPC_TABLES=3)
  int side2_dev = -1;
  std::vector<cudaEvent_t> sync_events;
  // CUDA graph of a whole run's launches, captured on the second identical call
  // (same plan, flags, scratch, stream, shard) and replayed after that
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap = nullptr;        // capture stream (the caller's may be the legacy default stream)
  int cap_dev = -1;
  std::string gkey, glast_key;
  uint32_t g_launches = 0;
  uint64_t default_cap_cache = 0;    // default_cap(), computed once
  uint64_t g_h2d = 0;
  map_kernel_stats g_stats{};
  std::vector<uint64_t> g_marks;     // profiled graph: (kind, event, event) per timed launch
  // timing and sync events, streams and the staging buffer go back to the pool
  void release_events() {
    ResourcePool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    for (cudaEvent_t e : events) P.timing.emplace_back(events_dev, e);
    for (cudaEvent_t e : sync_events) P.sync.emplace_back(events_dev, e);
    events.clear();
    sync_events.clear();
  }
  ~map_program() {
    if (gexec) cudaGraphExecDestroy(gexec);
    release_events();
    ResourcePool& P = pool();
    std::lock_guard<std::mutex> g(P.mu);
    if (side) P.streams.emplace_back(side_dev, side);
    if (side2) P.streams.emplace_back(side2_dev, side2);
    if (cap) P.streams.emplace_back(cap_dev, cap);
  }
};

namespace {

struct PhaseInfo {
  uint32_t phase;
  std::vector<size_t> inst;
  uint64_t per_block = 0;
  uint64_t ilo = ~0ull, ihi = 0;
  size_t ops = 0;
};

// Cluster units are opt-in (MAPC_CLUSTER=1): measured 2.7-9x SLOWER than the
// L2-resident direct tables on configs 4b/4c/4d.
bool cluster_units_enabled() {
  static const bool on = [] { const char* e = getenv("MAPC_CLUSTER"); return e && e[0] == '1'; }();
  return on;
}

bool layout_fits(const mapc::Compiled& C, uint32_t ph_span, uint64_t nb, uint64_t ilo, uint64_t ihi, MapcLayout* out) {
  MapcLayout L{};
  L.w_phase = bits_for(ph_span);
  L.w_array = bits_for(C.ast.arrays.size() - 1);
  L.w_block = bits_for(nb - 1);
  L.w_index = ilo <= ihi ? bits_for(ihi - ilo) : 0;
  L.w_tid = C.w_tid;
  L.pay_bits = C.w_tid + 1;
  L.sort_bits = L.w_phase + L.w_array + L.w_block + L.w_index;
  L.n_passes = (L.sort_bits + 7) / 8;
  L.idx_lo = ilo <= ihi ? ilo : 0;
  L.tb = 0;
  L.sort_lo = L.pay_bits;
  if (L.sort_bits + L.pay_bits > 64) return false;
  if (L.sort_bits + 2 * L.w_tid + 2 > 64) return false;
  if (out) *out = L;
  return true;
}

MapcOp lower_op_for_mode(MapcOp op, bool u32) {
  const uint32_t code = op.code & MAPC_CODE_MASK;
  if (u32 && (code == VM_DIV || code == VM_MOD) && (op.code & MAPC_B_IMM) && op.imm != 0 && op.imm < (1ull << 32)) {
    MapcFastDiv f = mapc::make_fastdiv((uint32_t)op.imm);
    if (!f.pow2) {
      MapcOp r = op;
      r.code = (uint8_t)((code == VM_DIV ? VM_DIVM : VM_MODM) | (op.code & MAPC_A_IMM));
      r.imm = ((uint64_t)f.d << 32) | f.m;
      r.aux = f.s;
      return r;
    }
  }
  return op;
}

void emit_chunk(const mapc::Compiled& C, const std::vector<PhaseInfo>& ph, size_t i0, size_t i1, uint64_t b_lo,
                uint64_t b_hi, const MapcLayout& L, Chunk* out) {
  Chunk ch;
  ch.phase_lo = ph[i0].phase;
  ch.phase_hi = ph[i1 - 1].phase;
  ch.b_lo = b_lo;
  ch.b_hi = b_hi;
  ch.lay = L;
  const uint64_t B = C.n_threads;
  for (size_t i = i0; i < i1; ++i) {
    for (size_t ii : ph[i].inst) {
      const mapc::InstanceInfo& in = C.inst[ii];
      for (const mapc::GroupProg& g : in.groups) {
        const uint32_t pb = (uint32_t)ch.ops.size();
        {
          mapj::JitProgram jp{pb, g.n_levels, g.ops};
          const uint64_t inner = (g.tid_inner || g.n_levels == 0) ? B : g.trips[g.n_levels - 1];
          jp.inner_range = inner;
          jp.tid_inner = g.tid_inner;
          ch.jit.programs.push_back(std::move(jp));
        }
        for (const MapcOp& op : g.ops) {
          ch.ops.push_back(lower_op_for_mode(op, C.u32_mode));
          const uint32_t code = op.code & MAPC_CODE_MASK;
          auto use = [&](uint32_t r) { ch.nreg = std::max(ch.nreg, r + 1); };
          if (code != VM_EMIT && code != VM_ACT) use(op.dst);
          if (!(op.code & MAPC_A_IMM) && code != VM_MOVI) use(op.a);
          const bool has_b = code != VM_BAND && code != VM_LNOT && code != VM_MOVI && code != VM_ACT && code != VM_EMIT;
          if (has_b && !(op.code & MAPC_B_IMM)) use(op.b);
          if (code == VM_MADK || (code == VM_TRIP && !(op.aux & MAPC_AUX_CONST))) use(op.aux);
        }
        ch.nreg = std::max(ch.nreg, (uint32_t)MAPC_REG_K0 + g.n_levels);
        const uint32_t pe = (uint32_t)ch.ops.size();
        const uint64_t tpb = g.tuples_per_block;
        const uint64_t per_seg = std::max<uint64_t>(1, 0xFFFFFFFFull / tpb);
        for (uint64_t b = b_lo; b < b_hi; b += per_seg) {
          const uint64_t nb = std::min(per_seg, b_hi - b);
          MapcSeg s{};
          s.tuple_begin = ch.total_tuples;
          s.n_tuples = nb * tpb;
          s.tile_begin = ch.total_tiles;
          ch.total_tiles += (s.n_tuples + MAPC_GEN_TILE - 1) / MAPC_GEN_TILE;
          if (g.dense) {
            s.key_begin = ch.dense_total;
            ch.dense_total += s.n_tuples * g.n_emits;
          } else {
            ch.max_emits = std::max(ch.max_emits, g.n_emits);
          }
          s.key_hi = (uint64_t)(in.phase - ch.phase_lo) << (L.w_array + L.w_block + L.w_index);
          s.prog_begin = pb;
          s.prog_end = pe;
          s.n_levels = g.n_levels;
          s.b0 = (uint32_t)b;
          s.lb0 = (uint32_t)(b - b_lo);
          s.n_emits = g.n_emits;
          s.dense = g.dense ? 1 : 0;
          s.tid_inner = g.tid_inner ? 1 : 0;
          for (uint32_t l = 0; l < g.n_levels; ++l) s.trip_div[l] = mapc::make_fastdiv((uint32_t)g.trips[l]);
          s.tid_div = mapc::make_fastdiv((uint32_t)B);
          ch.total_tuples += s.n_tuples;
          ch.bound += s.n_tuples * g.n_emits;
          ch.segs.push_back(s);
        }
      }
    }
  }
  // stride compression of the direct table: per local phase, the largest 2^k such
  // that every site's (index - idx_lo) has the same residue modulo 2^k (the compiler's
  // known low bits, GroupProg::site_kb/kv)
  if (L.sort_bits <= 31) {                   // 32-bit cell indices only (the compressed path's arithmetic)
    const uint32_t nph = ch.phase_hi - ch.phase_lo + 1;
    const uint32_t WI = L.w_index, WAB = L.w_array + L.w_block;
    std::vector<int> k(nph, -1);                 // -1: no site yet
    std::vector<uint64_t> r(nph, 0);
    for (size_t i = i0; i < i1; ++i)
      for (size_t ii : ph[i].inst) {
        const mapc::InstanceInfo& in = C.inst[ii];
        const uint32_t q = in.phase - ch.phase_lo;
        for (const mapc::GroupProg& g : in.groups)
          for (size_t e = 0; e < g.site_kb.size(); ++e) {
            uint32_t kb = std::min<uint32_t>(g.site_kb[e], WI);
            const uint64_t rv = (g.site_kv[e] - L.idx_lo) & (kb >= 64 ? ~0ull : ((1ull << kb) - 1));
            if (k[q] < 0) {
              k[q] = (int)kb;
              r[q] = rv;
            } else {
              kb = std::min<uint32_t>(kb, (uint32_t)k[q]);
              const uint64_t diff = (rv ^ r[q]) & ((1ull << kb) - 1);
              if (diff) kb = std::min<uint32_t>(kb, (uint32_t)__builtin_ctzll(diff));
              k[q] = (int)kb;
              r[q] &= (1ull << kb) - 1;
            }
          }
      }
    uint64_t cells = 0;
    ch.pcomp.assign(2 * (size_t)nph, 0);
    for (uint32_t q = 0; q < nph; ++q) {
      const uint32_t sh = k[q] < 0 ? WI : (uint32_t)k[q];
      ch.pcomp[2 * q] = cells;
      ch.pcomp[2 * q + 1] = (unsigned long long)sh | (r[q] << 8);
      cells += (1ull << WAB) << (WI - sh);
    }
    ch.comp_cells = cells;
    // worth it when the table shrinks at least 2x; 32-bit cell indices, <= 64 phases
    ch.comp_ok = L.sort_bits <= 31 && nph <= 64 && cells * 2 <= (1ull << L.sort_bits);
    ch.jit.comp = ch.comp_ok;
  }
  *out = std::move(ch);
}

// Greedy plan: consecutive phases while the bound, the layout and the
// constant-memory budget allow; an oversized phase is split by block ranges.
map_status make_plan(const mapc::Compiled& C, uint64_t cap, Plan* P, std::string* why) {
  std::vector<PhaseInfo> ph;
  for (size_t i = 0; i < C.inst.size(); ++i) {
    const mapc::InstanceInfo& in = C.inst[i];
    if (ph.empty() || ph.back().phase != in.phase) {
      ph.emplace_back();
      ph.back().phase = in.phase;
    }
    PhaseInfo& p = ph.back();
    p.inst.push_back(i);
    p.per_block += in.bound_per_block;
    for (auto& g : in.groups) {
      if (g.has_emit) {
        p.ilo = std::min(p.ilo, g.index.lo);
        p.ihi = std::max(p.ihi, g.index.hi);
      }
      p.ops += g.ops.size();
    }
  }
  Plan out;
  const uint64_t G = C.n_blocks;
  size_t i = 0;
  while (i < ph.size()) {
    size_t j = i;
    uint64_t acc = 0, ilo = ~0ull, ihi = 0;
    size_t ops = 0;
    MapcLayout L{}, Lok{};
    while (j < ph.size()) {
      const unsigned __int128 nb = (unsigned __int128)ph[j].per_block * G;
      if ((unsigned __int128)acc + nb > cap) break;
      const uint64_t nlo = std::min(ilo, ph[j].ilo), nhi = std::max(ihi, ph[j].ihi);
      if (!layout_fits(C, ph[j].phase - ph[i].phase, G, nlo, nhi, &L)) break;
      if (ops + ph[j].ops > MAPC_MAX_OPS) break;
      // Keep the direct-address table of a chunk L2-sized (<= 64 MiB of u32
      // cells) once the chunk is big enough to amortise its fixed cost (>= 2^23
      // accesses): the table's atomics then mostly hit L2 (4a: 92 -> 121 G acc/s,
      // profiles/r1n_chunking.jsonl).
      // (Not for chunks that will run on chip -- per-(phase, block) units that fit
      // shared memory and fill the GPU, §5.13 -- which have no table at all.)
      const uint64_t unit_cell_bytes = C.w_tid <= MAPC_CW16_MAX_WT ? 2 : 4;
      const uint64_t unit_bytes = L.w_array + L.w_index < 24 ? (1ull << (L.w_array + L.w_index)) * unit_cell_bytes : ~0ull;
      const bool on_chip = (unit_bytes <= MAPC_UNIT_MAX_BYTES && G >= 2 * 148) ||
                           (cluster_units_enabled() && unit_bytes <= (uint64_t)MAPC_CLUSTER_MAX * MAPC_CLUSTER_CTA_BYTES);
      if (j > i && acc >= (1ull << 23) && L.sort_bits >= 24 && !on_chip) break;
      acc += (uint64_t)nb;
      ilo = nlo; ihi = nhi; ops += ph[j].ops;
      Lok = L;
      ++j;
    }
    if (j > i) {
      out.chunks.emplace_back();
      emit_chunk(C, ph, i, j, 0, G, Lok, &out.chunks.back());
      i = j;
      continue;
    }
    // one phase does not fit whole: split its blocks
    if (ph[i].ops > MAPC_MAX_OPS) { *why = "one phase needs more bytecode than __constant__ holds"; return MAP_E_RANGE; }
    if (ph[i].per_block > cap) { *why = "one (phase, block) unit exceeds the chunk capacity"; return MAP_E_NOMEM; }
    uint64_t nb = std::max<uint64_t>(1, cap / std::max<uint64_t>(ph[i].per_block, 1));
    while (nb > 1 && !layout_fits(C, 0, nb, ph[i].ilo, ph[i].ihi, nullptr)) nb /= 2;
    if (!layout_fits(C, 0, nb, ph[i].ilo, ph[i].ihi, &L)) {
      *why = "the (phase, array, block, index, tid) key of one unit exceeds 64 bits";
      return MAP_E_RANGE;
    }
    for (uint64_t b = 0; b < G; b += nb) {
      const uint64_t be = std::min(G, b + nb);
      MapcLayout Lb;
      layout_fits(C, 0, be - b, ph[i].ilo, ph[i].ihi, &Lb);
      out.chunks.emplace_back();
      emit_chunk(C, ph, i, i + 1, b, be, Lb, &out.chunks.back());
    }
    ++i;
  }
  // capacities and scratch layout
  uint64_t kcap = 1;
  size_t stage = 0;
  for (auto& ch : out.chunks) {
    kcap = std::max(kcap, ch.bound);
    out.max_segs = std::max(out.max_segs, ch.segs.size());
    ch.stage_ops = stage;
    stage += align_up(std::max<size_t>(1, ch.ops.size()) * sizeof(MapcOp), 64);
    ch.stage_segs = stage;
    stage += align_up(seg_blob(ch), 64);
  }
  size_t dtab = 0;
  for (auto& ch : out.chunks) {
    ch.lay.cap = kcap;
    ch.jit.lay = ch.lay;
    ch.jit.max_emits = ch.max_emits;
    // segments baked into the specialised kernels as literals (fields fold to
    // constants; otherwise every tile loads its segment from global memory)
    if (ch.segs.size() <= MAPC_JIT_BAKE_SEGS) ch.jit.segs = ch.segs;
    // direct-address table: 2^S cells.  Worth it when its estimated time --
    // a fixed ~25 us, the table written (clear) and read (scan) at ~6 TB/s, the
    // generate at ~1.5 ps per access -- beats the keys pipelines' (~40 us fixed,
    // >= ~50 ps per access at these sizes incl. their passes and launches;
    // DESIGN.md §6, profiles/r1j_configs.jsonl).  Its size is bounded by key
    // buffer B (which it overlays) or 1 GiB.
    const uint32_t S = ch.lay.sort_bits;
    static const bool cell16 = [] { const char* e = getenv("MAPC_CELL16"); return !(e && e[0] == '0'); }();
    ch.cell_bytes = cell16 && ch.lay.w_tid <= MAPC_CW16_MAX_WT ? 2u : 2 * ch.lay.w_tid + 1 <= 32 ? 4u : 8u;
    if (S <= 40) {
      ch.cells = 1ull << S;
      const uint64_t tb = ch.cells * ch.cell_bytes;
      const double n = (double)std::max<uint64_t>(ch.bound, 1);
      const bool cheap = 25e-6 + 2.0 * (double)tb / 6e12 + 1.5e-12 * n <= 40e-6 + 50e-12 * n;
      const bool fits = tb <= kcap * 8 || tb <= (1ull << 30);
      ch.direct_ok = cheap && fits;
      if (ch.direct_ok) dtab = std::max<size_t>(dtab, tb);
    }
    // On-chip units: the cells of one (phase, block) -- (array, index) -- fit a
    // shared-memory table, and the chunk has enough units to fill the GPU (or is
    // small), so one CTA per unit does generate + fold + scan without HBM.
    {
      static const bool unit_env = [] { const char* e = getenv("MAPC_UNIT"); return !(e && e[0] == '0'); }();
      const bool cluster_env = cluster_units_enabled();
      const uint32_t wu = ch.lay.w_array + ch.lay.w_index;
      const uint64_t n_units = (uint64_t)(ch.phase_hi - ch.phase_lo + 1) * (ch.b_hi - ch.b_lo);
      const uint64_t ubytes = wu < 40 ? (1ull << wu) * ch.cell_bytes : ~0ull;
      // one CTA's shared memory, or a cluster of up to 16 CTAs (<= 192 KB each)
      uint32_t K = 1;
      if (ubytes > MAPC_UNIT_MAX_BYTES) {
        K = 2;
        while (K < MAPC_CLUSTER_MAX && ubytes / K > MAPC_CLUSTER_CTA_BYTES) K *= 2;
      }
      const bool fits = ubytes <= MAPC_UNIT_MAX_BYTES ||
                        (cluster_env && ubytes / K <= MAPC_CLUSTER_CTA_BYTES && ubytes % K == 0);
      ch.unit_ok = unit_env && ch.cell_bytes <= 4 && wu < 24 && fits && ch.segs.size() <= MAPC_UNIT_MAX_SEGS &&
                   (n_units * K >= 2 * 148 || ch.bound <= (1ull << 20) || K > 1) && ch.bound > 0;
      if (ch.unit_ok) {
        ch.jit.unit_segs = ch.segs;
        ch.jit.n_blocks = ch.b_hi - ch.b_lo;
        ch.jit.unit_cluster = K;
        ch.jit.unit_threads = K > 1 ? MAPC_CLUSTER_THREADS : MAPC_GEN_THREADS;
        ch.unit_smem = K > 1 ? ubytes / K : 0;
      }
    }
  }
  out.cap = kcap;
  const uint64_t sort_tiles = (kcap + mapc_sort_tile() - 1) / mapc_sort_tile();
  const uint64_t det_tiles = std::max<uint64_t>((kcap + mapc_detect_tile() - 1) / mapc_detect_tile(),
                                                MAPC_DETECT_MAX_UNITS);
  size_t off = 0;
  out.off_a = off; off += align_up(kcap * 8 + 64);     // + slack: bulk copies round up to 16 B
  out.off_b = off; off += align_up(kcap * 8 + 64);
  out.lb_bytes = sort_tiles * MAPC_RADIX * 8;
  out.off_lb = off; off += align_up(out.lb_bytes);
  out.off_ff = off; off += align_up(det_tiles * sizeof(MapcSegState));
  out.off_lf = off; off += align_up(det_tiles * sizeof(MapcSegState));
  {
    size_t blob = 0;
    for (auto& ch : out.chunks) blob = std::max(blob, seg_blob(ch));
    out.off_segs = off; off += align_up(blob);
  }
  out.off_ctrl = off; off += align_up(sizeof(MapcCtrl));
  out.off_res = off; off += align_up(std::max<size_t>(1, out.chunks.size()) * sizeof(MapcChunkResult));
  out.rh_bytes = (size_t)MAPC_MAX_PASSES * MAPC_MAX_RANGES * MAPC_RADIX * 4;
  out.off_rh = off; off += align_up(out.rh_bytes);
  out.off_xch = off; off += align_up(2 * 64 * sizeof(unsigned long long));   // exchange counts + cursors
  out.table_ctas = (uint32_t)std::min<uint64_t>(MAPC_TABLE_MAX_CTAS, (kcap + mapc_table_tile() - 1) / mapc_table_tile());
  out.off_tparts = off; off += align_up((size_t)2 * out.table_ctas * sizeof(MapcTablePart));
  out.off_tstore = off; off += align_up((size_t)2 * out.table_ctas * MAPC_TABLE_WORDS * 4);
  out.off_gate = off; off += align_up(64);
  out.off_ctrl2 = off; off += align_up(sizeof(MapcCtrl));
  out.off_allsegs = off;
  for (auto& ch : out.chunks) {
    ch.dev_segs = off - out.off_allsegs;
    off += align_up(seg_blob(ch));
  }
  out.dtab_bytes = dtab;
  if (dtab <= kcap * 8) {
    out.off_dtab = out.off_b;                 // the direct path never touches key buffer B
  } else {
    out.off_dtab = off; off += align_up(dtab);
  }
  out.total = off;
  out.stage_bytes = stage + align_up(std::max<size_t>(1, out.chunks.size()) * sizeof(MapcChunkResult), 64);
  *P = std::move(out);
  return MAP_OK;
}

// Detect path of a chunk (map_exec.flags, MAP_DETECT_*): the full LSD sort +
// segmented scan, or the partial sort + bucket tables (table.cu), which needs
// the keys to be dense enough in sf space that a bucket of 2^tb cells holds
// about a tile of keys or more.
MapcLayout effective_layout(const Chunk& ch, uint32_t flags, uint64_t n_keys = ~0ull) {
  const uint64_t nk = n_keys == ~0ull ? ch.bound : n_keys;
  MapcLayout L = ch.lay;
  const uint32_t sel = flags & MAP_DETECT_MASK;
  bool table = false;
  if (sel == MAP_DETECT_TABLE) {
    table = true;
  } else if (sel == MAP_DETECT_AUTO || sel == MAP_DETECT_DIRECT || sel == MAP_DETECT_UNIT) {
    const uint32_t S = L.sort_bits;
    table = nk >= (1ull << 16) && (S <= 1 || nk >= (1ull << (S - 1)));
  }
  if (table) {
    L.tb = std::min<uint32_t>(MAPC_TABLE_BITS_MAX, L.sort_bits);
    L.n_passes = (L.sort_bits - L.tb + 7) / 8;
    L.sort_lo = L.pay_bits + L.tb;
  }
  return L;
}

// Sort-free direct-address detect for this chunk (MAP_DETECT_AUTO or
// MAP_DETECT_DIRECT, and the chunk's table qualifies; direct.cu).
bool use_direct(const Chunk& ch, uint32_t flags) {
  const uint32_t sel = flags & MAP_DETECT_MASK;
  return (sel == MAP_DETECT_AUTO || sel == MAP_DETECT_DIRECT || sel == MAP_DETECT_UNIT) && ch.direct_ok;
}

// On-chip per-unit tables for this chunk (MAP_DETECT_AUTO or MAP_DETECT_UNIT,
// the specialised generate, and the chunk's units fit; MAPC_MODE_UNIT).
bool use_unit(const Chunk& ch, uint32_t flags, int gen_mode) {
  const uint32_t sel = flags & MAP_DETECT_MASK;
  return gen_mode == 1 && ch.unit_ok && (sel == MAP_DETECT_AUTO || sel == MAP_DETECT_UNIT);
}

// Whether a radix pass also accumulates the next pass's range table (k_rsweep
// RED_NEXT): on the bucket-table path the digits are high sort-field bits, which
// dense MAPs keep warp-uniform; the kernel falls back by itself otherwise.
int red_next(const MapcLayout& L) {
  static const bool off = getenv("MAPC_RED_NEXT") && getenv("MAPC_RED_NEXT")[0] == '0';
  return (!off && L.tb > 0) ? 1 : 0;
}

void put_diag(const std::string& d, char* diag, size_t cap) {
  if (!diag || !cap) return;
  size_t n = std::min(cap - 1, d.size());
  std::memcpy(diag, d.data(), n);
  diag[n] = 0;
}

map_status ensure_plan(map_program* p, uint64_t cap) {
  if (p->plan_for == cap) return MAP_OK;
  Plan P;
  map_status st = make_plan(p->C, cap, &P, &p->last_error);
  if (st != MAP_OK) return st;
  p->plan = std::move(P);
  p->plan_for = cap;
  return MAP_OK;
}

uint64_t default_cap(const map_program* p) {
  // default chunk: up to 2^30 keys (16 GiB of ping-pong buffers), never less
  // than the largest single (phase, block) unit; a plan of 2^25..2^31 accesses
  // is cut in (at least) two chunks so that the direct pipeline can overlap one
  // chunk's table scan with the other's generate (3b: 197 -> 218 G acc/s,
  // profiles/r1r_chunking.jsonl)
  if (p->default_cap_cache) return p->default_cap_cache;
  uint64_t want = std::min<uint64_t>(p->C.max_accesses, 1ull << 30);
  if (p->C.max_accesses >= (1ull << 25) && p->C.max_accesses <= (1ull << 31)) {
    // ... unless every chunk of the uncut plan runs on chip (unit mode: no table
    // scan to overlap, and one chunk saves its fixed launches; 3a 0.231 -> ms)
    bool all_unit = false;
    {
      Plan whole;
      std::string why;
      const uint64_t full = std::max<uint64_t>({want, p->C.max_unit, 1});
      if (make_plan(p->C, full, &whole, &why) == MAP_OK && !whole.chunks.empty()) {
        all_unit = true;
        for (const Chunk& ch : whole.chunks) all_unit = all_unit && ch.unit_ok;
      }
    }
    if (!all_unit) want = std::min<uint64_t>(want, (p->C.max_accesses + 1) / 2);
  }
  const_cast<map_program*>(p)->default_cap_cache = std::max<uint64_t>({want, p->C.max_unit, 1});
  return p->default_cap_cache;
}

// Default chunk capacity for a job sharded over `world` ranks: at least two
// chunks per rank where the plan's units allow it (every rank busy, and each
// rank can overlap one chunk's table scan with the next one's generate).
uint64_t default_cap_world(const map_program* p, uint32_t world) {
  const uint64_t base = default_cap(p);
  if (world <= 1) return base;
  const uint64_t want = (p->C.max_accesses + 2ull * world - 1) / (2ull * world);
  return std::max<uint64_t>({std::min(base, want), p->C.max_unit, 1});
}

// The chunks rank `rank` of `world` processes: a contiguous range, split where
// the running sum of chunk bounds crosses rank/world of the total (chunk c goes
// to the rank owning the midpoint of its bound), so ranks get equal work and
// each rank's chunks stay consecutive (the overlapped direct pipeline pairs
// neighbours).  Ranks beyond the chunk count get none.
std::vector<size_t> rank_chunks(const Plan& P, uint32_t rank, uint32_t world) {
  std::vector<size_t> mine;
  if (world <= 1) {
    for (size_t c = 0; c < P.chunks.size(); ++c) mine.push_back(c);
    return mine;
  }
  unsigned __int128 total = 0;
  for (const Chunk& ch : P.chunks) total += std::max<uint64_t>(ch.bound, 1);
  unsigned __int128 run = 0;
  for (size_t c = 0; c < P.chunks.size(); ++c) {
    const uint64_t b = std::max<uint64_t>(P.chunks[c].bound, 1);
    const unsigned __int128 mid2 = 2 * run + b;                      // 2 x midpoint
    uint32_t owner = (uint32_t)(mid2 * world / (2 * total));
    if (P.chunks.size() <= world) owner = (uint32_t)c;               // one chunk per rank
    if (owner >= world) owner = world - 1;
    if (owner == rank) mine.push_back(c);
    run += b;
  }
  return mine;
}

#define CK(expr)                                           \
  do {                                                     \
    cudaError_t e_ = (expr);                               \
    if (e_ != cudaSuccess) {                               \
      p->last_error = std::string(#expr) + ": " + cudaGetErrorString(e_); \
      return MAP_E_CUDA;                                   \
    }                                                      \
  } while (0)

void decode(const mapc::Compiled& C, const Chunk& ch, uint64_t w, map_witness* out) {
  const MapcLayout& L = ch.lay;
  const uint32_t wt = L.w_tid;
  const uint64_t tm = wt ? ((1ull << wt) - 1) : 0;
  const uint64_t sf = (2 * wt + 2) >= 64 ? 0 : (w >> (2 * wt + 2));
  out->tid_lo = (uint32_t)((w >> (wt + 2)) & tm);
  out->tid_hi = (uint32_t)((w >> 2) & tm);
  out->kind_lo = (uint8_t)((w >> 1) & 1);
  out->kind_hi = (uint8_t)(w & 1);
  auto field = [](uint64_t v, uint32_t lo, uint32_t bits) -> uint64_t {
    if (bits == 0) return 0;
    return (v >> lo) & ((bits >= 64) ? ~0ull : ((1ull << bits) - 1));
  };
  out->index = L.idx_lo + field(sf, 0, L.w_index);
  out->block = (uint32_t)(ch.b_lo + field(sf, L.w_index, L.w_block));
  out->array = (uint32_t)field(sf, L.w_index + L.w_block, L.w_array);
  out->phase = ch.phase_lo + (uint32_t)field(sf, L.w_index + L.w_block + L.w_array, L.w_phase);
  out->array_name = C.ast.arrays[out->array].c_str();
}

bool wit_less(const map_witness& a, const map_witness& b) {
  auto ta = std::make_tuple(a.phase, a.array, a.block, a.index, a.tid_lo, a.tid_hi, a.kind_lo, a.kind_hi);
  auto tb = std::make_tuple(b.phase, b.array, b.block, b.index, b.tid_lo, b.tid_hi, b.kind_lo, b.kind_hi);
  return ta < tb;
}

}  // namespace

extern "C" {

const char* map_status_str(map_status s) {
  switch (s) {
    case MAP_OK: return "ok";
    case MAP_E_PARSE: return "parse error";
    case MAP_E_SCOPE: return "scope error";
    case MAP_E_BARRIER: return "barrier placement error";
    case MAP_E_RANGE: return "range error";
    case MAP_E_ARITH: return "division by zero";
    case MAP_E_CUDA: return "CUDA error";
    case MAP_E_COMM: return "communication error";
    case MAP_E_ARG: return "bad argument";
    case MAP_E_NOMEM: return "scratch too small";
  }
  return "unknown status";
}

map_status map_compile(const char* src, size_t len, const map_instance* inst, map_program** out, char* diag,
                       size_t diag_cap) {
  if (!src || !inst || !out) return MAP_E_ARG;
  if (inst->n_params && (!inst->param_names || !inst->param_values)) return MAP_E_ARG;
  try {
    std::vector<std::string> names;
    std::vector<uint64_t> values;
    for (uint32_t i = 0; i < inst->n_params; ++i) {
      if (!inst->param_names[i]) return MAP_E_ARG;
      names.emplace_back(inst->param_names[i]);
      values.push_back(inst->param_values[i]);
    }
    std::unique_ptr<map_program> p(new map_program());
    p->C = mapc::compile_map(std::string(src, len), inst->grid, inst->block, names, values);
    *out = p.release();
    put_diag("", diag, diag_cap);
    return MAP_OK;
  } catch (const mapc::CompileError& e) {
    put_diag(e.msg, diag, diag_cap);
    return (map_status)e.status;
  } catch (const std::bad_alloc&) {
    put_diag("out of host memory", diag, diag_cap);
    return MAP_E_NOMEM;
  } catch (...) {
    put_diag("internal error", diag, diag_cap);
    return MAP_E_ARG;
  }
}

map_status map_info_get(const map_program* p, map_info* out) {
  if (!p || !out) return MAP_E_ARG;
  out->n_phases = p->C.n_phases;
  out->n_arrays = (uint32_t)p->C.ast.arrays.size();
  out->n_instances = (uint32_t)p->C.inst.size();
  out->n_groups = p->C.n_groups;
  out->max_accesses = p->C.max_accesses;
  out->max_unit_accesses = p->C.max_unit;
  out->u32_mode = p->C.u32_mode ? 1 : 0;
  out->bytecode_ops = p->C.total_ops;
  return MAP_OK;
}

size_t map_scratch_bytes(const map_program* cp, uint64_t chunk_max_accesses) {
  if (!cp) return 0;
  map_program* p = const_cast<map_program*>(cp);
  const uint64_t cap = chunk_max_accesses ? chunk_max_accesses : default_cap(p);
  if (ensure_plan(p, cap) != MAP_OK) return 0;
  return p->plan.total;
}

map_status map_check_races(map_program* p, const map_exec* ex, map_result* out) {
  if (!p || !ex || !out) return MAP_E_ARG;
  NvtxRange nvtx_run("map_check_races");
  p->have_witness = false;
  const uint32_t world = ex->world ? ex->world : 1;
  const uint32_t rank = ex->rank;
  if (rank >= world) return MAP_E_ARG;
  const uint64_t cap = ex->chunk_max_accesses ? ex->chunk_max_accesses : default_cap_world(p, world);
  map_status st = ensure_plan(p, cap);
  if (st != MAP_OK) return st;
  Plan& P = p->plan;
  if (!ex->scratch || ex->scratch_bytes < P.total) {
    p->last_error = "scratch too small: need " + std::to_string(P.total) + " bytes";
    return MAP_E_NOMEM;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    p->last_error = "no CUDA device";
    return MAP_E_CUDA;
  }
  CK(cudaSetDevice(ex->device));
  int n_sms = 0;
  CK(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, ex->device));
  cudaStream_t s = (cudaStream_t)ex->stream;
  if (p->pinned_bytes < P.stage_bytes) {
    // a captured graph reads the staging buffer: it dies with it
    if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
    p->gkey.clear();
    p->glast_key.clear();
    pool_release_pinned(p->pinned, p->pinned_bytes);
    p->pinned = nullptr;
    p->pinned_bytes = 0;
    size_t got = 0;
    p->pinned = pool_pinned(P.stage_bytes, &got);
    if (!p->pinned) {
      p->last_error = "cudaMallocHost failed";
      return MAP_E_CUDA;
    }
    p->pinned_bytes = got;
  }
  unsigned char* stage = (unsigned char*)p->pinned;
  for (auto& ch : P.chunks) {
    if (!ch.ops.empty()) std::memcpy(stage + ch.stage_ops, ch.ops.data(), ch.ops.size() * sizeof(MapcOp));
    if (!ch.segs.empty()) std::memcpy(stage + ch.stage_segs, ch.segs.data(), ch.segs.size() * sizeof(MapcSeg));
    if (!ch.pcomp.empty())
      std::memcpy(stage + ch.stage_segs + pcomp_off(ch), ch.pcomp.data(), ch.pcomp.size() * sizeof(unsigned long long));
  }
  MapcChunkResult* host_res = (MapcChunkResult*)(stage + P.stage_bytes -
                                                 align_up(std::max<size_t>(1, P.chunks.size()) * sizeof(MapcChunkResult), 64));
  unsigned char* base = (unsigned char*)ex->scratch;
  auto* bufA = (unsigned long long*)(base + P.off_a);
  auto* bufB = (unsigned long long*)(base + P.off_b);
  auto* lookback = (unsigned long long*)(base + P.off_lb);
  auto* ff = (MapcSegState*)(base + P.off_ff);
  auto* lf = (MapcSegState*)(base + P.off_lf);
  auto* segs = (MapcSeg*)(base + P.off_segs);
  auto* ctrl = (MapcCtrl*)(base + P.off_ctrl);
  auto* res = (MapcChunkResult*)(base + P.off_res);
  auto* rhist = (unsigned int*)(base + P.off_rh);
  auto* tparts = (MapcTablePart*)(base + P.off_tparts);
  auto* tstore = (uint32_t*)(base + P.off_tstore);
  static int sort_mode = -1;     // 1 = static-range passes (default), 0 = decoupled look-back onesweep
  if (sort_mode < 0) {
    const char* e = getenv("MAPC_SORT");
    sort_mode = (e && std::string(e) == "onesweep") ? 0 : 1;
  }
  const int G = mapc_rsweep_ranges(n_sms);
  // generate path: NVRTC-specialised kernels for large plans (compile cost
  // amortised), the bytecode VM otherwise (map_exec.flags, MAP_GEN_*).
  const uint32_t gsel = ex->flags & 3u;
  // (AUTO: the NVRTC compile, once per process, is amortised over plans of
  // >= 2^23 accesses needing at most 64 distinct kernels -- 4a/4b/4d run
  // 1.3-1.4x faster than on the VM, profiles/r1q_gen_vm_jit.jsonl; chunks that
  // differ only in unbaked data share a kernel (5a at T = 128: 128 chunks, 2
  // kernels); a plan needing thousands of distinct kernels stays on the VM)
  if (gsel == MAP_GEN_AUTO && P.jit_distinct == 0 && p->C.max_accesses >= (1ull << 23)) {
    std::vector<mapj::JitChunk> jc;
    jc.reserve(P.chunks.size());
    for (auto& ch : P.chunks) jc.push_back(ch.jit);
    P.jit_distinct = mapj::distinct_kernels(jc, p->C.u32_mode);
  }
  const int gen_mode = gsel == MAP_GEN_VM    ? 0
                       : gsel == MAP_GEN_JIT ? 1
                                             : (p->C.max_accesses >= (1ull << 23) && P.jit_distinct <= 64 ? 1 : 0);
  const std::vector<size_t> mine = rank_chunks(P, rank, world);   // this rank's chunks
  if (gen_mode == 1 && !mine.empty()) {
    // the kernels this run needs, per mode: keys (sort / table detect), direct +
    // filter (direct detect), for this rank's chunks only
    std::vector<char> want[5];
    bool any[5] = {false, false, false, false, false};
    for (uint32_t m = 0; m < 5; ++m) want[m].assign(P.chunks.size(), 0);
    for (size_t c : mine) {
      const bool un = use_unit(P.chunks[c], ex->flags, 1);
      const bool d = !un && use_direct(P.chunks[c], ex->flags);
      for (uint32_t m = 0; m < 5; ++m) {
        const bool w = un  ? (m == MAPC_MODE_UNIT || m == MAPC_MODE_UNITF)
                       : d ? (m == MAPC_MODE_DIRECT || m == MAPC_MODE_FILTER)
                           : m == MAPC_MODE_KEYS;
        const bool have = P.jit[m].kernels.size() == P.chunks.size() && P.jit[m].kernels[c] != nullptr;
        if (w && !have) { want[m][c] = 1; any[m] = true; }
      }
    }
    std::vector<mapj::JitChunk> jc;
    std::vector<uint32_t> cb;
    for (auto& ch : P.chunks) {
      jc.push_back(ch.jit);
      cb.push_back(ch.cell_bytes);
    }
    std::vector<std::thread> builders;
    std::string logs[5];
    int rcs[5] = {0, 0, 0, 0, 0};
    for (uint32_t m = 0; m < 5; ++m)
      if (any[m])
        builders.emplace_back(
            [&, m]() { rcs[m] = mapj::build_module(jc, p->C.u32_mode, m, cb, want[m], &P.jit[m], &logs[m]); });
    for (auto& t : builders) t.join();
    for (uint32_t m = 0; m < 5; ++m)
      if (rcs[m] != 0) {
        p->last_error = "specialised generate: " + logs[m];
        return MAP_E_CUDA;
      }
  }
  uint32_t passes_total = 0;
  for (auto& ch : P.chunks) passes_total += effective_layout(ch, ex->flags).n_passes;
  unsigned char* const dtab = base + P.off_dtab;
  auto* gate = (uint32_t*)(base + P.off_gate);
  if (p->last_lookback != (void*)lookback || p->device != ex->device || p->epoch + passes_total >= 0xFFFF) {
    CK(cudaMemsetAsync(lookback, 0, P.lb_bytes, s));
    p->epoch = 0;
    p->last_lookback = lookback;
    p->device = ex->device;
  }
  // events: 2 per timed launch group + 2 for the whole run
  const bool prof = ex->stats != nullptr;
  size_t need_ev = 2 + (prof ? mine.size() * (2 * (8 + MAPC_MAX_PASSES)) : 0);
  if (p->events_dev != ex->device) {   // events belong to the device current at creation
    if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; p->gkey.clear(); }
    p->release_events();
    p->events_dev = ex->device;
  }
  while (p->events.size() < need_ev) {
    cudaEvent_t e;
    CK(pool_event(ex->device, true, &e));
    p->events.push_back(e);
  }
  struct Mark { int kind; size_t e0, e1; };
  std::vector<Mark> marks;
  size_t ev = 2;
  uint32_t launches = 0;
  map_kernel_stats st_acc{};
  // per-launch timing events go to the stream the run is enqueued on (the caller's,
  // or the capture stream); inside a capture they become event-record nodes of the
  // graph (cudaEventRecordExternal), so a profiled run replays as a graph too
  cudaStream_t rec_s = s;
  bool capturing = false;
  auto rec = [&](size_t e, cudaStream_t st) {
    cudaEventRecordWithFlags(p->events[e], st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  };
  const bool gen_only = (ex->flags & MAP_EXEC_PROFILE_GENERATE) != 0;
  const bool sampled = gen_only && (ex->flags & MAP_EXEC_PROFILE_SAMPLED) != 0;
  size_t chunk_pos = 0;                              // position of the chunk being enqueued (sampling)
  auto timed = [&](int kind) {
    return prof && (!gen_only || kind == MAP_K_GENERATE || kind == MAP_K_DIRECT || kind == MAP_K_UNIT) &&
           (!sampled || chunk_pos % 4 == 2);
  };
  auto begin = [&](int kind) -> size_t {
    ++launches;
    st_acc.launches[kind]++;
    if (!timed(kind)) return 0;
    rec(ev, rec_s);
    st_acc.timed[kind]++;
    marks.push_back({kind, ev, ev + 1});
    ev += 2;
    return ev - 1;
  };
  auto end = [&](size_t e1) {
    if (prof && e1) rec(e1, rec_s);
  };
  auto begin_on = [&](int kind, cudaStream_t st) -> size_t {   // same, on another stream
    ++launches;
    st_acc.launches[kind]++;
    if (!timed(kind)) return 0;
    rec(ev, st);
    st_acc.timed[kind]++;
    marks.push_back({kind, ev, ev + 1});
    ev += 2;
    return ev - 1;
  };
  auto end_on = [&](size_t e1, cudaStream_t st) {
    if (prof && e1) rec(e1, st);
  };
  uint64_t h2d = 0;
  // Everything the run enqueues between the two timing events.  Without
  // per-kernel timing, the second identical call captures it into a CUDA graph
  // and later calls replay that graph (one launch instead of ~8 per chunk;
  // MAPC_GRAPHS=0 disables).
  auto enqueue = [&](cudaStream_t s) -> map_status {   // s: the caller's stream, or the capture stream
  CK(cudaMemsetAsync(gate, 0xFF, sizeof(uint32_t), s));
  // Overlapped direct pipeline: the direct generate is bound
  // by L2 atomics, not HBM, so chunk k's table scan + clear and witness run on a
  // library-owned side stream while chunk k+1's generate runs on the caller's
  // stream (two tables inside key buffer B, two control blocks, every chunk's
  // segment table resident).  The generate leaves room on every SM for the
  // side kernels' CTAs.  MAPC_OVERLAP=0 restores the sequential pipeline.
  static const int ovl_env = [] { const char* e = getenv("MAPC_OVERLAP"); return e ? atoi(e) : 1; }();
  // CTAs/SM of the generate and of the side stream's kernels: 8 / 4 when the
  // generate is row-jammed (fewer, heavier threads; profiles/r2zd_overlap_sweep.jsonl),
  // 12 / 3 otherwise (profiles/r2o_overlap_ctas_sweep.jsonl); the env overrides both
  static const int ovl_gen_env = [] { const char* e = getenv("MAPC_OVL_GEN_CTAS"); return e ? atoi(e) : 0; }();
  static const int ovl_side_env = [] { const char* e = getenv("MAPC_OVL_SIDE_CTAS"); return e ? atoi(e) : 0; }();
  bool jammed = false;
  for (size_t c : mine) jammed = jammed || mapj::jam_active(P.chunks[c].jit, P.chunks[c].cell_bytes);
  int ovl_gen_ctas = ovl_gen_env ? ovl_gen_env : jammed ? 8 : 12;
  const int ovl_side_ctas = ovl_side_env ? ovl_side_env : jammed ? 4 : 3;
  const size_t tab_stride = align_up(P.dtab_bytes);
  // tables in rotation: 2 (chunk k's scan then its clear for chunk k+2, both on the
  // side stream), or 3 (MAPC_TABLES=3: the clear of chunk k's table for chunk k+3 on
  // a second side stream, concurrent with chunk k+1's scan)
  // (default: 3 with the row-jammed generate, whose side stream is the critical path
  // -- profiles/r2zl_tables2.jsonl: 5a 1632 -> 1689 G acc/s, clears at 2 CTAs/SM; 2 otherwise)
  static const int tables_env = [] { const char* e = getenv("MAPC_TABLES"); return e ? atoi(e) : 0; }();
  const int NT = (tables_env ? tables_env == 3 : jammed) && mine.size() >= 3 && 3 * tab_stride <= P.cap * 8 ? 3 : 2;
  // with three tables: the generate 10 CTAs/SM, the scans 6 at 4 vectors in flight per
  // thread (fewer registers, so they co-reside with the generate), the clears 4
  // (profiles/r2zl_tables4.jsonl, r2zo_tables6.jsonl: 5a 1718 G acc/s; r2zn_tables5.jsonl
  // on a faster box: 1992)
  static const int clear_ctas_env = [] { const char* e = getenv("MAPC_OVL_CLEAR_CTAS"); return e ? atoi(e) : 0; }();
  static const int scan_unroll_env = [] { const char* e = getenv("MAPC_SCAN_UNROLL"); return e ? atoi(e) : 0; }();
  const int ovl_clear_ctas = clear_ctas_env ? clear_ctas_env : NT == 3 ? 4 : ovl_side_ctas;
  const int ovl_scan_ctas = ovl_side_env ? ovl_side_env : NT == 3 ? 6 : ovl_side_ctas;
  if (NT == 3 && !ovl_gen_env) ovl_gen_ctas = 10;   // the jammed kernel's occupancy cap (profiles/r2zo_tables6.jsonl)
  const int ovl_scan_unroll = scan_unroll_env ? scan_unroll_env : NT == 3 ? 4 : 8;
  bool ovl = ovl_env != 0 && !(ex->flags & MAP_EXEC_SEQUENTIAL) && gen_mode == 1 && mine.size() >= 2 &&
             P.off_dtab == P.off_b &&
             2 * tab_stride <= P.cap * 8;
  for (size_t c : mine) ovl = ovl && use_direct(P.chunks[c], ex->flags) && !use_unit(P.chunks[c], ex->flags, gen_mode);
  if (ovl) {
    auto own_stream = [&](cudaStream_t* st, int* dev) -> cudaError_t {
      if (*st && *dev == ex->device) return cudaSuccess;
      if (*st) {
        std::lock_guard<std::mutex> g(pool().mu);
        pool().streams.emplace_back(*dev, *st);
      }
      *st = nullptr;
      *dev = ex->device;
      return pool_stream(ex->device, st);
    };
    CK(own_stream(&p->side, &p->side_dev));
    if (NT == 3) CK(own_stream(&p->side2, &p->side2_dev));
    while (p->sync_events.size() < 12) {
      cudaEvent_t e;
      CK(pool_event(ex->device, false, &e));
      p->sync_events.push_back(e);
    }
    cudaStream_t s2 = p->side;
    cudaStream_t s3 = NT == 3 ? p->side2 : p->side;   // the clears
    cudaEvent_t ev_gen[2] = {p->sync_events[0], p->sync_events[1]};       // per control block
    cudaEvent_t ev_done[2] = {p->sync_events[2], p->sync_events[3]};
    cudaEvent_t ev_scanned[3] = {p->sync_events[4], p->sync_events[5], p->sync_events[6]};   // per table
    cudaEvent_t ev_cleared[3] = {p->sync_events[7], p->sync_events[8], p->sync_events[9]};
    cudaEvent_t ev_join = p->sync_events[10], ev_join3 = p->sync_events[11];
    auto* ctrl2 = (MapcCtrl*)(base + P.off_ctrl2);
    for (size_t c : mine) {
      const Chunk& ch = P.chunks[c];
      CK(cudaMemcpyAsync(base + P.off_allsegs + ch.dev_segs, stage + ch.stage_segs, seg_blob(ch),
                         cudaMemcpyHostToDevice, s));
      h2d += seg_blob(ch);
    }
    CK(cudaEventRecord(ev_join, s));                  // the side streams start after the gate reset and uploads
    CK(cudaStreamWaitEvent(s2, ev_join, 0));
    if (NT == 3) CK(cudaStreamWaitEvent(s3, ev_join, 0));
    // the other tables' first clears run under chunk 0's generate
    for (int t = 1; t < NT; ++t) {
      const Chunk& ct = P.chunks[mine[t]];
      size_t m = begin_on(MAP_K_CLEAR, s3);
      CK(mapc_launch_table_clear(dtab + t * tab_stride, dcells(ct, gen_mode) * ct.cell_bytes, n_sms, ovl_clear_ctas, s3));
      end_on(m, s3);
      CK(cudaEventRecord(ev_cleared[t], s3));
    }
    for (size_t i = 0; i < mine.size(); ++i) {
      const size_t c = mine[i];
      chunk_pos = i;
      NvtxRange nvtx_chunk("chunk " + std::to_string(c) + " direct (overlapped)");
      const Chunk& ch = P.chunks[c];
      const MapcLayout L = effective_layout(ch, ex->flags);
      const int b = (int)(i & 1);                     // control block
      const int t = (int)(i % NT);                    // table
      MapcCtrl* cb = b ? ctrl2 : ctrl;
      unsigned char* tb = dtab + t * tab_stride;
      auto* sg = (MapcSeg*)(base + P.off_allsegs + ch.dev_segs);
      const uint64_t tbytes = dcells(ch, gen_mode) * ch.cell_bytes;
      const auto* pc = comp_on(ch, gen_mode)
                           ? reinterpret_cast<const unsigned long long*>(reinterpret_cast<unsigned char*>(sg) + pcomp_off(ch))
                           : nullptr;
      if (i >= 2) CK(cudaStreamWaitEvent(s, ev_done[b], 0));   // chunk i-2 released control block b
      size_t m = begin(MAP_K_OTHER);
      CK(mapc_launch_chunk_init(cb, ch.dense_total, s));
      end(m);
      if (i == 0) {                                    // first use of table 0 in this run
        m = begin(MAP_K_CLEAR);
        CK(mapc_launch_table_clear(tb, tbytes, n_sms, 0, s));
        end(m);
      } else {
        CK(cudaStreamWaitEvent(s, ev_cleared[t], 0));   // table t cleared for this chunk
      }
      if (ch.total_tiles) {
        m = begin(MAP_K_DIRECT);
        CK(mapj::launch_chunk(P.jit[MAPC_MODE_DIRECT], c, sg, (int)ch.segs.size(), ch.total_tiles,
                              (unsigned long long*)tb, &cb->n, &cb->err, L.cap, &cb->wit_sf, n_sms,
                              ovl_gen_ctas, s, pc));
        end(m);
      }
      CK(cudaEventRecord(ev_gen[b], s));
      CK(cudaStreamWaitEvent(s2, ev_gen[b], 0));
      // scan, then clear table t when chunk i+NT uses it again (a scan that also
      // zeroes the cells it read was measured 2.5x slower: profiles/r1k_*, r2ze_*)
      // the last chunk's scan has no generate to share the GPU with: full grid
      const bool last = i + 1 == mine.size();
      m = begin_on(MAP_K_DETECT, s2);
      CK(mapc_launch_direct_scan(tb, dcells(ch, gen_mode), ch.cell_bytes, L.w_tid, cb, n_sms,
                                 last ? 0 : ovl_scan_ctas, s2, last ? 8 : ovl_scan_unroll));
      end_on(m, s2);

      if (i + NT < mine.size()) {
        // cleared for its next user, chunk i+NT, whose table may be larger
        const Chunk& nx = P.chunks[mine[i + NT]];
        if (NT == 3) {
          CK(cudaEventRecord(ev_scanned[t], s2));
          CK(cudaStreamWaitEvent(s3, ev_scanned[t], 0));
        }
        m = begin_on(MAP_K_CLEAR, s3);
        CK(mapc_launch_table_clear(tb, dcells(nx, gen_mode) * nx.cell_bytes, n_sms, ovl_clear_ctas, s3));
        end_on(m, s3);
        CK(cudaEventRecord(ev_cleared[t], s3));
      }
      m = begin_on(MAP_K_OTHER, s2);                  // gate (+ compressed-cell mapping) and witness + result
      launches += 1;
      st_acc.launches[MAP_K_OTHER] += 1;
      CK(mapc_launch_witness_gate(cb, gate, ch.phase_lo, ch.phase_hi, s2, pc, ch.phase_hi - ch.phase_lo + 1,
                                  L.w_array, L.w_block, L.w_index));
      if (ch.total_tiles) {
        ++launches;
        st_acc.launches[MAP_K_OTHER]++;
        CK(mapj::launch_chunk(P.jit[MAPC_MODE_FILTER], c, sg, (int)ch.segs.size(), ch.total_tiles, bufA, &cb->nf,
                              &cb->err, L.cap, &cb->wit_sf, n_sms, 0, s2));
      }
      CK(mapc_launch_witness_flat(bufA, cb, L.pay_bits, L.w_tid, L.cap, s2, res + c));
      end_on(m, s2);
      CK(cudaEventRecord(ev_done[b], s2));
    }
    CK(cudaEventRecord(ev_join, s2));                 // join the side streams back into the caller's
    CK(cudaStreamWaitEvent(s, ev_join, 0));
    if (NT == 3) {
      CK(cudaEventRecord(ev_join3, s3));
      CK(cudaStreamWaitEvent(s, ev_join3, 0));
    }
  }
  size_t seq_pos = 0;
  for (size_t c : mine) {
    if (ovl) break;
    chunk_pos = seq_pos++;
    const Chunk& ch = P.chunks[c];
    NvtxRange nvtx_chunk("chunk " + std::to_string(c) +
                         (use_unit(ch, ex->flags, gen_mode) ? " unit" : use_direct(ch, ex->flags) ? " direct" : " keys"));
    const MapcLayout L = effective_layout(ch, ex->flags);
    CK(mapc_upload_ops((const MapcOp*)(stage + ch.stage_ops), ch.ops.size(), s));
    CK(cudaMemcpyAsync(segs, stage + ch.stage_segs, seg_blob(ch), cudaMemcpyHostToDevice, s));
    h2d += ch.ops.size() * sizeof(MapcOp) + seg_blob(ch);
    size_t m = begin(MAP_K_OTHER);
    CK(mapc_launch_chunk_init(ctrl, ch.dense_total, s));
    end(m);
    if (use_unit(ch, ex->flags, gen_mode)) {
      // on-chip per-(phase, block) tables (jit.cpp, unit mode): generate, fold and
      // scan in one launch; then the witness cell's keys as on the direct path
      const uint64_t n_units = (uint64_t)(ch.phase_hi - ch.phase_lo + 1) * (ch.b_hi - ch.b_lo);
      m = begin(MAP_K_UNIT);
      CK(mapj::launch_units(P.jit[MAPC_MODE_UNIT], c, n_units, &ctrl->n, &ctrl->racy, &ctrl->racy_sf, &ctrl->err,
                            ch.jit.unit_cluster, ch.jit.unit_threads, ch.unit_smem, n_sms, s));
      end(m);
      m = begin(MAP_K_OTHER);
      launches += 1;
      st_acc.launches[MAP_K_OTHER] += 1;
      CK(mapc_launch_witness_gate(ctrl, gate, ch.phase_lo, ch.phase_hi, s, nullptr, 0, 0, 0, 0));
      if (ch.total_tiles) {
        ++launches;
        st_acc.launches[MAP_K_OTHER]++;
        CK(mapj::launch_unit_filter(P.jit[MAPC_MODE_UNITF], c, &ctrl->wit_sf, bufA, &ctrl->nf, L.cap, &ctrl->err,
                                    (ch.bound + n_units - 1) / std::max<uint64_t>(n_units, 1), n_sms, s));
      }
      CK(mapc_launch_witness_flat(bufA, ctrl, L.pay_bits, L.w_tid, L.cap, s, res + c));
      end(m);
      continue;
    }
    if (use_direct(ch, ex->flags)) {
      // sort-free direct-address detect (direct.cu): clear the table, fold every
      // access into its cell, scan the table, re-emit the witness cell's keys
      const uint64_t tbytes = dcells(ch, gen_mode) * ch.cell_bytes;
      const auto* pc = comp_on(ch, gen_mode)
                           ? reinterpret_cast<const unsigned long long*>(reinterpret_cast<unsigned char*>(segs) + pcomp_off(ch))
                           : nullptr;
      m = begin(MAP_K_CLEAR);
      CK(mapc_launch_table_clear(dtab, tbytes, n_sms, 0, s));
      end(m);
      if (ch.total_tiles) {
        m = begin(MAP_K_DIRECT);
        if (gen_mode == 1)
          CK(mapj::launch_chunk(P.jit[MAPC_MODE_DIRECT], c, segs, (int)ch.segs.size(), ch.total_tiles,
                                (unsigned long long*)dtab, &ctrl->n, &ctrl->err, L.cap, &ctrl->wit_sf, n_sms, 0, s, pc));
        else
          CK(mapc_launch_generate(segs, (int)ch.segs.size(), 0, ch.total_tiles, &L, p->C.u32_mode ? 1 : 0, bufA, ctrl,
                                  n_sms, ch.nreg, 0, 0, MAPC_MODE_DIRECT, dtab, ch.cell_bytes, s));
        end(m);
      }
      m = begin(MAP_K_DETECT);
      CK(mapc_launch_direct_scan(dtab, dcells(ch, gen_mode), ch.cell_bytes, L.w_tid, ctrl, n_sms, 0, s, 8));
      end(m);
      m = begin(MAP_K_OTHER);
      launches += 1;
      st_acc.launches[MAP_K_OTHER] += 1;
      CK(mapc_launch_witness_gate(ctrl, gate, ch.phase_lo, ch.phase_hi, s, pc, ch.phase_hi - ch.phase_lo + 1,
                                  L.w_array, L.w_block, L.w_index));
      if (ch.total_tiles) {
        ++launches;
        st_acc.launches[MAP_K_OTHER]++;
        if (gen_mode == 1)
          CK(mapj::launch_chunk(P.jit[MAPC_MODE_FILTER], c, segs, (int)ch.segs.size(), ch.total_tiles, bufA, &ctrl->nf,
                                &ctrl->err, L.cap, &ctrl->wit_sf, n_sms, 0, s));
        else
          CK(mapc_launch_generate(segs, (int)ch.segs.size(), 0, ch.total_tiles, &L, p->C.u32_mode ? 1 : 0, bufA, ctrl,
                                  n_sms, ch.nreg, MAPC_MAX_EMITS, 0, MAPC_MODE_FILTER, nullptr, ch.cell_bytes, s));
      }
      CK(mapc_launch_witness_flat(bufA, ctrl, L.pay_bits, L.w_tid, L.cap, s, res + c));
      end(m);
      continue;
    }
    if (ch.total_tiles) {
      m = begin(MAP_K_GENERATE);
      if (gen_mode == 1)
        CK(mapj::launch_chunk(P.jit[MAPC_MODE_KEYS], c, segs, (int)ch.segs.size(), ch.total_tiles, bufA, &ctrl->n,
                              &ctrl->err, L.cap, nullptr, n_sms, 0, s));
      else
        CK(mapc_launch_generate(segs, (int)ch.segs.size(), 0, ch.total_tiles, &L, p->C.u32_mode ? 1 : 0, bufA, ctrl,
                                n_sms, ch.nreg, ch.max_emits, 0, MAPC_MODE_KEYS, nullptr, 4, s));
      end(m);
    }
    if (sort_mode == 1) {
      if (L.n_passes) {
        CK(cudaMemsetAsync(rhist, 0, P.rh_bytes, s));
        m = begin(MAP_K_HIST);
        CK(mapc_launch_hist_ranges(bufA, ctrl, rhist, L.sort_lo, L.n_passes, G, s));
        end(m);
      }
      m = begin(MAP_K_SCAN);
      CK(mapc_launch_digit_scan(ctrl, L.n_passes, s));
      end(m);
      for (uint32_t pass = 0; pass < L.n_passes; ++pass) {
        // the pass's per-range table: pass 0 from k_hist_ranges; later passes from the
        // previous scatter (fused variants) or from one read of the pass's input
        if (pass > 0) {
          m = begin(MAP_K_HIST);
          CK(mapc_launch_range_hist(bufA, bufB, ctrl, rhist, pass, L.sort_lo, G, s));
          end(m);
        }
        m = begin(red_next(L) && pass + 1 < L.n_passes ? MAP_K_SORT_NEXT : MAP_K_ONESWEEP);
        CK(mapc_launch_rsweep(bufA, bufB, ctrl, rhist, pass, L.sort_lo, G, red_next(L), s));
        end(m);
      }
    } else {
      if (L.n_passes) {
        m = begin(MAP_K_HIST);
        CK(mapc_launch_hist(bufA, ctrl, L.sort_lo, L.n_passes, ch.bound, n_sms, s));
        end(m);
      }
      m = begin(MAP_K_SCAN);
      CK(mapc_launch_digit_scan(ctrl, L.n_passes, s));
      end(m);
      for (uint32_t pass = 0; pass < L.n_passes; ++pass) {
        ++p->epoch;
        m = begin(MAP_K_ONESWEEP);
        CK(mapc_launch_onesweep(bufA, bufB, ctrl, lookback, pass, L.sort_lo + 8 * pass, p->epoch, ch.bound, n_sms, s));
        end(m);
      }
    }
    m = begin(MAP_K_DETECT);
    ++launches;                        // detect + fixup
    st_acc.launches[MAP_K_DETECT]++;
    if (L.tb)
      CK(mapc_launch_detect_table(bufA, bufB, ctrl, L.n_passes, L.pay_bits, L.tb, L.w_tid, tparts, tstore, ch.bound,
                                  n_sms, s));
    else
      CK(mapc_launch_detect(bufA, bufB, ctrl, L.n_passes, L.pay_bits, L.w_tid, ff, lf, ch.bound, n_sms, s));
    CK(mapc_launch_witness(bufA, bufB, ctrl, L.n_passes, L.pay_bits, L.tb, L.w_tid, s));
    end(m);
    m = begin(MAP_K_OTHER);
    CK(mapc_launch_chunk_finish(ctrl, L.n_passes, res + c, s));
    end(m);
  }
  return MAP_OK;
  };
  static const bool graphs_env = [] { const char* e = getenv("MAPC_GRAPHS"); return !(e && e[0] == '0'); }();
  std::string gkey;
  {
    auto put = [&](const void* v, size_t n) { gkey.append(reinterpret_cast<const char*>(v), n); };
    const uint64_t plan_for = p->plan_for;
    put(&plan_for, 8); put(&ex->flags, 4); put(&ex->scratch, sizeof(void*)); put(&ex->scratch_bytes, 8);
    put(&ex->stream, sizeof(void*)); put(&ex->device, 4); put(&rank, 4); put(&world, 4); put(&gen_mode, 4);
    put(&p->pinned, sizeof(void*));
    const uint8_t pf = prof;
    put(&pf, 1);
  }
  // (not with the look-back onesweep variant: its epochs must advance every run)
  const bool use_graph = graphs_env && !mine.empty() && sort_mode == 1;
  if (use_graph && p->gexec && p->gkey == gkey) {            // replay
    CK(cudaEventRecord(p->events[0], s));
    CK(cudaGraphLaunch(p->gexec, s));
    launches = p->g_launches;
    h2d = p->g_h2d;
    st_acc = p->g_stats;
    marks.clear();
    for (size_t i = 0; i + 3 <= p->g_marks.size(); i += 3)
      marks.push_back({(int)p->g_marks[i], (size_t)p->g_marks[i + 1], (size_t)p->g_marks[i + 2]});
  } else if (use_graph && p->glast_key == gkey) {            // second identical call: capture
    if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; p->gkey.clear(); }
    if (!p->cap || p->cap_dev != ex->device) {
      if (p->cap) {
        std::lock_guard<std::mutex> g(pool().mu);
        pool().streams.emplace_back(p->cap_dev, p->cap);
      }
      p->cap = nullptr;
      CK(pool_stream(ex->device, &p->cap));
      p->cap_dev = ex->device;
    }
    CK(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    rec_s = p->cap;
    capturing = true;
    const map_status est = enqueue(p->cap);
    capturing = false;
    rec_s = s;
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(p->cap, &graph);
    if (est != MAP_OK) { if (graph) cudaGraphDestroy(graph); return est; }
    if (ce != cudaSuccess) {
      p->last_error = std::string("graph capture: ") + cudaGetErrorString(ce);
      return MAP_E_CUDA;
    }
    const cudaError_t ie = cudaGraphInstantiate(&p->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      p->gexec = nullptr;
      p->last_error = std::string("graph instantiate: ") + cudaGetErrorString(ie);
      return MAP_E_CUDA;
    }
    p->gkey = gkey;
    p->g_launches = launches;
    p->g_h2d = h2d;
    p->g_stats = st_acc;
    p->g_marks.clear();
    for (const Mark& mk : marks) p->g_marks.insert(p->g_marks.end(), {(uint64_t)mk.kind, mk.e0, mk.e1});
    CK(cudaEventRecord(p->events[0], s));
    CK(cudaGraphLaunch(p->gexec, s));
  } else {
    CK(cudaEventRecord(p->events[0], s));
    const map_status est = enqueue(s);
    if (est != MAP_OK) return est;
    p->glast_key = gkey;
  }
  CK(cudaEventRecord(p->events[1], s));
  if (!P.chunks.empty())
    CK(cudaMemcpyAsync(host_res, res, P.chunks.size() * sizeof(MapcChunkResult), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, p->events[0], p->events[1]);

  map_result r{};
  r.n_chunks = (int32_t)mine.size();
  r.device_ms = ms;
  r.gpu_launches = launches;
  r.h2d_bytes = h2d;
  r.d2h_bytes = P.chunks.size() * sizeof(MapcChunkResult);
  uint32_t err = 0;
  bool have = false;
  map_witness best{};
  for (size_t c : mine) {
    const MapcChunkResult& cr = host_res[c];
    r.n_accesses += cr.n;
    r.racy_segments += cr.racy;
    err |= cr.err;
    if (use_unit(P.chunks[c], ex->flags, gen_mode)) {
      // on-chip units: no algorithmic HBM traffic (the kernel is ALU / shared-memory bound)
    } else if (use_direct(P.chunks[c], ex->flags)) {
      // direct path: the fused generate reads and writes every cell of the
      // table once (the per-access reductions happen in L2), the clear writes
      // it and the scan reads it
      const uint64_t tbytes = dcells(P.chunks[c], gen_mode) * P.chunks[c].cell_bytes;
      st_acc.bytes[MAP_K_DIRECT] += 2 * tbytes;
      st_acc.bytes[MAP_K_CLEAR] += tbytes;
      st_acc.bytes[MAP_K_DETECT] += tbytes;
    } else {
    st_acc.bytes[MAP_K_GENERATE] += 8 * cr.n;
    // the histogram reads that ran: k_hist_ranges, and k_range_hist per later pass
    // whose table the previous scatter did not accumulate
    st_acc.bytes[MAP_K_HIST] += 8 * cr.n * cr.table_reads;
    // a pass builds the next pass's range table only when a later pass is active
    {
      const MapcLayout Lc = effective_layout(P.chunks[c], ex->flags);
      for (uint32_t q = 0; q < Lc.n_passes; ++q) {
        if (!((cr.active_mask >> q) & 1u)) continue;
        const bool later = (cr.active_mask >> (q + 1)) != 0;
        st_acc.bytes[red_next(Lc) && later ? MAP_K_SORT_NEXT : MAP_K_ONESWEEP] += 16ull * cr.n;
      }
    }
    st_acc.bytes[MAP_K_DETECT] += 8 * cr.n;
    }
    if (cr.witness != ~0ull) {
      map_witness w{};
      decode(p->C, P.chunks[c], cr.witness, &w);
      if (!have || wit_less(w, best)) best = w;
      have = true;
    }
  }
  if (prof) {
    for (const Mark& mk : marks) {
      float t = 0;
      cudaEventElapsedTime(&t, p->events[mk.e0], p->events[mk.e1]);
      st_acc.ms[mk.kind] += t;
    }
    *ex->stats = st_acc;
  }
  if (err & MAPC_ERR_DIV0) {
    p->last_error = "division or modulo by zero on a reached path";
    return MAP_E_ARITH;
  }
  if (err) {
    p->last_error = "internal consistency check failed (err bits " + std::to_string(err) + ")";
    return MAP_E_RANGE;
  }
  // a racy chunk may skip its witness (k_witness_gate) when an earlier racy
  // chunk of this run must hold a smaller one
  r.verdict = (have || r.racy_segments) ? 1 : 0;
  p->have_witness = have;
  p->wit = best;
  *out = r;
  return MAP_OK;
}

map_status map_witness_get(const map_program* p, map_witness* out) {
  if (!p || !out) return MAP_E_ARG;
  if (!p->have_witness) return MAP_E_ARG;
  *out = p->wit;
  return MAP_OK;
}

void map_program_free(map_program* p) {
  if (!p) return;
  pool_release_pinned(p->pinned, p->pinned_bytes);
  delete p;
}

uint64_t map_default_chunk(const map_program* p, uint32_t world) {
  return p ? default_cap_world(p, world) : 0;
}

map_status map_rank_chunks(const map_program* cp, uint64_t chunk_max_accesses, uint32_t rank, uint32_t world,
                           uint32_t* out, uint32_t cap, uint32_t* n) {
  if (!cp || !n || (cap && !out) || (world && rank >= world)) return MAP_E_ARG;
  map_program* p = const_cast<map_program*>(cp);
  const uint32_t w = world ? world : 1;
  map_status st = ensure_plan(p, chunk_max_accesses ? chunk_max_accesses : default_cap_world(p, w));
  if (st != MAP_OK) return st;
  const std::vector<size_t> mine = rank_chunks(p->plan, rank, w);
  for (size_t i = 0; i < mine.size() && i < cap; ++i) out[i] = (uint32_t)mine[i];
  *n = (uint32_t)mine.size();
  return MAP_OK;
}

map_status map_chunk_count(const map_program* cp, uint64_t chunk_max_accesses, uint32_t* n_chunks) {
  if (!cp || !n_chunks) return MAP_E_ARG;
  map_program* p = const_cast<map_program*>(cp);
  map_status st = ensure_plan(p, chunk_max_accesses ? chunk_max_accesses : default_cap(p));
  if (st != MAP_OK) return st;
  *n_chunks = (uint32_t)p->plan.chunks.size();
  return MAP_OK;
}

}  // extern "C"

namespace {

// Device pointers of the scratch layout (shared by the stage API entry points).
struct Dev {
  unsigned long long *bufA, *bufB, *lookback;
  MapcSegState *ff, *lf;
  MapcSeg* segs;
  MapcCtrl* ctrl;
  MapcChunkResult* res;
  unsigned int* rhist;
  unsigned long long* xch;
  MapcTablePart* tparts;
  uint32_t* tstore;
  int n_sms, G;
  cudaStream_t s;
};

map_status stage_setup(map_program* p, const map_exec* ex, uint32_t chunk, Dev* d) {
  if (!p || !ex) return MAP_E_ARG;
  const uint64_t cap = ex->chunk_max_accesses ? ex->chunk_max_accesses : default_cap(p);
  map_status st = ensure_plan(p, cap);
  if (st != MAP_OK) return st;
  Plan& P = p->plan;
  if (chunk >= P.chunks.size()) return MAP_E_ARG;
  if (!ex->scratch || ex->scratch_bytes < P.total) {
    p->last_error = "scratch too small: need " + std::to_string(P.total) + " bytes";
    return MAP_E_NOMEM;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    p->last_error = "no CUDA device";
    return MAP_E_CUDA;
  }
  CK(cudaSetDevice(ex->device));
  CK(cudaDeviceGetAttribute(&d->n_sms, cudaDevAttrMultiProcessorCount, ex->device));
  d->G = mapc_rsweep_ranges(d->n_sms);
  d->s = (cudaStream_t)ex->stream;
  unsigned char* base = (unsigned char*)ex->scratch;
  d->bufA = (unsigned long long*)(base + P.off_a);
  d->bufB = (unsigned long long*)(base + P.off_b);
  d->lookback = (unsigned long long*)(base + P.off_lb);
  d->ff = (MapcSegState*)(base + P.off_ff);
  d->lf = (MapcSegState*)(base + P.off_lf);
  d->segs = (MapcSeg*)(base + P.off_segs);
  d->ctrl = (MapcCtrl*)(base + P.off_ctrl);
  d->res = (MapcChunkResult*)(base + P.off_res);
  d->rhist = (unsigned int*)(base + P.off_rh);
  d->xch = (unsigned long long*)(base + P.off_xch);
  d->tparts = (MapcTablePart*)(base + P.off_tparts);
  d->tstore = (uint32_t*)(base + P.off_tstore);
  return MAP_OK;
}

}  // namespace

extern "C" {

map_status map_chunk_info(const map_program* cp, uint64_t chunk_max_accesses, uint32_t chunk, map_chunk_desc* out) {
  if (!cp || !out) return MAP_E_ARG;
  map_program* p = const_cast<map_program*>(cp);
  map_status st = ensure_plan(p, chunk_max_accesses ? chunk_max_accesses : default_cap(p));
  if (st != MAP_OK) return st;
  if (chunk >= p->plan.chunks.size()) return MAP_E_ARG;
  const Chunk& ch = p->plan.chunks[chunk];
  out->phase_lo = ch.phase_lo;
  out->phase_hi = ch.phase_hi;
  out->block_lo = (uint32_t)ch.b_lo;
  out->block_hi = (uint32_t)ch.b_hi;
  out->bound = ch.bound;
  out->sort_bits = ch.lay.sort_bits;
  out->n_passes = ch.lay.n_passes;
  return MAP_OK;
}

// Rank `rank` of `world` generates the generate tiles [rank*T/world, (rank+1)*T/world)
// of chunk `chunk` (all keys compacted, VM path) and lays them out by destination
// rank dest = hi64(splitmix64(sort field) * world) in keys_out (device, >= the
// chunk's bound); counts_out[world] (host) receives the per-destination counts.
map_status map_generate_bucketed(map_program* p, const map_exec* ex, uint32_t rank, uint32_t world, uint32_t chunk,
                                 void* keys_out, uint64_t* counts_out) {
  if (!keys_out || !counts_out || world == 0 || rank >= world || (int)world > mapc_bucket_max_world()) return MAP_E_ARG;
  Dev d;
  map_status st = stage_setup(p, ex, chunk, &d);
  if (st != MAP_OK) return st;
  Plan& P = p->plan;
  const Chunk& ch = P.chunks[chunk];
  const MapcLayout& L = ch.lay;
  CK(cudaMemcpyAsync(d.segs, ch.segs.data(), ch.segs.size() * sizeof(MapcSeg), cudaMemcpyHostToDevice, d.s));
  CK(mapc_upload_ops(ch.ops.data(), ch.ops.size(), d.s));
  CK(mapc_launch_chunk_init(d.ctrl, 0, d.s));
  const uint64_t t0 = ch.total_tiles * rank / world, t1 = ch.total_tiles * (rank + 1) / world;
  CK(mapc_launch_generate(d.segs, (int)ch.segs.size(), t0, t1, &L, p->C.u32_mode ? 1 : 0, d.bufA, d.ctrl, d.n_sms,
                          ch.nreg, MAPC_MAX_EMITS, 1, MAPC_MODE_KEYS, nullptr, 4, d.s));
  CK(cudaMemsetAsync(d.xch, 0, 2 * 64 * sizeof(unsigned long long), d.s));
  CK(mapc_launch_bucket_count(d.bufA, d.ctrl, L.pay_bits, world, d.xch, d.n_sms, d.s));
  std::vector<unsigned long long> cnt(world);
  CK(cudaMemcpyAsync(cnt.data(), d.xch, world * sizeof(unsigned long long), cudaMemcpyDeviceToHost, d.s));
  CK(cudaStreamSynchronize(d.s));
  std::vector<unsigned long long> cur(world);
  unsigned long long acc = 0;
  for (uint32_t r = 0; r < world; ++r) { cur[r] = acc; acc += cnt[r]; }
  CK(cudaMemcpyAsync(d.xch + 64, cur.data(), world * sizeof(unsigned long long), cudaMemcpyHostToDevice, d.s));
  CK(mapc_launch_bucket_scatter(d.bufA, d.ctrl, L.pay_bits, world, d.xch + 64, (unsigned long long*)keys_out, d.n_sms,
                                d.s));
  MapcChunkResult r{};
  CK(mapc_launch_chunk_finish(d.ctrl, 0, d.res + chunk, d.s));
  CK(cudaMemcpyAsync(&r, d.res + chunk, sizeof(r), cudaMemcpyDeviceToHost, d.s));
  CK(cudaStreamSynchronize(d.s));
  if (r.err & MAPC_ERR_DIV0) { p->last_error = "division or modulo by zero on a reached path"; return MAP_E_ARITH; }
  if (r.err) { p->last_error = "internal consistency check failed"; return MAP_E_RANGE; }
  for (uint32_t q = 0; q < world; ++q) counts_out[q] = cnt[q];
  return MAP_OK;
}

// Sort + detect n keys (device) of chunk `chunk`, e.g. the keys a rank received
// in the exchange; the chunk's packed canonical witness (UINT64_MAX = DRF) and
// racy-segment count are written to the host.
map_status map_sort_detect(map_program* p, const map_exec* ex, uint32_t chunk, void* keys, uint64_t n,
                           uint64_t* packed_witness, uint64_t* racy_segments) {
  if ((!keys && n) || !packed_witness || !racy_segments) return MAP_E_ARG;
  Dev d;
  map_status st = stage_setup(p, ex, chunk, &d);
  if (st != MAP_OK) return st;
  Plan& P = p->plan;
  const Chunk& ch = P.chunks[chunk];
  const MapcLayout L = effective_layout(ch, ex->flags, n);
  if (n > P.cap) return MAP_E_NOMEM;
  CK(mapc_launch_chunk_init(d.ctrl, n, d.s));
  if (n) CK(cudaMemcpyAsync(d.bufA, keys, n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, d.s));
  if (L.n_passes) {
    CK(cudaMemsetAsync(d.rhist, 0, P.rh_bytes, d.s));
    CK(mapc_launch_hist_ranges(d.bufA, d.ctrl, d.rhist, L.sort_lo, L.n_passes, d.G, d.s));
  }
  CK(mapc_launch_digit_scan(d.ctrl, L.n_passes, d.s));
  for (uint32_t pass = 0; pass < L.n_passes; ++pass) {
    if (pass > 0) CK(mapc_launch_range_hist(d.bufA, d.bufB, d.ctrl, d.rhist, pass, L.sort_lo, d.G, d.s));
    CK(mapc_launch_rsweep(d.bufA, d.bufB, d.ctrl, d.rhist, pass, L.sort_lo, d.G, red_next(L), d.s));
  }
  if (L.tb)
    CK(mapc_launch_detect_table(d.bufA, d.bufB, d.ctrl, L.n_passes, L.pay_bits, L.tb, L.w_tid, d.tparts, d.tstore,
                                std::max<uint64_t>(n, 1), d.n_sms, d.s));
  else
    CK(mapc_launch_detect(d.bufA, d.bufB, d.ctrl, L.n_passes, L.pay_bits, L.w_tid, d.ff, d.lf,
                          std::max<uint64_t>(n, 1), d.n_sms, d.s));
  CK(mapc_launch_witness(d.bufA, d.bufB, d.ctrl, L.n_passes, L.pay_bits, L.tb, L.w_tid, d.s));
  CK(mapc_launch_chunk_finish(d.ctrl, L.n_passes, d.res + chunk, d.s));
  MapcChunkResult r{};
  CK(cudaMemcpyAsync(&r, d.res + chunk, sizeof(r), cudaMemcpyDeviceToHost, d.s));
  CK(cudaStreamSynchronize(d.s));
  if (r.err) { p->last_error = "internal consistency check failed"; return MAP_E_RANGE; }
  *packed_witness = r.witness;
  *racy_segments = r.racy;
  return MAP_OK;
}

// All racy segments (NEXT-4): per chunk, generate (bytecode VM) + full LSD sort,
// then two listing passes write every racy segment's packed canonical witness
// in sort-field order into the chunk's free key buffer; the host decodes them
// and merges the chunks' lists in canonical order (a phase split by block
// ranges interleaves arrays, so chunk order alone is not canonical).
map_status map_list_races(map_program* p, const map_exec* ex, map_witness* out, uint64_t cap, uint64_t* n_total) {
  if (!p || !ex || !n_total || (cap && !out)) return MAP_E_ARG;
  Dev d0;
  map_status st = stage_setup(p, ex, 0, &d0);
  if (st == MAP_E_ARG && p->plan.chunks.empty()) {          // no accesses at all
    *n_total = 0;
    return MAP_OK;
  }
  if (st != MAP_OK) return st;
  Plan& P = p->plan;
  std::vector<map_witness> all;
  uint64_t total = 0;
  for (uint32_t c = 0; c < P.chunks.size(); ++c) {
    Dev d;
    st = stage_setup(p, ex, c, &d);
    if (st != MAP_OK) return st;
    const Chunk& ch = P.chunks[c];
    const MapcLayout L = effective_layout(ch, MAP_DETECT_SORT);
    CK(mapc_upload_ops(ch.ops.data(), ch.ops.size(), d.s));
    CK(cudaMemcpyAsync(d.segs, ch.segs.data(), ch.segs.size() * sizeof(MapcSeg), cudaMemcpyHostToDevice, d.s));
    CK(mapc_launch_chunk_init(d.ctrl, ch.dense_total, d.s));
    if (ch.total_tiles)
      CK(mapc_launch_generate(d.segs, (int)ch.segs.size(), 0, ch.total_tiles, &L, p->C.u32_mode ? 1 : 0, d.bufA,
                              d.ctrl, d.n_sms, ch.nreg, ch.max_emits, 0, MAPC_MODE_KEYS, nullptr, 4, d.s));
    if (L.n_passes) {
      CK(cudaMemsetAsync(d.rhist, 0, P.rh_bytes, d.s));
      CK(mapc_launch_hist_ranges(d.bufA, d.ctrl, d.rhist, L.sort_lo, L.n_passes, d.G, d.s));
    }
    CK(mapc_launch_digit_scan(d.ctrl, L.n_passes, d.s));
    for (uint32_t pass = 0; pass < L.n_passes; ++pass) {
      if (pass > 0) CK(mapc_launch_range_hist(d.bufA, d.bufB, d.ctrl, d.rhist, pass, L.sort_lo, d.G, d.s));
      CK(mapc_launch_rsweep(d.bufA, d.bufB, d.ctrl, d.rhist, pass, L.sort_lo, d.G, red_next(L), d.s));
    }
    CK(mapc_launch_chunk_finish(d.ctrl, L.n_passes, d.res + c, d.s));
    MapcChunkResult r{};
    unsigned int sel = 0;
    CK(cudaMemcpyAsync(&r, d.res + c, sizeof(r), cudaMemcpyDeviceToHost, d.s));
    CK(cudaMemcpyAsync(&sel, &d.ctrl->sel[L.n_passes], sizeof(sel), cudaMemcpyDeviceToHost, d.s));
    CK(cudaStreamSynchronize(d.s));
    if (r.err & MAPC_ERR_DIV0) { p->last_error = "division or modulo by zero on a reached path"; return MAP_E_ARITH; }
    if (r.err) { p->last_error = "internal consistency check failed"; return MAP_E_RANGE; }
    if (r.n == 0) continue;
    unsigned long long* free_buf = sel ? d.bufA : d.bufB;       // the buffer not holding the sorted keys
    const uint64_t dev_cap = std::min<uint64_t>(cap, P.cap);
    auto* counts = reinterpret_cast<unsigned long long*>(d.ff);
    CK(mapc_launch_list_racy(d.bufA, d.bufB, d.ctrl, L.n_passes, L.pay_bits, L.w_tid, counts, MAPC_DETECT_MAX_UNITS,
                             free_buf, dev_cap, d.xch, r.n, d.n_sms, d.s));
    unsigned long long nr = 0;
    CK(cudaMemcpyAsync(&nr, d.xch, sizeof(nr), cudaMemcpyDeviceToHost, d.s));
    CK(cudaStreamSynchronize(d.s));
    total += nr;
    const uint64_t take = std::min<uint64_t>(nr, dev_cap);
    std::vector<unsigned long long> packed(take);
    if (take) {
      CK(cudaMemcpyAsync(packed.data(), free_buf, take * sizeof(unsigned long long), cudaMemcpyDeviceToHost, d.s));
      CK(cudaStreamSynchronize(d.s));
    }
    for (unsigned long long w : packed) {
      map_witness mw{};
      decode(p->C, ch, w, &mw);
      all.push_back(mw);
    }
  }
  std::sort(all.begin(), all.end(), wit_less);
  const uint64_t k = std::min<uint64_t>(cap, all.size());
  for (uint64_t i = 0; i < k; ++i) out[i] = all[i];
  *n_total = total;
  return MAP_OK;
}

map_status map_unpack_witness(const map_program* p, uint32_t chunk, uint64_t packed, map_witness* out) {
  if (!p || !out || chunk >= p->plan.chunks.size() || packed == ~0ull) return MAP_E_ARG;
  decode(p->C, p->plan.chunks[chunk], packed, out);
  return MAP_OK;
}

const char* map_array_name(const map_program* p, uint32_t idx) {
  if (!p || idx >= p->C.ast.arrays.size()) return nullptr;
  return p->C.ast.arrays[idx].c_str();
}

// Human-readable listing of the lowered programs (debugging / tests).
size_t map_debug_dump(const map_program* p, char* buf, size_t cap) {
  if (!p) return 0;
  static const char* names[] = {"add", "sub", "mul", "div", "mod", "shl", "shr", "min", "max", "divm", "modm",
                                "band", "eq", "ne", "lt", "le", "gt", "ge", "land", "lor", "lnot", "trip",
                                "madk", "act", "emit", "movi", "nop"};
  std::string out;
  for (size_t i = 0; i < p->C.inst.size(); ++i) {
    const auto& in = p->C.inst[i];
    for (size_t g = 0; g < in.groups.size(); ++g) {
      const auto& G = in.groups[g];
      out += "instance " + std::to_string(i) + " phase " + std::to_string(in.phase) + " group " + std::to_string(g) +
             " levels " + std::to_string(G.n_levels) + " trips";
      for (uint32_t l = 0; l < G.n_levels; ++l) out += " " + std::to_string(G.trips[l]);
      out += std::string(G.dense ? " dense" : "") + (G.tid_inner ? " tid_inner" : "") + " emits " + std::to_string(G.n_emits);
      // per site: index mod 2^kb == kv (the known low bits behind the stride compression)
      for (size_t e = 0; e < G.site_kb.size(); ++e)
        out += " known" + std::to_string(e) + "=" + std::to_string(G.site_kb[e]) + ":" + std::to_string(G.site_kv[e]);
      out += "\n";
      for (const MapcOp& op : G.ops) {
        const uint32_t c = op.code & MAPC_CODE_MASK;
        out += "  r" + std::to_string(op.dst) + " = " + (c <= VM_NOP ? names[c] : "?") + " ";
        out += (op.code & MAPC_A_IMM) ? ("#" + std::to_string(op.imm)) : ("r" + std::to_string(op.a));
        out += ", ";
        out += (op.code & MAPC_B_IMM) ? ("#" + std::to_string(op.imm)) : ("r" + std::to_string(op.b));
        out += " aux=" + std::to_string(op.aux) + "\n";
      }
    }
  }
  if (buf && cap) {
    size_t n = std::min(cap - 1, out.size());
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return out.size();
}

// Generate + NVRTC-compile the specialised generate module without loading it
// (no GPU needed): 0 on success, else writes the compiler log.  Test hook.
// The specialised generate source of one chunk (debugging / SASS inspection).
size_t map_debug_jit_source(const map_program* cp, uint64_t chunk_max_accesses, uint32_t chunk, char* out,
                            size_t cap) {
  map_program* p = const_cast<map_program*>(cp);
  if (!p || ensure_plan(p, chunk_max_accesses ? chunk_max_accesses : default_cap(p)) != MAP_OK) return 0;
  if (chunk >= p->plan.chunks.size()) return 0;
  std::vector<mapj::JitChunk> one{p->plan.chunks[chunk].jit};
  const char* mode_env = getenv("MAPC_DEBUG_JIT_MODE");          // 0 keys, 1 direct, 2 filter
  const uint32_t mode = mode_env ? (uint32_t)atoi(mode_env) : MAPC_MODE_KEYS;
  const std::string src = mapj::module_source(one, p->C.u32_mode, mode, p->plan.chunks[chunk].cell_bytes);
  put_diag(src, out, cap);
  return src.size();
}

int map_debug_jit_check(const map_program* cp, uint64_t chunk_max_accesses, char* log, size_t cap) {
  map_program* p = const_cast<map_program*>(cp);
  if (!p) return -1;
  if (ensure_plan(p, chunk_max_accesses ? chunk_max_accesses : default_cap(p)) != MAP_OK) return -1;
  std::string l;
  int r = 0;
  std::vector<std::thread> pool;
  std::mutex mu;
  std::atomic<size_t> next{0};
  auto& chunks = p->plan.chunks;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (unsigned w = 0; w < std::min<size_t>(hw, chunks.size()); ++w)
    pool.emplace_back([&]() {
      for (size_t i = next++; i < chunks.size(); i = next++) {
        std::vector<char> cubin;
        std::string li;
        std::vector<mapj::JitChunk> one{chunks[i].jit};
        bool bad = false;
        for (uint32_t mode = 0; mode < 5 && !bad; ++mode)
          if ((mode != MAPC_MODE_UNIT && mode != MAPC_MODE_UNITF) || chunks[i].unit_ok)
            bad = mapj::compile_cubin(mapj::module_source(one, p->C.u32_mode, mode, chunks[i].cell_bytes), &cubin,
                                    &li) != 0;
        if (bad) {
          std::lock_guard<std::mutex> g(mu);
          r = 1;
          l = li;
        }
      }
    });
  for (auto& t : pool) t.join();
  put_diag(l, log, cap);
  return r;
}

// Last error text of a program (diagnostics for the Python binding).
const char* map_last_error(const map_program* p) { return p ? p->last_error.c_str() : ""; }

// Host-side self test of the invariant-divisor parameters (CPU tests).
uint32_t mapc_test_fastdiv(uint32_t n, uint32_t d) { return mapc::fastdiv_apply(n, mapc::make_fastdiv(d)); }

}  // extern "C"

// ---- internal: the MAP's access keys in a global layout (execute.cpp) --------
// Every chunk of the plan (chunk_max_accesses of ex; all chunks, no shard) is
// generated with the bytecode VM in keys mode and its keys are re-packed into
// the global layout [phase | array | block | index | tid | kind] of widths
// w_out[4] (phase, array, block, index; the payload w_tid + 1 is the program's)
// and appended to out[cap] (device).  *n = the keys generated (even beyond cap);
// *n_outside = keys whose index the output layout cannot hold (written as ~0).
extern "C" cudaError_t mapc_launch_bc_repack(const unsigned long long* in, unsigned long long n, const uint32_t* w_in,
                                             const unsigned long long* offs, const uint32_t* w_out,
                                             unsigned long long* out, unsigned long long* n_outside, cudaStream_t s);

extern "C" map_status mapc_internal_lambda_keys(map_program* p, const map_exec* ex, const uint32_t* w_out,
                                                unsigned long long* out, uint64_t cap, unsigned long long* n_outside,
                                                uint64_t* n) {
  if (!p || !ex || !w_out || !out || !n || !n_outside) return MAP_E_ARG;
  uint64_t total = 0;
  map_status st0 = ensure_plan(p, ex->chunk_max_accesses ? ex->chunk_max_accesses : default_cap(p));
  if (st0 != MAP_OK) return st0;
  for (uint32_t c = 0; c < p->plan.chunks.size(); ++c) {
    Dev d;
    map_status st = stage_setup(p, ex, c, &d);
    if (st != MAP_OK) return st;
    const Chunk& ch = p->plan.chunks[c];
    const MapcLayout& L = ch.lay;
    CK(mapc_upload_ops(ch.ops.data(), ch.ops.size(), d.s));
    CK(cudaMemcpyAsync(d.segs, ch.segs.data(), ch.segs.size() * sizeof(MapcSeg), cudaMemcpyHostToDevice, d.s));
    CK(mapc_launch_chunk_init(d.ctrl, ch.dense_total, d.s));
    if (ch.total_tiles)
      CK(mapc_launch_generate(d.segs, (int)ch.segs.size(), 0, ch.total_tiles, &L, p->C.u32_mode ? 1 : 0, d.bufA,
                              d.ctrl, d.n_sms, ch.nreg, ch.max_emits, 0, MAPC_MODE_KEYS, nullptr, 4, d.s));
    MapcCtrl hc{};
    CK(cudaMemcpyAsync(&hc, d.ctrl, sizeof(hc), cudaMemcpyDeviceToHost, d.s));
    CK(cudaStreamSynchronize(d.s));
    if (hc.err & MAPC_ERR_DIV0) { p->last_error = "division or modulo by zero on a reached path"; return MAP_E_ARITH; }
    if (hc.err) { p->last_error = "internal consistency check failed"; return MAP_E_RANGE; }
    if (total + hc.n <= cap) {
      const uint32_t w_in[5] = {L.w_phase, L.w_array, L.w_block, L.w_index, L.pay_bits};
      const unsigned long long offs[3] = {ch.phase_lo, ch.b_lo, L.idx_lo};
      CK(mapc_launch_bc_repack(d.bufA, hc.n, w_in, offs, w_out, out + total, n_outside, d.s));
    }
    total += hc.n;
  }
  *n = total;
  return MAP_OK;
}

// internal: static facts of a compiled program the executor needs
extern "C" map_status mapc_internal_index_hull(const map_program* p, uint64_t* max_index, uint32_t* n_phases) {
  if (!p || !max_index || !n_phases) return MAP_E_ARG;
  uint64_t hi = 0;
  bool any = false;
  for (const auto& in : p->C.inst)
    for (const auto& g : in.groups)
      if (g.has_emit) { hi = std::max(hi, g.index.hi); any = true; }
  *max_index = any ? hi : 0;
  *n_phases = p->C.n_phases;
  return MAP_OK;
}
