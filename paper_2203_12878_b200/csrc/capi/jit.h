// jit.h -- NVRTC-specialised generate kernels (see jit.cpp).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../devabi.h"

namespace mapj {

struct JitProgram {
  uint32_t prog_begin;            // case label: the program's offset in the chunk's bytecode
  uint32_t n_levels;
  std::vector<MapcOp> ops;        // mode-independent ops (divisions by constants left to NVRTC)
  // range of the innermost tuple coordinate (tid when tid_inner or without loops,
  // else the innermost loop counter): when a multiple of G, the G tuples from a
  // multiple of G differ only in that coordinate (+0..G-1), no carry
  uint64_t inner_range = 0;
  bool tid_inner = false;
};

struct JitChunk {
  MapcLayout lay;
  uint32_t max_emits;
  std::vector<JitProgram> programs;
  std::vector<MapcSeg> segs;      // baked as literals when few (tuple decode and slots fold to constants)
  // unit mode (MAPC_MODE_UNIT): every segment baked, and the chunk's unit grid
  std::vector<MapcSeg> unit_segs;
  uint64_t n_blocks = 0;          // blocks of the chunk (b_hi - b_lo)
  uint32_t unit_cluster = 1;      // CTAs per unit: 1 = the unit's table in one CTA's shared memory,
                                  // K > 1 = spread over a K-CTA cluster (distributed shared memory)
  uint32_t unit_threads = 128;    // threads per CTA of the unit kernel
  bool comp = false;              // direct mode: stride-compressed table (pcomp, mapcheck.cpp Chunk)
};

struct JitHandle {
  std::vector<cudaKernel_t> kernels;   // one per chunk
};

// mode: MAPC_MODE_KEYS (keys -> key buffer), MAPC_MODE_DIRECT (red.or into the
// direct-address table passed as `keys`, cells of cell_bytes), MAPC_MODE_FILTER
// (only keys with sort field *target, compacted; n_ctr counts them).
std::string chunk_kernel_source(const JitChunk& ch, int index, bool u32, uint32_t mode, uint32_t cell_bytes);
std::string module_source(const std::vector<JitChunk>& chunks, bool u32, uint32_t mode, uint32_t cell_bytes);
int compile_cubin(const std::string& src, std::vector<char>* cubin, std::string* log);
// Compile (or fetch from the process-wide cache) the kernels of the chunks with
// want[i] != 0 for one mode; out->kernels has one entry per chunk (null = not built).
// The direct-mode kernel of this chunk is row-jammed (jit.cpp jam_rows).
bool jam_active(const JitChunk& ch, uint32_t cell_bytes);
// Number of distinct specialised kernels the chunks need (chunks that differ only
// in data the kernel does not bake share one; build_module compiles each once).
size_t distinct_kernels(const std::vector<JitChunk>& chunks, bool u32);
int build_module(const std::vector<JitChunk>& chunks, bool u32, uint32_t mode, const std::vector<uint32_t>& cell_bytes,
                 const std::vector<char>& want, JitHandle* out, std::string* log);
cudaError_t launch_chunk(const JitHandle& h, size_t chunk, const MapcSeg* segs, int n_segs,
                         unsigned long long total_tiles, unsigned long long* keys, unsigned long long* n_ctr,
                         unsigned int* err_flag, unsigned long long cap, const unsigned long long* target,
                         int n_sms, int max_ctas_per_sm, cudaStream_t s, const unsigned long long* pcomp = nullptr);
// Unit mode (MAPC_MODE_UNIT): n_units (phase, block) units of the chunk, one CTA
// each at a time; counts into n_ctr (guarded accesses), racy, racy_sf (atomicMin).
// cluster = CTAs per unit (thread-block cluster, DSMEM table when > 1), threads per
// CTA, smem = dynamic shared bytes per CTA (cluster > 1).
cudaError_t launch_units(const JitHandle& h, size_t chunk, unsigned long long n_units, unsigned long long* n_ctr,
                         unsigned long long* racy, unsigned long long* racy_sf, unsigned int* err_flag,
                         uint32_t cluster, uint32_t threads, size_t smem, int n_sms, cudaStream_t s);
// Unit filter (MAPC_MODE_UNITF): the keys of cell *target from its unit's tuples
// (unit_accesses bounds them; sets the grid), appended to keys[cap], counted in *n_ctr.
cudaError_t launch_unit_filter(const JitHandle& h, size_t chunk, const unsigned long long* target,
                               unsigned long long* keys, unsigned long long* n_ctr, unsigned long long cap,
                               unsigned int* err_flag, unsigned long long unit_accesses, int n_sms, cudaStream_t s);

}  // namespace mapj
