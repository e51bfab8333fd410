// Is the direct generate bound by the NUMBER of global reductions?  The 5a phase
// pattern with 16-bit cells folded in aligned quads (one red.or.b64 per 4 cells):
//   A  one red per site per quad: rows r-1, r, r+1 of the read half and row r of
//      the write half -> 4 reds per 16 accesses (what the JIT generate does);
//   B  a thread walks U consecutive rows of one column quad and ORs a read-half
//      row's three touches (as rows r+1, r, r-1 of iterations r, r+1, r+2) in a
//      register before ONE red -> (U + 2 + U) reds per 16 U accesses.
// Both over a 1 GiB table (2^29 16-bit cells) in plain and in compressible memory,
// cleared before every launch (as the pipeline does).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared \
//        scripts/quad_red_microbench.cu -lcuda -o /tmp/quad_red_microbench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                    \
  do {                                                                           \
    auto e_ = (x);                                                               \
    if (e_ != 0) {                                                               \
      std::printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__);           \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

constexpr uint32_t NT = 1024, R = 256, C = 1024, H = NT * R, Q = C / 4;   // quads per row
constexpr uint64_t HALF = (uint64_t)H * C;                                  // cells per half (2^28)

__device__ __forceinline__ uint64_t code4(uint32_t tid, uint32_t kind) {
  const uint64_t c = (tid & 0x3FFu) | (kind << 14);
  return c | (c << 16) | (c << 32) | (c << 48);
}

// A: item = (tid, r, quad), linear in that order; blocked CTA ranges
__global__ void __launch_bounds__(128, 12) k_a(unsigned long long* tab) {
  const uint64_t n = (uint64_t)NT * R * Q;
  const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t q = (uint32_t)(i % Q), r = (uint32_t)((i / Q) % R), tid = (uint32_t)(i / ((uint64_t)Q * R));
    const uint32_t row = tid * R + r;
    const uint64_t rd = code4(tid, 0), wr = code4(tid, 1);
    atomicOr(tab + ((uint64_t)((row + H - 1) % H) * Q + q), rd);
    atomicOr(tab + ((uint64_t)row * Q + q), rd);
    atomicOr(tab + ((uint64_t)((row + 1) % H) * Q + q), rd);
    atomicOr(tab + (HALF / 4 + (uint64_t)row * Q + q), wr);
  }
}

// B: item = (tid, row block of U, quad); the thread walks the U rows keeping the
// read-half codes of rows row-1 .. row+1 in registers
template <int U>
__global__ void __launch_bounds__(128, 12) k_b(unsigned long long* tab) {
  const uint64_t n = (uint64_t)NT * (R / U) * Q;
  const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t q = (uint32_t)(i % Q), rb = (uint32_t)((i / Q) % (R / U)), tid = (uint32_t)(i / ((uint64_t)Q * (R / U)));
    const uint64_t rd = code4(tid, 0), wr = code4(tid, 1);
    const uint32_t row0 = tid * R + rb * U;
    // rows row0-1 .. row0+U: each read row's OR is one red (its touches by this thread)
#pragma unroll
    for (int j = -1; j <= U; ++j) {
      const uint32_t row = (row0 + H + j) % H;
      atomicOr(tab + ((uint64_t)row * Q + q), rd);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) atomicOr(tab + (HALF / 4 + (uint64_t)(row0 + u) * Q + q), wr);
  }
}

__global__ void k_clear(uint4* t, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    t[i] = make_uint4(0, 0, 0, 0);
}

template <class F>
float best_of(F launch, void* tab, int sms) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e9f;
  for (int rep = 0; rep < 5; ++rep) {
    k_clear<<<sms * 8, 256>>>((uint4*)tab, (2 * HALF * 2) / 16);
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep && ms < best) best = ms;
  }
  return best;
}

void run(const char* mem, void* tab, int sms) {
  auto* t = (unsigned long long*)tab;
  const double acc = (double)NT * R * C * 4;
  const float a = best_of([&] { k_a<<<sms * 12, 128>>>(t); }, tab, sms);
  std::printf("%-13s A  4 reds / 16 acc          %.4f ms  %.1f G acc/s\n", mem, a, acc / a / 1e6);
  const float b2 = best_of([&] { k_b<2><<<sms * 12, 128>>>(t); }, tab, sms);
  std::printf("%-13s B2 %d reds / %d acc         %.4f ms  %.1f G acc/s\n", mem, 2 + 2 + 2, 32, b2, acc / b2 / 1e6);
  const float b4 = best_of([&] { k_b<4><<<sms * 12, 128>>>(t); }, tab, sms);
  std::printf("%-13s B4 %d reds / %d acc        %.4f ms  %.1f G acc/s\n", mem, 4 + 2 + 4, 64, b4, acc / b4 / 1e6);
  const float b8 = best_of([&] { k_b<8><<<sms * 12, 128>>>(t); }, tab, sms);
  std::printf("%-13s B8 %d reds / %d acc       %.4f ms  %.1f G acc/s\n", mem, 8 + 2 + 8, 128, b8, acc / b8 / 1e6);
}

int main() {
  CK(cudaFree(0));
  CUdevice dev;
  CK(cuCtxGetDevice(&dev));
  int sms = 0;
  CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  const size_t bytes = 2 * HALF * 2;   // 2^29 16-bit cells
  void* plain;
  CK(cudaMalloc(&plain, bytes));
  run("cudaMalloc", plain, sms);
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.allocFlags.compressionType = CU_MEM_ALLOCATION_COMP_GENERIC;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CK(cuMemCreate(&h, sz, &prop, 0));
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, sz, 0, 0, 0));
  CK(cuMemMap(va, sz, 0, h, 0));
  CUmemAccessDesc ad = {};
  ad.location = prop.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(va, sz, &ad, 1));
  run("compressible", (void*)va, sms);
  return 0;
}
