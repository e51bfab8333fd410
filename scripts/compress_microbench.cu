// Does generic memory compression (cuMemCreate, CU_MEM_ALLOCATION_COMP_GENERIC)
// cut the DRAM cost of the direct table's cycle clear -> red.or -> scan?
// The cleared table is all zeros, which compressible memory can hold in
// compressed form, so the clear's writes and the red's line fills may shrink.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared \
//        scripts/compress_microbench.cu -lcuda -o /tmp/compress_microbench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
  do {                                                                              \
    auto e_ = (x);                                                                  \
    if (e_ != 0) {                                                                  \
      std::printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__);              \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

__global__ void k_clear(uint4* t, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    t[i] = make_uint4(0, 0, 0, 0);
}

// 5a-like: every 8-byte word of the table gets `reps` red.or.b64 of a nonzero code
// (16-bit lanes), warps on consecutive words, each CTA a contiguous block.
__global__ void k_red(unsigned long long* t, size_t n8, int reps) {
  const size_t per = (n8 + gridDim.x - 1) / gridDim.x;
  const size_t lo = blockIdx.x * per, hi = min(n8, lo + per);
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    for (int r = 0; r < reps; ++r) {
      const unsigned long long c = 0x0007000700070007ull << (r & 7);
      asm volatile("red.global.or.b64 [%0], %1;" ::"l"(t + i), "l"(c) : "memory");
    }
}

__global__ void k_scan(const uint4* t, size_t n16, unsigned long long* out) {
  unsigned long long acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = t[i];
    acc += (v.x & v.y) ^ (v.z | v.w);
  }
  if (acc == 0x123456789ull) *out = acc;
}

static void cycle(const char* name, void* p, size_t bytes, unsigned long long* out, int sms) {
  cudaEvent_t e[4];
  for (auto& x : e) CK(cudaEventCreate(&x));
  float best[3] = {1e9f, 1e9f, 1e9f};
  for (int it = 0; it < 6; ++it) {
    CK(cudaEventRecord(e[0]));
    k_clear<<<sms * 8, 256>>>((uint4*)p, bytes / 16);
    CK(cudaEventRecord(e[1]));
    k_red<<<sms * 12, 128>>>((unsigned long long*)p, bytes / 8, 2);
    CK(cudaEventRecord(e[2]));
    k_scan<<<sms * 8, 256>>>((const uint4*)p, bytes / 16, out);
    CK(cudaEventRecord(e[3]));
    CK(cudaEventSynchronize(e[3]));
    for (int k = 0; k < 3; ++k) {
      float ms;
      CK(cudaEventElapsedTime(&ms, e[k], e[k + 1]));
      if (it > 0 && ms < best[k]) best[k] = ms;
    }
  }
  const double gb = bytes / 1e9;
  std::printf("%-12s clear %.4f ms (%.0f GB/s)  red x2 %.4f ms (%.0f GB/s payload)  scan %.4f ms (%.0f GB/s)  cycle %.4f ms\n",
              name, best[0], gb / best[0] * 1e3, best[1], 2 * gb / best[1] * 1e3, best[2], gb / best[2] * 1e3,
              best[0] + best[1] + best[2]);
}

int main() {
  CK(cudaFree(0));
  CUdevice dev;
  CK(cuCtxGetDevice(&dev));
  int sms = 0, comp = 0;
  CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  CK(cuDeviceGetAttribute(&comp, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, dev));
  std::printf("sms %d generic_compression_supported %d\n", sms, comp);
  const size_t bytes = 1ull << 30;
  unsigned long long* out;
  CK(cudaMalloc(&out, 8));

  void* plain;
  CK(cudaMalloc(&plain, bytes));
  cycle("cudaMalloc", plain, bytes, out, sms);

  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.allocFlags.compressionType = CU_MEM_ALLOCATION_COMP_GENERIC;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CUresult r = cuMemCreate(&h, sz, &prop, 0);
  if (r != CUDA_SUCCESS) {
    std::printf("cuMemCreate(compressible) failed: %d\n", (int)r);
    return 0;
  }
  CUmemAllocationProp got = {};
  CK(cuMemGetAllocationPropertiesFromHandle(&got, h));
  std::printf("granularity %zu compression granted %d\n", gran, (int)got.allocFlags.compressionType);
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, sz, 0, 0, 0));
  CK(cuMemMap(va, sz, 0, h, 0));
  CUmemAccessDesc ad = {};
  ad.location = prop.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(va, sz, &ad, 1));
  cycle("compressible", (void*)va, bytes, out, sms);
  cycle("cudaMalloc", plain, bytes, out, sms);
  cycle("compressible", (void*)va, bytes, out, sms);
  return 0;
}
