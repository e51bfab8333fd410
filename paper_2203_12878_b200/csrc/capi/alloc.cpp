// alloc.cpp -- optional device-memory helper for the caller's scratch
// (include/mapcheck.h map_scratch_alloc / map_scratch_free).
//
// The library never allocates its scratch; this helper lets a
// caller put it in *compressible* device memory (cuMemCreate with
// CU_MEM_ALLOCATION_COMP_GENERIC).  The direct path clears its tables to zero
// before every chunk and the generate's atomics then fill those lines from DRAM:
// all-zero lines compress, so the clear and the fills move fewer DRAM bytes
// (5a 1262 -> 1391 G acc/s).  The driver API is reached through
// cudaGetDriverEntryPoint, so libmapcheck.so does not link libcuda (it still
// loads on a machine without a driver; the helper then returns MAP_E_CUDA).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>

#include "../../../include/mapcheck.h"

namespace {

struct Fns {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemGetAllocationPropertiesFromHandle) props = nullptr;
  decltype(&cuDeviceGetAttribute) attribute = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* out) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p)
    return false;
  *out = reinterpret_cast<F>(p);
  return true;
}

const Fns& fns() {
  static const Fns f = [] {
    Fns r;
    r.ok = entry("cuMemCreate", &r.create) && entry("cuMemRelease", &r.release) &&
           entry("cuMemAddressReserve", &r.reserve) && entry("cuMemAddressFree", &r.addr_free) &&
           entry("cuMemMap", &r.map) && entry("cuMemUnmap", &r.unmap) && entry("cuMemSetAccess", &r.set_access) &&
           entry("cuMemGetAllocationGranularity", &r.granularity) &&
           entry("cuMemGetAllocationPropertiesFromHandle", &r.props) &&
           entry("cuDeviceGetAttribute", &r.attribute);
    return r;
  }();
  return f;
}

struct Block {
  CUmemGenericAllocationHandle h;
  size_t size;
  bool vmm;       // cuMemCreate mapping (else cudaMalloc)
};
std::mutex g_mu;
std::map<uintptr_t, Block> g_blocks;

}  // namespace

extern "C" map_status map_scratch_alloc(int device, uint64_t bytes, uint32_t flags, void** ptr, uint64_t* size,
                                        uint32_t* compressed) {
  if (!ptr || bytes == 0 || (flags & ~MAP_ALLOC_COMPRESSIBLE) != 0) return MAP_E_ARG;
  *ptr = nullptr;
  if (size) *size = 0;
  if (compressed) *compressed = 0;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return MAP_E_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return MAP_E_CUDA;
  const Fns& f = fns();
  int comp_ok = 0;
  if ((flags & MAP_ALLOC_COMPRESSIBLE) && f.ok)
    f.attribute(&comp_ok, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, (CUdevice)device);
  if (comp_ok) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    prop.allocFlags.compressionType = CU_MEM_ALLOCATION_COMP_GENERIC;
    size_t gran = 0;
    if (f.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && gran) {
      const size_t sz = (bytes + gran - 1) / gran * gran;
      CUmemGenericAllocationHandle h;
      if (f.create(&h, sz, &prop, 0) == CUDA_SUCCESS) {
        CUmemAllocationProp got = {};
        f.props(&got, h);
        CUdeviceptr va = 0;
        bool mapped = false;
        if (f.reserve(&va, sz, 0, 0, 0) == CUDA_SUCCESS) {
          if (f.map(va, sz, 0, h, 0) == CUDA_SUCCESS) {
            CUmemAccessDesc ad = {};
            ad.location = prop.location;
            ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            if (f.set_access(va, sz, &ad, 1) == CUDA_SUCCESS) {
              mapped = true;
            } else {
              f.unmap(va, sz);
            }
          }
          if (!mapped) f.addr_free(va, sz);
        }
        if (mapped) {
          std::lock_guard<std::mutex> g(g_mu);
          g_blocks[(uintptr_t)va] = Block{h, sz, true};
          *ptr = (void*)va;
          if (size) *size = sz;
          if (compressed) *compressed = got.allocFlags.compressionType == CU_MEM_ALLOCATION_COMP_GENERIC;
          return MAP_OK;
        }
        f.release(h);
      }
    }
  }
  // plain device memory: no compression requested, supported or granted
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return MAP_E_NOMEM;
  }
  std::lock_guard<std::mutex> g(g_mu);
  g_blocks[(uintptr_t)p] = Block{0, (size_t)bytes, false};
  *ptr = p;
  if (size) *size = bytes;
  return MAP_OK;
}

extern "C" map_status map_scratch_free(void* ptr) {
  if (!ptr) return MAP_OK;
  Block b;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_blocks.find((uintptr_t)ptr);
    if (it == g_blocks.end()) return MAP_E_ARG;
    b = it->second;
    g_blocks.erase(it);
  }
  if (!b.vmm) return cudaFree(ptr) == cudaSuccess ? MAP_OK : MAP_E_CUDA;
  // the caller has synchronised its work on this memory (as for cudaFree)
  const Fns& f = fns();
  if (cudaDeviceSynchronize() != cudaSuccess) return MAP_E_CUDA;
  bool ok = f.unmap((CUdeviceptr)ptr, b.size) == CUDA_SUCCESS;
  ok = f.addr_free((CUdeviceptr)ptr, b.size) == CUDA_SUCCESS && ok;
  ok = f.release(b.h) == CUDA_SUCCESS && ok;
  return ok ? MAP_OK : MAP_E_CUDA;
}
