// exchange.cu -- destination bucketing for the key-exchange multi-GPU mode.
//
// When one (phase, block) unit must be split across GPUs,
// every rank generates a slice of the chunk's tuples and routes each key to
// rank dest = hi64(splitmix64(sort field) * world): all accesses of a segment
// share the sort field, hence the destination, so each rank's local sort +
// detect is exact.  The exchange itself is one all_to_all_single over NCCL
// (paper_2203_12878_b200/dist.py); these kernels lay the keys out by
// destination.
#include "common.cuh"

namespace mapk {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint32_t dest_of(unsigned long long key, uint32_t pay_bits, uint32_t world) {
  return (uint32_t)__umul64hi(splitmix64(key >> pay_bits), (unsigned long long)world);
}

constexpr int BK_THREADS = 256;
constexpr int BK_MAX_WORLD = 64;

__global__ void __launch_bounds__(BK_THREADS)
k_bucket_count(const unsigned long long* __restrict__ keys, const MapcCtrl* __restrict__ ctrl, uint32_t pay_bits,
               uint32_t world, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int c[BK_MAX_WORLD];
  for (int i = threadIdx.x; i < BK_MAX_WORLD; i += BK_THREADS) c[i] = 0;
  __syncthreads();
  const unsigned long long n = ctrl->n;
  for (unsigned long long i = (unsigned long long)blockIdx.x * BK_THREADS + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * BK_THREADS)
    atomicAdd(&c[dest_of(keys[i], pay_bits, world)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < (int)world; i += BK_THREADS)
    if (c[i]) atomicAdd(&counts[i], (unsigned long long)c[i]);
}

// cursors[d] starts at the exclusive prefix of counts; order inside a bucket is arbitrary
__global__ void __launch_bounds__(BK_THREADS)
k_bucket_scatter(const unsigned long long* __restrict__ keys, const MapcCtrl* __restrict__ ctrl, uint32_t pay_bits,
                 uint32_t world, unsigned long long* __restrict__ cursors, unsigned long long* __restrict__ out) {
  const unsigned long long n = ctrl->n;
  for (unsigned long long i = (unsigned long long)blockIdx.x * BK_THREADS + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * BK_THREADS) {
    const unsigned long long k = keys[i];
    out[atomicAdd(&cursors[dest_of(k, pay_bits, world)], 1ull)] = k;
  }
}

}  // namespace mapk

extern "C" int mapc_bucket_max_world() { return mapk::BK_MAX_WORLD; }

extern "C" cudaError_t mapc_launch_bucket_count(const unsigned long long* keys, const MapcCtrl* ctrl, uint32_t pay_bits,
                                                uint32_t world, unsigned long long* counts, int n_sms, cudaStream_t s) {
  mapk::k_bucket_count<<<n_sms * 4, mapk::BK_THREADS, 0, s>>>(keys, ctrl, pay_bits, world, counts);
  return cudaGetLastError();
}

extern "C" cudaError_t mapc_launch_bucket_scatter(const unsigned long long* keys, const MapcCtrl* ctrl,
                                                  uint32_t pay_bits, uint32_t world, unsigned long long* cursors,
                                                  unsigned long long* out, int n_sms, cudaStream_t s) {
  mapk::k_bucket_scatter<<<n_sms * 4, mapk::BK_THREADS, 0, s>>>(keys, ctrl, pay_bits, world, cursors, out);
  return cudaGetLastError();
}
