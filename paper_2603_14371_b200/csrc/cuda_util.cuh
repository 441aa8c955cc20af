// CUDA helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "common.h"

#define OXY_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) oxy::fail(OXY_ECUDA, "%s failed: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

namespace oxy {
// kernels launched by this library (read by bench.py as gpu_launches)
extern unsigned long long g_launches;
// scratch reallocations (invalidates captured CUDA graphs)
extern unsigned long long g_devbuf_reallocs;
}

#define OXY_LAUNCH_CHECK()                                  \
  do {                                                      \
    __atomic_fetch_add(&oxy::g_launches, 1ull, __ATOMIC_RELAXED); \
    OXY_CUDA(cudaGetLastError());                           \
  } while (0)

namespace oxy {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// draw i (0-based) of SplitMix64(seed).uniform(), bit-exact with the reference
__host__ __device__ inline double splitmix_uniform(uint64_t seed, uint64_t i) {
  return (double)(mix64(seed + (i + 1) * kGamma) >> 11) * 0x1.0p-53;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: every F2 kernel starts with pdl_wait(), so it
// may be scheduled while its predecessor drains; the wait blocks until the
// predecessor grid has completed and its writes are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Allow the dependent grid to be scheduled now (it still waits in pdl_wait()
// for our completion before touching anything we write).
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// 2^x on the SFU (ex2.approx.ftz, ~2 ulp; results below 2^-126 flush to 0,
// 2^-inf = 0).  Branch-free: exp2f's denormal-range fix-up, combined with a
// per-element "row fully masked" test, made the compiler emit one divergent
// region per score and serialise the SFU latency (2 us per 64-key tile).
__device__ __forceinline__ float exp2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OXY_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
}

// launch_pdl with a thread-block cluster shape (cluster (1,1,1): a plain launch)
template <typename... KArgs, typename... Args>
inline void launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               dim3 cluster, Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster.x;
  attr[1].val.clusterDim.y = cluster.y;
  attr[1].val.clusterDim.z = cluster.z;
  cfg.attrs = attr;
  cfg.numAttrs = cluster.x * cluster.y * cluster.z > 1 ? 2 : 1;
  OXY_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
}

// Grow-only device scratch buffer.
struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
  void *get(size_t need) {
    if (need > bytes) {
      ++g_devbuf_reallocs;
      if (ptr) cudaFree(ptr);
      size_t cap = need + need / 2 + 256;
      OXY_CUDA(cudaMalloc(&ptr, cap));
      bytes = cap;
    }
    return ptr;
  }
  template <typename T>
  T *as(size_t n) { return static_cast<T *>(get(n * sizeof(T))); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

template <typename T>
__device__ inline T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ inline T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block reductions (fixed shuffle tree, then warp 0).
template <typename T>
__device__ inline T block_sum(T v, T *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  T r = lane < nw ? red[lane] : T(0);
  r = warp_sum(r);
  return r;
}

template <typename T>
__device__ inline T block_max(T v, T *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  T r = lane < nw ? red[lane] : red[0];
  r = warp_max(r);
  return r;
}

}  // namespace oxy
