// Per-SM HBM ingest probe: how many GB/s can one SM pull when only N SMs stream?
// (the decode lane runs on a 68-SM partition and measured ~43 GB/s per SM through
// its TMA pipelines).  Streams a 4 GB buffer with N CTAs (one per SM: 200 KB smem
// each) three ways:
//   ldg  : 16 warps, 16-byte ld.global.nc loads, 8 in flight per thread
//   tma  : one thread issues 1-D cp.async.bulk global->shared copies of 16 KB into a
//          ring of `stages` slots (mbarrier complete_tx), consumer warps release slots
//   tma2d: the GEMM's A-operand pattern — 2-D tensor-map boxes of 64 bf16 x 128 rows
//          (128-byte swizzle) out of a row-major [rows, K = 2048] weight matrix, each
//          box 128 segments of 128 B one 4 KB row stride apart
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ingest_probe tools/ingest_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) ldg_kernel(const uint4 *src, size_t n16, unsigned long long *sink) {
  const size_t per = n16 / gridDim.x;
  const uint4 *p = src + blockIdx.x * per;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < per; i += (size_t)blockDim.x * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t j = i + (size_t)u * blockDim.x;
      if (j < per) asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
      else v[u] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

constexpr int CHUNK = 16384;
__global__ void __launch_bounds__(128, 1) tma_kernel(const uint8_t *src, size_t bytes, int stages,
                                                     unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + stages * CHUNK);
  uint64_t *empty = full + stages;
  const size_t per = bytes / gridDim.x / CHUNK * CHUNK;
  const uint8_t *p = src + blockIdx.x * per;
  const int n = (int)(per / CHUNK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      asm volatile(
          "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(
              smem_u32(empty + s)),
          "r"(ph ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sm + s * CHUNK)),
                   "l"(p + (size_t)i * CHUNK), "r"(CHUNK), "r"(smem_u32(full + s)));
    }
  } else if (threadIdx.x == 32) {
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      asm volatile(
          "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(
              smem_u32(full + s)),
          "r"(ph));
      acc ^= reinterpret_cast<const uint32_t *>(sm + s * CHUNK)[0];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + s)));
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}

__global__ void __launch_bounds__(128, 1) tma2d_kernel(const __grid_constant__ CUtensorMap map, int rows, int kb,
                                                       int stages, unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(base + stages * CHUNK);
  uint64_t *empty = full + stages;
  const int mtiles = rows / 128;
  const int per = mtiles / gridDim.x;  // whole 128-row tiles per CTA
  const int n = per * kb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      const int mt = blockIdx.x * per + i / kb, k = i % kb;
      asm volatile(
          "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(
              smem_u32(empty + s)),
          "r"(ph ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(CHUNK));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(base + s * CHUNK)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(full + s)), "r"(k * 64), "r"(mt * 128));
    }
  } else if (threadIdx.x == 32) {
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      asm volatile(
          "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(
              smem_u32(full + s)),
          "r"(ph));
      acc ^= reinterpret_cast<const uint32_t *>(base + s * CHUNK)[0];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + s)));
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}

int main() {
  const size_t bytes = 4ull << 30;
  uint8_t *buf;
  unsigned long long *sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(ldg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int sms : {32, 68, 80, 148}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      ldg_kernel<<<sms, 512, 200 * 1024>>>(reinterpret_cast<const uint4 *>(buf), bytes / 16, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("ldg  %3d SMs: %7.1f GB/s total, %6.1f GB/s per SM\n", sms, bytes / ms / 1e6, bytes / ms / 1e6 / sms);
    }
    for (int stages : {4, 8, 12}) {
      const size_t smem = (size_t)stages * CHUNK + 2 * stages * 8 + 64;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        tma_kernel<<<sms, 128, smem>>>(buf, bytes, stages, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep)
          printf("tma  %3d SMs, %2d x 16 KB in flight: %7.1f GB/s total, %6.1f GB/s per SM\n", sms, stages,
                 bytes / ms / 1e6, bytes / ms / 1e6 / sms);
      }
    }
  }
  // 2-D tensor boxes over a [rows, 2048] bf16 matrix (the decode gate/up weight shape)
  {
    const int K = 2048, rows = (int)(bytes / (K * 2)) / (148 * 128) * (148 * 128);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    cudaFuncSetAttribute(tma2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const double mb = (double)rows * K * 2;
    for (int sms : {68, 148}) {
      for (int stages : {5, 8, 12}) {
        const size_t smem = 1024 + (size_t)stages * CHUNK + 2 * stages * 8 + 64;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          tma2d_kernel<<<sms, 128, smem>>>(map, rows, K / 64, stages, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double moved = (double)(rows / 128 / sms) * sms * 128 * K * 2;
          if (rep)
            printf("tma2d %3d SMs, %2d x 16 KB boxes in flight: %7.1f GB/s total, %6.1f GB/s per SM\n", sms, stages,
                   moved / ms / 1e6, moved / ms / 1e6 / sms);
        }
      }
    }
    (void)mb;
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
