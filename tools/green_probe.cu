// Feasibility probe: SM partitions (green contexts) for the two execution lanes.
// Splits the GPU's SMs into two green contexts, creates a stream in each, launches
// kernels through the RUNTIME API onto those streams (eagerly and from a captured
// CUDA graph), and reports which SMs each launch ran on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/green_probe tools/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                  \
      const char *s_;                                                          \
      cuGetErrorString(r_, &s_);                                               \
      printf("%s failed: %s\n", #x, s_);                                       \
      return 1;                                                                \
    }                                                                          \
  } while (0)
#define RK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s failed: %s\n", #x, cudaGetErrorString(e_));                  \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void smid_kernel(int *out, long long spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

static std::set<int> sms_of(const std::vector<int> &v) { return std::set<int>(v.begin(), v.end()); }

int main(int argc, char **argv) {
  const int want = argc > 1 ? atoi(argv[1]) : 72;
  RK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all, parts[2], rest;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned n = 1;
  CK(cuDevSmResourceSplitByCount(parts, &n, &all, &rest, 0, want));
  printf("device SMs %u -> partition %u SMs + remainder %u SMs\n", all.sm.smCount, parts[0].sm.smCount,
         rest.sm.smCount);
  CUdevResourceDesc d0, d1;
  CK(cuDevResourceGenerateDesc(&d0, &parts[0], 1));
  CK(cuDevResourceGenerateDesc(&d1, &rest, 1));
  CUgreenCtx g0, g1;
  CK(cuGreenCtxCreate(&g0, d0, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s0, s1;
  CK(cuGreenCtxStreamCreate(&s0, g0, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
  const int blocks = 1024;
  int *d;
  RK(cudaMalloc(&d, 3 * blocks * sizeof(int)));
  std::vector<int> h(blocks);
  // (1) eager runtime-API launches on the green streams (primary context current)
  smid_kernel<<<blocks, 64, 0, (cudaStream_t)s0>>>(d, 2000);
  smid_kernel<<<blocks, 64, 0, (cudaStream_t)s1>>>(d + blocks, 2000);
  RK(cudaGetLastError());
  RK(cudaDeviceSynchronize());
  RK(cudaMemcpy(h.data(), d, blocks * sizeof(int), cudaMemcpyDeviceToHost));
  auto a = sms_of(h);
  RK(cudaMemcpy(h.data(), d + blocks, blocks * sizeof(int), cudaMemcpyDeviceToHost));
  auto b = sms_of(h);
  int both = 0;
  for (int x : a) both += b.count(x);
  printf("eager: lane0 on %zu SMs, lane1 on %zu SMs, shared %d\n", a.size(), b.size(), both);
  // (2) a graph captured on a green stream, replayed on it and on a primary stream
  cudaGraph_t g;
  cudaGraphExec_t ge;
  RK(cudaStreamBeginCapture((cudaStream_t)s0, cudaStreamCaptureModeRelaxed));
  smid_kernel<<<blocks, 64, 0, (cudaStream_t)s0>>>(d + 2 * blocks, 2000);
  RK(cudaStreamEndCapture((cudaStream_t)s0, &g));
  RK(cudaGraphInstantiate(&ge, g, 0));
  RK(cudaGraphLaunch(ge, (cudaStream_t)s0));
  RK(cudaDeviceSynchronize());
  RK(cudaMemcpy(h.data(), d + 2 * blocks, blocks * sizeof(int), cudaMemcpyDeviceToHost));
  auto c = sms_of(h);
  int inpart = 0;
  for (int x : c) inpart += a.count(x);
  printf("graph replay on lane0 stream: %zu SMs, %d of them in lane0's partition\n", c.size(), inpart);
  cudaStream_t prim;
  RK(cudaStreamCreateWithFlags(&prim, cudaStreamNonBlocking));
  RK(cudaGraphLaunch(ge, prim));
  RK(cudaDeviceSynchronize());
  RK(cudaMemcpy(h.data(), d + 2 * blocks, blocks * sizeof(int), cudaMemcpyDeviceToHost));
  auto e = sms_of(h);
  inpart = 0;
  for (int x : e) inpart += a.count(x);
  printf("same graph replayed on a primary-context stream: %zu SMs, %d in lane0's partition\n", e.size(), inpart);
  // (3) isolation: a long kernel filling lane1 while lane0 runs short kernels
  cudaEvent_t t0, t1;
  RK(cudaEventCreate(&t0));
  RK(cudaEventCreate(&t1));
  RK(cudaEventRecord(t0, (cudaStream_t)s0));
  for (int i = 0; i < 100; ++i) smid_kernel<<<64, 64, 0, (cudaStream_t)s0>>>(d, 100);
  RK(cudaEventRecord(t1, (cudaStream_t)s0));
  RK(cudaDeviceSynchronize());
  float alone;
  RK(cudaEventElapsedTime(&alone, t0, t1));
  smid_kernel<<<100000, 256, 0, (cudaStream_t)s1>>>(d + blocks, 200000);
  RK(cudaEventRecord(t0, (cudaStream_t)s0));
  for (int i = 0; i < 100; ++i) smid_kernel<<<64, 64, 0, (cudaStream_t)s0>>>(d, 100);
  RK(cudaEventRecord(t1, (cudaStream_t)s0));
  RK(cudaDeviceSynchronize());
  float busy;
  RK(cudaEventElapsedTime(&busy, t0, t1));
  printf("100 short launches on lane0: alone %.3f ms, with lane1 saturated %.3f ms\n", alone, busy);
  return 0;
}
