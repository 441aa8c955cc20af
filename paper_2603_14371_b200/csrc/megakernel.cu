// Persistent layer-program kernel: see megakernel.cuh for the design.
#include <algorithm>
#include <cstring>

#include "attn_device.cuh"
#include "cuda_util.cuh"
#include "gemm_device.cuh"
#include "megakernel.cuh"

namespace oxy {
namespace mk {

using gemm::A_STAGE_BYTES;
using gemm::BK;
using gemm::BM;

constexpr int STAGE_BYTES = A_STAGE_BYTES + MK_MAX_BN * BK * 2;  // 32 KB
constexpr int RING_BYTES = MK_STAGES * STAGE_BYTES;              // 192 KB (>= 5 flash tiles, 169 KB)
static_assert(RING_BYTES >= (int)pi05::FaCfg<256>::SMEM, "flash tiles must fit the GEMM ring");
constexpr int BAR_BYTES = (2 * MK_STAGES + 4) * 8 + 16;

size_t mk_smem_bytes() { return 1024 + RING_BYTES + BAR_BYTES; }

#ifndef MK_POLL_NS
#define MK_POLL_NS 100
#endif

// ------------------------------------------------------------------ grid barrier
// Monotonic arrival counter (zeroed before the launch); phase i completes when
// all CTAs have arrived i + 1 times.  Writers' generic-proxy stores are fenced
// for the async proxy (the next phase's TMA reads them).
__device__ __forceinline__ void grid_barrier(unsigned *sync, unsigned target, unsigned long long *arrive) {
  asm volatile("fence.proxy.async;" ::: "memory");  // generic <-> async proxy, global and shared
  __syncthreads();
  if (threadIdx.x == 0) {
    if (arrive) {
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      *arrive = ns;
    }
    // release: the CTA's writes (ordered before us by bar.sync) become visible
    // to every CTA that acquires the counter value that includes our arrival
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(sync) : "memory");
    unsigned v;
    // back off between polls: 148 pollers hammering one L2 line slow down every
    // other request that lands on that L2 slice (the working CTAs' loads)
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sync) : "memory");
      if (v >= target) break;
      __nanosleep(MK_POLL_NS);
    }
  }
  __syncthreads();
}

struct Pipe {
  int it_p = 0;           // producer k-block counter
  int it_m = 0, lt_m = 0;  // MMA k-block / tile counters
  int lt_e = 0;           // epilogue tile counter
};

// ------------------------------------------------------------------ phases

__device__ __forceinline__ void gemm_phase(const GemmPh &g, int items, uint8_t *ring, uint32_t full0,
                                           uint32_t empty0, uint32_t tfull0, uint32_t tempty0, uint32_t tmem,
                                           const CUtensorMap *maps, Pipe &pp, int &s_last) {
  using namespace gemm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bn = g.bn, b_bytes = bn * BK * 2;
  const int per_m = g.splits * g.n_tiles;
  if (warp == 0) {
    if (lane == 0) {
      const CUtensorMap *ma = maps + g.map_a, *mb = maps + g.map_b;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(ma)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mb)) : "memory");
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int mt = item / per_m, rem = item % per_m, split = rem / g.n_tiles, nt = rem % g.n_tiles;
        const int kb0 = split * g.kb_per_split;
        const int nkb = min(g.kb_total, kb0 + g.kb_per_split) - kb0;
        for (int i = 0; i < nkb; ++i, ++pp.it_p) {
          const int s = pp.it_p % MK_STAGES;
          const uint32_t ph = (pp.it_p / MK_STAGES) & 1;
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          mbar_expect_tx(full0 + 8 * s, A_STAGE_BYTES + b_bytes);
          const int kc = (kb0 + i) * BK;
          uint8_t *st = ring + s * STAGE_BYTES;
          tma_load_2d(ma, full0 + 8 * s, smem_u32(st), kc, mt * BM);
          tma_load_2d(mb, full0 + 8 * s, smem_u32(st + A_STAGE_BYTES), kc, nt * bn);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++pp.lt_m) {
        const int rem = item % per_m, split = rem / g.n_tiles;
        const int kb0 = split * g.kb_per_split;
        const int nkb = min(g.kb_total, kb0 + g.kb_per_split) - kb0;
        const int acc = pp.lt_m & 1;
        mbar_wait(tempty0 + 8 * acc, ((pp.lt_m >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)acc * MK_MAX_BN;
        for (int i = 0; i < nkb; ++i, ++pp.it_m) {
          const int s = pp.it_m % MK_STAGES;
          const uint32_t ph = (pp.it_m / MK_STAGES) & 1;
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint32_t a = smem_u32(ring + s * STAGE_BYTES), b = a + A_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_bf16(d, make_sdesc(a + kk * 32), make_sdesc(b + kk * 32), idesc, (i | kk) != 0 ? 1u : 0u);
          mma_commit(empty0 + 8 * s);
        }
        mma_commit(tfull0 + 8 * acc);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++pp.lt_e) {
      const int mt = item / per_m, rem = item % per_m, split = rem / g.n_tiles, nt = rem % g.n_tiles;
      const int acc = pp.lt_e & 1;
      mbar_wait(tfull0 + 8 * acc, (pp.lt_e >> 1) & 1);
      tc_fence_after();
      const int f = mt * BM + q * 32 + lane;
      const uint32_t trow = tmem + (uint32_t)acc * MK_MAX_BN + ((uint32_t)(q * 32) << 16);
      epi_tile(g, trow, 0, bn, nt * bn, f, split, g.splits > 1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(tempty0 + 8 * acc);
    }
  }
  (void)s_last;
}

// fixed-order split-K sum + epilogue, one thread per feature pair (grid-stride)
__device__ __forceinline__ void reduce_epi_phase(const ReducePh &r) {
  const int pairs = (r.n + 1) >> 1;
  const int64_t total = (int64_t)r.t * pairs;
  for (int64_t idx = blockIdx.x * (int64_t)MK_THREADS + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * MK_THREADS) {
    const int t = (int)(idx / pairs), f = (int)(idx % pairs) * 2;
    const bool two = f + 1 < r.n;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
    for (int s = 0; s < r.splits; ++s) {
      const float *row = r.ws + ((size_t)s * r.t + t) * r.n;
      a0 += __ldcg(row + f);
      a1 += two ? __ldcg(row + f + 1) : 0.f;
    }
    gemm::epilogue_store(r.epi, t, f, r.n, a0, a1);
    if (two) gemm::epilogue_store(r.epi, t, f + 1, r.n, a1, a0);
  }
}

constexpr int NORM_MAXV = 12;  // rows of up to 12 * 192 = 2304 features

__device__ __forceinline__ void res_norm_phase(const NormPh &p, float *red) {
  for (int row = blockIdx.x; row < p.t; row += gridDim.x) {
    float v[NORM_MAXV];
#pragma unroll
    for (int j = 0; j < NORM_MAXV; ++j) v[j] = 0.f;
    if (p.ws) {
      for (int s0 = 0; s0 < p.splits; s0 += 4) {  // 4 splits x 12 features of loads in flight
        float u[4][NORM_MAXV];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const float *wrow = p.ws + ((size_t)(s0 + s) * p.t + row) * p.n;
#pragma unroll
          for (int j = 0; j < NORM_MAXV; ++j) {
            const int f = threadIdx.x + j * MK_THREADS;
            u[s][j] = (f < p.n && s0 + s < p.splits) ? __ldcg(wrow + f) : 0.f;
          }
        }
#pragma unroll
        for (int s = 0; s < 4; ++s)  // split order 0..S-1 per element
#pragma unroll
          for (int j = 0; j < NORM_MAXV; ++j) v[j] += u[s][j];
      }
    }
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NORM_MAXV; ++j) {
      const int f = threadIdx.x + j * MK_THREADS;
      if (f < p.n) {
        float xv = p.x[(size_t)row * p.ldx + f];
        if (p.ws) {
          xv += p.gate ? p.gate[f] * v[j] : v[j];
          p.x[(size_t)row * p.ldx + f] = xv;
        }
        v[j] = xv;
        ss += xv * xv;
      }
    }
    ss = block_sum(ss, red);
    const float inv = rsqrtf(ss / (float)p.n + p.eps);
#pragma unroll
    for (int j = 0; j < NORM_MAXV; ++j) {
      const int f = threadIdx.x + j * MK_THREADS;
      if (f < p.n) {
        const float o = p.w ? v[j] * inv * (1.f + p.w[f]) : v[j] * inv * (1.f + p.ms[f]) + p.mb[f];
        p.y[(size_t)row * p.ldy + f] = __float2bfloat16(o);
      }
    }
    __syncthreads();  // red[] is reused by the next row
  }
}

__device__ __forceinline__ void attn_phase(const AttnPh &a, int items, uint8_t *ring) {
  if (threadIdx.x >= pi05::FA_THREADS) return;  // warps 4-5 sit this phase out
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int split = item % a.splits, rest = item / a.splits;
    const int qt = rest % a.q_tiles, gi = rest / a.q_tiles;
    const pi05::AttnGroup g = a.groups[gi];
    pi05::flash_item<256>(g, qt, split, a.splits, a.kpool, a.vpool, a.scale_log2, a.ws_o, a.ws_ml, a.ws_rows,
                          reinterpret_cast<bf16 *>(ring), threadIdx.x);
  }
}

// Split-order merge: one thread per (query row, column pair), grid-stride; the
// per-row split weights are recomputed per thread from the (m, l) rows (L1 hits).
__device__ __forceinline__ void attn_merge_phase(const AttnPh &a) {
  constexpr int HDP = 256, PAIRS = HDP / 2;
  const int64_t total = (int64_t)a.n_groups * a.max_nq * PAIRS;
  const size_t mstride = (size_t)a.ws_rows * 2, ostride = (size_t)a.ws_rows * HDP;
  for (int64_t idx = blockIdx.x * (int64_t)MK_THREADS + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * MK_THREADS) {
    const int c = (int)(idx % PAIRS) * 2;
    const int64_t rr = idx / PAIRS;
    const int gi = (int)(rr / a.max_nq), r = (int)(rr % a.max_nq);
    const pi05::AttnGroup &g = a.groups[gi];
    if (r >= g.nq) continue;
    const size_t row0 = (size_t)g.wrow0 + r;
    float M = -INFINITY;
#pragma unroll 8
    for (int s = 0; s < a.splits; ++s) M = fmaxf(M, __ldcg(a.ws_ml + row0 * 2 + s * mstride));
    float a0 = 0.f, a1 = 0.f, L = 0.f;
#pragma unroll 8
    for (int s = 0; s < a.splits; ++s) {  // split order
      const float ms = __ldcg(a.ws_ml + row0 * 2 + s * mstride);
      const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
      const float l = __ldcg(a.ws_ml + row0 * 2 + s * mstride + 1);
      const float2 v = __ldcg(reinterpret_cast<const float2 *>(a.ws_o + row0 * HDP + c + s * ostride));
      L += l * w;
      a0 += v.x * w;
      a1 += v.y * w;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    *reinterpret_cast<__nv_bfloat162 *>(g.o + (size_t)r * g.ldo + c) = __floats2bfloat162_rn(a0 * inv, a1 * inv);
  }
}

__device__ __forceinline__ void euler_phase(const EulerPh &e) {
  for (int i = blockIdx.x * MK_THREADS + threadIdx.x; i < e.n; i += gridDim.x * MK_THREADS) {
    const float v = e.a[i] + e.dt * e.v[i];
    e.a[i] = v;
    e.ab[i] = __float2bfloat16(v);
  }
}

// ------------------------------------------------------------------ kernel

__global__ void __launch_bounds__(MK_THREADS, 1)
    mk_kernel(const Phase *__restrict__ prog, int n_phases, const CUtensorMap *__restrict__ maps, unsigned *sync,
              unsigned long long *times) {
  using namespace gemm;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(ring + RING_BYTES);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * MK_STAGES + 4);
  __shared__ float red[40];
  __shared__ int s_last;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + MK_STAGES),
                 tfull0 = smem_u32(bars + 2 * MK_STAGES), tempty0 = smem_u32(bars + 2 * MK_STAGES + 2);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < MK_STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * MK_MAX_BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  Pipe pp;
  for (int ph = 0; ph < n_phases; ++ph) {
    const Phase &P = prog[ph];
    const int type = P.type, items = P.items;
    switch (type) {
      case PH_GEMM: gemm_phase(P.g, items, ring, full0, empty0, tfull0, tempty0, tmem, maps, pp, s_last); break;
      case PH_REDUCE_EPI: reduce_epi_phase(P.r); break;
      case PH_RES_NORM: res_norm_phase(P.nm, red); break;
      case PH_ATTN: attn_phase(P.at, items, ring); break;
      case PH_ATTN_MERGE: attn_merge_phase(P.at); break;
      case PH_EULER: euler_phase(P.eu); break;
      default: break;
    }
    if (ph + 1 < n_phases)
      grid_barrier(sync, (unsigned)(ph + 1) * gridDim.x,
                   times ? times + n_phases + (size_t)ph * gridDim.x + blockIdx.x : nullptr);
    if (times && blockIdx.x == 0 && threadIdx.x == 0) {  // optional per-phase timeline (profiling)
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      times[ph] = ns;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * MK_MAX_BN)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host

Program::~Program() {
  cudaFree(d_times);
  cudaFree(d_phases);
  cudaFree(d_maps);
  cudaFree(d_sync);
}

int Program::map(const void *ptr, int rows, int k, int box_rows) {
  for (size_t i = 0; i < map_keys.size(); ++i)
    if (map_keys[i] == ptr && map_meta[3 * i] == rows && map_meta[3 * i + 1] == k && map_meta[3 * i + 2] == box_rows)
      return (int)i;
  maps.push_back(gemm::make_map(ptr, rows, k, box_rows));
  map_keys.push_back(ptr);
  map_meta.insert(map_meta.end(), {rows, k, box_rows});
  return (int)maps.size() - 1;
}

int gemm_splits(int n_out, int k, int t, int sms) {
  const int kb_total = (k + BK - 1) / BK, m_tiles = (n_out + BM - 1) / BM;
  const int bn = std::min(MK_MAX_BN, std::max(16, (t + 15) / 16 * 16));
  const int base = m_tiles * ((t + bn - 1) / bn);
  int splits = std::max(1, std::min(sms / base, kb_total / 2));
  splits = std::max(1, std::min(splits, kb_total));
  const int per = (kb_total + splits - 1) / splits;
  return (kb_total + per - 1) / per;
}

int Program::gemm(const bf16 *w, const bf16 *x, int n_out, int k, int t, const gemm::EpiParams &epi, float *ws,
                  int sms, int force_splits) {
  Phase p{};
  p.type = PH_GEMM;
  GemmPh &g = p.g;
  g.n_out = n_out;
  g.k = k;
  g.t = t;
  g.kb_total = (k + BK - 1) / BK;
  g.m_tiles = (n_out + BM - 1) / BM;
  g.bn = std::min(MK_MAX_BN, std::max(16, (t + 15) / 16 * 16));
  g.n_tiles = (t + g.bn - 1) / g.bn;
  const int base = g.m_tiles * g.n_tiles;
  int splits = force_splits > 0 ? force_splits : gemm_splits(n_out, k, t, sms);
  splits = std::max(1, std::min(splits, g.kb_total));
  g.kb_per_split = (g.kb_total + splits - 1) / splits;
  g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  if (g.splits > 1 && !ws) fail(OXY_EINVAL, "megakernel split-K GEMM needs a workspace");
  g.epi = epi;
  g.ws = ws;
  g.map_a = map(w, n_out, k, BM);
  g.map_b = map(x, t, k, g.bn);
  p.items = base * g.splits;
  phases.push_back(p);
  return g.splits;
}

void Program::reduce_epi(const float *ws, int splits, int t, int n, const gemm::EpiParams &epi) {
  Phase p{};
  p.type = PH_REDUCE_EPI;
  p.r = ReducePh{ws, splits, t, n, epi};
  p.items = 0;
  phases.push_back(p);
}

void Program::res_norm(const float *ws, int splits, int t, int n, const float *gate, float *x, int ldx, bf16 *y,
                       int ldy, const float *w, const float *ms, const float *mb, float eps) {
  if (n > NORM_MAXV * MK_THREADS) fail(OXY_EINVAL, "megakernel norm rows are limited to %d", NORM_MAXV * MK_THREADS);
  Phase p{};
  p.type = PH_RES_NORM;
  p.nm = NormPh{ws, splits, t, n, gate, x, ldx, y, ldy, w, ms, mb, eps};
  p.items = t;
  phases.push_back(p);
}

void Program::attention(const pi05::AttnGroup *groups_d, int n_groups, int q_tiles, int max_nq, int splits,
                        int ws_rows, const bf16 *kpool, const bf16 *vpool, float scale, float *ws_o, float *ws_ml) {
  Phase p{};
  p.type = PH_ATTN;
  p.at = AttnPh{groups_d, n_groups, q_tiles, splits, ws_rows, max_nq, kpool, vpool, scale * 1.4426950408889634f,
                ws_o, ws_ml};
  p.items = n_groups * q_tiles * splits;
  phases.push_back(p);
  if (splits > 1) {
    if (splits > 32) fail(OXY_EINVAL, "megakernel attention merge handles <= 32 splits");
    Phase m = p;
    m.type = PH_ATTN_MERGE;
    m.items = n_groups * max_nq;
    phases.push_back(m);
  }
}

void Program::euler(float *a, const float *v, bf16 *ab, int n, float dt) {
  Phase p{};
  p.type = PH_EULER;
  p.eu = EulerPh{a, v, ab, n, dt};
  p.items = 0;
  phases.push_back(p);
}

void Program::upload(cudaStream_t st) {
  if (phases.size() > cap_phases) {
    cudaFree(d_times);
    d_times = nullptr;
    cudaFree(d_phases);
    cap_phases = phases.size() + 64;
    OXY_CUDA(cudaMalloc(&d_phases, cap_phases * sizeof(Phase)));
  }
  if (maps.size() > cap_maps || !d_maps) {
    cudaFree(d_maps);
    cap_maps = maps.size() + 16;
    OXY_CUDA(cudaMalloc(&d_maps, cap_maps * sizeof(CUtensorMap)));
  }
  if (!d_sync) OXY_CUDA(cudaMalloc(&d_sync, 64));
  OXY_CUDA(cudaMemcpyAsync(d_phases, phases.data(), phases.size() * sizeof(Phase), cudaMemcpyHostToDevice, st));
  if (!maps.empty())
    OXY_CUDA(cudaMemcpyAsync(d_maps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, st));
}

void Program::launch(cudaStream_t st) {
  static bool attr = false;
  static int sms = 0;
  if (!attr) {
    OXY_CUDA(cudaFuncSetAttribute(mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mk_smem_bytes()));
    int dev = 0;
    OXY_CUDA(cudaGetDevice(&dev));
    OXY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    attr = true;
  }
  if (phases.empty()) return;
  const int g = grid > 0 ? std::min(grid, sms) : sms;
  OXY_CUDA(cudaMemsetAsync(d_sync, 0, sizeof(unsigned), st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(MK_THREADS);
  cfg.dynamicSmemBytes = mk_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (profile && !d_times) OXY_CUDA(cudaMalloc(&d_times, cap_phases * (1 + 160) * sizeof(unsigned long long)));
  OXY_CUDA(cudaLaunchKernelEx(&cfg, mk_kernel, (const Phase *)d_phases, (int)phases.size(),
                              (const CUtensorMap *)d_maps, d_sync, profile ? d_times : nullptr));
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
}

}  // namespace mk
}  // namespace oxy
