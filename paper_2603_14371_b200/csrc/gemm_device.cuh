// Device-side building blocks of the tcgen05 GEMM shared by the stand-alone
// kernels (gemm_sm100.cu) and the persistent layer kernel (megakernel.cu):
// PTX wrappers (mbarrier, TMA, tcgen05, cluster), the fused epilogues, and the
// deterministic split-K fix-up.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "cuda_util.cuh"
#include "gemm_sm100.cuh"

namespace oxy {
namespace gemm {

// ------------------------------------------------------------------ PTX

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t"
      "}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// One lane of a converged warp (elect.sync).  The MMA-issuing loops run on the whole
// warp and issue from the elected lane: with the loop warp-uniform the compiler keeps
// descriptors and addresses in uniform registers; a loop under `if (lane == 0)` had
// every tcgen05.mma wrapped in an R2UR.BROADCAST / elect re-convergence loop.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// A long wait (an epilogue warp waiting for the next accumulator): poll with a sleep
// between probes so the waiting warps do not compete with the tensor pipe's shared-
// memory traffic.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, int ns) {
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint32_t bar, uint32_t dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// K-major, 128-byte swizzle: 8-row atoms of 1024 B (SBO), version 1 (sm100).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;            // descriptor version
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- cluster / CTA-pair helpers (cta_group::2)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// pair TMA: the bytes land in this CTA's smem, completion is counted on the
// leader CTA's barrier (bar_leader = shared::cluster address in CTA 0)
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap *map, uint32_t bar_leader, uint32_t dst, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_leader), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}
// arrive on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

// Epilogue arithmetic is written with explicit rounding intrinsics (no FMA
// contraction or re-association left to the compiler, which may decide
// differently in each kernel it inlines into): every kernel variant (one-tile,
// persistent 1-/2-CTA) and every epilogue path (direct, staged bf16, split
// reduce, split fix-up) then computes an output element bit-identically — the
// batch-invariant plans (gemm::policy_splits) rely on it.
//
// GELU (tanh form) on the SFU: tanh.approx.f32 (rel. error ~2^-11, far below
// the bf16 rounding of the stored activation)
__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  const float x3 = __fmul_rn(__fmul_rn(x, x), x);
  const float u = __fmul_rn(c, __fmaf_rn(0.044715f, x3, x));
  float th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(u));
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.f, th));
}
__device__ __forceinline__ float geglu(float g, float up) { return __fmul_rn(gelu_tanh(g), up); }
__device__ __forceinline__ float swish(float x) { return __fdiv_rn(x, __fadd_rn(1.f, __expf(-x))); }
// rotary pair: x1' = x1 c - x2 s (first), x2' = x2 c + x1 s (second)
__device__ __forceinline__ float rope_rot(bool second, float acc, float pair, float cs, float sn) {
  return __fmaf_rn(acc, cs, second ? __fmul_rn(pair, sn) : -__fmul_rn(pair, sn));
}

// RoPE + q / k / v routing of one accumulator (rotary pairs interleaved in the
// weight rows), with (cs, sn) of this token's position already loaded
__device__ __forceinline__ void rope_store(const QkvRope &r, int t, int f, float acc, float pair, float cs,
                                           float sn) {
  const int h = f >> 8, j = f & 255, i = j >> 1;
  if (h < 9) {  // q heads 0..7, k head 8: rotate the (x1, x2) pair
    const bool second = j & 1;  // this lane holds x2 (dim i + 128)
    const float v = rope_rot(second, acc, pair, cs, sn);
    const int dim = second ? i + 128 : i;
    if (h < 8) {
      r.q_out[(size_t)t * 2048 + h * 256 + dim] = __float2bfloat16(v);
    } else {
      const int s = r.slot ? r.slot[t] : t;
      if (s >= 0) r.k_dst[(size_t)s * 256 + dim] = __float2bfloat16(v);
    }
  } else {  // v head
    const int s = r.slot ? r.slot[t] : t;
    if (s >= 0) r.v_dst[(size_t)s * 256 + j] = __float2bfloat16(acc);
  }
}

// rope_store with the k / v destination slot already loaded (s < 0: dropped)
__device__ __forceinline__ void rope_store_slot(const QkvRope &r, int t, int s, int f, float acc, float pair,
                                                float cs, float sn) {
  const int h = f >> 8, j = f & 255, i = j >> 1;
  if (h < 9) {
    const bool second = j & 1;
    const float v = rope_rot(second, acc, pair, cs, sn);
    const int dim = second ? i + 128 : i;
    if (h < 8) r.q_out[(size_t)t * 2048 + h * 256 + dim] = __float2bfloat16(v);
    else if (s >= 0) r.k_dst[(size_t)s * 256 + dim] = __float2bfloat16(v);
  } else if (s >= 0) {
    r.v_dst[(size_t)s * 256 + j] = __float2bfloat16(acc);
  }
}

__device__ __forceinline__ float2 rope_cs(const QkvRope &r, int pos, int i) {
  if (r.cs && pos < ROPE_TABLE_POS) return __ldg(r.cs + (size_t)pos * 128 + i);
  float sn, cs;
  sincosf(__fmul_rn((float)pos, r.inv_freq[i]), &sn, &cs);
  return make_float2(cs, sn);
}

// Shared epilogue.  `pair` is the accumulator of feature f^1 (GeGLU, RoPE).
// MODE >= 0 fixes the mode at compile time; MODE < 0 dispatches on e.mode.
template <int MODE = -1>
__device__ __forceinline__ void epilogue_store(const EpiParams &e, int t, int f, int n_out, float acc,
                                               float pair) {
  if (e.bias) acc = __fadd_rn(acc, e.bias[f]);
  switch (MODE >= 0 ? MODE : e.mode) {
    case EPI_F32:
      static_cast<float *>(e.out)[(size_t)t * e.ldo + f] = acc;
      break;
    case EPI_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] = __float2bfloat16(acc);
      break;
    case EPI_ADD_F32:
      static_cast<float *>(e.out)[(size_t)t * e.ldo + f] = __fadd_rn(static_cast<float *>(e.out)[(size_t)t * e.ldo + f], acc);
      break;
    case EPI_GEGLU_BF16:
      if ((f & 1) == 0) {
        const float up = __fadd_rn(pair, e.bias ? e.bias[f + 1] : 0.f);
        static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + (f >> 1)] = __float2bfloat16(geglu(acc, up));
      }
      break;
    case EPI_GELU_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] = __float2bfloat16(gelu_tanh(acc));
      break;
    case EPI_ADD_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] =
          __float2bfloat16(__fadd_rn(acc, e.res[(size_t)t * e.ldr + f]));
      break;
    case EPI_ADD_GATED_F32:
      static_cast<float *>(e.out)[(size_t)t * e.ldo + f] =
          __fmaf_rn(e.gate[f], acc, static_cast<float *>(e.out)[(size_t)t * e.ldo + f]);
      break;
    case EPI_SWISH_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] =
          __float2bfloat16(swish(acc));
      break;
    case EPI_QKV_ROPE: {
      const QkvRope &r = e.rope;
      const float2 c = rope_cs(r, r.pos[t], (f & 255) >> 1);
      rope_store(r, t, f, acc, pair, c.x, c.y);
      break;
    }
  }
}

// Staged bf16 store of one 16-token chunk.  Lane l of the warp holds y[j] for
// feature f0 + l and token j; the warp transposes the chunk through a private
// smem tile (16 rows x 36 floats: conflict-free row writes and float4 reads)
// and each lane then writes 16-byte vectors of consecutive output columns of
// one token, instead of 16 two-byte stores per lane.  KIND 0: column f (32
// columns from f0); 1: GeGLU, column f/2 from the even lanes (16 columns);
// 2: RoPE q, dims i0.. from the even lanes and 128 + i0.. from the odd ones.
// out0 = the chunk's first token row at the warp's first column; ncols =
// valid columns from there (KIND 0 / 1).  Returns after the warp's stores.
constexpr int STG_LD = 36;
template <int KIND>
__device__ __forceinline__ void stage_store_bf16(float *stg, const float (&y)[16], int nvt, __nv_bfloat16 *out0,
                                                 size_t ld, int ncols) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 16; ++j) stg[j * STG_LD + lane] = y[j];
  __syncwarp();
  const int j = lane >> 1, h = lane & 1;
  if (j >= nvt) return;
  const float *row = stg + j * STG_LD;
  constexpr int N = KIND == 1 ? 8 : 16;
  float x[16];
  int col;
  if constexpr (KIND == 0) {
    col = 16 * h;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 a = *reinterpret_cast<const float4 *>(row + 16 * h + 4 * q);
      x[4 * q] = a.x;
      x[4 * q + 1] = a.y;
      x[4 * q + 2] = a.z;
      x[4 * q + 3] = a.w;
    }
  } else if constexpr (KIND == 1) {
    col = 8 * h;
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = row[2 * (8 * h + k)];
  } else {
    col = 128 * h;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = row[2 * k + h];
  }
  __nv_bfloat16 *dst = out0 + (size_t)j * ld + col;
  uint32_t w[8];
#pragma unroll
  for (int k = 0; k < N / 2; ++k) {
    __nv_bfloat162 b = __floats2bfloat162_rn(x[2 * k], x[2 * k + 1]);
    w[k] = *reinterpret_cast<uint32_t *>(&b);
  }
  const bool full = KIND == 2 || col + N <= ncols;
  if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    if constexpr (N == 16) *reinterpret_cast<uint4 *>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (KIND == 2 || col + k < ncols) dst[k] = __float2bfloat16(x[k]);
  }
}

// Epilogue over this thread's output feature f and the tile's BN token columns
// (TMEM lane = f).  MODE < 0 writes split-K partials.  Per 16-token chunk every
// load (per-feature bias / gate once, the chunk's residual or RoPE operands)
// is issued before any store, and stores are predicated, not branched: the
// compiler cannot prove the outputs do not alias the operands, so a
// load-after-store per token serialised the epilogue on L2 latency, and one
// divergent region per token cost ~1 us per 16-token chunk (tools/gemm_prof.py).
// Accumulator sources of epi_loop: src(c, nv, v) fills v[0..16) with the fp32
// accumulators (as bits) of tile columns c..c+15 of this thread's feature
// (entries >= nv are don't-care).  TmemSrc is warp-collective.
struct TmemSrc {
  uint32_t trow;
  __device__ __forceinline__ void operator()(int c, int, uint32_t (&v)[16]) const { tmem_ld16(trow + (uint32_t)c, v); }
};

// Cluster split-K: the sum of the S split partials ws[s, t, f] in split order
// 0..S-1 (the order every other reduction path uses).  The loads of one round
// are all issued before any add; the round shape follows the chunk width so a
// slice of T/S tokens costs one L2 round trip whatever S is.
struct SplitSumSrc {
  const float *ws;
  int splits, t, n_out, n0, f;
  bool fok;
  template <int J, int U>
  __device__ __forceinline__ void rounds(int t0, int nv, float (&a)[16]) const {
    for (int s0 = 0; s0 < splits; s0 += U) {
      float v[U][J];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < J; ++j)
          v[u][j] = (fok && j < nv && s0 + u < splits)
                        ? __ldcg(ws + ((size_t)(s0 + u) * t + t0 + j) * n_out + f)
                        : 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < J; ++j)
          if (s0 + u < splits) a[j] = __fadd_rn(a[j], v[u][j]);
    }
  }
  __device__ __forceinline__ void operator()(int c, int nv, uint32_t (&v)[16]) const {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = 0.f;
    const int t0 = n0 + c;
    if (nv <= 4) rounds<4, 8>(t0, nv, a);
    else if (nv <= 8) rounds<8, 4>(t0, nv, a);
    else rounds<16, 2>(t0, nv, a);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(a[j]);
  }
};

template <int MODE, typename P, typename SRC>
__device__ __forceinline__ void epi_loop(const P &p, const SRC &src, int c_begin, int c_end, int n0, int f, int split,
                                         float *stg = nullptr) {
  const bool fok = f < p.n_out;
  const EpiParams &e = p.epi;
  if constexpr (MODE == EPI_QKV_ROPE) {
    const QkvRope &r = e.rope;
    const int i = (f & 255) >> 1;
    const bool kv = (f >> 8) >= 8;  // k / v head rows: routed through the slot table
    for (int c = c_begin; c < c_end; c += 16) {
      uint32_t v[16];
      const int t0 = n0 + c;
      const int nvt = max(0, min(min(16, c_end - c), p.t - t0));  // valid tokens of the chunk
      const int nv = fok ? nvt : 0;
      src(c, nv, v);
      int pos[16], sl[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        pos[j] = j < nv ? __ldg(r.pos + t0 + j) : 0;
        sl[j] = kv && j < nv ? (r.slot ? r.slot[t0 + j] : t0 + j) : -1;
      }
      // one chunk-uniform table test, then 16 independent table loads (a
      // per-token table-or-sincosf branch serialised them: 14 us per chunk)
      int pmax = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) pmax = max(pmax, pos[j]);
      float2 csn[16];
      if (r.cs && pmax < ROPE_TABLE_POS) {
#pragma unroll
        for (int j = 0; j < 16; ++j) csn[j] = __ldg(r.cs + (size_t)pos[j] * 128 + i);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) csn[j] = rope_cs(r, pos[j], i);
      }
      if (stg && !kv) {  // q heads (warp-uniform: a warp's 32 features lie in one head)
        const int hd = f >> 8, second = f & 1;
        float y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float acc = __uint_as_float(v[j]);
          const float pair = __shfl_xor_sync(0xffffffffu, acc, 1);
          y[j] = rope_rot(second, acc, pair, csn[j].x, csn[j].y);
        }
        const int i0 = ((f - (threadIdx.x & 31)) & 255) >> 1;
        stage_store_bf16<2>(stg, y, nvt, r.q_out + (size_t)t0 * 2048 + hd * 256 + i0, 2048, 0);
        continue;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float acc = __uint_as_float(v[j]);
        const float pair = __shfl_xor_sync(0xffffffffu, acc, 1);
        if (j < nv) rope_store_slot(r, t0 + j, sl[j], f, acc, pair, csn[j].x, csn[j].y);
      }
    }
  } else {
    const float bias = (MODE >= 0 && e.bias && fok) ? __ldg(e.bias + f) : 0.f;
    const float bias_up = (MODE == EPI_GEGLU_BF16 && e.bias && fok) ? __ldg(e.bias + (f | 1)) : 0.f;
    const float gate = (MODE == EPI_ADD_GATED_F32 && fok) ? __ldg(e.gate + f) : 0.f;
    for (int c = c_begin; c < c_end; c += 16) {
      uint32_t v[16];
      const int t0 = n0 + c;
      const int nvt = max(0, min(min(16, c_end - c), p.t - t0));  // valid tokens of the chunk
      const int nv = fok ? nvt : 0;
      src(c, nv, v);
      if constexpr (MODE < 0) {
        float *dst = p.ws + ((size_t)split * p.t + t0) * p.n_out + f;
        const size_t ld = p.n_out;
        if (nv == 16) {  // full chunk: straight-line stores
#pragma unroll
          for (int j = 0; j < 16; ++j) dst[j * ld] = __uint_as_float(v[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nv) dst[j * ld] = __uint_as_float(v[j]);
        }
      } else if constexpr (MODE == EPI_ADD_F32 || MODE == EPI_ADD_GATED_F32 || MODE == EPI_ADD_BF16) {
        const float *src = MODE == EPI_ADD_BF16 ? e.res + (size_t)t0 * e.ldr + f
                                                : static_cast<const float *>(e.out) + (size_t)t0 * e.ldo + f;
        const int lds = MODE == EPI_ADD_BF16 ? e.ldr : e.ldo;
        float old[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) old[j] = j < nv ? src[(size_t)j * lds] : 0.f;
        auto put = [&](int j) {
          const float acc = __fadd_rn(__uint_as_float(v[j]), bias);
          const size_t o = (size_t)(t0 + j) * e.ldo + f;
          if constexpr (MODE == EPI_ADD_F32) static_cast<float *>(e.out)[o] = __fadd_rn(old[j], acc);
          else if constexpr (MODE == EPI_ADD_GATED_F32) static_cast<float *>(e.out)[o] = __fmaf_rn(gate, acc, old[j]);
          else static_cast<__nv_bfloat16 *>(e.out)[o] = __float2bfloat16(__fadd_rn(acc, old[j]));
        };
        if (nv == 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) put(j);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nv) put(j);
        }
      } else if (MODE != EPI_F32 && stg != nullptr && (e.ldo & 7) == 0) {  // bf16 outputs, staged
        const int f0 = f - (int)(threadIdx.x & 31);
        float y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float acc = __fadd_rn(__uint_as_float(v[j]), bias);
          if constexpr (MODE == EPI_GEGLU_BF16) {
            const float pr = __shfl_xor_sync(0xffffffffu, __uint_as_float(v[j]), 1);
            y[j] = geglu(acc, __fadd_rn(pr, bias_up));
          } else if constexpr (MODE == EPI_GELU_BF16) {
            y[j] = gelu_tanh(acc);
          } else if constexpr (MODE == EPI_SWISH_BF16) {
            y[j] = swish(acc);
          } else {
            y[j] = acc;
          }
        }
        __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(e.out) + (size_t)t0 * e.ldo;
        if constexpr (MODE == EPI_GEGLU_BF16)
          stage_store_bf16<1>(stg, y, nvt, o + (f0 >> 1), e.ldo, (p.n_out - f0) >> 1);
        else
          stage_store_bf16<0>(stg, y, nvt, o + f0, e.ldo, p.n_out - f0);
      } else {
        float pair[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pair[j] = MODE == EPI_GEGLU_BF16 ? __shfl_xor_sync(0xffffffffu, __uint_as_float(v[j]), 1) : 0.f;
        auto put = [&](int j) {
          const float acc = __fadd_rn(__uint_as_float(v[j]), bias);
          const size_t o = (size_t)(t0 + j) * e.ldo + f;
          if constexpr (MODE == EPI_F32) {
            static_cast<float *>(e.out)[o] = acc;
          } else if constexpr (MODE == EPI_BF16) {
            static_cast<__nv_bfloat16 *>(e.out)[o] = __float2bfloat16(acc);
          } else if constexpr (MODE == EPI_GEGLU_BF16) {
            if ((f & 1) == 0)
              static_cast<__nv_bfloat16 *>(e.out)[(size_t)(t0 + j) * e.ldo + (f >> 1)] =
                  __float2bfloat16(geglu(acc, __fadd_rn(pair[j], bias_up)));
          } else if constexpr (MODE == EPI_GELU_BF16) {
            static_cast<__nv_bfloat16 *>(e.out)[o] = __float2bfloat16(gelu_tanh(acc));
          } else if constexpr (MODE == EPI_SWISH_BF16) {
            static_cast<__nv_bfloat16 *>(e.out)[o] = __float2bfloat16(swish(acc));
          }
        };
        if (nv == 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) put(j);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nv) put(j);
        }
      }
    }
  }
}

// the mode switch sits outside the column loop: one tight loop per epilogue.
// Columns [c_begin, c_end) of the tile (chunks of 16 from c_begin).
template <typename P, typename SRC>
__device__ __forceinline__ void epi_tile_src(const P &p, const SRC &src, int c_begin, int c_end, int n0, int f,
                                             int split, bool split_out, float *stg = nullptr) {
  switch (split_out ? -1 : p.epi.mode) {
    case -1: epi_loop<-1>(p, src, c_begin, c_end, n0, f, split); break;
    case EPI_F32: epi_loop<EPI_F32>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_BF16: epi_loop<EPI_BF16>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_ADD_F32: epi_loop<EPI_ADD_F32>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_GEGLU_BF16: epi_loop<EPI_GEGLU_BF16>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_GELU_BF16: epi_loop<EPI_GELU_BF16>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_ADD_BF16: epi_loop<EPI_ADD_BF16>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_ADD_GATED_F32: epi_loop<EPI_ADD_GATED_F32>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_SWISH_BF16: epi_loop<EPI_SWISH_BF16>(p, src, c_begin, c_end, n0, f, split, stg); break;
    case EPI_QKV_ROPE: epi_loop<EPI_QKV_ROPE>(p, src, c_begin, c_end, n0, f, split, stg); break;
  }
}
template <typename P>
__device__ __forceinline__ void epi_tile(const P &p, uint32_t trow, int c_begin, int c_end, int n0, int f, int split,
                                         bool split_out, float *stg = nullptr) {
  epi_tile_src(p, TmemSrc{trow}, c_begin, c_end, n0, f, split, split_out, stg);
}

// Deterministic split-K fix-up, run by the epilogue warps (named barrier 1 over
// bar_threads threads; `leader` does the tile-counter atomic) after they wrote
// this CTA's partials: the last CTA of the tile to arrive sums the partials in
// split order 0..S-1 (columns [c_begin, c_end) of feature f per thread) and
// applies the epilogue (mode fixed at compile time, as in epi_loop).
template <int MODE, typename P>
__device__ __forceinline__ void fixup_sum(const P &p, int n0, int c_begin, int c_end, int f) {
  const int ce = min(c_end, p.t - n0);
  const bool fok = f < p.n_out;
  for (int c0 = c_begin; c0 < ce; c0 += 16) {
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
    for (int s = 0; s < p.splits; ++s) {  // split order 0..S-1; 16 loads in flight per split
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = (fok && c0 + j < ce) ? __ldcg(p.ws + ((size_t)s * p.t + n0 + c0 + j) * p.n_out + f) : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] += v[j];
    }
    if constexpr (MODE == EPI_QKV_ROPE) {
      const QkvRope &r = p.epi.rope;
      const int i = (f & 255) >> 1;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = n0 + c0 + j;
        const float pair = __shfl_xor_sync(0xffffffffu, acc[j], 1);
        if (fok && c0 + j < ce) {
          const float2 c = rope_cs(r, __ldg(r.pos + t), i);
          rope_store(r, t, f, acc[j], pair, c.x, c.y);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float pair = __shfl_xor_sync(0xffffffffu, acc[j], 1);
        if (fok && c0 + j < ce) epilogue_store<MODE>(p.epi, n0 + c0 + j, f, p.n_out, acc[j], pair);
      }
    }
  }
}

template <typename P>
__device__ __forceinline__ void splitk_fixup(const P &p, int tile, int n0, int c_begin, int c_end, int f, int &s_last,
                                             int bar_threads, int leader) {
  // the CTA's partial stores are ordered before the leader's release by bar.sync
  // (cumulativity); the leader's acquire + bar.sync orders the reads after every
  // other split's release
  asm volatile("bar.sync 1, %0;" ::"r"(bar_threads) : "memory");
  if ((int)threadIdx.x == leader) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(p.counters + tile) : "memory");
    s_last = old == p.splits - 1;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(bar_threads) : "memory");
  if (s_last) {
    switch (p.epi.mode) {
      case EPI_F32: fixup_sum<EPI_F32>(p, n0, c_begin, c_end, f); break;
      case EPI_BF16: fixup_sum<EPI_BF16>(p, n0, c_begin, c_end, f); break;
      case EPI_ADD_F32: fixup_sum<EPI_ADD_F32>(p, n0, c_begin, c_end, f); break;
      case EPI_GEGLU_BF16: fixup_sum<EPI_GEGLU_BF16>(p, n0, c_begin, c_end, f); break;
      case EPI_GELU_BF16: fixup_sum<EPI_GELU_BF16>(p, n0, c_begin, c_end, f); break;
      case EPI_ADD_BF16: fixup_sum<EPI_ADD_BF16>(p, n0, c_begin, c_end, f); break;
      case EPI_ADD_GATED_F32: fixup_sum<EPI_ADD_GATED_F32>(p, n0, c_begin, c_end, f); break;
      case EPI_SWISH_BF16: fixup_sum<EPI_SWISH_BF16>(p, n0, c_begin, c_end, f); break;
      case EPI_QKV_ROPE: fixup_sum<EPI_QKV_ROPE>(p, n0, c_begin, c_end, f); break;
      default: break;
    }
    if ((int)threadIdx.x == leader) p.counters[tile] = 0;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(bar_threads) : "memory");  // s_last is reused by the next tile
}

}  // namespace gemm
}  // namespace oxy
