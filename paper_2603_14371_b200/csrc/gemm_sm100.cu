// tcgen05 + TMA + TMEM GEMM for sm_100a (see gemm_sm100.cuh for the contract).
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM allocator + single-thread
// MMA issuer, warps 2-5 epilogue (warp w reads TMEM lanes 32*(w%4)..+31, i.e.
// output features, and loops over the BN token columns).  Stage ring of
// {A 128x64, B BNx64} bf16 tiles with full/empty mbarriers; tcgen05.commit
// releases a stage when the MMAs that read it retire.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

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

__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * x * (1.f + tanhf(c * (x + 0.044715f * x * x * x)));
}

// Shared epilogue.  `pair` is the accumulator of feature f^1 (GeGLU, RoPE).
// MODE >= 0 fixes the mode at compile time; MODE < 0 dispatches on e.mode.
template <int MODE = -1>
__device__ __forceinline__ void epilogue_store(const EpiParams &e, int t, int f, int n_out, float acc,
                                               float pair) {
  if (e.bias) acc += e.bias[f];
  switch (MODE >= 0 ? MODE : e.mode) {
    case EPI_F32:
      static_cast<float *>(e.out)[(size_t)t * e.ldo + f] = acc;
      break;
    case EPI_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] = __float2bfloat16(acc);
      break;
    case EPI_ADD_F32:
      static_cast<float *>(e.out)[(size_t)t * e.ldo + f] += acc;
      break;
    case EPI_GEGLU_BF16:
      if ((f & 1) == 0) {
        float up = pair + (e.bias ? e.bias[f + 1] : 0.f);
        static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + (f >> 1)] =
            __float2bfloat16(gelu_tanh(acc) * up);
      }
      break;
    case EPI_GELU_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] = __float2bfloat16(gelu_tanh(acc));
      break;
    case EPI_ADD_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] =
          __float2bfloat16(acc + e.res[(size_t)t * e.ldr + f]);
      break;
    case EPI_ADD_GATED_F32:
      static_cast<float *>(e.out)[(size_t)t * e.ldo + f] += e.gate[f] * acc;
      break;
    case EPI_SWISH_BF16:
      static_cast<__nv_bfloat16 *>(e.out)[(size_t)t * e.ldo + f] =
          __float2bfloat16(acc / (1.f + __expf(-acc)));
      break;
    case EPI_QKV_ROPE: {
      const QkvRope &r = e.rope;
      const int h = f >> 8, j = f & 255, i = j >> 1;
      if (h < 9) {  // q heads 0..7, k head 8: rotate the (x1, x2) pair
        float sn, cs;
        sincosf((float)r.pos[t] * r.inv_freq[i], &sn, &cs);
        const bool second = j & 1;  // this lane holds x2 (dim i + 128)
        const float v = second ? acc * cs + pair * sn : acc * cs - pair * sn;
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
      break;
    }
  }
}

struct KParams {
  int n_out, k, t, bn, stages, kb_total, splits, kb_per_split;
  EpiParams epi;
  float *ws;
  int *counters;  // one per (m, n) tile; self-resetting
  int fixup;      // 1: last-arriving split CTA reduces; 0: separate reduce kernel
  int prefetch;   // 1: issue the first ring of weight tiles before griddepcontrol.wait
  int trigger;    // 1: launch_dependents once all operand loads are issued
};

// Epilogue over this thread's output feature f and the tile's BN token columns
// (TMEM lane = f).  MODE < 0 writes split-K partials.
template <int MODE>
__device__ __forceinline__ void epi_loop(const KParams &p, uint32_t trow, int bn, int n0, int f, int split) {
  const bool fok = f < p.n_out;
  for (int c = 0; c < bn; c += 16) {
    uint32_t v[16];
    tmem_ld16(trow + (uint32_t)c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int t = n0 + c + j;
      const float acc = __uint_as_float(v[j]);
      float pair = 0.f;
      if (MODE == EPI_GEGLU_BF16 || MODE == EPI_QKV_ROPE) pair = __shfl_xor_sync(0xffffffffu, acc, 1);
      if (t >= p.t || !fok) continue;
      if (MODE < 0) p.ws[((size_t)split * p.t + t) * p.n_out + f] = acc;
      else epilogue_store<(MODE < 0 ? 0 : MODE)>(p.epi, t, f, p.n_out, acc, pair);
    }
  }
}

// Launch-time knobs (env, read once): OXY_SPLITK=fixup|kernel, OXY_PDL=0|1,
// OXY_GEMM_SMEM_KB=<per-CTA smem budget>.  Used for A/B measurements.
struct Knobs {
  int fixup = 0, pdl = 1, smem_kb = 100;  // 2 CTAs per SM (measured best)
  // early PDL (weight prefetch + trigger) for skinny / wide GEMMs: -1 = default policy
  int early_skinny = 1, early_wide = 0;
  Knobs() {
    if (const char *s = getenv("OXY_PDL_EARLY_SKINNY")) early_skinny = atoi(s);
    if (const char *s = getenv("OXY_PDL_EARLY_WIDE")) early_wide = atoi(s);
    if (const char *s = getenv("OXY_SPLITK")) fixup = std::string(s) == "fixup";
    if (const char *s = getenv("OXY_PDL")) pdl = atoi(s);
    if (const char *s = getenv("OXY_GEMM_SMEM_KB")) smem_kb = std::max(64, std::min(200, atoi(s)));
  }
};
static const Knobs &knobs() {
  static Knobs k;
  return k;
}

// Fixed-order split-K reduction + epilogue; one thread per feature pair.
__global__ void splitk_reduce_kernel(const float *ws, int splits, int t_rows, int n_out, EpiParams e) {
  pdl_trigger();
  pdl_wait();
  const int pairs = (n_out + 1) >> 1;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)t_rows * pairs) return;
  const int t = (int)(idx / pairs), f = (int)(idx % pairs) * 2;
  float a0 = 0.f, a1 = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float *row = ws + ((size_t)s * t_rows + t) * n_out;
    a0 += row[f];
    if (f + 1 < n_out) a1 += row[f + 1];
  }
  epilogue_store(e, t, f, n_out, a0, a1);
  if (f + 1 < n_out) epilogue_store(e, t, f + 1, n_out, a1, a0);
}

__global__ void __launch_bounds__(192, 2)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                KParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  const int bn = p.bn, stages = p.stages;
  const int b_bytes = bn * BK * 2;
  uint8_t *sA = smem;
  uint8_t *sB = smem + stages * A_STAGE_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + stages * b_bytes);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * MAX_STAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // token tiles fastest: the CTAs sharing one weight tile run in the same wave
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * bn, split = blockIdx.z;
  __shared__ int s_last;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kb_total, kb0 + p.kb_per_split) - kb0;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + MAX_STAGES),
                 done = smem_u32(bars + 2 * MAX_STAGES);
  uint32_t ncols = 32;
  while (ncols < (uint32_t)bn) ncols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      // Weights never depend on the previous kernel: stream the first ring of
      // weight tiles before waiting on it, activations after.
      const int pre = p.prefetch ? min(nkb, stages) : 0;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(full0 + 8 * i, A_STAGE_BYTES + b_bytes);
        tma_load_2d(&tmA, full0 + 8 * i, smem_u32(sA + i * A_STAGE_BYTES), (kb0 + i) * BK, m0);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(&tmB, full0 + 8 * i, smem_u32(sB + i * b_bytes), (kb0 + i) * BK, n0);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (i / stages) & 1;
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        mbar_expect_tx(full0 + 8 * s, A_STAGE_BYTES + b_bytes);
        const int kc = (kb0 + i) * BK;
        tma_load_2d(&tmA, full0 + 8 * s, smem_u32(sA + s * A_STAGE_BYTES), kc, m0);
        tma_load_2d(&tmB, full0 + 8 * s, smem_u32(sB + s * b_bytes), kc, n0);
      }
      // all operand loads are in flight: let the next kernel start its
      // prologue and weight prefetch while this CTA drains
      if (p.trigger) pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % stages;
        const uint32_t ph = (i / stages) & 1;
        mbar_wait(full0 + 8 * s, ph);
        tc_fence_after();
        const uint32_t a = smem_u32(sA + s * A_STAGE_BYTES), b = smem_u32(sB + s * b_bytes);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          mma_bf16(tmem, make_sdesc(a + kk * 32), make_sdesc(b + kk * 32), idesc,
                   (i | kk) != 0 ? 1u : 0u);
        mma_commit(empty0 + 8 * s);
      }
      mma_commit(done);
    }
    __syncwarp();
  } else {
    pdl_wait();  // the epilogue reads bias/residual/gates and writes outputs
    mbar_wait(done, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int f = m0 + q * 32 + lane;
    const bool split_out = p.splits > 1;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    // the mode switch sits outside the column loop: one tight loop per epilogue
    switch (split_out ? -1 : p.epi.mode) {
      case -1: epi_loop<-1>(p, trow, bn, n0, f, split); break;
      case EPI_F32: epi_loop<EPI_F32>(p, trow, bn, n0, f, split); break;
      case EPI_BF16: epi_loop<EPI_BF16>(p, trow, bn, n0, f, split); break;
      case EPI_ADD_F32: epi_loop<EPI_ADD_F32>(p, trow, bn, n0, f, split); break;
      case EPI_GEGLU_BF16: epi_loop<EPI_GEGLU_BF16>(p, trow, bn, n0, f, split); break;
      case EPI_GELU_BF16: epi_loop<EPI_GELU_BF16>(p, trow, bn, n0, f, split); break;
      case EPI_ADD_BF16: epi_loop<EPI_ADD_BF16>(p, trow, bn, n0, f, split); break;
      case EPI_ADD_GATED_F32: epi_loop<EPI_ADD_GATED_F32>(p, trow, bn, n0, f, split); break;
      case EPI_SWISH_BF16: epi_loop<EPI_SWISH_BF16>(p, trow, bn, n0, f, split); break;
      case EPI_QKV_ROPE: epi_loop<EPI_QKV_ROPE>(p, trow, bn, n0, f, split); break;
    }
    if (split_out && p.fixup) {
      // Deterministic split-K fix-up: the last CTA of this tile to arrive sums
      // the partials in split order 0..S-1 and applies the epilogue.
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int tile = blockIdx.y * gridDim.x + blockIdx.x;
      if (threadIdx.x == 64) s_last = atomicAdd(p.counters + tile, 1) == p.splits - 1;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (s_last) {
        __threadfence();
        const int ncols = min(bn, p.t - n0);
        const bool fok = f < p.n_out;
        for (int c0 = 0; c0 < ncols; c0 += 4) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (int s0 = 0; s0 < p.splits; s0 += 8) {
            float v[8][4];  // 32 independent L2 loads in flight per thread
#pragma unroll
            for (int s = 0; s < 8; ++s)
#pragma unroll
              for (int j = 0; j < 4; ++j)
                v[s][j] = (fok && s0 + s < p.splits && c0 + j < ncols)
                              ? __ldcg(p.ws + ((size_t)(s0 + s) * p.t + n0 + c0 + j) * p.n_out + f)
                              : 0.f;
#pragma unroll
            for (int s = 0; s < 8; ++s)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[j] += v[s][j];  // split order 0..S-1
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float pair = __shfl_xor_sync(0xffffffffu, acc[j], 1);
            if (fok && c0 + j < ncols) epilogue_store(p.epi, n0 + c0 + j, f, p.n_out, acc[j], pair);
          }
        }
        if (threadIdx.x == 64) p.counters[tile] = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    OXY_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) fail(OXY_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// rows x k bf16 row-major, box (64 x box_rows), 128-byte swizzle
CUtensorMap make_map(const void *ptr, int rows, int k, int box_rows) {
  if ((k * 2) % 16 != 0) fail(OXY_EINVAL, "GEMM K=%d: row stride must be a multiple of 16 bytes", k);
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) fail(OXY_EINVAL, "GEMM operand not 16-byte aligned");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(OXY_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return map;
}

Plan make_plan(int n_out, int k, int t, int sms, int force_splits) {
  Plan p{};
  p.kb_total = (k + BK - 1) / BK;
  p.m_tiles = (n_out + BM - 1) / BM;
  p.n_tiles = (t + MAX_BN - 1) / MAX_BN;
  // wide token dims (prefill): narrower token tiles until the grid fills the SMs
  while (t > 64 && p.m_tiles * p.n_tiles < sms && (t + p.n_tiles) / (p.n_tiles + 1) >= 48) ++p.n_tiles;
  int per = (t + p.n_tiles - 1) / p.n_tiles;
  p.bn = std::max(16, (per + 15) / 16 * 16);
  p.n_tiles = (t + p.bn - 1) / p.bn;
  const int base = p.m_tiles * p.n_tiles;
  int splits = 1;
  if (force_splits > 0) {
    splits = force_splits;
  } else if (base < sms && t <= 64) {  // skinny (decode / denoise): split K, tiny fix-up
    splits = std::max(1, std::min(sms / base, p.kb_total / 4));
  }
  splits = std::max(1, std::min(splits, p.kb_total));
  const int per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + per_split - 1) / per_split;
  p.stages = std::max(2, std::min(MAX_STAGES, knobs().smem_kb * 1024 / (A_STAGE_BYTES + p.bn * BK * 2)));
  return p;
}

static size_t smem_bytes(const Plan &p) {
  return 1024 + (size_t)p.stages * (A_STAGE_BYTES + p.bn * BK * 2) + (2 * MAX_STAGES + 1) * 8 + 16;
}

void launch(const void *w, const void *x, int n_out, int k, int t, const EpiParams &epi,
            const Plan &plan, float *ws, int *counters, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    OXY_CUDA(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  226 * 1024));  // + static smem stays under 227 KB
    attr_set = true;
  }
  if (t <= 0) return;
  if (plan.splits > 1 && (!ws || !counters)) fail(OXY_EINVAL, "split-K GEMM needs a workspace");
  if (plan.splits > 1 && plan.m_tiles * plan.n_tiles > MAX_TILES) fail(OXY_EINVAL, "too many split-K tiles");
  CUtensorMap ma = make_map(w, n_out, k, BM);
  CUtensorMap mb = make_map(x, t, k, plan.bn);
  KParams kp;
  kp.n_out = n_out;
  kp.k = k;
  kp.t = t;
  kp.bn = plan.bn;
  kp.stages = plan.stages;
  kp.kb_total = plan.kb_total;
  kp.splits = plan.splits;
  kp.kb_per_split = (plan.kb_total + plan.splits - 1) / plan.splits;
  kp.epi = epi;
  kp.ws = ws;
  kp.counters = counters;
  kp.fixup = knobs().fixup;
  kp.prefetch = kp.trigger = t <= 64 ? knobs().early_skinny : knobs().early_wide;
  dim3 grid(plan.n_tiles, plan.m_tiles, plan.splits);
  if (knobs().pdl) {
    launch_pdl(gemm_kernel, grid, dim3(192), smem_bytes(plan), st, ma, mb, kp);
  } else {
    gemm_kernel<<<grid, 192, smem_bytes(plan), st>>>(ma, mb, kp);
    OXY_LAUNCH_CHECK();
  }
  if (plan.splits > 1 && !kp.fixup && epi.mode != EPI_PARTIALS) {
    const int64_t n = (int64_t)t * ((n_out + 1) / 2);
    if (knobs().pdl) {
      launch_pdl(splitk_reduce_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, ws, plan.splits, t,
                 n_out, epi);
    } else {
      splitk_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ws, plan.splits, t, n_out, epi);
      OXY_LAUNCH_CHECK();
    }
  }
}

// one 1024-thread CTA per token row (memory-level parallelism for the skinny
// decode/denoise rows); thread owns features tid, tid+1024 (coalesced)
constexpr int RN_THREADS = 1024, RN_MAXV = 2;  // n <= 2048
__global__ void __launch_bounds__(RN_THREADS)
    splitk_residual_norm_kernel(const float *ws, int splits, int t_rows, int n, const float *gate, float *x,
                                int ldx, __nv_bfloat16 *y, int ldy, const float *w, const float *ms,
                                const float *mb, float eps) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int t = blockIdx.x;
  float v[RN_MAXV] = {0.f, 0.f};
#pragma unroll 8
  for (int s = 0; s < splits; ++s) {  // split order 0..S-1 per element
    const float *row = ws + ((size_t)s * t_rows + t) * n;
#pragma unroll
    for (int i = 0; i < RN_MAXV; ++i) {
      const int f = threadIdx.x + i * RN_THREADS;
      if (f < n) v[i] += row[f];
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < RN_MAXV; ++i) {
    const int f = threadIdx.x + i * RN_THREADS;
    if (f < n) {
      float xv = x[(size_t)t * ldx + f];
      xv += gate ? gate[f] * v[i] : v[i];
      x[(size_t)t * ldx + f] = xv;
      v[i] = xv;
      ss += xv * xv;
    }
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / (float)n + eps);
#pragma unroll
  for (int i = 0; i < RN_MAXV; ++i) {
    const int f = threadIdx.x + i * RN_THREADS;
    if (f < n) {
      const float o = w ? v[i] * inv * (1.f + w[f]) : v[i] * inv * (1.f + ms[f]) + mb[f];
      y[(size_t)t * ldy + f] = __float2bfloat16(o);
    }
  }
}

void splitk_residual_norm(const float *ws, int splits, int t, int n, const float *gate, float *x, int ldx,
                          __nv_bfloat16 *y, int ldy, const float *w, const float *mod_scale,
                          const float *mod_shift, float eps, cudaStream_t st) {
  if (t <= 0) return;
  if (n > RN_THREADS * RN_MAXV) fail(OXY_EINVAL, "fused residual norm supports rows of at most 2048");
  launch_pdl(splitk_residual_norm_kernel, dim3(t), dim3(RN_THREADS), 0, st, ws, splits, t, n, gate, x, ldx, y, ldy, w,
             mod_scale, mod_shift, eps);
}

int *counters_for_abi() {
  static int *c = nullptr;
  if (!c) {
    OXY_CUDA(cudaMalloc(&c, MAX_TILES * sizeof(int)));
    OXY_CUDA(cudaMemset(c, 0, MAX_TILES * sizeof(int)));
  }
  return c;
}

}  // namespace gemm
}  // namespace oxy

extern "C" int oxy_gemm_bf16(const void *w_d, const void *x_d, int32_t n_out, int32_t k, int32_t t,
                             int32_t mode, void *out_d, int32_t ldo, const float *bias_d,
                             const float *res_d, int32_t ldr, int32_t splits, float *ws_d,
                             int64_t ws_floats, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(n_out > 0 && k > 0 && t >= 0, "bad GEMM shape");
  OXY_REQUIRE(mode >= 0 && mode <= 5, "unknown epilogue mode %d (0-5 via the C ABI)", mode);
  int dev = 0, sms = 148;
  OXY_CUDA(cudaGetDevice(&dev));
  OXY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  oxy::gemm::Plan plan = oxy::gemm::make_plan(n_out, k, t, sms, splits);
  if (plan.splits > 1)
    OXY_REQUIRE(ws_d && ws_floats >= (int64_t)plan.splits * t * n_out,
                "split-K workspace too small (%lld floats needed)",
                (long long)plan.splits * t * n_out);
  oxy::gemm::EpiParams e{mode, out_d, ldo, bias_d, res_d, ldr, nullptr};
  oxy::gemm::launch(w_d, x_d, n_out, k, t, e, plan, ws_d, oxy::gemm::counters_for_abi(),
                    oxy::as_stream(stream));
  OXY_API_END
}

extern "C" int oxy_gemm_plan(int32_t n_out, int32_t k, int32_t t, int32_t splits, int32_t *out6) {
  OXY_API_BEGIN
  oxy::gemm::Plan p = oxy::gemm::make_plan(n_out, k, t, 148, splits);
  out6[0] = p.bn;
  out6[1] = p.n_tiles;
  out6[2] = p.m_tiles;
  out6[3] = p.splits;
  out6[4] = p.stages;
  out6[5] = p.kb_total;
  OXY_API_END
}
