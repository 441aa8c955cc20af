// tcgen05 + TMA + TMEM GEMM for sm_100a (see gemm_sm100.cuh for the contract).
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM allocator + single-thread
// MMA issuer, warps 2-5 epilogue (warp w reads TMEM lanes 32*(w%4)..+31, i.e.
// output features, and loops over the BN token columns).  Stage ring of
// {A 128x64, B BNx64} bf16 tiles with full/empty mbarriers; tcgen05.commit
// releases a stage when the MMAs that read it retire.
#include <algorithm>
#include <array>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "cuda_util.cuh"
#include "gemm_sm100.cuh"
#include "gemm_device.cuh"

namespace oxy {
namespace gemm {

struct KParams {
  int n_out, k, t, bn, stages, kb_total, splits, kb_per_split;
  EpiParams epi;
  float *ws;
  int *counters;  // one per (m, n) tile; self-resetting
  int fixup;      // 1: last-arriving split CTA reduces; 0: separate reduce kernel
  int prefetch;   // 1: issue the first ring of weight tiles before griddepcontrol.wait
  int trigger;    // 1: launch_dependents once all operand loads are issued
  int csk;        // 1: cluster split-K — the split CTAs of a tile are one cluster (along z)
  int tma_ws;     // 1: split partials leave through a TMA tensor store (tmW) instead of st.global
  int kmulti;     // > 1: all K partitions of the tile in this CTA, region r = k-block / kb_per_split
  int bm;         // weight rows per tile: 128, or 64 (Plan::bm; epilogue warps 4-5 idle)
  int b_box;      // token rows per B TMA box: bn, or T when one token tile covers T (rows past
                  // it stay stale in smem; their accumulator columns are never stored)
};

// One residual row's RMSNorm / adaRMSNorm by one warp (NormFuse): lane l owns
// float4 columns l, l + 32, ...; the sum of squares runs in that fixed order and
// then a fixed butterfly, so the fused tail and rownorm_kernel agree bit for bit.
constexpr int NORM_MAX_V4 = 16;  // rows of up to 2048 features
constexpr int NORM_V4_PASS = 8;  // float4 per lane held at once (register budget of gemm_kernel)
__device__ __forceinline__ void warp_rownorm(const float *xrow, int n, const NormFuse &nf, __nv_bfloat16 *yrow) {
  const int lane = threadIdx.x & 31, nv4 = n >> 7;
  const float4 *xr = reinterpret_cast<const float4 *>(xrow);
  float ss = 0.f;
  for (int i0 = 0; i0 < nv4; i0 += NORM_V4_PASS) {
    float4 xv[NORM_V4_PASS];
#pragma unroll
    for (int i = 0; i < NORM_V4_PASS; ++i)
      if (i0 + i < nv4) xv[i] = __ldcg(xr + (i0 + i) * 32 + lane);
#pragma unroll
    for (int i = 0; i < NORM_V4_PASS; ++i)
      if (i0 + i < nv4) {
        ss = __fmaf_rn(xv[i].x, xv[i].x, ss);
        ss = __fmaf_rn(xv[i].y, xv[i].y, ss);
        ss = __fmaf_rn(xv[i].z, xv[i].z, ss);
        ss = __fmaf_rn(xv[i].w, xv[i].w, ss);
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  const float inv = rsqrtf(__fadd_rn(__fdiv_rn(ss, (float)n), nf.eps));
#pragma unroll 4
  for (int i = 0; i < nv4; ++i) {
    const int c = (i * 32 + lane) * 4;
    const float4 x4 = __ldcg(xr + i * 32 + lane);
    float o[4] = {x4.x, x4.y, x4.z, x4.w};
    if (nf.w) {
      const float4 w = __ldg(reinterpret_cast<const float4 *>(nf.w + c));
      const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = __fmul_rn(__fmul_rn(o[k], inv), __fadd_rn(1.f, wv[k]));
    } else {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(nf.ms + c));
      const float4 b = __ldg(reinterpret_cast<const float4 *>(nf.mb + c));
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = __fadd_rn(__fmul_rn(__fmul_rn(o[k], inv), __fadd_rn(1.f, av[k])), bv[k]);
    }
    __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t *>(&h0);
    u.y = *reinterpret_cast<uint32_t *>(&h1);
    *reinterpret_cast<uint2 *>(yrow + c) = u;
  }
}

__global__ void __launch_bounds__(256) rownorm_kernel(const float *x, int ldx, int t, int n, NormFuse nf) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r < t) warp_rownorm(x + (size_t)r * ldx, n, nf, nf.y + (size_t)r * nf.ldy);
}

void rownorm(const float *x, int ldx, int t, int n, const NormFuse &nf, cudaStream_t st) {
  if (t <= 0) return;
  if (n % 128 != 0 || n > 128 * NORM_MAX_V4 || ldx % 4 != 0 || nf.ldy % 4 != 0)
    fail(OXY_EINVAL, "row norm: rows of 128..2048 features (multiple of 128), strides multiple of 4");
  launch_pdl(rownorm_kernel, dim3((t + 7) / 8), dim3(256), 0, st, x, ldx, t, n, nf);
}

// Launch-time knobs (env, read once): OXY_SPLITK=fixup|kernel, OXY_PDL=0|1,
// OXY_GEMM_SMEM_KB=<per-CTA smem budget>.  Used for A/B measurements.
struct Knobs {
  int fixup = 0, pdl = 1, smem_kb = 100;  // 2 CTAs per SM (measured best)
  int tma_ws = 0;  // split partials via TMA tensor store (OXY_GEMM_TMA_WS=1; neutral in the frame)
  int bbox_exact = 1;  // B boxes of T rows when T < bn (OXY_GEMM_BBOX_EXACT=0: padded boxes)
  // prefill band tile width as a cap on the generic tiling: ViT o-proj / fc2 go from 72 /
  // 108 to 144 CTAs (prefill 6.14 -> 5.97 ms, profiles/r02/prefill_ab2.txt; =0: off)
  int band_cap = 1;
  int wide_fixup = 0;  // persistent kernel: in-kernel split fix-up instead of the reduce launch (A/B)
  int chain_max_splits = 0;  // cap on the decode / denoise split-K policy (OXY_CHAIN_MAX_SPLITS, A/B)
  int chain_bigk_splits = 0;  // decode down projection (K >= 8192) split count (OXY_CHAIN_BIGK_SPLITS, A/B)
  int kdual = 1;  // split-2 plans on the persistent kernel accumulate both K halves in-CTA (OXY_KDUAL=0: off)
  int kdual_bn = 0;  // cap on the token tile of kdual plans (128 keeps two accumulators; A/B)
  int kmulti = 1;    // chain plans at >= KMULTI_MIN_T tokens: 2-4 splits in-CTA (OXY_KMULTI=0: off)
  std::vector<std::array<int, 3>> split_overrides;  // OXY_SPLITS="n,k,s;...": chain split count per shape,
                                                    // n < 0: prefill entry for |n| (A/B)
  // early PDL (weight prefetch + trigger) for skinny / wide GEMMs: -1 = default policy
  // (T > 64 on the one-tile-per-CTA kernel: neutral at 1 stream, 0 to -1.3 ms per
  // 8-stream frame and 0 to -1 ms at 16 across same-session A/Bs)
  int early_skinny = 1, early_wide = 1;
  // persistent wide kernel for T > 64: -1 auto (cost model), 0 off, 1 / 2 force CTA group
  int wide = -1, wide_bn = 0, wide_splits = 0;  // -1 auto (see make_plan), 0 off, 1 / 2 force
  int wide_cl = 0;  // 0 auto, 1 / 2 force the pairs per cluster
  int wide_min_k = 0;  // > 0: also take the wide kernel for K >= this at T >= 256 (A/B knob)
  int wide_stages = 0;  // > 0: cap the persistent kernel's smem stages (A/B knob)
  int wide_diag = 0;    // timing diagnosis only (wrong results): 1 skip the MMAs, 2 skip the operand loads
  int wide_units = 0;   // > 0: cap the persistent grid at this many CTA pairs (diagnosis)
  int wide_nofence = 0; // 1: no tcgen05.fence::after_thread_sync per k-block in the MMA loop (A/B)
  int wide_sleep = 0;   // > 0: epilogue warps poll the accumulator barrier with this ns sleep (A/B)
  int prefill_kmulti = 0;  // 1: prefill split plans accumulate their splits in-CTA (A/B; 5.66 -> 7.71 ms prefill)
  int wide_min_n = 16384;  // the persistent kernel from T = 256 for n_out >= this (A/B knob)
  int split_slots = 1;  // skinny split-K fills split_slots CTAs per SM (A/B knob)
  // 64-row weight tiles for skinny (T <= 64) plans whose 64-row grid still fits
  // half_m CTAs per SM (OXY_GEMM_HALF; 0: off)
  int half_m = 0;
  int bigk_min = 0, bigk_bn = 0, bigk_splits = 0;  // OXY_GEMM_BIGK=kmin,bn,splits (A/B knob)
  // split K (fixed-order reduction) for token counts up to this when the tiles do not fill
  // the SMs: the multi-stream denoise (T = 50 x streams); 8 streams 67.9 -> 61.1 ms/frame
  int split_t = 1024;
  Knobs() {
    if (const char *s = getenv("OXY_GEMM_SPLIT_T")) split_t = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE")) wide = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_BN")) wide_bn = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_SPLITS")) wide_splits = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_CL")) wide_cl = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_MIN_K")) wide_min_k = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_STAGES")) wide_stages = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_DIAG")) wide_diag = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_UNITS")) wide_units = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_NOFENCE")) wide_nofence = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_SLEEP")) wide_sleep = atoi(s);
    if (const char *s = getenv("OXY_PREFILL_KMULTI")) prefill_kmulti = atoi(s);
    if (const char *s = getenv("OXY_GEMM_WIDE_MIN_N")) wide_min_n = atoi(s);
    if (const char *s = getenv("OXY_GEMM_SPLIT_SLOTS")) split_slots = std::max(1, atoi(s));
    if (const char *s = getenv("OXY_GEMM_HALF")) half_m = atoi(s);
    if (const char *s = getenv("OXY_GEMM_BIGK")) sscanf(s, "%d,%d,%d", &bigk_min, &bigk_bn, &bigk_splits);
    if (const char *s = getenv("OXY_PDL_EARLY_SKINNY")) early_skinny = atoi(s);
    if (const char *s = getenv("OXY_PDL_EARLY_WIDE")) early_wide = atoi(s);
    if (const char *s = getenv("OXY_SPLITK")) fixup = std::string(s) == "fixup";
    if (const char *s = getenv("OXY_PDL")) pdl = atoi(s);
    if (const char *s = getenv("OXY_GEMM_SMEM_KB")) smem_kb = std::max(64, std::min(200, atoi(s)));
    if (const char *s = getenv("OXY_GEMM_TMA_WS")) tma_ws = atoi(s);
    if (const char *s = getenv("OXY_GEMM_BBOX_EXACT")) bbox_exact = atoi(s);
    if (const char *s = getenv("OXY_GEMM_BAND_CAP")) band_cap = atoi(s);
    if (const char *s = getenv("OXY_WIDE_FIXUP")) wide_fixup = atoi(s);
    if (const char *s = getenv("OXY_CHAIN_MAX_SPLITS")) chain_max_splits = atoi(s);
    if (const char *s = getenv("OXY_CHAIN_BIGK_SPLITS")) chain_bigk_splits = atoi(s);
    if (const char *s = getenv("OXY_KDUAL")) kdual = atoi(s);
    if (const char *s = getenv("OXY_KDUAL_BN")) kdual_bn = atoi(s);
    if (const char *s = getenv("OXY_KMULTI")) kmulti = atoi(s);
    if (const char *s = getenv("OXY_SPLITS")) {
      std::string v(s);
      size_t pos = 0;
      while (pos < v.size()) {
        size_t e = v.find(';', pos);
        if (e == std::string::npos) e = v.size();
        std::array<int, 3> o{};
        if (sscanf(v.substr(pos, e - pos).c_str(), "%d,%d,%d", &o[0], &o[1], &o[2]) == 3) split_overrides.push_back(o);
        pos = e + 1;
      }
    }
  }
};
// per-enqueue override of the skinny early-PDL policy (-1: knob); set by the
// model around one lane's enqueue (host calls are serial)
int g_early_override = -1;
// per-enqueue token tiling by K band {k_min, bn, splits} x 2 (first matching band; k_min 0:
// off), same discipline
int g_deepk[6] = {0, 0, 0, 0, 0, 0};
long long g_plan_counts[PC_COUNT] = {};

static const Knobs &knobs() {
  static Knobs k;
  return k;
}

// Fixed-order split-K reduction + epilogue; one thread per feature pair.  All
// split partials are loaded before any is summed (16 in flight), and the RoPE
// position / (cos, sin) entry — host-planned, not produced by the previous
// kernel — is fetched before the PDL wait.
constexpr int RD_CHUNK = 8;
__global__ void splitk_reduce_v1_kernel(const float *ws, int splits, int t_rows, int n_out, EpiParams e) {
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

__global__ void splitk_reduce_kernel(const float *ws, int splits, int t_rows, int n_out, EpiParams e) {
  pdl_trigger();
  const int pairs = (n_out + 1) >> 1;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)t_rows * pairs) return;
  const int t = (int)(idx / pairs), f = (int)(idx % pairs) * 2;
  const bool rope = e.mode == EPI_QKV_ROPE;
  float2 csn = make_float2(1.f, 0.f);
  if (rope) csn = rope_cs(e.rope, __ldg(e.rope.pos + t), (f & 255) >> 1);
  pdl_wait();
  const bool vec = (n_out & 1) == 0;
  float a0 = 0.f, a1 = 0.f;
  for (int s0 = 0; s0 < splits; s0 += RD_CHUNK) {
    float2 p[RD_CHUNK];
#pragma unroll
    for (int s = 0; s < RD_CHUNK; ++s) {
      if (s0 + s >= splits) continue;
      const float *row = ws + ((size_t)(s0 + s) * t_rows + t) * n_out + f;
      p[s] = vec ? __ldcg(reinterpret_cast<const float2 *>(row))
                 : make_float2(__ldcg(row), f + 1 < n_out ? __ldcg(row + 1) : 0.f);
    }
#pragma unroll
    for (int s = 0; s < RD_CHUNK; ++s)
      if (s0 + s < splits) {
        a0 += p[s].x;
        a1 += p[s].y;
      }
  }
  if (rope) {  // f even, f + 1 is its rotary pair (interleaved weight rows)
    rope_store(e.rope, t, f, a0, a1, csn.x, csn.y);
    rope_store(e.rope, t, f + 1, a1, a0, csn.x, csn.y);
    return;
  }
  epilogue_store(e, t, f, n_out, a0, a1);
  if (f + 1 < n_out) epilogue_store(e, t, f + 1, n_out, a1, a0);
}

#ifdef OXY_GEMM_PROF
// timing builds: %globaltimer at pipeline events of weight tile 0 / token tile 0
// of the launches matching (n_out, k) set by oxy_debug_gemm_prof_select, one row
// per split (the last matching launch wins)
__device__ unsigned long long g_gemm_prof[32][24];
__device__ int g_gemm_prof_sel[2];
// (the selection is read once per CTA into gprof_on: a global load per event put an
// L2 round trip into every probed step and skewed the timelines)
#define GPROF_INIT()                                                                                 \
  const bool gprof_on = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z < 32 &&                     \
                        p.n_out == g_gemm_prof_sel[0] && p.k == g_gemm_prof_sel[1]
#define GPROF(ev)                                                                             \
  do {                                                                                        \
    if (gprof_on) {                                                                           \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      g_gemm_prof[blockIdx.z][ev] = t_;                                                       \
    }                                                                                         \
  } while (0)
// persistent wide kernel: per CTA 0..3 and local tile 0..15: [0] MMA warp starts the
// tile (accumulator free), [1] last k-block issued, [2] epilogue warp 2 sees the
// accumulator, [3] epilogue warp 2 done; row 16: [0] entry [1] setup done [2] exit
__device__ unsigned long long g_wide_prof[4][17][6];
#define WPROF(cta, lt, ev)                                                                     \
  do {                                                                                         \
    if (gprof_on && (cta) < 4 && (lt) < 17) {                                                  \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      g_wide_prof[cta][lt][ev] = t_;                                                           \
      if ((ev) < 2) g_wide_prof[cta][lt][4 + (ev)] = clock64();                                \
    }                                                                                          \
  } while (0)
#define WPROF_INIT() const bool gprof_on = p.n_out == g_gemm_prof_sel[0] && p.k == g_gemm_prof_sel[1]
#else
#define WPROF(cta, lt, ev) \
  do {                     \
  } while (0)
#define WPROF_INIT() \
  do {               \
  } while (0)
#define GPROF_INIT() \
  do {               \
  } while (0)
#define GPROF(ev) \
  do {            \
  } while (0)
#endif

// The `n` K-partition accumulators of a kmulti tile, `stride` columns apart, summed in
// partition order r0 + r1 + ... (the split reduce's order).
struct MultiTmemSrc {
  uint32_t t0;
  int n, stride;
  __device__ __forceinline__ void operator()(int c, int, uint32_t (&v)[16]) const {
    tmem_ld16(t0 + (uint32_t)c, v);
    for (int r = 1; r < n; ++r) {
      uint32_t w[16];
      tmem_ld16(t0 + (uint32_t)(c + r * stride), w);
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__fadd_rn(__uint_as_float(v[e]), __uint_as_float(w[e])));
    }
  }
};

// Greedy-decode epilogue of the LM head (EPI_ARGMAX): per 16-token chunk each
// warp folds its 32 vocabulary rows per token (butterfly: every lane ends with
// the warp's (max, lowest id)), the 4 warps meet in smem, and one (max, id) per
// (token, weight tile) is stored.  The order-free rule — larger value wins,
// equal values go to the lower id, NaN never wins — is the reference's
// lowest-id tie-break (kvweaver/backend.py:387-388), so the fold order does not
// matter and the result equals an argmax over the materialised logits.
__device__ __forceinline__ void amax_better(float &bv, int &bi, float v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}
__device__ __forceinline__ void argmax_epilogue(const KParams &p, const TmemSrc &src, int bn, int n0, int f,
                                                int tile, float (*s_v)[16], int (*s_i)[16]) {
  const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3;
  for (int c = 0; c < bn; c += 16) {
    uint32_t v[16];
    src(c, 16, v);
    const int t0 = n0 + c;
    float bv[16];
    int bi[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      bv[j] = (f < p.n_out && t0 + j < p.t) ? __uint_as_float(v[j]) : -INFINITY;
      bi[j] = f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv[j], o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi[j], o);
        amax_better(bv[j], bi[j], ov, oi);
      }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        s_v[q][j] = bv[j];
        s_i[q][j] = bi[j];
      }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (q == 0 && lane < 16 && t0 + lane < p.t) {
      float b = s_v[0][lane];
      int i = s_i[0][lane];
      for (int w = 1; w < 4; ++w) amax_better(b, i, s_v[w][lane], s_i[w][lane]);
      const size_t o = (size_t)(t0 + lane) * p.epi.ldo + tile;
      static_cast<float *>(p.epi.out)[o] = b;
      p.epi.amax_idx[o] = i;
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
  }
}

// 128 registers: two CTAs per SM still leave register room for the next
// kernel's early (PDL) CTAs and the other lane's kernels (168 registers, the
// compiler's free choice with the cluster split-K tail, filled the register file
// and serialised the chain)
__global__ void __maxnreg__(128)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmW, KParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  const int bn = p.bn, stages = p.stages;
  const int b_bytes = bn * BK * 2;
  const uint32_t stage_tx = (p.bm * BK + p.b_box * BK) * 2;  // bytes one stage's two TMA boxes deliver
  uint8_t *sA = smem;
  uint8_t *sB = smem + stages * A_STAGE_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + stages * b_bytes);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * MAX_STAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // token tiles fastest: the CTAs sharing one weight tile run in the same wave
  const int m0 = blockIdx.y * p.bm, n0 = blockIdx.x * bn, split = blockIdx.z;
  __shared__ int s_last;
  const int kb0 = p.kmulti > 1 ? 0 : split * p.kb_per_split;
  const int nkb = p.kmulti > 1 ? p.kb_total : min(p.kb_total, kb0 + p.kb_per_split) - kb0;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + MAX_STAGES),
                 done = smem_u32(bars + 2 * MAX_STAGES);
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(bn * (p.kmulti > 1 ? p.kmulti : 1))) ncols <<= 1;
  GPROF_INIT();
  if (threadIdx.x == 0) GPROF(0);

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
  if (threadIdx.x == 0) GPROF(1);
  if (warp == 0) {
    // the whole warp walks the loads (uniform registers); the elected lane issues them
    // Weights never depend on the previous kernel: stream the first ring of
    // weight tiles before waiting on it, activations after.
    const int pre = p.prefetch ? min(nkb, stages) : 0;
    if (elect_one()) {
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(full0 + 8 * i, stage_tx);
        tma_load_2d(&tmA, full0 + 8 * i, smem_u32(sA + i * A_STAGE_BYTES), (kb0 + i) * BK, m0);
#ifdef OXY_GEMM_PROF_PREB  // timing experiment only (races the previous kernel): B before the wait too
        tma_load_2d(&tmB, full0 + 8 * i, smem_u32(sB + i * b_bytes), (kb0 + i) * BK, n0);
#endif
      }
    }
    __syncwarp();
    if (lane == 0) GPROF(2);
    pdl_wait();
    if (lane == 0) GPROF(3);
#ifndef OXY_GEMM_PROF_PREB
    if (elect_one())
      for (int i = 0; i < pre; ++i)
        tma_load_2d(&tmB, full0 + 8 * i, smem_u32(sB + i * b_bytes), (kb0 + i) * BK, n0);
    __syncwarp();
#endif
    for (int i = pre; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      mbar_wait(empty0 + 8 * s, ph ^ 1);
      const int kc = (kb0 + i) * BK;
      if (elect_one()) {
        mbar_expect_tx(full0 + 8 * s, stage_tx);
        tma_load_2d(&tmA, full0 + 8 * s, smem_u32(sA + s * A_STAGE_BYTES), kc, m0);
        tma_load_2d(&tmB, full0 + 8 * s, smem_u32(sB + s * b_bytes), kc, n0);
      }
      __syncwarp();
    }
    // all operand loads are in flight: let the next kernel start its
    // prologue and weight prefetch while this CTA drains
    if (lane == 0) GPROF(4);
    if (p.trigger && lane == 0) pdl_trigger();
  } else if (warp == 1) {
    // the whole warp walks the k-loop (uniform registers); the elected lane issues
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      mbar_wait(full0 + 8 * s, ph);
      tc_fence_after();
      if (lane == 0) {
        if (i == 0) GPROF(5);
        if (i > 0 && i < 4) GPROF(15 + i);
      }
      const uint32_t a = smem_u32(sA + s * A_STAGE_BYTES), b = smem_u32(sB + s * b_bytes);
      // kmulti: k-block i accumulates into region i / kb_per_split, each region from zero
      const int reg = p.kmulti > 1 ? i / p.kb_per_split : 0, i0 = i - reg * p.kb_per_split;
      const uint32_t d = tmem + (uint32_t)(reg * bn);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          mma_bf16(d, make_sdesc(a + kk * 32), make_sdesc(b + kk * 32), idesc, (i0 | kk) != 0 ? 1u : 0u);
        mma_commit(empty0 + 8 * s);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(done);
    __syncwarp();
    if (lane == 0) GPROF(6);
  }
  const int q = warp & 3;
  const int f = m0 + q * 32 + lane;
  // the operand ring is idle once `done` fired: 4 x 2.3 KB transpose tiles for the bf16 epilogues
  float *stg = reinterpret_cast<float *>(sA) + q * (16 * STG_LD);
  if (warp >= 2) {
    // kmulti: the summed partitions take the real epilogue, or leave as ONE partial slab
    const bool split_out = p.kmulti > 1 ? p.epi.mode == EPI_PARTIALS : p.splits > 1;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    pdl_wait();  // the epilogue reads bias/residual/gates and writes outputs
    if (threadIdx.x == 64) GPROF(7);
    mbar_wait(done, 0);
    tc_fence_after();
    if (threadIdx.x == 64) GPROF(8);
    if (p.epi.mode == EPI_ARGMAX) {
      __shared__ float s_amv[4][16];
      __shared__ int s_ami[4][16];
      argmax_epilogue(p, TmemSrc{trow}, bn, n0, f, blockIdx.y, s_amv, s_ami);
    } else if (split_out && p.tma_ws) {
      // split-K partials through one TMA tensor store: the 128 x bn fp32 tile is
      // staged token-major in the idle operand ring (thread = feature column, so
      // a warp's 32 stores per token row are conflict-free) and written by a
      // single bulk copy instead of 16 x bn/16 per-thread store instructions;
      // token rows past T and features past N_out are clipped by the 3-D map
      float *stage = reinterpret_cast<float *>(sA);
      const int col = q * 32 + lane;
      const TmemSrc src{trow};
      for (int c = 0; c < bn; c += 16) {
        uint32_t v[16];
        src(c, 16, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) stage[(c + j) * BM + col] = __uint_as_float(v[j]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (threadIdx.x == 64) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                         reinterpret_cast<uint64_t>(&tmW)),
                     "r"(m0), "r"(n0), "r"(split), "r"(smem_u32(stage))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem released once read
      }
    } else
#ifdef OXY_GEMM_PROF
    if (bn > 32) {
      epi_tile(p, trow, 0, 16, n0, f, split, split_out, stg);
      if (threadIdx.x == 64) GPROF(11);
      epi_tile(p, trow, 16, 32, n0, f, split, split_out, stg);
      if (threadIdx.x == 64) GPROF(12);
      epi_tile(p, trow, 32, bn, n0, f, split, split_out, stg);
    } else
#endif
    if (q * 32 >= p.bm) {
      // 64-row tile: these accumulator lanes came from stale A rows — nothing to store
    } else if (p.kmulti > 1) epi_tile_src(p, MultiTmemSrc{trow, p.kmulti, bn}, 0, bn, n0, f, 0, split_out, stg);
    else epi_tile(p, trow, 0, bn, n0, f, split, split_out, stg);
    if (threadIdx.x == 64) GPROF(9);
    if (split_out && p.fixup) splitk_fixup(p, blockIdx.y * gridDim.x + blockIdx.x, n0, 0, bn, f, s_last, 128, 64);
  }
  if (p.csk) {
    // Cluster split-K: every split CTA of this tile is in the cluster.  Once all
    // partials are stored, CTA r reduces token slice r of the tile (split order
    // 0..S-1) and runs the real epilogue on it — no reduce launch.
    __syncwarp();
    cluster_sync_all();
    if (threadIdx.x == 64) GPROF(13);
    const int valid = min(bn, p.t - n0);
    const int per = (valid + p.splits - 1) / p.splits;
    const int cb = min(valid, split * per), ce = min(valid, cb + per);
    if (warp >= 2 && cb < ce)
      epi_tile_src(p, SplitSumSrc{p.ws, p.splits, p.t, p.n_out, n0, f, f < p.n_out}, cb, ce, n0, f, split, false,
                   stg);
    if (threadIdx.x == 64) GPROF(14);
    if (p.epi.norm.y) {
      // Residual RMSNorm: the last cluster to finish (a grid-wide arrival count,
      // kept by cluster rank 0) normalises every row.  Each thread's fence plus
      // the cluster barrier order its residual stores before rank 0's release.
      __shared__ int s_norm_last;
      __threadfence();
      __syncwarp();
      cluster_sync_all();
      if (split == 0 && threadIdx.x == 64) {
        int old;
        int *ctr = p.counters + (MAX_TILES - 1);
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
        const int last = old == (int)(gridDim.x * gridDim.y) - 1;
        if (last) *ctr = 0;  // self-resetting for the next launch on this lane
        s_norm_last = last;
      }
      cluster_sync_all();
      int last;
      asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(last) : "r"(map_to_rank(smem_u32(&s_norm_last), 0)));
      if (last) {
        const int nw = blockDim.x >> 5;
        for (int r = split * nw + warp; r < p.t; r += p.splits * nw)
          warp_rownorm(static_cast<const float *>(p.epi.out) + (size_t)r * p.epi.ldo, p.n_out, p.epi.norm,
                       p.epi.norm.y + (size_t)r * p.epi.norm.ldy);
      }
      if (threadIdx.x == 64) GPROF(15);
      cluster_sync_all();  // rank 0's flag is read by the peers before it exits
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) GPROF(10);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols)
                 : "memory");
  }
}

__device__ __forceinline__ void tma_load_2d_pair_mc(const CUtensorMap *map, uint32_t bar_leader, uint32_t dst, int c0,
                                                    int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_leader), "h"(mask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mask(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

// ------------------------------------------------------------------ wide (prefill) GEMM
//
// Persistent, one CTA per SM (or one CTA pair per TPC with CG = 2), static
// tile schedule with the token tiles of one weight tile adjacent (they run in
// the same wave and share the weight tile through L2).  Two TMEM accumulators:
// the epilogue of tile i overlaps the mainloop of tile i+1.  With CG = 2 the
// pair computes a 256-feature x BN-token tile with tcgen05.mma.cta_group::2:
// each CTA stages its 128 weight rows and BN/2 token rows per stage, so the
// smem/L2 bytes per MAC halve against the 1-CTA tile.
// The two K-half accumulators of a kdual tile, summed p0 + p1 (the split reduce's order).
struct DualTmemSrc {
  uint32_t t0, t1;
  __device__ __forceinline__ void operator()(int c, int, uint32_t (&v)[16]) const {
    uint32_t w[16];
    tmem_ld16(t0 + (uint32_t)c, v);
    tmem_ld16(t1 + (uint32_t)c, w);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__fadd_rn(__uint_as_float(v[e]), __uint_as_float(w[e])));
  }
};

struct WParams {
  int n_out, k, t, bn, stages, kb_total;
  int m_tiles, n_tiles, splits, kb_per_split, tiles;
  int kdual;  // splits == 2 done in-CTA: tiles are (m, n) only, K half h -> accumulator region h
  int diag;   // OXY_GEMM_WIDE_DIAG (timing diagnosis): 1 no MMAs, 2 no operand loads
  int sleep_ns;  // > 0: the epilogue's accumulator wait sleeps between probes
  EpiParams epi;
  float *ws;
  int *counters;  // one per (tile, CTA of the pair); self-resetting
};

constexpr int WIDE_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 per TMEM lane quadrant)

// CL = 2 (with CG = 2): a cluster of two CTA pairs works on two adjacent token
// tiles of one weight tile; each CTA TMA-loads half of its 128 weight rows and
// multicasts them to the same-rank CTA of the other pair, halving the weight
// bytes read from L2 (the prefill GEMMs are L2-bandwidth bound at ~10 TB/s).
// Stage reuse then needs both pairs' MMA commits (empty count = CL).
template <int CG, int CL = 1>
__global__ void __launch_bounds__(WIDE_THREADS, 1)
    gemm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, WParams p) {
  static_assert(CL == 1 || CG == 2, "A multicast across pairs needs CTA pairs");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  const int bn = p.bn, stages = p.stages;
  const int b_rows = bn / CG;
  const int b_bytes = b_rows * BK * 2;
  uint8_t *sA = smem;
  uint8_t *sB = smem + stages * A_STAGE_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + stages * b_bytes);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * MAX_STAGES + 4);
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WPROF_INIT();
  if (threadIdx.x == 0) WPROF(blockIdx.x, 16, 0);
  const uint32_t crank = CG == 2 ? cluster_rank() : 0;
  const uint32_t rank = crank & 1, pp = crank >> 1;  // CTA within its pair, pair within the cluster
  const int unit = blockIdx.x / (CG * CL), units = gridDim.x / (CG * CL);
  const int ngr = (p.n_tiles + CL - 1) / CL;  // token-tile groups (one tile per pair)
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + MAX_STAGES),
                 tfull0 = smem_u32(bars + 2 * MAX_STAGES), tempty0 = smem_u32(bars + 2 * MAX_STAGES + 2);
  // two accumulators (tile i's epilogue overlaps tile i+1's mainloop); kdual: two regions
  // (K halves) each — for bn > 128 only one accumulator then (no epilogue overlap)
  const int nbuf = p.kdual && bn > 128 ? 1 : 2;
  const uint32_t ncols = p.kdual ? (bn <= 64 ? 256u : 512u) : bn <= 128 ? (bn <= 64 ? 128u : 256u) : 512u;
  const uint32_t acc_stride = ncols / nbuf, half_stride = acc_stride / 2;
  const int per_m_split = p.kdual ? 1 : p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, CL);  // one MMA commit per pair reading this stage's multicast A
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 8 * CG);  // one arrival per epilogue warp of each CTA of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int per_m = per_m_split * ngr;
  if (threadIdx.x == 0) WPROF(blockIdx.x, 16, 1);

  if (warp == 0) {
    // the whole warp walks the loads (uniform registers); the elected lane issues them
    // completion is counted on the pair leader's barrier: the cvta address of
    // a cluster CTA carries its rank in bits 24+, so clearing bit 24 names it
    const uint32_t full_l = full0 & ~(1u << 24);
    const uint16_t a_mask = (uint16_t)((1u << rank) | (1u << (2 + rank)));  // same rank in both pairs
    int it = 0;
    bool waited = false;
    for (int tile = unit; tile < p.tiles; tile += units) {
      if (tile + units >= p.tiles && lane == 0) pdl_trigger();  // last tile: let the next kernel get scheduled
      const int mt = tile / per_m, rem = tile % per_m, split = rem / ngr, nt = (rem % ngr) * CL + (int)pp;
      const int kb0 = p.kdual ? 0 : split * p.kb_per_split;
      const int nkb = p.kdual ? p.kb_total : min(p.kb_total, kb0 + p.kb_per_split) - kb0;
      const int arow = mt * BM * CG + (int)rank * BM + (CL == 2 ? (int)pp * (BM / 2) : 0),
                brow = nt * bn + (int)rank * b_rows;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % stages;
        const uint32_t ph = (it / stages) & 1;
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        if ((p.diag & 3) == 2) {  // diagnosis: the pipeline without operand traffic
          if (rank == 0 && elect_one()) mbar_arrive_local(full0 + 8 * s);
          __syncwarp();
          if (!waited) { pdl_wait(); waited = true; }
          continue;
        }
        const int kc = (kb0 + i) * BK;
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(full0 + 8 * s, CG * (A_STAGE_BYTES + b_bytes));
          if (CL == 2) {  // half of this CTA's weight rows, to both pairs
            tma_load_2d_pair_mc(&tmA, full_l + 8 * s, smem_u32(sA + s * A_STAGE_BYTES + (int)pp * (A_STAGE_BYTES / 2)),
                                kc, arow, a_mask);
          } else if (CG == 2) {
            tma_load_2d_pair(&tmA, full_l + 8 * s, smem_u32(sA + s * A_STAGE_BYTES), kc, arow);
          } else {
            tma_load_2d(&tmA, full0 + 8 * s, smem_u32(sA + s * A_STAGE_BYTES), kc, arow);
          }
        }
        __syncwarp();
        if (!waited) { pdl_wait(); waited = true; }  // activations come from the previous kernel
        if (elect_one()) {
          if (CG == 2) tma_load_2d_pair(&tmB, full_l + 8 * s, smem_u32(sB + s * b_bytes), kc, brow);
          else tma_load_2d(&tmB, full0 + 8 * s, smem_u32(sB + s * b_bytes), kc, brow);
        }
        __syncwarp();
      }
    }
    if (!waited) pdl_wait();
  } else if (warp == 1) {
    if (rank == 0) {  // the whole warp walks the loop; the elected lane issues
      // kind::f16, bf16 x bf16 -> f32, K-major A/B, N = bn, M = 128 * CG
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) |
                             ((uint32_t)((BM * CG) >> 4) << 24);
      const uint16_t all_mask = (uint16_t)((1u << (CG * CL)) - 1), pair_mask = (uint16_t)(3u << (2 * pp));
      int it = 0, lt = 0;
      for (int tile = unit; tile < p.tiles; tile += units, ++lt) {
        const int rem = tile % per_m, split = rem / ngr;
        const int kb0 = p.kdual ? 0 : split * p.kb_per_split;
        const int nkb = p.kdual ? p.kb_total : min(p.kb_total, kb0 + p.kb_per_split) - kb0;
        const int acc = lt % nbuf;
        mbar_wait(tempty0 + 8 * acc, ((lt / nbuf) & 1) ^ 1);
        tc_fence_after();
        WPROF(blockIdx.x, lt, 0);
        const uint32_t d0 = tmem + (uint32_t)acc * acc_stride;
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % stages;
          const uint32_t ph = (it / stages) & 1;
          mbar_wait(full0 + 8 * s, ph);
          if (!(p.diag & 4)) tc_fence_after();
          const uint32_t a = smem_u32(sA + s * A_STAGE_BYTES), b = smem_u32(sB + s * b_bytes);
          // kdual: k-blocks of the second K half accumulate into the second region, each
          // half from zero — the split-2 partials, kept in TMEM
          const bool hi = p.kdual && i >= p.kb_per_split;
          const uint32_t d = d0 + (hi ? half_stride : 0u);
          const int i0 = hi ? i - p.kb_per_split : i;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              if ((p.diag & 3) == 1) break;  // diagnosis: the pipeline without MMAs
              if (CG == 2)
                mma_bf16_pair(d, make_sdesc(a + kk * 32), make_sdesc(b + kk * 32), idesc, (i0 | kk) != 0 ? 1u : 0u);
              else
                mma_bf16(d, make_sdesc(a + kk * 32), make_sdesc(b + kk * 32), idesc, (i0 | kk) != 0 ? 1u : 0u);
            }
            if (CG == 2) mma_commit_mask(empty0 + 8 * s, all_mask);  // both pairs may refill the stage
            else mma_commit(empty0 + 8 * s);
          }
          __syncwarp();
        }
        if (elect_one()) {
          if (CG == 2) mma_commit_mask(tfull0 + 8 * acc, pair_mask);
          else mma_commit(tfull0 + 8 * acc);
        }
        __syncwarp();
        WPROF(blockIdx.x, lt, 1);
      }
    }
    __syncwarp();
  } else {
    pdl_wait();  // the epilogue reads bias/residual/gates and writes outputs
    // two warps per TMEM lane quadrant, each taking half of the tile's 16-column chunks
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int chunks = bn / 16, c_mid = ((chunks + 1) / 2) * 16;
    const int cb = half ? c_mid : 0, ce = half ? bn : c_mid;
    // kdual: the summed halves take the real epilogue, or leave as ONE partial slab
    const bool split_out = p.kdual ? p.epi.mode == EPI_PARTIALS : p.splits > 1;
    const uint32_t tempty_l = CG == 2 ? map_to_rank(tempty0, 2 * pp) : tempty0;
    int lt = 0;
    for (int tile = unit; tile < p.tiles; tile += units, ++lt) {
      const int mt = tile / per_m, rem = tile % per_m, split = rem / ngr, nt = (rem % ngr) * CL + (int)pp;
      const int acc = lt % nbuf;
      if (p.sleep_ns > 0) mbar_wait_sleep(tfull0 + 8 * acc, (lt / nbuf) & 1, p.sleep_ns);
      else mbar_wait(tfull0 + 8 * acc, (lt / nbuf) & 1);
      tc_fence_after();
      if (threadIdx.x == 64) WPROF(blockIdx.x, lt, 2);
      const int f = mt * BM * CG + (int)rank * BM + q * 32 + lane;
      const int n0 = nt * bn;
      const uint32_t trow = tmem + (uint32_t)acc * acc_stride + ((uint32_t)(q * 32) << 16);
      if (p.kdual) epi_tile_src(p, DualTmemSrc{trow, trow + half_stride}, cb, ce, n0, f, 0, split_out);
      else epi_tile(p, trow, cb, ce, n0, f, split, split_out);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(tempty_l + 8 * acc);
        else mbar_arrive_local(tempty0 + 8 * acc);
      }
      if (threadIdx.x == 64) WPROF(blockIdx.x, lt, 3);
      if (!p.kdual && split_out && p.epi.mode != EPI_PARTIALS && nt < p.n_tiles)  // (the odd pair of a ragged group idles)
        splitk_fixup(p, (mt * p.n_tiles + nt) * CG + (int)rank, n0, cb, ce, f, s_last, WIDE_THREADS - 64, 64);
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (threadIdx.x == 0) WPROF(blockIdx.x, 16, 2);
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
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

constexpr int WIDE_SMEM = 220 * 1024;

static int wide_stages(int bn, int cg) {
  const int s = std::min(MAX_STAGES, (WIDE_SMEM - 2048) / (A_STAGE_BYTES + bn / cg * BK * 2));
  return knobs().wide_stages > 0 ? std::min(s, knobs().wide_stages) : s;
}

// Cost model (SM cycles) of the persistent wide kernel.  Per k-block a CTA
// needs max(MMA, operand ingest): MMA = 128 x bn x 64 MACs at 4096 MAC/cycle/SM;
// ingest = (16 KB of weights + bn/CG token rows of 128 B) at ~33 B/cycle/SM
// (measured: the 2-CTA GEMM at T=800 streams 32-35 B/cycle/SM whether 80 or
// 148 SMs are active).  Split-K pays a partial-sum round trip and a fix-up.
static double wide_cost(int n_out, int kb_total, int t, int units, int cg, int bn, int splits, int cl = 1) {
  const int m_tiles = (n_out + BM * cg - 1) / (BM * cg), n_tiles = (t + bn - 1) / bn;
  const int tiles = m_tiles * ((n_tiles + cl - 1) / cl) * splits;
  const int waves = (tiles + units - 1) / units;
  const int kbs = (kb_total + splits - 1) / splits;
  // weight bytes per CTA and k-block are read from L2 once per cluster (multicast)
  const double mma = 2.0 * bn, bytes = A_STAGE_BYTES / cl + (double)bn / cg * BK * 2;
  const double per_tile = kbs * std::max(mma, bytes / 33.0) + 600.0;
  double c = 3000.0 + waves * per_tile + 60.0 * bn;
  if (splits > 1) c += 2.0 * bn * 128 * 4 * splits / 33.0 + 1500.0;
  if (cl > 1 && n_tiles % cl) c *= 1.0 + 0.5 / n_tiles;  // an idle pair on ragged token groups
  return c;
}

static void wide_attrs() {
  static bool done = false;
  if (done) return;
  OXY_CUDA(cudaFuncSetAttribute(gemm_wide_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  OXY_CUDA(cudaFuncSetAttribute(gemm_wide_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  OXY_CUDA(cudaFuncSetAttribute(gemm_wide_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  done = true;
}

static int device_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    OXY_CUDA(cudaGetDevice(&dev));
    OXY_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// Work units (CTA pairs, or clusters of two pairs) the persistent wide kernel keeps
// co-resident on `sms` SMs.  A 4-CTA cluster needs two TPCs of one GPC, so fewer than
// sms / 4 fit at once: a grid of sms / 4 clusters ran its last clusters as a second
// wave (the round-1 CL = 2 measurement, 1139 vs 651 us).  The cluster count comes from
// the occupancy query; CL = 2 only on the whole device (not inside an SM partition,
// where clusters above 8 CTAs and the GPC split are not ours to know).
static int wide_units(int cg, int cl, int sms) {
  if (cl == 1) return sms / cg;
  static int cap = -1;
  if (cap < 0) {
    wide_attrs();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(device_sms());
    cfg.blockDim = dim3(WIDE_THREADS);
    cfg.dynamicSmemBytes = WIDE_SMEM;
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = 4;
    a.val.clusterDim.y = 1;
    a.val.clusterDim.z = 1;
    cfg.attrs = &a;
    cfg.numAttrs = 1;
    int n = 0;
    OXY_CUDA(cudaOccupancyMaxActiveClusters(&n, gemm_wide_kernel<2, 2>, &cfg));
    cap = n;
  }
  return sms == device_sms() ? std::min(cap, sms / 4) : 0;
}

static bool wide_plan(Plan &p, int n_out, int k, int t, int sms, int req_splits) {
  const Knobs &kn = knobs();
  double best = 1e30;
  for (int cg = 1; cg <= 2; ++cg) {
    if (kn.wide > 0 && cg != kn.wide) continue;
    for (int cl = 1; cl <= (cg == 2 ? 2 : 1); ++cl) {
      // two pairs per cluster multicasting the weight tile: only when forced (A/B)
      if (kn.wide_cl ? cl != kn.wide_cl : cl != 1) continue;
      const int units = wide_units(cg, cl, sms);
      if (units <= 0) continue;
      for (int bn = 32; bn <= MAX_BN; bn += 16) {
        if (kn.wide_bn && bn != kn.wide_bn) continue;
        if (cl == 2 && (t + bn - 1) / bn < 2) continue;
        for (int splits = 1; splits <= std::max(4, req_splits); ++splits) {
          if (req_splits > 0 ? splits != req_splits
                             : ((kn.wide_splits && splits != kn.wide_splits) || (splits > 1 && p.kb_total / splits < 4)))
            continue;
          const double c = wide_cost(n_out, p.kb_total, t, units, cg, bn, splits, cl);
          if (c < best * 0.999) {
            best = c;
            p.cg = cg;
            p.cl = cl;
            p.bn = bn;
            p.splits = splits;
          }
        }
      }
    }
  }
  if (best >= 1e30) return false;
  p.m_tiles = (n_out + BM * p.cg - 1) / (BM * p.cg);
  p.n_tiles = (t + p.bn - 1) / p.bn;
  const int per_split = (p.kb_total + p.splits - 1) / p.splits;
  p.splits = (p.kb_total + per_split - 1) / per_split;
  // a fixed split-2 partition (prefill deep-K policy) on the persistent kernel: both K
  // halves in one CTA (pair), two TMEM regions per accumulator -> token tiles <= 128
  p.kdual = kn.kdual && req_splits == 2 && p.splits == 2 && p.cl == 1;
  if (p.kdual && kn.kdual_bn > 0 && p.bn > kn.kdual_bn) {
    p.bn = kn.kdual_bn;
    p.n_tiles = (t + p.bn - 1) / p.bn;
  }
  p.stages = wide_stages(p.bn, p.cg);
  return true;
}

// split-K workspace [splits][t][n_out] fp32 as a 3-D map, box 128 features x bn tokens x 1
// split, no swizzle (the staged tile is dense token-major)
static CUtensorMap make_map_ws(const float *ws, int splits, int t, int n_out, int bn) {
  if (reinterpret_cast<uintptr_t>(ws) % 16 != 0) fail(OXY_EINVAL, "split-K workspace not 16-byte aligned");
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)n_out, (cuuint64_t)t, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)n_out * 4, (cuuint64_t)t * n_out * 4};
  cuuint32_t box[3] = {(cuuint32_t)BM, (cuuint32_t)bn, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(ws), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(OXY_ECUDA, "cuTensorMapEncodeTiled (split-K workspace) failed (%d)", (int)r);
  return map;
}

// rows x cols fp32 row-major, box (box_cols x box_rows), 128-byte swizzle (box_cols * 4 == 128)
CUtensorMap make_map_f32(const void *ptr, int rows, int cols, int box_cols, int box_rows) {
  if ((cols * 4) % 16 != 0 || reinterpret_cast<uintptr_t>(ptr) % 16 != 0) fail(OXY_EINVAL, "fp32 map alignment");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(OXY_ECUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", (int)r);
  return map;
}

int policy_splits(int phase, int n_out, int k, int sms) {
  const int kb = (k + BK - 1) / BK;
  int s;
  if (phase == PH_PREFILL) {
    // deep-K projections (Gemma qkv / o / down, ViT fc2) split K in two: with the
    // 128-token tiles of the deep-K band both CTA slots per SM stay busy and the o /
    // down residual + RMSNorm fuse into the split reduce; the gate/up projections
    // (n_out >= 16384) run on the persistent 2-CTA kernel unsplit
    s = (k >= 2048 && n_out < 16384) ? 2 : 1;
    for (const auto &o : knobs().split_overrides)  // OXY_SPLITS="-n,k,s": prefill entries (A/B)
      if (o[0] == -n_out && o[1] == k) s = o[2];
  } else {
    // skinny chains: split K until the weight tiles of one token tile fill the SMs.
    // Inside the PDL chain every split CTA streams its weight ring before
    // griddepcontrol.wait, so more splits hide more of the weight read behind the
    // previous kernel (profiles/r01_gemm_splits.md)
    const int m_tiles = (n_out + BM - 1) / BM;
    s = std::max(1, std::min(knobs().split_slots * sms / m_tiles, kb / 4));
    if (knobs().chain_max_splits > 0) s = std::min(s, knobs().chain_max_splits);
    if (knobs().chain_bigk_splits > 0 && k >= 8192) s = knobs().chain_bigk_splits;
    // measured per-shape choice for the action expert's gate/up 8192 x 1024 (the
    // partitioned 1-stream denoise and the 8-stream frame, profiles/r02/split_ab*.txt):
    // unsplit, the GeGLU epilogue in the GEMM and no reduce launch.  (qkv in 8 was
    // 0.02 ms faster at 1 stream but takes it off the in-CTA split path at >= 16
    // streams, where its 8 fp32 partial slabs cost 3-10 ms per frame.)
    if (k == 1024 && n_out == 8192) s = 1;
    for (const auto &o : knobs().split_overrides)  // OXY_SPLITS="n,k,s;..." (A/B)
      if (o[0] == n_out && o[1] == k) s = o[2];
  }
  s = std::max(1, std::min(s, kb));
  const int per = (kb + s - 1) / s;
  return (kb + per - 1) / per;
}

Plan make_plan(int n_out, int k, int t, int sms, int force_splits) {
  Plan p{};
  p.sms = sms;
  p.kb_total = (k + BK - 1) / BK;
  // persistent 2-CTA kernel: in-frame it wins for the gate/up projections from
  // T = 256 and for every projection once T >= 2048 (multi-stream prefill);
  // at 1-stream T = 800 the narrower shapes stay on the one-tile-per-CTA kernel
  // (profiles/r01_gemm_wide.md).  OXY_GEMM_WIDE: -1 auto, 0 off, 1 / 2 force.
  // (K >= 8192 projections at T = 800 — the prefill down projection, 73.7 vs 98 us
  // stand-alone with split-K 2 — measured slower in the frame: 9.37 vs 9.27 ms prefill)
  const bool wide_ok =
      knobs().wide > 0 || (knobs().wide < 0 && ((n_out >= knobs().wide_min_n && t >= 256) || t >= 2048 ||
                                                (knobs().wide_min_k > 0 && k >= knobs().wide_min_k && t >= 256)));
  if (t > 64 && wide_ok && wide_plan(p, n_out, k, t, sms, force_splits)) return p;
  p.cg = 0;
  p.cl = 1;
  p.m_tiles = (n_out + BM - 1) / BM;
  p.n_tiles = (t + MAX_BN - 1) / MAX_BN;
  // wide token dims (prefill): narrower token tiles until the grid (with its K
  // splits) fills the SMs (one past: "at most one CTA per SM" plans measured slower
  // in the frame, 9.60 vs 9.27 ms prefill — the second CTA slot keeps the PDL chain
  // overlapping).  Token tiling never changes a result; only the K partition does.
  const int sp_hint = force_splits > 0 ? force_splits : 1;
  while (t > 64 && p.m_tiles * p.n_tiles * sp_hint < sms && (t + p.n_tiles) / (p.n_tiles + 1) >= 48) ++p.n_tiles;
  int per = (t + p.n_tiles - 1) / p.n_tiles;
  p.bn = std::max(16, (per + 15) / 16 * 16);
  // deep-K projections at prefill token counts: wider token tiles (half the weight
  // re-reads through L2) and split-K 2 to keep both CTA slots per SM busy
  const int *dk = knobs().bigk_min > 0 ? &knobs().bigk_min : g_deepk;
  if (knobs().bigk_min <= 0 && dk[0] > 0 && k < dk[0] && dk[3] > 0) dk += 3;  // second band
  if (dk[0] > 0 && k >= dk[0] && t >= 256) {
    p.band = dk == g_deepk + 3 ? 2 : 1;
    // the band's tile width is a cap when the generic tiling already needed narrower
    // tiles to fill the SMs (ViT o-proj / fc2: 72 / 108 CTAs at the band width)
    if (dk[1] > 0) p.bn = knobs().band_cap ? std::min(p.bn, std::min(MAX_BN, dk[1])) : std::min(MAX_BN, dk[1]);
    if (dk[2] > 0 && force_splits <= 0) force_splits = dk[2];
  }
  p.n_tiles = (t + p.bn - 1) / p.bn;
  const int base = p.m_tiles * p.n_tiles;
  int splits = 1;
  if (force_splits > 0) {
    splits = force_splits;
  } else if (base < sms && t <= knobs().split_t) {
    // skinny (decode / denoise): split K to fill the SMs.  Stand-alone, fewer
    // splits look cheaper (no reduce), but inside the PDL chain every split CTA
    // streams its weight ring before griddepcontrol.wait, so more splits hide
    // more of the weight read behind the previous kernel: measured in-frame,
    // this policy beats 'split only past 16 k-blocks' by 2.4 ms per denoise
    // (profiles/r01_gemm_splits.md)
    splits = std::max(1, std::min(knobs().split_slots * sms / base, p.kb_total / 4));
  }
  splits = std::max(1, std::min(splits, p.kb_total));
  const int per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + per_split - 1) / per_split;
  p.stages = std::max(2, std::min(MAX_STAGES, knobs().smem_kb * 1024 / (A_STAGE_BYTES + p.bn * BK * 2)));
  p.bm = BM;
  if (knobs().half_m > 0 && t <= 64 && n_out % 64 == 0 &&
      2 * p.m_tiles * p.n_tiles * p.splits <= knobs().half_m * sms) {
    p.bm = 64;
    p.m_tiles = n_out / 64;
  }
  return p;
}

// the plan's split partition accumulated in-CTA (kmulti) where the one-tile kernel
// can hold the splits' accumulators (2-4 regions of <= 256 / splits columns)
static void to_kmulti(Plan &p, int t) {
  if (p.cg == 0 && p.splits >= 2 && p.splits <= 4) {
    const int max_bn = 256 / p.splits / 16 * 16;
    if (p.bn > max_bn) {
      p.bn = max_bn;
      p.n_tiles = (t + p.bn - 1) / p.bn;
    }
    p.kmulti = p.splits;
    p.stages = std::max(2, std::min(MAX_STAGES, knobs().smem_kb * 1024 / (A_STAGE_BYTES + p.bn * BK * 2)));
  }
}

Plan make_chain_plan(int n_out, int k, int t, int sms, int splits) {
  Plan p = make_plan(n_out, k, t, sms, splits);
  if (knobs().kmulti && t >= KMULTI_MIN_T) to_kmulti(p, t);
  return p;
}

Plan make_prefill_plan(int n_out, int k, int t, int sms, int splits) {
  Plan p = make_plan(n_out, k, t, sms, splits);
  if (knobs().prefill_kmulti) to_kmulti(p, t);
  return p;
}

static size_t smem_bytes(const Plan &p) {
  return 1024 + (size_t)p.stages * (A_STAGE_BYTES + p.bn * BK * 2) + (2 * MAX_STAGES + 1) * 8 + 16;
}

static size_t wide_smem_bytes(const Plan &p) {
  return 1024 + (size_t)p.stages * (A_STAGE_BYTES + p.bn / p.cg * BK * 2) + (2 * MAX_STAGES + 4) * 8 + 16;
}

// Fixed-order split-K reduction + the real epilogue over [splits][t][n_out] partials.
static void launch_split_reduce(const float *ws, int splits, int t, int n_out, const EpiParams &epi, cudaStream_t st) {
  const int64_t n = (int64_t)t * ((n_out + 1) / 2);
  if (knobs().pdl) {
    // RoPE: the variant that fetches positions / (cos, sin) before the PDL wait
    // and keeps all split loads in flight; GeGLU / plain: the simple loop measured
    // faster in the denoise chain (8.94 vs 9.24 ms per denoise)
    static const int v = getenv("OXY_REDUCE_V") ? atoi(getenv("OXY_REDUCE_V")) : -1;
    const bool pre = v < 0 ? epi.mode == EPI_QKV_ROPE : v == 2;
    launch_pdl(pre ? splitk_reduce_kernel : splitk_reduce_v1_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0,
               st, ws, splits, t, n_out, epi);
  } else {
    splitk_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ws, splits, t, n_out, epi);
    OXY_LAUNCH_CHECK();
  }
}

static void launch_wide(const void *w, const void *x, int n_out, int k, int t, const EpiParams &epi,
                        const Plan &plan, float *ws, int *counters, cudaStream_t st) {
  wide_attrs();
  const int cg = plan.cg, cl = plan.cl > 0 ? plan.cl : 1;
  CUtensorMap ma = make_map(w, n_out, k, cl == 2 ? BM / 2 : BM);  // CL = 2: each CTA loads half its rows
  CUtensorMap mb = make_map(x, t, k, plan.bn / cg);
  WParams wp;
  wp.n_out = n_out;
  wp.k = k;
  wp.t = t;
  wp.bn = plan.bn;
  wp.stages = plan.stages;
  wp.kb_total = plan.kb_total;
  wp.m_tiles = plan.m_tiles;
  wp.n_tiles = plan.n_tiles;
  wp.splits = plan.splits;
  wp.kb_per_split = (plan.kb_total + plan.splits - 1) / plan.splits;
  wp.kdual = plan.kdual;
  wp.diag = knobs().wide_diag | (knobs().wide_nofence ? 4 : 0);
  wp.sleep_ns = knobs().wide_sleep;
  wp.tiles = plan.m_tiles * ((plan.n_tiles + cl - 1) / cl) * (plan.kdual ? 1 : plan.splits);
  wp.epi = epi;
  wp.ws = ws;
  wp.counters = counters;
  // split K with a real epilogue: partials only, then the parallel fixed-order reduce
  // kernel (bit-identical to the in-kernel fix-up, where the last-arriving CTA of a
  // tile sums and applies the epilogue alone: 487 vs ~50 us for the Gemma qkv + RoPE
  // and 320 vs ~45 us for the ViT fc2 at T = 6400; OXY_WIDE_FIXUP=1 restores it)
  const bool reduce_after = plan.splits > 1 && !plan.kdual && epi.mode != EPI_PARTIALS && !knobs().wide_fixup;
  if (reduce_after) wp.epi.mode = EPI_PARTIALS;
  int units = std::min(wp.tiles, std::max(1, wide_units(cg, cl, cl == 2 ? device_sms() : plan.sms)));
  if (knobs().wide_units > 0) units = std::min(units, knobs().wide_units);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * cg * cl);
  cfg.blockDim = dim3(WIDE_THREADS);
  cfg.dynamicSmemBytes = wide_smem_bytes(plan);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (knobs().pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cg == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2 * cl;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cg == 2 && cl == 2) OXY_CUDA(cudaLaunchKernelEx(&cfg, gemm_wide_kernel<2, 2>, ma, mb, wp));
  else if (cg == 2) OXY_CUDA(cudaLaunchKernelEx(&cfg, gemm_wide_kernel<2>, ma, mb, wp));
  else OXY_CUDA(cudaLaunchKernelEx(&cfg, gemm_wide_kernel<1>, ma, mb, wp));
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  if (reduce_after) launch_split_reduce(ws, plan.splits, t, n_out, epi, st);
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
  if (plan.splits > 1 && plan.m_tiles * plan.n_tiles * 2 > MAX_TILES) fail(OXY_EINVAL, "too many split-K tiles");
  if (plan.cg > 0) {
    if (epi.mode == EPI_ARGMAX) fail(OXY_EINVAL, "argmax LM head: one-tile-per-CTA plans only");
    ++g_plan_counts[plan.cg == 2 ? PC_WIDE_2CTA : PC_WIDE_1CTA];
    launch_wide(w, x, n_out, k, t, epi, plan, ws, counters, st);
    return;
  }
  if (epi.mode == EPI_ARGMAX) ++g_plan_counts[PC_ARGMAX_HEAD];
  ++g_plan_counts[plan.band == 1 ? PC_BAND_DEEPK
                  : plan.band == 2 ? PC_BAND_MIDK
                  : plan.splits > 1 ? PC_SKINNY_SPLIT
                                    : PC_SKINNY];
  // 64-row tiles only on the per-warp epilogue paths (argmax / TMA-stored partials /
  // fix-up / cluster split-K use all four epilogue warps)
  const int bm = plan.bm == 64 && epi.mode != EPI_ARGMAX && !knobs().tma_ws && !knobs().fixup && !plan.csk &&
                         !(plan.kmulti > 1)
                     ? 64
                     : BM;
  const int m_tiles = (n_out + bm - 1) / bm;
  CUtensorMap ma = make_map(w, n_out, k, bm);
  // one token tile covering T < bn: a T-row box (no out-of-bounds zero fill; fewer bytes,
  // neutral in the frame — profiles/r02_skinny_gemm.md)
  const int b_box = plan.n_tiles == 1 && t < plan.bn && knobs().bbox_exact ? t : plan.bn;
  CUtensorMap mb = make_map(x, t, k, b_box);
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
  kp.prefetch = kp.trigger = t <= 64 ? (g_early_override >= 0 ? g_early_override : knobs().early_skinny)
                                     : knobs().early_wide;
  kp.b_box = b_box;
  kp.bm = bm;
  kp.kmulti = plan.kmulti > 1 && plan.cg == 0 ? plan.kmulti : 0;
  if (kp.kmulti && (plan.bn * kp.kmulti > 256 || kp.kmulti != plan.splits))
    fail(OXY_EINVAL, "in-CTA split-K: %d partitions x %d token columns", kp.kmulti, plan.bn);
  kp.csk = plan.csk && plan.splits > 1 && !plan.kmulti;
  if (epi.mode == EPI_ARGMAX && (plan.splits != 1 || !epi.amax_idx))
    fail(OXY_EINVAL, "argmax LM head: unsplit plan and an index buffer required");
  if (epi.norm.y && !(kp.csk && t <= NORM_FUSE_MAX_T && (epi.mode == EPI_ADD_F32 || epi.mode == EPI_ADD_GATED_F32)))
    fail(OXY_EINVAL, "fused row norm needs a cluster split-K residual GEMM of <= %d rows", NORM_FUSE_MAX_T);
  if (epi.norm.y && (n_out % 128 != 0 || n_out > 128 * NORM_MAX_V4 || epi.ldo % 4 != 0 || epi.norm.ldy % 4 != 0))
    fail(OXY_EINVAL, "fused row norm: rows of 128..2048 features (multiple of 128), strides multiple of 4");
  // TMA-stored partials: [splits][t][n_out] fp32, box 128 features x bn tokens x 1 split
  // (staged in the operand ring, which must hold the 128 x bn fp32 tile)
  kp.tma_ws = plan.splits > 1 && !kp.kmulti && !kp.fixup && !kp.csk && knobs().tma_ws &&
              (size_t)BM * plan.bn * 4 <= (size_t)plan.stages * (A_STAGE_BYTES + plan.bn * BK * 2) &&
              (n_out * 4) % 16 == 0;
  const CUtensorMap mw = kp.tma_ws ? make_map_ws(ws, plan.splits, t, n_out, plan.bn) : ma;
  dim3 grid(plan.n_tiles, m_tiles, kp.kmulti ? 1 : plan.splits);
  if (kp.csk) {
    if (plan.splits > CSK_MAX) fail(OXY_EINVAL, "cluster split-K: at most %d splits", CSK_MAX);
    static bool np_set = false;
    if (!np_set) {
      OXY_CUDA(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      np_set = true;
    }
    ++g_plan_counts[PC_CSK];
    if (epi.norm.y) ++g_plan_counts[PC_CSK_NORM];
    launch_pdl_cluster(gemm_kernel, grid, dim3(192), smem_bytes(plan), st, dim3(1, 1, plan.splits), ma, mb, mw, kp);
    return;
  }
  if (knobs().pdl) {
    launch_pdl(gemm_kernel, grid, dim3(192), smem_bytes(plan), st, ma, mb, mw, kp);
  } else {
    gemm_kernel<<<grid, 192, smem_bytes(plan), st>>>(ma, mb, mw, kp);
    OXY_LAUNCH_CHECK();
  }
  if (plan.splits > 1 && !kp.kmulti && !kp.fixup && epi.mode != EPI_PARTIALS)
    launch_split_reduce(ws, plan.splits, t, n_out, epi, st);
}

// One CTA per token row, one thread per 4 consecutive features (n / 4 threads):
// every load of the row — all split partials, the residual, gate and norm
// weights — is issued before any arithmetic, so the kernel costs one L2 round
// trip plus the block reduction.  Split order 0..S-1 per element.
constexpr int RN_CHUNK = 16;  // split partials in flight per thread
__global__ void __launch_bounds__(512)
    splitk_residual_norm_kernel(const float *ws, int splits, int t_rows, int n, const float *gate, float *x,
                                int ldx, __nv_bfloat16 *y, int ldy, const float *w, const float *ms,
                                const float *mb, float eps) {
  pdl_trigger();
  const int t = blockIdx.x, f = threadIdx.x * 4;
  // weights do not depend on the previous kernel: fetch them before the wait
  float4 wv = make_float4(0.f, 0.f, 0.f, 0.f), sv = wv, bv = wv, gv = make_float4(1.f, 1.f, 1.f, 1.f);
  if (w) wv = __ldg(reinterpret_cast<const float4 *>(w + f));
  else {
    sv = __ldg(reinterpret_cast<const float4 *>(ms + f));
    bv = __ldg(reinterpret_cast<const float4 *>(mb + f));
  }
  if (gate) gv = __ldg(reinterpret_cast<const float4 *>(gate + f));
  pdl_wait();
  __shared__ float red[32];
  float4 xv = *reinterpret_cast<const float4 *>(x + (size_t)t * ldx + f);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s0 = 0; s0 < splits; s0 += RN_CHUNK) {
    float4 p[RN_CHUNK];
#pragma unroll
    for (int s = 0; s < RN_CHUNK; ++s)
      if (s0 + s < splits) p[s] = __ldcg(reinterpret_cast<const float4 *>(ws + ((size_t)(s0 + s) * t_rows + t) * n + f));
#pragma unroll
    for (int s = 0; s < RN_CHUNK; ++s)
      if (s0 + s < splits) {
        a.x += p[s].x;
        a.y += p[s].y;
        a.z += p[s].z;
        a.w += p[s].w;
      }
  }
  xv.x += gv.x * a.x;
  xv.y += gv.y * a.y;
  xv.z += gv.z * a.z;
  xv.w += gv.w * a.w;
  *reinterpret_cast<float4 *>(x + (size_t)t * ldx + f) = xv;
  float ss = xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / (float)n + eps);
  float o0, o1, o2, o3;
  if (w) {
    o0 = xv.x * inv * (1.f + wv.x), o1 = xv.y * inv * (1.f + wv.y);
    o2 = xv.z * inv * (1.f + wv.z), o3 = xv.w * inv * (1.f + wv.w);
  } else {
    o0 = xv.x * inv * (1.f + sv.x) + bv.x, o1 = xv.y * inv * (1.f + sv.y) + bv.y;
    o2 = xv.z * inv * (1.f + sv.z) + bv.z, o3 = xv.w * inv * (1.f + sv.w) + bv.w;
  }
  __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
  uint2 out;
  out.x = *reinterpret_cast<uint32_t *>(&h0);
  out.y = *reinterpret_cast<uint32_t *>(&h1);
  *reinterpret_cast<uint2 *>(y + (size_t)t * ldy + f) = out;
}

void splitk_residual_norm(const float *ws, int splits, int t, int n, const float *gate, float *x, int ldx,
                          __nv_bfloat16 *y, int ldy, const float *w, const float *mod_scale,
                          const float *mod_shift, float eps, cudaStream_t st) {
  ++g_plan_counts[PC_SPLIT_RES_NORM];
  if (t <= 0) return;
  if (n % 128 != 0 || n > 2048) fail(OXY_EINVAL, "fused residual norm: rows of 128..2048 features (multiple of 128)");
  if (ldx % 4 != 0 || ldy % 4 != 0) fail(OXY_EINVAL, "fused residual norm: row strides must be multiples of 4");
  launch_pdl(splitk_residual_norm_kernel, dim3(t), dim3(n / 4), 0, st, ws, splits, t, n, gate, x, ldx, y, ldy, w,
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

extern "C" int oxy_gemm_policy_splits(int32_t phase, int32_t n_out, int32_t k, int32_t *splits) {
  OXY_API_BEGIN
  OXY_REQUIRE(splits && n_out > 0 && k > 0 && (phase == 0 || phase == 1), "bad policy query");
  int dev = 0, sms = 148;
  OXY_CUDA(cudaGetDevice(&dev));
  OXY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  *splits = oxy::gemm::policy_splits(phase, n_out, k, sms);
  OXY_API_END
}

extern "C" int oxy_plan_counts(int64_t *out, int32_t n, int32_t reset) {
  OXY_API_BEGIN
  OXY_REQUIRE(n >= 0 && (n == 0 || out), "bad plan-count buffer");
  for (int i = 0; i < n && i < oxy::gemm::PC_COUNT; ++i) out[i] = oxy::gemm::g_plan_counts[i];
  if (reset)
    for (auto &c : oxy::gemm::g_plan_counts) c = 0;
  OXY_API_END
}

extern "C" int oxy_gemm_plan(int32_t n_out, int32_t k, int32_t t, int32_t splits, int32_t *out6) {
  OXY_API_BEGIN
  oxy::gemm::Plan p = oxy::gemm::make_plan(n_out, k, t, oxy::gemm::device_sms(), splits);
  out6[0] = p.bn;
  out6[1] = p.n_tiles;
  out6[2] = p.m_tiles;
  out6[3] = p.splits;
  out6[4] = p.stages;
  out6[5] = p.kb_total;
  OXY_API_END
}

#ifdef OXY_GEMM_PROF
extern "C" int oxy_debug_gemm_prof_select(int n_out, int k) {
  const int v[2] = {n_out, k};
  return cudaMemcpyToSymbol(oxy::gemm::g_gemm_prof_sel, v, sizeof(v)) == cudaSuccess ? 0 : -1;
}
extern "C" int oxy_debug_wide_prof(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, oxy::gemm::g_wide_prof, sizeof(oxy::gemm::g_wide_prof)) == cudaSuccess ? 0 : -1;
}
extern "C" int oxy_debug_gemm_prof(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, oxy::gemm::g_gemm_prof, sizeof(oxy::gemm::g_gemm_prof)) == cudaSuccess ? 0 : -1;
}
#endif
