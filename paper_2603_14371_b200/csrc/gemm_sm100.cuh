// tcgen05 GEMM for sm_100a: Y[t, f] (op)= sum_k W[f, k] * X[t, k].
//
// Weights are the UMMA A operand (M = 128 output features per tile) and the
// activations the B operand (N = BN tokens per tile, 16..256, runtime), both
// bf16 K-major, loaded by TMA with 128-byte swizzle into a multi-stage smem
// ring; fp32 accumulators live in TMEM.  Putting the weights on M keeps the
// same kernel efficient from 1-token decode (BN = 16) to 800-token prefill:
// a weight tile is streamed from HBM once per token tile.  Split-K spreads
// skinny (decode / denoise) GEMMs over all 148 SMs; partial sums are reduced
// in a fixed order so results do not depend on timing.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace oxy {
namespace gemm {

enum Epi : int {
  EPI_F32 = 0,        // out_f32[t, f] = acc (+ bias)
  EPI_BF16 = 1,       // out_bf16[t, f] = acc (+ bias)
  EPI_ADD_F32 = 2,    // out_f32[t, f] += acc (+ bias)          residual stream
  EPI_GEGLU_BF16 = 3, // rows (2j, 2j+1) = (gate_j, up_j): out_bf16[t, j] = gelu_tanh(g) * u
  EPI_GELU_BF16 = 4,  // out_bf16[t, f] = gelu_tanh(acc + bias)
  EPI_ADD_BF16 = 5,   // out_bf16[t, f] = bf16(acc + bias + res_f32[t, f])  (no in-place)
  EPI_ADD_GATED_F32 = 6,  // out_f32[t, f] += gate[f] * (acc + bias)     adaRMS gated residual
  EPI_SWISH_BF16 = 7,     // out_bf16[t, f] = swish(acc + bias)
  EPI_QKV_ROPE = 8,       // fused QKV projection: RoPE on q/k (rotary pairs interleaved in the
                          // weight rows), q -> bf16 [T, 2048], k/v -> pool slot rows or dense rows
  EPI_PARTIALS = 9,       // split-K partials only; the caller launches its own fused reduction
  EPI_ARGMAX = 10,        // greedy LM head: no logits; per (token, 128-row weight tile) the max
                          // accumulator and its lowest row id -> out_f32[t, tile] / amax_idx[t, tile]
                          // (ldo = tiles per token row); unsplit one-tile-per-CTA plans only
};

// Fused split-K reduction + residual + RMSNorm (one CTA per token row):
//   x[t, :] += (gate ? gate : 1) * sum_s ws[s, t, :]          (fixed split order)
//   y[t, :] = bf16( x * rsqrt(mean(x^2) + eps) * (1 + w) )       (w != null)
//           = bf16( x * rsqrt(...) * (1 + mod_scale) + mod_shift ) (adaRMS)
void splitk_residual_norm(const float *ws, int splits, int t, int n, const float *gate, float *x, int ldx,
                          __nv_bfloat16 *y, int ldy, const float *w, const float *mod_scale,
                          const float *mod_shift, float eps, cudaStream_t st);

// Extra state of EPI_QKV_ROPE (8 q heads + 1 k + 1 v head of 256).
constexpr int ROPE_TABLE_POS = 16384;  // positions covered by the cos/sin table
struct QkvRope {
  const float *inv_freq;  // [128]
  const float2 *cs;       // [ROPE_TABLE_POS][128] (cos, sin) of fp32(pos * inv_freq), or null
  const int *pos;         // [T]
  const int *slot;        // [T] pool slot (<0: skip k/v) or null: dense k/v rows
  __nv_bfloat16 *q_out;   // [T, 2048]
  __nv_bfloat16 *k_dst, *v_dst;  // pool layer base (slot rows) or dense [T, 256]
};

// RMSNorm / adaRMSNorm of the finished residual rows, fused into a cluster
// split-K GEMM with an EPI_ADD_F32 / EPI_ADD_GATED_F32 epilogue (y != null):
//   y[t, :] = bf16( x * rsqrt(mean(x^2) + eps) * (1 + w) )            (w != null)
//           = bf16( x * rsqrt(mean(x^2) + eps) * (1 + ms) + mb )      (adaRMS)
// over the whole row x[t, 0..N) (x = the epilogue's out, N = n_out).
struct NormFuse {
  __nv_bfloat16 *y = nullptr;
  int ldy = 0;
  const float *w = nullptr, *ms = nullptr, *mb = nullptr;
  float eps = 1e-6f;
};

struct EpiParams {
  int mode;
  void *out;
  int ldo;              // row stride of out (elements)
  const float *bias;    // [N] or null
  const float *res;     // EPI_ADD_BF16 residual input [T, ldr]
  int ldr;
  const float *gate;    // EPI_ADD_GATED_F32 per-feature gate [N]
  QkvRope rope;         // EPI_QKV_ROPE
  NormFuse norm{};      // cluster split-K residual modes only
  int *amax_idx = nullptr;  // EPI_ARGMAX row ids
};

// The row norm of NormFuse as a stand-alone kernel (one warp per row), bit-identical
// to the fused one: used when the rows are too many for the fused tail.
void rownorm(const float *x, int ldx, int t, int n, const NormFuse &nf, cudaStream_t st);
constexpr int NORM_FUSE_MAX_T = 64;  // rows the last cluster normalises in-kernel
constexpr int CSK_MAX = 16;          // cluster split-K: splits per cluster (non-portable above 8)

// Row permutation that puts rotary pair (i, i + 128) of every q/k head at rows
// (2i, 2i + 1): new row -> canonical row.  V rows (f >= 2304) are unchanged.
__host__ __device__ inline int qkv_rope_row(int f) {
  if (f >= 9 * 256) return f;
  const int h = f >> 8, j = f & 255;
  return (h << 8) + ((j & 1) ? (j >> 1) + 128 : (j >> 1));
}

constexpr int BM = 128;        // weight rows per tile (UMMA M)
constexpr int BK = 64;         // K per stage: 64 bf16 = one 128-byte swizzle row
constexpr int MAX_BN = 256;
constexpr int MAX_STAGES = 8;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int SMEM_BUDGET = 200 * 1024;
constexpr int MAX_TILES = 1 << 16;  // split-K tile counters

struct Plan {
  int bn, n_tiles, m_tiles, splits, stages, kb_total;
  int cg;  // 0: one-tile-per-CTA kernel (skinny); 1 / 2: persistent wide kernel, 1-CTA / CTA-pair tiles
  int cl;  // wide kernel: CTA pairs per cluster sharing (multicasting) the weight tile (1 or 2)
  int band;  // prefill token-tile band applied: 0 none, 1 deep-K, 2 mid-K
  int csk;   // 1: the split CTAs of a tile form one cluster and reduce in-kernel (no reduce launch)
  int kdual; // persistent kernel, 2 K splits: one CTA (pair) accumulates both K halves of a tile
             // into two TMEM accumulators and sums them (p0 + p1) in its epilogue — the
             // split-2 result bit for bit, without the fp32 partial round trip
  int kmulti;  // one-tile kernel: the `splits` K partitions of a tile accumulated by ONE CTA into
              // `splits` TMEM regions and summed in split order in its epilogue (no partials,
              // no reduce launch; bit-identical to split CTAs + reduce).  0 = split CTAs.
  int bm;      // one-tile kernel: weight rows per CTA tile — 128, or 64 for skinny chains whose
              // 128-row grid leaves CTA slots idle (the MMA stays M = 128: rows 64..127 of the
              // A stage are stale and their accumulator lanes are never stored, so every output
              // element is computed bit for bit as with 128-row tiles); 0 = 128
  int sms;     // SMs the plan was made for (the persistent kernel's grid; an SM partition's size)
  int partials() const { return kdual || kmulti ? 1 : splits; }  // partial slabs an EPI_PARTIALS launch writes
};

// Plan classes counted at enqueue time (eager runs and graph captures; replays are
// not re-counted) so tests can assert which code paths a call exercised.
enum PlanClass {
  PC_SKINNY = 0,      // gemm_kernel, whole K
  PC_SKINNY_SPLIT,    // gemm_kernel, split K
  PC_BAND_DEEPK,      // gemm_kernel with the deep-K prefill band (128-token tiles)
  PC_BAND_MIDK,       // gemm_kernel with the mid-K prefill band (96-token tiles)
  PC_WIDE_1CTA,       // persistent gemm_wide_kernel<1>
  PC_WIDE_2CTA,       // persistent gemm_wide_kernel<2> (cta_group::2)
  PC_SPLIT_RES_NORM,  // split reduce + residual + RMSNorm fused
  PC_ATTN_CMERGE,     // tcgen05 attention, key splits merged over a cluster
  PC_ATTN_WSMERGE,    // tcgen05 attention, key splits merged through the workspace
  PC_ATTN_ONE,        // tcgen05 attention, one split
  PC_CSK,             // gemm_kernel, cluster split-K (in-kernel reduction)
  PC_CSK_NORM,        // ... with the residual RMSNorm fused into the last cluster
  PC_ARGMAX_HEAD,     // LM head with the greedy argmax epilogue (no logits in HBM)
  PC_VIT_TC,          // SigLIP attention on tcgen05 (vit_attn_tc_kernel)
  PC_COUNT
};
extern long long g_plan_counts[PC_COUNT];

// Skinny-GEMM early PDL (weight prefetch before the wait + early dependent
// launch) for the launches that follow: -1 = knob default, 0 / 1 = force.
extern int g_early_override;
extern int g_deepk[6];

// Batch-invariant split-K policy.  The K partition of a projection — and so the
// fp32 summation order of every output element — is a function of (phase, N_out,
// K) only, never of the token count: a row's result is the same whether it is
// projected alone or inside any batch (decode rows, lock-stepped streams).  The
// token tiling (BN, tiles, 1- or 2-CTA kernel) may vary freely: tcgen05 computes
// each output element from its own row and column only.
enum Phase { PH_PREFILL = 0, PH_CHAIN = 1 };
int policy_splits(int phase, int n_out, int k, int sms);

// Host: build a plan for (N_out, K, T) on `sms` SMs.  force_splits > 0 fixes the K
// partition (every kernel variant honours it); 0 = pick for speed (C ABI tests).
Plan make_plan(int n_out, int k, int t, int sms, int force_splits = 0);
// chain-phase variant: for token counts >= KMULTI_MIN_T (>= 11 streams) and 2..4 splits,
// accumulate the splits in-CTA (Plan::kmulti) with token tiles of <= 256 / splits
Plan make_chain_plan(int n_out, int k, int t, int sms, int splits);
Plan make_prefill_plan(int n_out, int k, int t, int sms, int splits);
constexpr int KMULTI_MIN_T = 512;

// Host: launch.  ws must hold splits * T * N_out floats when splits > 1.
void launch(const void *w, const void *x, int n_out, int k, int t, const EpiParams &epi,
            const Plan &plan, float *ws, int *counters, cudaStream_t st);
// 2-D TMA map over a row-major bf16 [rows, k] matrix, box (64 cols x box_rows), 128-byte swizzle
CUtensorMap make_map(const void *ptr, int rows, int k, int box_rows);
// 2-D TMA map over a row-major fp32 [rows, cols] matrix, box (box_cols x box_rows), 128-byte swizzle
CUtensorMap make_map_f32(const void *ptr, int rows, int cols, int box_cols, int box_rows);
// self-resetting split-K tile counters for launches made through the C ABI
int *counters_for_abi();

}  // namespace gemm
}  // namespace oxy
