// F2 (pi0.5-shaped) kernels other than the GEMM.  See pi05_kernels.cu.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace oxy {
namespace pi05 {

using bf16 = __nv_bfloat16;

constexpr int KV_BLOCK = 64;   // pool block size (positions) = one attention key tile
constexpr int HEAD_DIM = 256;  // Gemma head dim (pool row)
constexpr int Q_HEADS = 8;     // Gemma query heads per KV head (MQA)

// ---- norms / elementwise --------------------------------------------------
// y[r] = bf16( x[r] * rsqrt(mean(x[r]^2) + eps) * (1 + w) )            (w != null)
//      = bf16( x[r] * rsqrt(...) * (1 + mod_scale) + mod_shift )       (adaRMS)
void rmsnorm(const float *x, int ldx, bf16 *y, int ldy, const float *w, const float *mod_scale,
             const float *mod_shift, int rows, int D, float eps, cudaStream_t st);
// y[r] = bf16( (x - mean) * rstd * w + b )
void layernorm(const float *x, int ldx, bf16 *y, int ldy, const float *w, const float *b, int rows,
               int D, float eps, cudaStream_t st);
// x[r] = float(table[tok[r]]) * scale (rows with active[r]==0 skipped if active)
void embed_rows(float *x, int ldx, const bf16 *table, const int *tok, const int *active, int rows,
                int D, float scale, cudaStream_t st);
// dst[f, :] = src[gemm::qkv_rope_row(f), :] (rotary-pair interleaved QKV weights)
void permute_rows(bf16 *dst, const bf16 *src, int rows, int cols, cudaStream_t st);
// (cos, sin) of fp32(pos * inv_freq[i]) for pos < n_pos (sin/cos evaluated in fp64)
void rope_table(float2 *cs, const float *inv_freq, int n_pos, cudaStream_t st);
// images uint8 [n, 224, 224, 3] -> patches bf16 [n*256, kpad] (x/127.5 - 1, (dy,dx,c) order)
void patchify(const uint8_t *img, int n, bf16 *patches, int kpad, cudaStream_t st);
// dst[i*ld + j] = src[(i % period) * ld_src + j] (broadcast of per-image tables)
void tile_rows(float *dst, int ld, const float *src, int ld_src, int rows, int period, int D,
               cudaStream_t st);
void f32_to_bf16(const float *x, bf16 *y, int64_t n, cudaStream_t st);
// a += dt * v (fp32), and a_bf16 = bf16(a)
void euler_step(float *a, const float *v, bf16 *a_bf, int64_t n, float dt, cudaStream_t st);
// standard normal noise from splitmix64 (Box-Muller, counter form)
void normal_noise(float *out, int64_t n, uint64_t seed, cudaStream_t st);
// bf16 weights from splitmix64 counter: U(-bound, bound) in draw order starting at `offset`
void init_uniform_bf16(bf16 *out, int64_t n, uint64_t seed, uint64_t offset, float bound,
                       cudaStream_t st);
void init_uniform_f32(float *out, int64_t n, uint64_t seed, uint64_t offset, float bound,
                      float center, cudaStream_t st);
// copy-on-write of shared tail blocks (cow[r] = {src, dst, n}) for all layers
void cow_blocks(bf16 *pool, const int *cow, int rows, int L, size_t layer_stride,
                size_t kv_stride, cudaStream_t st);
// slot of each active row's next position
void next_slots(int *slot, const int *pos, const int *active, const int *bt, int bt_stride,
                int rows, cudaStream_t st);

// ---- attention -------------------------------------------------------------
struct AttnGroup {
  const bf16 *q;   // query row r at q + r * ldq
  bf16 *o;         // output row r at o + r * ldo
  int ldq, ldo, nq;
  const int *bt;   // segment A: paged keys [0, nka) through this block table
  int nka;
  const bf16 *kb, *vb;  // segment B: dense keys [0, nkb), row stride ldkv
  int ldkv, nkb;
  int wrow0;       // first workspace row of this group (split-KV)
};

// Bidirectional (prefix-LM / suffix / ViT) flash attention, mma.sync bf16.
// head_dim 256 (paged allowed) or 72 (dense only).  splits > 1 uses ws.
void flash_attention(const AttnGroup *groups_d, int n_groups, int max_q_tiles, int head_dim,
                     const bf16 *kpool, const bf16 *vpool, float scale, int splits,
                     int max_key_tiles, float *ws_o, float *ws_ml, int ws_rows, cudaStream_t st);

// tcgen05 flash attention, head dim 256 (attn_tc.cu): groups' q rows are rows of
// q_base viewed as [q_rows, 256]; paged keys through kpool/vpool maps (box 64x64),
// dense keys g.kb/g.vb rows of kd_base/vd_base [kd_rows, 256] (null: none).
// q_tiles = ceil(max nq / 128).  Key splits are per group: attn_group_splits(tiles,
// tps) — a function of the group's own key count, so a group's output does not
// depend on the other groups of the call; `splits` (grid y) is the largest group's
// count.  Groups with more than one split write ws (merged in-kernel over a
// cluster when cmerge, else by flash_merge; both merges do identical arithmetic).
// kv_ready: the paged K/V were not written by the previous kernel on the stream
// (the expert suffix over an earlier prefill), so they are prefetched before the PDL wait.
__host__ __device__ inline int attn_group_splits(int tiles, int tps, int &per) {
  per = tps > 0 ? tps : 1;
  if ((tiles + per - 1) / per > 32) per = (tiles + 31) / 32;  // the merges take <= 32 splits
  return tiles > 0 ? (tiles + per - 1) / per : 1;
}
void flash_attention_tc(const AttnGroup *groups_d, int n_groups, int q_tiles, int splits, int tps, const bf16 *q_base,
                        int q_rows, const CUtensorMap &kpool_map, const CUtensorMap &vpool_map, const bf16 *kd_base,
                        const bf16 *vd_base, int kd_rows, float scale, float *ws_o, float *ws_ml, int ws_rows,
                        bool kv_ready, bool cmerge, cudaStream_t st, int lane_sms = 0);
// largest split count merged inside the attention kernel over DSMEM (clusters of
// `splits` CTAs); larger counts use the workspace + flash_merge.  OXY_ATTN_CMERGE:
// the cap (default 16; 0 or 1 = always the workspace merge)
int attn_cluster_merge_max();
// split-order merge of the tcgen05 kernel's bf16 head-dim-256 partials (ws rows as in flash_attention)
// SigLIP self-attention on tcgen05: 256 tokens per image, `heads` heads of dim 72,
// q/k/v read from the fused qkv rows [n_images * 256, 3 * 72 heads], output
// [n_images * 256, 72 heads] bf16.  One CTA per (image, head, 128 queries).
void vit_attention_tc(const bf16 *qkv, bf16 *out, int n_images, int heads, cudaStream_t st);
void flash_merge(const AttnGroup *groups_d, int n_groups, int max_rows, int splits, int tps, const bf16 *ws_o,
                 const float *ws_ml, int ws_rows, cudaStream_t st);

// Decode-attention key chunking of one row: chunks of `cb_min` pool blocks, widened
// only when the row's own context would need more than 64 chunks.  A function of the
// row's own length, never of the batch (rows, longest context): batch-invariant.
constexpr int DECODE_CHUNK_BLOCKS = 2;
__host__ __device__ inline int decode_row_chunk(int nb, int cb_min) {
  return nb > 64 * cb_min ? (nb + 63) / 64 : cb_min;
}
// Paged decode attention: rows x 8 q-heads vs 1 KV head, keys [0, pos[r]].  A
// persistent grid (<= 2 CTAs per SM) streams work items — whole rows, or (row,
// chunk) pairs when there are too few rows to fill the SMs — through a TMA-fed ring;
// chunk partials are folded in chunk order (in registers, or by a fold kernel).
// kmap/vmap: 2-D tensor maps over one layer's K / V pool viewed as [num_blocks*64, 256]
// (box 64 x 64, 128-byte swizzle; gemm::make_map).  ws: rows*max_blocks*8*(256+2) floats.
constexpr int MAX_DECODE_ROWS_ABI = 8192;
void decode_attention_v3(const CUtensorMap &kmap, const CUtensorMap &vmap, const bf16 *q, bf16 *out, const int *bt,
                         int bt_stride, const int *pos, const int *active, int rows, int max_blocks, float scale,
                         float *ws, int sms, cudaStream_t st);

// Greedy token + continuous-batching state update over logits [rows, V].
// part: rows * 64 (val, idx) scratch.
// no-cache recompute route: dense fp32 attention with the prefix-LM mask (q [T, 8*256],
// k / v [T, 256] bf16 rows; keys [0, P) for t < P, else [0, t])
void prefix_lm_attention_ref(const bf16 *q, const bf16 *k, const bf16 *v, bf16 *out, int T, int P, float scale,
                             cudaStream_t st);
// fold of the LM head's EPI_ARGMAX partials ([rows][tiles] max / id) + the same state update
void argmax_tiles_update(int rows, int tiles, const float *pv, const int *pi, int step, int k, int eos, int *active,
                         int *tok, int *pos, int *count, const int *budget, int *out_tokens, cudaStream_t st);
void argmax_update(const float *logits, int rows, int V, int step, int k, int eos, int *active,
                   int *tok, int *pos, int *count, const int *budget, int *out_tokens,
                   float *part_val, int *part_idx, cudaStream_t st);
}  // namespace pi05
}  // namespace oxy
