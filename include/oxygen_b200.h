/*
 * oxygen_b200.h — C ABI of the B200 unified-KV hot path (liboxygen_b200.so).
 *
 * The reference (kvweaver, pure Python) has no FFI: its plugin boundary is the
 * duck-typed backend protocol + KvManager.  This ABI sits
 * UNDER that Python surface; paper_2603_14371_b200/_lib.py binds it with
 * ctypes.  Each entry point names the reference interface it replaces.
 *
 * Conventions: every function returns int status (OXY_OK = 0); on failure
 * oxy_last_error() returns a thread-local message.  Plain pointers and sizes
 * only; "stream" is a cudaStream_t passed as void* (NULL = legacy stream).
 * Host pointers are marked _h, device pointers _d.  Not thread-safe per
 * object: one scheduler thread owns a pool/model.
 */
#ifndef OXYGEN_B200_H
#define OXYGEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OXY_OK 0
#define OXY_EINVAL 1     /* bad argument (maps to ValueError)            */
#define OXY_ENOBLOCKS 2  /* KV pool out of blocks (maps to MemoryError)  */
#define OXY_ECUDA 3      /* CUDA runtime/driver failure (RuntimeError)   */
#define OXY_ESTATE 4     /* allocator invariant violated (RuntimeError)  */

const char *oxy_last_error(void);
int oxy_abi_version(void);

/* ------------------------------------------------------------------------
 * Deterministic paged-KV block allocator (host side, no CUDA).
 * Replaces the per-request numpy copies owned by kvweaver/kv_manager.py:35-105
 * with shared refcounted blocks.  Semantics are pinned in oracle/paged_alloc.py
 * (lowest free id first; refcount; per-block fill watermark; copy-on-write of
 * a shared partially-filled tail).
 * ---------------------------------------------------------------------- */
typedef struct oxy_alloc oxy_alloc;

int oxy_alloc_create(int32_t num_blocks, int32_t block_size, oxy_alloc **out);
int oxy_alloc_destroy(oxy_alloc *a);
/* fresh sequence of n_tokens positions (prefill, kvweaver/backend.py:309-314);
 * writes ceil(n_tokens/B) block ids */
int oxy_alloc_seq(oxy_alloc *a, int32_t n_tokens, int32_t *blocks_h);
int oxy_alloc_incref(oxy_alloc *a, const int32_t *blocks_h, int32_t n);
int oxy_alloc_decref(oxy_alloc *a, const int32_t *blocks_h, int32_t n);
/* extend a handle (blocks, seq_len) by up to n_new positions (decode append,
 * kvweaver/backend.py:389-411).  Writes ceil((seq_len+n_new)/B) ids to
 * new_blocks_h and cow_h[3] = {src, dst, n_slots} (src = -1: no copy). */
int oxy_alloc_reserve(oxy_alloc *a, const int32_t *blocks_h, int32_t seq_len, int32_t n_new,
                      int32_t *new_blocks_h, int32_t *cow_h);
/* after the decode: keep ceil((seq_len+n_actual)/B) blocks, free the rest,
 * lower the tail watermark to what was written */
/* blocks oxy_alloc_reserve(blocks_h, seq_len, n_new) would take from the free
 * list right now (new tail blocks + a copy-on-write copy); allocates nothing.
 * Admission control (paged.BlockAllocator) uses it to keep decode from ever
 * running out of blocks for admitted requests. */
int oxy_alloc_reserve_need(const oxy_alloc *a, const int32_t *blocks_h, int32_t seq_len, int32_t n_new,
                           int32_t *need);
int oxy_alloc_settle(oxy_alloc *a, const int32_t *blocks_h, int32_t seq_len,
                     int32_t n_reserved, int32_t n_actual, int32_t *n_blocks_out);
int oxy_alloc_num_free(const oxy_alloc *a, int32_t *out);
/* full state for parity tests: refcount[nb], fill[nb], sorted free ids */
int oxy_alloc_snapshot(const oxy_alloc *a, int32_t *refcount_h, int32_t *fill_h,
                       int32_t *free_h, int32_t *n_free);
/* slot(p) = blocks[p / B] * B + p % B for p in [start, start+count) */
int oxy_build_slot_mapping(const int32_t *blocks_h, int32_t block_size, int32_t start,
                           int32_t count, int32_t *slots_h);

/* ------------------------------------------------------------------------
 * F1: the reference toy transformer on the GPU (kvweaver/backend.py:235-420),
 * fp32 verification mode (dtype 0) or fp64 (dtype 1).  KV pool per layer:
 * K and V [num_blocks, block_size, d_model] in the model dtype.
 * ---------------------------------------------------------------------- */
typedef struct oxy_toy oxy_toy;

typedef struct oxy_toy_config {
  int32_t L, d_model, n_heads, vocab, eos_token, action_dim, H;
  uint64_t seed;
} oxy_toy_config;

/* ToyBackend.__init__ (kvweaver/backend.py:238-267): weights drawn on device
 * from the splitmix64 counter form, in the reference draw order. */
int oxy_toy_create(const oxy_toy_config *cfg, int32_t dtype, int32_t num_blocks,
                   int32_t block_size, void *stream, oxy_toy **out);
int oxy_toy_destroy(oxy_toy *m);
/* read (write=0) or overwrite (write=1) one weight tensor as float64:
 * which 0 embed,1 wq,2 wk,3 wv,4 wo,5 w1,6 w2,7 unembed,8 action_head */
int oxy_toy_weight(oxy_toy *m, int32_t which, int32_t layer, double *host, int64_t n,
                   int32_t write, void *stream);
/* prefill (kvweaver/backend.py:276-314): causal pass, K/V into the pool blocks */
int oxy_toy_prefill(oxy_toy *m, const int32_t *tokens_h, int32_t T, const int32_t *blocks_h,
                    void *stream);
/* recompute_logits (kvweaver/backend.py:301-304): no-cache pass, last row */
int oxy_toy_recompute_logits(oxy_toy *m, const int32_t *tokens_h, int32_t T,
                             double *logits_h, void *stream);
/* action_denoise (kvweaver/backend.py:316-332): reads the cache, S Euler steps */
int oxy_toy_denoise(oxy_toy *m, const int32_t *blocks_h, int32_t seq_len, int32_t S,
                    double *actions_h, void *stream);
/* batched_language_decode (kvweaver/backend.py:334-420): up to k greedy steps
 * for m rows; per-row stop on EOS / budget on device.  block_tables_h [m*max_blocks],
 * cow_h [m*3] from oxy_alloc_reserve.  out_tokens_h [m*k], out_count_h [m]. */
int oxy_toy_decode(oxy_toy *m, int32_t rows, int32_t k, const int32_t *block_tables_h,
                   int32_t max_blocks, const int32_t *seq_lens_h, const int32_t *last_tokens_h,
                   const int32_t *budgets_h, const int32_t *cow_h, int32_t *out_tokens_h,
                   int32_t *out_count_h, void *stream);
/* materialise one layer's K,V rows [seq_len, d_model] as float64 (KvLayer view) */
int oxy_toy_read_kv(oxy_toy *m, const int32_t *blocks_h, int32_t seq_len, int32_t layer,
                    double *keys_h, double *values_h, void *stream);

/* inverse of oxy_toy_read_kv: write rows [0, seq_len) of one layer into the
 * handle's blocks (adopting a host KvCache into the pool; fault injection) */
int oxy_toy_write_kv(oxy_toy *m, const int32_t *blocks_h, int32_t seq_len, int32_t layer,
                     const double *keys_h, const double *values_h, void *stream);

/* ------------------------------------------------------------------------
 * tcgen05 GEMM (the pi0.5 projections): Y[t, f] (op)= sum_k W[f, k] X[t, k],
 * W [n_out, k] and X [t, k] bf16 row-major on device.  mode: 0 f32 store,
 * 1 bf16 store, 2 f32 +=, 3 GeGLU (row pairs gate/up -> bf16 [t, n_out/2]),
 * 4 GELU bf16, 5 bf16(acc + res_f32).  splits: 0 = auto (split-K needs
 * ws_d of splits*t*n_out floats).  No reference counterpart (the reference's
 * numpy matmuls, kvweaver/backend.py:290-297).
 * ---------------------------------------------------------------------- */
int oxy_gemm_bf16(const void *w_d, const void *x_d, int32_t n_out, int32_t k, int32_t t,
                  int32_t mode, void *out_d, int32_t ldo, const float *bias_d,
                  const float *res_d, int32_t ldr, int32_t splits, float *ws_d,
                  int64_t ws_floats, void *stream);
/* plan the launch: out6 = {bn, n_tiles, m_tiles, splits, stages, k_blocks} */
int oxy_gemm_plan(int32_t n_out, int32_t k, int32_t t, int32_t splits, int32_t *out6);
/* the batch-invariant split-K count the model uses for an (n_out, k) projection in
 * a phase (0 = prefill, 1 = skinny decode / denoise chains); a function of
 * (phase, n_out, k) only — never of the token count (gemm_sm100.cuh) */
int oxy_gemm_policy_splits(int32_t phase, int32_t n_out, int32_t k, int32_t *splits);
/* launches enqueued per plan class since the last reset (eager runs and CUDA
 * graph captures; replays are not re-counted): out[0..n) = {skinny, skinny
 * split-K, prefill deep-K band, prefill mid-K band, persistent 1-CTA, persistent
 * 2-CTA (cta_group::2), fused split reduce + residual + RMSNorm, attention with
 * cluster merge, attention with workspace merge, attention unsplit}.  Test and
 * profiling aid: lets a parity test assert which kernel plans it exercised. */
int oxy_plan_counts(int64_t *out, int32_t n, int32_t reset);

/* Paged decode attention (the language-decode hot kernel; replaces the padded
 * dense re-materialisation of kvweaver/backend.py:365-384): rows x 8 query
 * heads (q_d bf16 [rows, 2048]) over 1 KV head of dim 256 read through the
 * block table from one layer's pool (bf16 [num_blocks, 64, 256] K and V),
 * keys [0, pos[r]]; out_d bf16 [rows, 2048].  ws_d: rows*max_blocks*8*258
 * floats.  Device pointers; scale 1/16.  Pools hold num_blocks blocks. */
int oxy_paged_decode_attention(const void *q_d, void *out_d, const void *kpool_d,
                               const void *vpool_d, int32_t num_blocks, const int32_t *bt_d,
                               int32_t bt_stride, const int32_t *pos_d, int32_t rows,
                               int32_t max_blocks, float *ws_d, void *stream);

/* tcgen05 prefix attention (prefill prefix-LM / action-expert suffix; replaces
 * the masked softmax attention of kvweaver/backend.py:287-295 for head dim 256):
 * nq query rows (q_d bf16 [nq, 256]: tokens x 8 heads of one MQA group),
 * bidirectional over paged keys [0, nka) read through bt_d from the pools
 * (bf16 [num_blocks, 64, 256]) followed by dense keys kd_d / vd_d bf16
 * [nkb, 256]; out_d bf16 [nq, 256]; scale 1/16.  splits > 1 splits the keys
 * and merges them in split order: splits <= 16 inside the kernel over
 * distributed shared memory (ws_o / ws_ml unused, may be NULL), larger counts
 * through the workspace (ws_o: at least splits * ceil(nq/128)*128 * 256 bf16,
 * i.e. half that many floats; ws_ml: splits * ceil(nq/128)*128 * 2 floats). */
int oxy_prefix_attention(const void *q_d, void *out_d, const void *kpool_d, const void *vpool_d,
                         int32_t num_blocks, const int32_t *bt_d, int32_t nka, const void *kd_d,
                         const void *vd_d, int32_t nkb, int32_t nq, int32_t splits, float *ws_o,
                         float *ws_ml, void *stream);

/* tcgen05 SigLIP self-attention (the vision tower of the pi0.5 prefix, SURVEY.md
 * §8f rank 1; the reference stands patches in as token ids, kvweaver/backend.py:56-66):
 * qkv_d bf16 [n_images * 256, 3 * 72 * heads] (q | k | v, head-major 72-dim
 * slices, the fused projection's rows), out_d bf16 [n_images * 256, 72 * heads];
 * each image's 256 tokens attend to each other, scale 1/sqrt(72).
 * Device pointers, 16-byte aligned. */
int oxy_vit_attention(const void *qkv_d, void *out_d, int32_t n_images, int32_t heads, void *stream);

/* kernels launched by this library so far (process-wide counter) */
int64_t oxy_launch_count(void);

/* ------------------------------------------------------------------------
 * F2: pi0.5-shaped VLA (Gemma-2B prefix + Gemma-300M action expert + SigLIP),
 * bf16 on tcgen05, one unified paged KV pool (block 64 x 256 per layer).
 * The three calls replace the backend protocol of kvweaver/backend.py:309-420
 * for this model family; pool blocks come from oxy_alloc_*.
 * ---------------------------------------------------------------------- */
typedef struct oxy_pi05 oxy_pi05;

typedef struct oxy_pi05_config {
  int32_t width, depth, mlp, vocab;
  int32_t expert_width, expert_mlp;
  int32_t vit_width, vit_depth, vit_mlp, vit_heads;
  int32_t H, action_dim, eos_token;
  uint64_t seed;
} oxy_pi05_config;

int oxy_pi05_create(const oxy_pi05_config *cfg, int32_t num_blocks, void *stream,
                    oxy_pi05 **out);
int oxy_pi05_destroy(oxy_pi05 *m);
int oxy_pi05_num_tensors(oxy_pi05 *m, int32_t *n);
int oxy_pi05_tensor_info(oxy_pi05 *m, int32_t i, char *name64, int64_t *shape2,
                         int32_t *dtype, uint64_t *offset, float *bound, float *center);
int oxy_pi05_tensor_read(oxy_pi05 *m, int32_t i, void *host, int64_t nbytes, void *stream);
/* shared prefix prefill of n_obs observations (prefill, kvweaver/backend.py:309-314):
 * prefix i = [n_img_h[i] camera images (uint8 [224,224,3] each, device, in order);
 * n_txt_h[i] prompt tokens]; K/V of every layer written to blocks_h (concatenated
 * per observation, ceil(P_i/64) ids each). */
int oxy_pi05_prefill(oxy_pi05 *m, int32_t n_obs, const int32_t *n_img_h,
                     const int32_t *n_txt_h, const int32_t *tokens_h, const uint8_t *images_d,
                     const int32_t *blocks_h, void *stream);
/* action expert (action_denoise, kvweaver/backend.py:316-332): S Euler steps for
 * n streams reading each stream's prefix blocks; actions_d f32 [n, H, A]. */
int oxy_pi05_denoise(oxy_pi05 *m, int32_t n, const int32_t *prefix_lens_h,
                     const int32_t *blocks_h, int32_t S, float *actions_d, void *stream);
/* Same as oxy_pi05_denoise but enqueued on the model's action-expert lane
 * without making `stream` wait for it, so a following oxy_pi05_decode on
 * `stream` overlaps it (OxyGen's cross-task parallelism inside a frame,
 * kvweaver/scheduler.py:117-171 runs the two stages back to back).
 * actions_d is valid only after oxy_pi05_join(stream). */
int oxy_pi05_denoise_async(oxy_pi05 *m, int32_t n, const int32_t *prefix_lens_h,
                           const int32_t *blocks_h, int32_t S, float *actions_d, void *stream);
/* make `stream` wait for the last oxy_pi05_denoise(_async) */
int oxy_pi05_join(oxy_pi05 *m, void *stream);
/* device time of the last denoise (waits for it to finish) */
int oxy_pi05_denoise_elapsed_us(oxy_pi05 *m, double *us);
/* continuous-batched greedy decode (batched_language_decode,
 * kvweaver/backend.py:334-420); same contract as oxy_toy_decode; logits_h
 * (optional) receives [k, rows, vocab] f32. */
int oxy_pi05_decode(oxy_pi05 *m, int32_t rows, int32_t k, const int32_t *block_tables_h,
                    int32_t max_blocks, const int32_t *seq_lens_h, const int32_t *last_tokens_h,
                    const int32_t *budgets_h, const int32_t *cow_h, int32_t *out_tokens_h,
                    int32_t *out_count_h, float *logits_h, void *stream);
/* no-cache logits of the last of n tokens (replaces kvweaver/backend.py:301-304,
 * the oracle route of suite_reference, kvweaver/verify.py:152-181): one dense
 * forward over the whole sequence, positions [0, prefix_len) bidirectional
 * (prefix-LM), later positions causal; plain fp32 attention, no pool or block
 * tables.  logits_h: host f32 [vocab]. */
int oxy_pi05_recompute_logits(oxy_pi05 *m, const int32_t *tokens_h, int32_t n, int32_t prefix_len,
                              float *logits_h, void *stream);
int oxy_pi05_read_kv(oxy_pi05 *m, const int32_t *blocks_h, int32_t seq_len, int32_t layer,
                     float *keys_h, float *values_h, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* OXYGEN_B200_H */
