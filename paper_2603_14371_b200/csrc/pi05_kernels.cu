// F2 kernels: norms, RoPE + paged KV append, flash attention over
// [paged prefix || dense suffix], paged decode attention, greedy argmax.
#include <cmath>

#include "cuda_util.cuh"
#include "gemm_sm100.cuh"
#include "pi05_kernels.cuh"
#include "attn_device.cuh"

namespace oxy {
namespace pi05 {

// ============================================================ elementwise

// Row norms: one CTA per row, one thread per 4 features (D / 4 threads), the
// row held in registers (one load per element, all in flight), the scale /
// shift weights fetched before the PDL wait.
__global__ void rmsnorm_kernel(const float *x, int ldx, bf16 *y, int ldy, const float *w,
                               const float *ms, const float *mb, int D, float eps) {
  pdl_trigger();
  const int j = threadIdx.x * 4;
  const bool act = j < D;  // the block is rounded up to whole warps
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 sv = z, bv = z;
  if (act) {
    if (w) sv = __ldg(reinterpret_cast<const float4 *>(w + j));
    else {
      sv = __ldg(reinterpret_cast<const float4 *>(ms + j));
      bv = __ldg(reinterpret_cast<const float4 *>(mb + j));
    }
  }
  pdl_wait();
  __shared__ float red[32];
  const float4 v = act ? *reinterpret_cast<const float4 *>(x + (size_t)blockIdx.x * ldx + j) : z;
  const float ss = block_sum(v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w, red);
  const float inv = rsqrtf(ss / (float)D + eps);
  // (1 + w) for RMSNorm, (1 + scale) and + shift for adaRMS
  const float o0 = v.x * inv * (1.f + sv.x) + bv.x, o1 = v.y * inv * (1.f + sv.y) + bv.y;
  const float o2 = v.z * inv * (1.f + sv.z) + bv.z, o3 = v.w * inv * (1.f + sv.w) + bv.w;
  __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
  uint2 out;
  out.x = *reinterpret_cast<uint32_t *>(&h0);
  out.y = *reinterpret_cast<uint32_t *>(&h1);
  if (act) *reinterpret_cast<uint2 *>(y + (size_t)blockIdx.x * ldy + j) = out;
}

void rmsnorm(const float *x, int ldx, bf16 *y, int ldy, const float *w, const float *ms,
             const float *mb, int rows, int D, float eps, cudaStream_t st) {
  if (rows <= 0) return;
  if (D % 4 != 0 || D > 4096 || ldx % 4 != 0 || ldy % 4 != 0) fail(OXY_EINVAL, "rmsnorm: D %% 4 == 0, D <= 4096");
  launch_pdl(rmsnorm_kernel, dim3(rows), dim3((D / 4 + 31) / 32 * 32), 0, st, x, ldx, y, ldy, w, ms, mb, D, eps);
}

__global__ void layernorm_kernel(const float *x, int ldx, bf16 *y, int ldy, const float *w,
                                 const float *b, int D, float eps) {
  pdl_trigger();
  const int j = threadIdx.x * 4;
  const bool act = j < D;  // the block is rounded up to whole warps
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 wv = act ? __ldg(reinterpret_cast<const float4 *>(w + j)) : z;
  const float4 bv = act ? __ldg(reinterpret_cast<const float4 *>(b + j)) : z;
  pdl_wait();
  __shared__ float red[32];
  const float4 v = act ? *reinterpret_cast<const float4 *>(x + (size_t)blockIdx.x * ldx + j) : z;
  const float mean = block_sum(v.x + v.y + v.z + v.w, red) / (float)D;
  const float d0 = act ? v.x - mean : 0.f, d1 = act ? v.y - mean : 0.f, d2 = act ? v.z - mean : 0.f,
              d3 = act ? v.w - mean : 0.f;
  __syncthreads();  // red[] is reused
  const float rstd = rsqrtf(block_sum(d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3, red) / (float)D + eps);
  __nv_bfloat162 h0 = __floats2bfloat162_rn(d0 * rstd * wv.x + bv.x, d1 * rstd * wv.y + bv.y);
  __nv_bfloat162 h1 = __floats2bfloat162_rn(d2 * rstd * wv.z + bv.z, d3 * rstd * wv.w + bv.w);
  uint2 out;
  out.x = *reinterpret_cast<uint32_t *>(&h0);
  out.y = *reinterpret_cast<uint32_t *>(&h1);
  if (act) *reinterpret_cast<uint2 *>(y + (size_t)blockIdx.x * ldy + j) = out;
}

void layernorm(const float *x, int ldx, bf16 *y, int ldy, const float *w, const float *b, int rows,
               int D, float eps, cudaStream_t st) {
  if (rows <= 0) return;
  if (D % 4 != 0 || D > 4096 || ldx % 4 != 0 || ldy % 4 != 0) fail(OXY_EINVAL, "layernorm: D %% 4 == 0, D <= 4096");
  launch_pdl(layernorm_kernel, dim3(rows), dim3((D / 4 + 31) / 32 * 32), 0, st, x, ldx, y, ldy, w, b, D, eps);
}

__global__ void embed_kernel(float *x, int ldx, const bf16 *table, const int *tok,
                             const int *active, int D, float scale) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (active && !active[r]) return;
  const bf16 *row = table + (size_t)tok[r] * D;
  for (int j = threadIdx.x; j < D; j += blockDim.x)
    x[(size_t)r * ldx + j] = __bfloat162float(row[j]) * scale;
}

void embed_rows(float *x, int ldx, const bf16 *table, const int *tok, const int *active, int rows,
                int D, float scale, cudaStream_t st) {
  if (rows <= 0) return;
  launch_pdl(embed_kernel, dim3(rows), dim3(256), 0, st, x, ldx, table, tok, active, D, scale);
}

__global__ void permute_rows_kernel(bf16 *dst, const bf16 *src, int cols) {
  const int f = blockIdx.x;
  const bf16 *s = src + (size_t)gemm::qkv_rope_row(f) * cols;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) dst[(size_t)f * cols + j] = s[j];
}

void permute_rows(bf16 *dst, const bf16 *src, int rows, int cols, cudaStream_t st) {
  permute_rows_kernel<<<rows, 256, 0, st>>>(dst, src, cols);
  OXY_LAUNCH_CHECK();
}

__global__ void rope_table_kernel(float2 *cs, const float *inv_freq, int n) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const float ang = __fmul_rn((float)(idx >> 7), inv_freq[idx & 127]);  // as the fp32 oracle
  double s, c;
  sincos((double)ang, &s, &c);
  cs[idx] = make_float2((float)c, (float)s);
}

void rope_table(float2 *cs, const float *inv_freq, int n_pos, cudaStream_t st) {
  const int n = n_pos * 128;
  rope_table_kernel<<<(n + 255) / 256, 256, 0, st>>>(cs, inv_freq, n);
  OXY_LAUNCH_CHECK();
}

__global__ void patchify_kernel(const uint8_t *img, bf16 *patches, int kpad) {
  pdl_trigger();
  pdl_wait();
  const int p = blockIdx.x;  // image * 256 + patch
  const int im = p >> 8, py = (p & 255) >> 4, px = p & 15;
  const uint8_t *base = img + (size_t)im * 224 * 224 * 3;
  for (int e = threadIdx.x; e < kpad; e += blockDim.x) {
    float v = 0.f;
    if (e < 588) {
      const int dy = e / 42, rem = e % 42, dx = rem / 3, c = rem % 3;
      const int y = py * 14 + dy, x = px * 14 + dx;
      v = (float)base[((size_t)y * 224 + x) * 3 + c] / 127.5f - 1.f;
    }
    patches[(size_t)p * kpad + e] = __float2bfloat16(v);
  }
}

void patchify(const uint8_t *img, int n, bf16 *patches, int kpad, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(patchify_kernel, dim3(n * 256), dim3(128), 0, st, img, patches, kpad);
}

__global__ void tile_rows_kernel(float *dst, int ld, const float *src, int ld_src, int period, int D) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const float *s = src + (size_t)(r % period) * ld_src;
  for (int j = threadIdx.x; j < D; j += blockDim.x) dst[(size_t)r * ld + j] = s[j];
}

void tile_rows(float *dst, int ld, const float *src, int ld_src, int rows, int period, int D,
               cudaStream_t st) {
  if (rows <= 0) return;
  launch_pdl(tile_rows_kernel, dim3(rows), dim3(256), 0, st, dst, ld, src, ld_src, period, D);
}

__global__ void f32_to_bf16_kernel(const float *x, bf16 *y, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16(x[i]);
}

void f32_to_bf16(const float *x, bf16 *y, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  f32_to_bf16_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(x, y, n);
  OXY_LAUNCH_CHECK();
}

__global__ void euler_kernel(float *a, const float *v, bf16 *ab, int64_t n, float dt) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = a[i] + dt * v[i];
    a[i] = x;
    ab[i] = __float2bfloat16(x);
  }
}

void euler_step(float *a, const float *v, bf16 *ab, int64_t n, float dt, cudaStream_t st) {
  euler_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(a, v, ab, n, dt);
  OXY_LAUNCH_CHECK();
}

// Box-Muller on consecutive splitmix64 uniforms: pair i uses draws 2i, 2i+1.
__global__ void noise_kernel(float *out, int64_t n, uint64_t seed) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double u1 = splitmix_uniform(seed, 2 * i), u2 = splitmix_uniform(seed, 2 * i + 1);
    double r = sqrt(-2.0 * log(1.0 - u1)), th = 6.283185307179586 * u2;
    out[2 * i] = (float)(r * cos(th));
    if (2 * i + 1 < n) out[2 * i + 1] = (float)(r * sin(th));
  }
}

void normal_noise(float *out, int64_t n, uint64_t seed, cudaStream_t st) {
  noise_kernel<<<(unsigned)std::min<int64_t>((n / 2 + 256) / 256, 1024), 256, 0, st>>>(out, n, seed);
  OXY_LAUNCH_CHECK();
}

__global__ void init_bf16_kernel(bf16 *out, int64_t n, uint64_t seed, uint64_t offset, float bound) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double u = splitmix_uniform(seed, offset + (uint64_t)i);
    out[i] = __float2bfloat16((float)((2.0 * u - 1.0) * (double)bound));
  }
}

void init_uniform_bf16(bf16 *out, int64_t n, uint64_t seed, uint64_t offset, float bound, cudaStream_t st) {
  init_bf16_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64), 256, 0, st>>>(out, n, seed, offset, bound);
  OXY_LAUNCH_CHECK();
}

__global__ void init_f32_kernel(float *out, int64_t n, uint64_t seed, uint64_t offset, float bound, float center) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double u = splitmix_uniform(seed, offset + (uint64_t)i);
    out[i] = (float)((double)center + (2.0 * u - 1.0) * (double)bound);
  }
}

void init_uniform_f32(float *out, int64_t n, uint64_t seed, uint64_t offset, float bound, float center,
                      cudaStream_t st) {
  init_f32_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(out, n, seed, offset, bound, center);
  OXY_LAUNCH_CHECK();
}

__global__ void cow_kernel(bf16 *pool, const int *cow, size_t layer_stride, size_t kv_stride) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, l = blockIdx.y;
  const int src = cow[r * 3], dst = cow[r * 3 + 1], n = cow[r * 3 + 2];
  if (src < 0) return;
  const size_t elems = (size_t)n * HEAD_DIM / 8;  // int4 chunks
  for (int kv = 0; kv < 2; ++kv) {
    const int4 *s = reinterpret_cast<const int4 *>(pool + l * layer_stride + kv * kv_stride +
                                                   (size_t)src * KV_BLOCK * HEAD_DIM);
    int4 *d = reinterpret_cast<int4 *>(pool + l * layer_stride + kv * kv_stride +
                                       (size_t)dst * KV_BLOCK * HEAD_DIM);
    for (size_t i = threadIdx.x; i < elems; i += blockDim.x) d[i] = s[i];
  }
}

void cow_blocks(bf16 *pool, const int *cow, int rows, int L, size_t layer_stride, size_t kv_stride,
                cudaStream_t st) {
  if (rows <= 0) return;
  cow_kernel<<<dim3(rows, L), 256, 0, st>>>(pool, cow, layer_stride, kv_stride);
  OXY_LAUNCH_CHECK();
}

__global__ void next_slot_kernel(int *slot, const int *pos, const int *active, const int *bt,
                                 int bt_stride, int rows) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (!active[r]) { slot[r] = -1; return; }
  const int p = pos[r];
  slot[r] = bt[(size_t)r * bt_stride + p / KV_BLOCK] * KV_BLOCK + p % KV_BLOCK;
}

void next_slots(int *slot, const int *pos, const int *active, const int *bt, int bt_stride, int rows,
                cudaStream_t st) {
  launch_pdl(next_slot_kernel, dim3((rows + 127) / 128), dim3(128), 0, st, slot, pos, active, bt, bt_stride, rows);
}

// ============================================================ flash attention

template <int HD>
__global__ void __launch_bounds__(128)
    flash_attn_kernel(const AttnGroup *groups, int max_q_tiles, const bf16 *kpool, const bf16 *vpool,
                      float scale_log2, int splits, float *ws_o, float *ws_ml, int ws_rows) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char fa_smem[];
  const AttnGroup g = groups[blockIdx.x / max_q_tiles];
  flash_item<HD>(g, blockIdx.x % max_q_tiles, blockIdx.y, splits, kpool, vpool, scale_log2, ws_o, ws_ml, ws_rows,
                 reinterpret_cast<bf16 *>(fa_smem), threadIdx.x);
}

// Combine split-KV partials in split order (log2 domain).  CTA = one query
// row, thread = one column pair (warp 0 computes the split weights once).
// A variant with every thread loading all (m, l) and O pairs up front measured
// slower in the denoise chain (9.0 vs 8.8 ms per denoise).  CTA = one query
// row, thread = one column pair; split loads unrolled for memory parallelism.
__device__ __forceinline__ float2 ld_pair(const float *p) { return *reinterpret_cast<const float2 *>(p); }
__device__ __forceinline__ float2 ld_pair(const bf16 *p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(p));
}

// PT: partial element type (fp32 from the mma.sync kernel, bf16 from the tcgen05 one).
// tps > 0: per-group split counts (attn_group_splits, the tcgen05 kernel); 0: `splits`
// for every group.  The arithmetic is the tcgen05 cluster merge's, op for op (split
// weights exp2(m_s - M) / L summed in split order, then sum_s w_s * O_s in split
// order), so a group merged here equals the same group merged over DSMEM.
template <int HD, typename PT>
__global__ void fa_merge_kernel(const AttnGroup *groups, int splits, int tps, const PT *ws_o, const float *ws_ml,
                                int ws_rows) {
  pdl_trigger();
  pdl_wait();
  using C = FaCfg<HD>;
  __shared__ float wsh[32];
  const AttnGroup g = groups[blockIdx.y];
  const int r = blockIdx.x;
  if (r >= g.nq) return;
  int gs = splits;
  if (tps > 0) {
    int per;
    gs = attn_group_splits((g.nka + 63) / 64 + (g.nkb + 63) / 64, tps, per);
    if (gs <= 1) return;  // written directly by the attention kernel
  }
  const size_t row0 = (size_t)g.wrow0 + r;
  const size_t mstride = (size_t)ws_rows * 2;
  if (threadIdx.x == 0) {  // split weights, sequentially in split order (splits <= 32)
    float m[32], M = -INFINITY;
    for (int s = 0; s < gs; ++s) {
      m[s] = ws_ml[row0 * 2 + s * mstride];
      M = fmaxf(M, m[s]);
    }
    float L = 0.f;
    for (int s = 0; s < gs; ++s) {
      m[s] = m[s] == -INFINITY ? 0.f : exp2f(m[s] - M);
      L += ws_ml[row0 * 2 + s * mstride + 1] * m[s];
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    for (int s = 0; s < gs; ++s) wsh[s] = m[s] * inv;
  }
  __syncthreads();
  const int c = threadIdx.x * 2;
  if (c >= HD) return;
  const PT *o = ws_o + row0 * C::HDP + c;
  const size_t ostride = (size_t)ws_rows * C::HDP;
  float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
  for (int s = 0; s < gs; ++s) {  // split order; independent loads
    const float2 v = ld_pair(o + s * ostride);
    a0 += wsh[s] * v.x;
    a1 += wsh[s] * v.y;
  }
  *reinterpret_cast<__nv_bfloat162 *>(g.o + (size_t)r * g.ldo + c) = __floats2bfloat162_rn(a0, a1);
}

template <int HD>
static void flash_launch(const AttnGroup *groups_d, int n_groups, int max_q_tiles, const bf16 *kpool,
                         const bf16 *vpool, float scale, int splits, float *ws_o, float *ws_ml,
                         int ws_rows, cudaStream_t st) {
  using C = FaCfg<HD>;
  static bool attr = false;
  if (!attr) {
    OXY_CUDA(cudaFuncSetAttribute(flash_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM));
    attr = true;
  }
  const float scale_log2 = scale * 1.4426950408889634f;
  dim3 grid(n_groups * max_q_tiles, splits);
  launch_pdl(flash_attn_kernel<HD>, dim3(grid), dim3(128), C::SMEM, st, groups_d, max_q_tiles, kpool, vpool, scale_log2, splits, ws_o, ws_ml, ws_rows);
  if (splits > 1) {
    launch_pdl(fa_merge_kernel<HD, float>, dim3(max_q_tiles * FA_BQ, n_groups), dim3((HD / 2 + 31) / 32 * 32), 0, st,
               groups_d, splits, 0, ws_o, ws_ml, ws_rows);
  }
}

void flash_merge(const AttnGroup *groups_d, int n_groups, int max_rows, int splits, int tps, const bf16 *ws_o,
                 const float *ws_ml, int ws_rows, cudaStream_t st) {
  if (splits <= 1 || n_groups <= 0) return;
  launch_pdl(fa_merge_kernel<256, bf16>, dim3(max_rows, n_groups), dim3(128), 0, st, groups_d, splits, tps, ws_o,
             ws_ml, ws_rows);
}

void flash_attention(const AttnGroup *groups_d, int n_groups, int max_q_tiles, int head_dim,
                     const bf16 *kpool, const bf16 *vpool, float scale, int splits, int max_key_tiles,
                     float *ws_o, float *ws_ml, int ws_rows, cudaStream_t st) {
  (void)max_key_tiles;
  if (n_groups <= 0 || max_q_tiles <= 0) return;
  if (head_dim == 256)
    flash_launch<256>(groups_d, n_groups, max_q_tiles, kpool, vpool, scale, splits, ws_o, ws_ml, ws_rows, st);
  else if (head_dim == 72)
    flash_launch<72>(groups_d, n_groups, max_q_tiles, kpool, vpool, scale, splits, ws_o, ws_ml, ws_rows, st);
  else
    fail(OXY_EINVAL, "flash_attention: unsupported head_dim %d", head_dim);
}

// ============================================================ decode attention

constexpr int DA_PART = Q_HEADS * (HEAD_DIM + 2);

// Persistent paged decode attention.  Work item = (row, chunk of cb pool
// blocks; decode_row_chunk: a function of the row's own length).  Grid = up to
// 2 CTAs per SM, each looping over items blockIdx.x, +gridDim.x, ... so the KV
// stream never drains between items.  5 warps:
//   warp 4     producer (one thread): per block, the K tile then the V tile
//              (64 keys x 256 dims bf16 = 32 KB, four 64-column TMA boxes,
//              128-byte swizzle) into a ring of D4_SLOTS 32 KB slots
//              (full / empty mbarriers); 2 CTAs x 96 KB in flight per SM;
//   warps 0-3  S = Q K^T split by keys (warp w: keys 16w..16w+15 of the block,
//              mma.sync bf16, the 8 query heads as MMA rows), scores staged in
//              smem; every warp then runs the same online softmax over all 64
//              keys (4 lanes per head, shuffle reductions) and computes
//              O += P V for ITS 64 of the 256 output dims — no cross-warp merge
//              at the end of an item: a single-chunk row is written directly,
//              a chunk's unnormalised O and (m, l) go to the workspace and
//              decode_merge3_kernel combines the chunks in chunk order.
// Pool slots past a sequence's length are masked (-inf scores).
constexpr int D4_SLOTS = 3;
constexpr int D4_SUB = KV_BLOCK * 128;           // one 64-key x 64-dim bf16 box: 8 KB
constexpr int D4_TILE = 4 * D4_SUB;              // K or V tile of one pool block: 32 KB
constexpr int D4_SLD = 72;                       // score row stride (floats)
constexpr int D4_THREADS = 160;
constexpr size_t D4_SMEM = 1024 + D4_SLOTS * D4_TILE + 2 * Q_HEADS * D4_SLD * 4 + 32 + 2 * D4_SLOTS * 8 + 64;

// 16-byte chunk c (0..31) of row `row` in a tile of 4 swizzled 64-col sub-tiles
__device__ __forceinline__ uint32_t tile16(uint32_t base, int rows_per_sub, int row, int c) {
  return base + (c >> 3) * (rows_per_sub * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4);
}

__device__ __forceinline__ void d3_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void d3_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// consumer release of a ring slot (the callers first store a value that depends on
// every MMA fed from the slot, see decode_attn_v4_kernel)
__device__ __forceinline__ void d3_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void d3_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void d3_tma(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

// item -> (row, its chunking, the chunks [ca, cb) this item covers); false: nothing
// to do.  row_mode: an item is a whole row (all its chunks, folded in registers);
// else one chunk (partials folded by decode_fold_kernel).
struct D4Item {
  int r, n_keys, nb, cb, n_chunks, ca, ce;
};
// one lane of the converged producer warp (elect.sync): the warp walks the items with
// its values in uniform registers, the elected lane issues the TMA loads
__device__ __forceinline__ bool d4_elect() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ bool d4_item(int item, int row_mode, int max_chunks, int cb_min, const int *pos,
                                        const int *active, D4Item &it) {
  it.r = row_mode ? item : item / max_chunks;
  if (active && !active[it.r]) return false;
  it.n_keys = pos[it.r] + 1;
  it.nb = (it.n_keys + KV_BLOCK - 1) / KV_BLOCK;
  it.cb = decode_row_chunk(it.nb, cb_min);
  it.n_chunks = (it.nb + it.cb - 1) / it.cb;
  if (row_mode) {
    it.ca = 0;
    it.ce = it.n_chunks;
    return true;
  }
  it.ca = item % max_chunks;
  it.ce = it.ca + 1;
  return it.ca < it.n_chunks;
}

// fold of chunk partials (m_c, l_c, O_c) in chunk order; out = O * (1 / L)
__device__ __forceinline__ void d4_fold(float &M, float &L, float mc, float lc, float &fa, float &fb) {
  const float mn = fmaxf(M, mc);
  fa = M == -INFINITY ? 0.f : exp2f(M - mn);
  fb = exp2f(mc - mn);
  L = __fmaf_rn(lc, fb, __fmul_rn(L, fa));
  M = mn;
}

__global__ void __launch_bounds__(D4_THREADS, 2)
    decode_attn_v4_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                          const bf16 *q, const int *bt, int bt_stride, const int *pos, const int *active, int cb_min,
                          int max_chunks, int n_items, int row_mode, float scale_log2, float *ws, bf16 *out) {
  pdl_trigger();
  extern __shared__ unsigned char d3_raw[];
  // 1024-byte alignment in the SHARED address space (the 128-byte swizzle the TMA
  // applies and the ldmatrix addressing below assume it)
  const uint32_t raw_s = smem_addr(d3_raw);
  unsigned char *smem = d3_raw + (((raw_s + 1023u) & ~1023u) - raw_s);
  const uint32_t ring = smem_addr(smem);
  float *sS = reinterpret_cast<float *>(smem + D4_SLOTS * D4_TILE);  // [2][8][D4_SLD]
  float *sSink = sS + 2 * Q_HEADS * D4_SLD;                           // [4] slot-release dependencies
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + D4_SLOTS * D4_TILE + 2 * Q_HEADS * D4_SLD * 4 + 32);
  const uint32_t full0 = smem_addr(bars), empty0 = full0 + 8 * D4_SLOTS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < D4_SLOTS; ++s) {
      d3_mbar_init(full0 + 8 * s, 1);
      d3_mbar_init(empty0 + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
  }
  __syncthreads();
  // positions / activity come from the previous decode step and Q from the
  // QKV projection right before us: wait for the whole chain
  pdl_wait();
  D4Item it;
  if (warp == 4) {
    // the whole warp walks the items (uniform registers); the elected lane issues the loads
    int t = 0;  // tiles issued (K and V alternate)
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      if (!d4_item(item, row_mode, max_chunks, cb_min, pos, active, it)) continue;
      const int *btr = bt + (size_t)it.r * bt_stride;
      const int b_end = min(it.nb, it.ce * it.cb);
      for (int b = it.ca * it.cb; b < b_end; ++b) {
        const int row0 = btr[b] * KV_BLOCK;
#pragma unroll
        for (int kv = 0; kv < 2; ++kv, ++t) {
          const int s = t % D4_SLOTS;
          d3_wait(empty0 + 8 * s, ((t / D4_SLOTS) & 1) ^ 1);
          const uint32_t dst = ring + s * D4_TILE;
          if (d4_elect()) {
            d3_expect_tx(full0 + 8 * s, D4_TILE);
#pragma unroll
            for (int j = 0; j < 4; ++j) d3_tma(kv ? &vmap : &kmap, full0 + 8 * s, dst + j * D4_SUB, 64 * j, row0);
          }
          __syncwarp();
        }
      }
    }
    return;
  }
  const int g = lane >> 2, c = lane & 3;  // MMA row (= query head) and column pair of this lane
  const int krow = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
  int t = 0, nbk = 0;  // tiles consumed, blocks processed (score buffer parity)
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    if (!d4_item(item, row_mode, max_chunks, cb_min, pos, active, it)) continue;
    const int r = it.r, n_keys = it.n_keys;
    // Q of this row as MMA A fragments: head g, dims 16ks + 2c (+1), +8 (rows 8-15 are zero).
    // L2-coherent loads (ld.global.cg), not the non-coherent path: the QKV projection
    // rewrites this buffer every layer, and under PDL an SM's L1 can still hold the
    // previous layer's lines (measured: stale Q with __ldg once CTAs loop over items)
    const uint32_t *qg = reinterpret_cast<const uint32_t *>(q + (size_t)r * Q_HEADS * HEAD_DIM + g * HEAD_DIM);
    uint32_t qa0[16], qa2[16];
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      qa0[ks] = __ldcg(qg + 8 * ks + c);
      qa2[ks] = __ldcg(qg + 8 * ks + 4 + c);
    }
    // fold state of the row (row mode, or a single-chunk row): M, L per head g, O for
    // this warp's 64 dims (MMA rows 0-7)
    float FM = -INFINITY, FL = 0.f, fo[8][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) fo[nt][0] = fo[nt][1] = 0.f;
    const bool fold = row_mode || it.n_chunks == 1;
    for (int chunk = it.ca; chunk < it.ce; ++chunk) {
      const int b0 = chunk * it.cb, nblk = min(it.nb, b0 + it.cb) - b0;
      float o[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m_run = -INFINITY, l_run = 0.f;
      for (int i = 0; i < nblk; ++i, ++nbk) {
        // ---- S = Q K^T for this warp's 16 keys
        int s = t % D4_SLOTS;
        d3_wait(full0 + 8 * s, (t / D4_SLOTS) & 1);
        const uint32_t kb = ring + s * D4_TILE;
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  #pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          uint32_t k0, k1, k2, k3;
          ldsm_x4(tile16(kb, 64, krow, ks * 2 + ((lane >> 3) & 1)), k0, k1, k2, k3);
          mma16816(sc[0], qa0[ks], 0u, qa2[ks], 0u, k0, k1);
          mma16816(sc[1], qa0[ks], 0u, qa2[ks], 0u, k2, k3);
        }
        float *Sb = sS + (nbk & 1) * Q_HEADS * D4_SLD;
        const int kbase = (b0 + i) * KV_BLOCK;
  #pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int kl = warp * 16 + nt * 8 + 2 * c;
          float2 v;
          v.x = kbase + kl < n_keys ? sc[nt][0] * scale_log2 : -INFINITY;
          v.y = kbase + kl + 1 < n_keys ? sc[nt][1] * scale_log2 : -INFINITY;
          *reinterpret_cast<float2 *>(Sb + g * D4_SLD + kl) = v;
        }
        // release the K slot only after a store that depends on every S MMA (and so
        // on every ldmatrix of the slot): an mbarrier arrive right after the last
        // ldmatrix does not wait for its read, and the next TMA into the slot raced it
        __syncwarp();
        if (lane == 0) d3_arrive(empty0 + 8 * s);
        ++t;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // ---- online softmax over the block's 64 keys (identical in every warp)
        float p[4][4], mx = m_run;
  #pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float2 a = *reinterpret_cast<const float2 *>(Sb + g * D4_SLD + kk * 16 + 2 * c);
          const float2 b = *reinterpret_cast<const float2 *>(Sb + g * D4_SLD + kk * 16 + 8 + 2 * c);
          p[kk][0] = a.x;
          p[kk][1] = a.y;
          p[kk][2] = b.x;
          p[kk][3] = b.y;
          mx = fmaxf(mx, fmaxf(fmaxf(a.x, a.y), fmaxf(b.x, b.y)));
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float corr = mx == -INFINITY ? 1.f : exp2f(m_run - mx);
        const float mxs = mx == -INFINITY ? 0.f : mx;
        float ls = 0.f;
  #pragma unroll
        for (int kk = 0; kk < 4; ++kk)
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            p[kk][e] = exp2_approx(p[kk][e] - mxs);
            ls += p[kk][e];
          }
        ls += __shfl_xor_sync(0xffffffffu, ls, 1);
        ls += __shfl_xor_sync(0xffffffffu, ls, 2);
        l_run = l_run * corr + ls;
        m_run = mx;
  #pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          o[nt][0] *= corr;
          o[nt][1] *= corr;
        }
        // ---- O[:, 64 warp .. 64 warp + 63] += P V
        s = t % D4_SLOTS;
        d3_wait(full0 + 8 * s, (t / D4_SLOTS) & 1);
        const uint32_t vb = ring + s * D4_TILE;
  #pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t pa0 = pack_bf16(p[kk][0], p[kk][1]), pa2 = pack_bf16(p[kk][2], p[kk][3]);
  #pragma unroll
          for (int np = 0; np < 4; ++np) {
            uint32_t v0, v1, v2, v3;
            ldsm_x4_t(tile16(vb, 64, kk * 16 + (lane & 15), warp * 8 + np * 2 + (lane >> 4)), v0, v1, v2, v3);
            mma16816(o[2 * np], pa0, 0u, pa2, 0u, v0, v1);
            mma16816(o[2 * np + 1], pa0, 0u, pa2, 0u, v2, v3);
          }
        }
        // same for the V slot: a store depending on every PV MMA's result first
        if (lane == 0) {
          float dep = 0.f;
  #pragma unroll
          for (int nt = 0; nt < 8; ++nt) dep += o[nt][0];
          sSink[warp] = dep;
        }
        __syncwarp();
        if (lane == 0) d3_arrive(empty0 + 8 * s);
        ++t;
      }
      // ---- this warp's 64 dims of the item's result (MMA rows 0-7 = heads)
      if (fold) {
        float fa, fb;
        d4_fold(FM, FL, m_run, l_run, fa, fb);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          fo[nt][0] = __fmaf_rn(o[nt][0], fb, __fmul_rn(fo[nt][0], fa));
          fo[nt][1] = __fmaf_rn(o[nt][1], fb, __fmul_rn(fo[nt][1], fa));
        }
      } else {  // one chunk of a multi-chunk row: unnormalised O and (m, l) to the workspace
        float *part = ws + ((size_t)r * max_chunks + chunk) * DA_PART + g * (HEAD_DIM + 2);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
          *reinterpret_cast<float2 *>(part + warp * 64 + nt * 8 + 2 * c) = make_float2(o[nt][0], o[nt][1]);
        if (warp == 0 && c == 0) {
          part[HEAD_DIM] = m_run;
          part[HEAD_DIM + 1] = l_run;
        }
      }
    }
    if (fold) {
      const float inv = 1.f / FL;
      bf16 *orow = out + (size_t)r * Q_HEADS * HEAD_DIM + g * HEAD_DIM + warp * 64 + 2 * c;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
        *reinterpret_cast<__nv_bfloat162 *>(orow + nt * 8) =
            __floats2bfloat162_rn(__fmul_rn(fo[nt][0], inv), __fmul_rn(fo[nt][1], inv));
    }
  }
}

// Fold of a multi-chunk row's partials (chunk mode): CTA = (row, head), thread =
// output dim; the same fold, in chunk order, as the in-register one of row mode, so
// a row's result does not depend on which mode its batch ran in.
__global__ void decode_fold_kernel(const float *ws, bf16 *out, const int *pos, const int *active, int cb_min,
                                   int max_chunks) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  if (active && !active[r]) return;
  const int nb = (pos[r] + KV_BLOCK) / KV_BLOCK;
  const int cb = decode_row_chunk(nb, cb_min);
  const int n_chunks = (nb + cb - 1) / cb;
  if (n_chunks == 1) return;  // written by the attention kernel
  const float *pr = ws + (size_t)r * max_chunks * DA_PART + h * (HEAD_DIM + 2);
  float M = -INFINITY, L = 0.f, acc = 0.f;
  for (int c0 = 0; c0 < n_chunks; c0 += 8) {
    float mc[8], lc[8], v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float *pc = pr + (size_t)min(c0 + j, n_chunks - 1) * DA_PART;
      mc[j] = __ldcg(pc + HEAD_DIM);
      lc[j] = __ldcg(pc + HEAD_DIM + 1);
      v[j] = __ldcg(pc + d);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (c0 + j >= n_chunks) break;
      float fa, fb;
      d4_fold(M, L, mc[j], lc[j], fa, fb);
      acc = __fmaf_rn(v[j], fb, __fmul_rn(acc, fa));
    }
  }
  out[(size_t)r * Q_HEADS * HEAD_DIM + h * HEAD_DIM + d] = __float2bfloat16(__fmul_rn(acc, 1.f / L));
}

void decode_attention_v3(const CUtensorMap &kmap, const CUtensorMap &vmap, const bf16 *q, bf16 *out, const int *bt,
                         int bt_stride, const int *pos, const int *active, int rows, int max_blocks, float scale,
                         float *ws, int sms, cudaStream_t st) {
  if (rows <= 0) return;
  static bool attr = false;
  if (!attr) {
    OXY_CUDA(cudaFuncSetAttribute(decode_attn_v4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)D4_SMEM));
    attr = true;
  }
  static const int knob_grid = [] {  // A/B knob: CTAs of the persistent grid (0: 2 per SM)
    const char *e = getenv("OXY_DA_GRID");
    return e ? atoi(e) : 0;
  }();
  static const int knob_rows = [] {  // A/B knob: row mode from this many rows (0: default)
    const char *e = getenv("OXY_DA_ROW_MODE_ROWS");
    return e ? atoi(e) : 0;
  }();
  const int cb = DECODE_CHUNK_BLOCKS;
  const int max_chunks = std::min(64, (max_blocks + cb - 1) / cb);
  // From a quarter of the SMs' worth of rows: whole rows per item, chunks folded in
  // registers (no partials, no fold launch; 256 x 1024: 0.66 of HBM vs 0.50); fewer
  // rows: chunk items for parallelism (6 rows: 16.6 vs 22 us), folded by
  // decode_fold_kernel.  Both fold the same chunk partials in the same order, so the
  // mode (a function of the batch) never changes a row's result.
  const int row_mode = rows >= (knob_rows > 0 ? knob_rows : std::max(1, sms / 4)) ? 1 : 0;
  const int n_items = row_mode ? rows : rows * max_chunks;
  const int grid = std::min(n_items, knob_grid > 0 ? knob_grid : 2 * sms);
  launch_pdl(decode_attn_v4_kernel, dim3(grid), dim3(D4_THREADS), D4_SMEM, st, kmap, vmap, q, bt, bt_stride, pos,
             active, cb, max_chunks, n_items, row_mode, scale * 1.4426950408889634f, ws, out);
  if (!row_mode && max_chunks > 1)
    launch_pdl(decode_fold_kernel, dim3(rows, Q_HEADS), dim3(HEAD_DIM), 0, st, ws, out, pos, active, cb, max_chunks);
}

// ============================================================ no-cache recompute attention
// The oracle route of suite_reference (kvweaver/verify.py:152-181): plain fp32
// softmax attention over dense rows with the prefix-LM mask — query t sees keys
// [0, P) and, past the prefix, [P, t] — deliberately independent of the tiled
// kernels, the paged pool and the decode path.  CTA = (query, head), thread = dim.
__global__ void prefix_lm_attention_ref_kernel(const bf16 *q, const bf16 *k, const bf16 *v, bf16 *out, int T, int P,
                                               float scale) {
  extern __shared__ float ra_sh[];
  float *qs = ra_sh, *sc = ra_sh + HEAD_DIM, *red = sc + T;
  const int t = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  qs[d] = __bfloat162float(q[(size_t)t * Q_HEADS * HEAD_DIM + h * HEAD_DIM + d]);
  __syncthreads();
  const int nk = t < P ? P : t + 1;
  float mx = -INFINITY;
  for (int j = d; j < nk; j += blockDim.x) {
    const bf16 *kr = k + (size_t)j * HEAD_DIM;
    float acc = 0.f;
    for (int e = 0; e < HEAD_DIM; ++e) acc = fmaf(qs[e], __bfloat162float(kr[e]), acc);
    sc[j] = acc * scale;
    mx = fmaxf(mx, sc[j]);
  }
  const float M = block_max(mx, red);
  float sum = 0.f;
  for (int j = d; j < nk; j += blockDim.x) {
    const float e = expf(sc[j] - M);
    sc[j] = e;
    sum += e;
  }
  const float L = block_sum(sum, red + 32);
  __syncthreads();
  float o = 0.f;
  for (int j = 0; j < nk; ++j) o = fmaf(sc[j], __bfloat162float(v[(size_t)j * HEAD_DIM + d]), o);
  out[(size_t)t * Q_HEADS * HEAD_DIM + h * HEAD_DIM + d] = __float2bfloat16(o / L);
}

void prefix_lm_attention_ref(const bf16 *q, const bf16 *k, const bf16 *v, bf16 *out, int T, int P, float scale,
                             cudaStream_t st) {
  const size_t smem = (HEAD_DIM + (size_t)T + 64) * sizeof(float);
  OXY_REQUIRE(smem <= 200 * 1024, "recompute sequence of %d positions too long", T);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    OXY_CUDA(cudaFuncSetAttribute(prefix_lm_attention_ref_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = smem;
  }
  prefix_lm_attention_ref_kernel<<<dim3(T, Q_HEADS), HEAD_DIM, smem, st>>>(q, k, v, out, T, P, scale);
  OXY_LAUNCH_CHECK();
}

// ============================================================ argmax

constexpr int AM_CHUNKS = 64;

__device__ __forceinline__ void better(float &bv, int &bi, float v, int i) {
  if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

__global__ void argmax_partial_kernel(const float *logits, int V, const int *active, float *pv, int *pi) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sv[32];
  __shared__ int si[32];
  const int r = blockIdx.x, c = blockIdx.y;
  if (active && !active[r]) return;
  const int per = (V + AM_CHUNKS - 1) / AM_CHUNKS;
  const int j0 = c * per, j1 = min(V, j0 + per);
  const float *lg = logits + (size_t)r * V;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) better(bv, bi, lg[j], j);
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) better(bv, bi, sv[i], si[i]);
    pv[r * AM_CHUNKS + c] = bv;
    pi[r * AM_CHUNKS + c] = bi;
  }
}

__global__ void argmax_final_kernel(int rows, const float *pv, const int *pi, int step, int k, int eos,
                                    int *active, int *tok, int *pos, int *count, const int *budget,
                                    int *out_tokens) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (active && !active[r]) return;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = 0; c < AM_CHUNKS; ++c) better(bv, bi, pv[r * AM_CHUNKS + c], pi[r * AM_CHUNKS + c]);
  if (bi == 0x7fffffff) bi = 0;
  out_tokens[(size_t)r * k + step] = bi;
  tok[r] = bi;
  pos[r] += 1;
  const int c = ++count[r];
  if (bi == eos || c == budget[r]) active[r] = 0;
}

// Greedy step from the LM head's EPI_ARGMAX partials: one (max, lowest id) per
// (row, 128-row weight tile), folded per row by one CTA with the same order-free
// rule, then the same per-row state update as argmax_final_kernel.
__global__ void __launch_bounds__(256) argmax_tiles_final_kernel(int tiles, const float *pv, const int *pi, int step,
                                                                 int k, int eos, int *active, int *tok, int *pos,
                                                                 int *count, const int *budget, int *out_tokens) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sv[8];
  __shared__ int si[8];
  const int r = blockIdx.x;
  if (active && !active[r]) return;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = threadIdx.x; c < tiles; c += blockDim.x)
    better(bv, bi, __ldcg(pv + (size_t)r * tiles + c), __ldcg(pi + (size_t)r * tiles + c));
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sv[w] = bv;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) better(bv, bi, sv[i], si[i]);
  if (bi == 0x7fffffff) bi = 0;
  out_tokens[(size_t)r * k + step] = bi;
  tok[r] = bi;
  pos[r] += 1;
  const int c = ++count[r];
  if (bi == eos || c == budget[r]) active[r] = 0;
}

void argmax_tiles_update(int rows, int tiles, const float *pv, const int *pi, int step, int k, int eos, int *active,
                         int *tok, int *pos, int *count, const int *budget, int *out_tokens, cudaStream_t st) {
  launch_pdl(argmax_tiles_final_kernel, dim3(rows), dim3(256), 0, st, tiles, pv, pi, step, k, eos, active, tok, pos,
             count, budget, out_tokens);
}

void argmax_update(const float *logits, int rows, int V, int step, int k, int eos, int *active, int *tok,
                   int *pos, int *count, const int *budget, int *out_tokens, float *pv, int *pi,
                   cudaStream_t st) {
  launch_pdl(argmax_partial_kernel, dim3(rows, AM_CHUNKS), dim3(256), 0, st, logits, V, active, pv, pi);
  launch_pdl(argmax_final_kernel, dim3((rows + 63) / 64), dim3(64), 0, st, rows, pv, pi, step, k, eos, active, tok, pos, count, budget, out_tokens);
}

}  // namespace pi05
}  // namespace oxy

extern "C" int oxy_paged_decode_attention(const void *q_d, void *out_d, const void *kpool_d,
                                          const void *vpool_d, int32_t num_blocks, const int32_t *bt_d,
                                          int32_t bt_stride, const int32_t *pos_d, int32_t rows,
                                          int32_t max_blocks, float *ws_d, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(rows >= 1 && rows <= oxy::pi05::MAX_DECODE_ROWS_ABI && max_blocks >= 1 && bt_stride >= max_blocks &&
                  num_blocks >= 1,
              "bad decode-attention shape");
  using oxy::pi05::bf16;
  int dev = 0, sms = 148;
  OXY_CUDA(cudaGetDevice(&dev));
  OXY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const CUtensorMap km = oxy::gemm::make_map(kpool_d, num_blocks * oxy::pi05::KV_BLOCK, oxy::pi05::HEAD_DIM,
                                             oxy::pi05::KV_BLOCK);
  const CUtensorMap vm = oxy::gemm::make_map(vpool_d, num_blocks * oxy::pi05::KV_BLOCK, oxy::pi05::HEAD_DIM,
                                             oxy::pi05::KV_BLOCK);
  oxy::pi05::decode_attention_v3(km, vm, static_cast<const bf16 *>(q_d), static_cast<bf16 *>(out_d), bt_d,
                                 bt_stride, pos_d, nullptr, rows, max_blocks, 1.f / 16.f, ws_d, sms,
                                 oxy::as_stream(stream));
  OXY_API_END
}
