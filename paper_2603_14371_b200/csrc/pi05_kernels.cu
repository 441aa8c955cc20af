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

// CTA = (row, chunk of `cb` pool blocks), 4 warps, 1 CTA/SM.  One thread
// streams each block's K and V (2 x 32 KB) with 8 TMA tensor copies (64-column
// sub-tiles, 128-byte swizzle) into a 3-stage mbarrier ring, so the SM keeps up
// to 192 KB of KV in flight with a handful of instructions.  Warp w owns keys
// 16w..16w+15 of every block (S = QK^T and O = PV on mma.sync bf16, online
// softmax in registers); the 4 warps merge once per chunk; chunks of a row are
// merged by decode_merge3_kernel in chunk order (deterministic).
constexpr int D3_STAGES = 3;
constexpr int D3_SUB = KV_BLOCK * 128;              // one 64-row x 64-col bf16 sub-tile: 8 KB
constexpr int D3_STAGE_BYTES = 8 * D3_SUB;          // K (4 sub-tiles) + V (4 sub-tiles)
constexpr size_t D3_SMEM = 1024 + 4 * 16 * 128 + D3_STAGES * D3_STAGE_BYTES + 64;

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

__global__ void __launch_bounds__(128, 1)
    decode_attn_v3_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                          const bf16 *q, const int *bt, int bt_stride, const int *pos, const int *active, int cb,
                          int max_chunks, float scale_log2, float *ws, bf16 *out) {
  pdl_trigger();
  extern __shared__ unsigned char d3_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(d3_raw) + 1023) &
                                                          ~static_cast<uintptr_t>(1023));
  const uint32_t sQ = smem_addr(smem);                    // 4 sub-tiles x 16 rows x 128 B
  const uint32_t sKV = sQ + 4 * 16 * 128;                 // stages
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 4 * 16 * 128 + D3_STAGES * D3_STAGE_BYTES);
  const uint32_t full0 = smem_addr(bars);
  if (threadIdx.x == 0) {
    for (int s = 0; s < D3_STAGES; ++s) d3_mbar_init(full0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
  }
  __syncthreads();
  // pos / active / block table come from earlier steps (argmax update, host
  // plan), not from the kernel right before us (the QKV projection): read them
  // and prefetch every pool block but the one holding this step's position
  // before the PDL wait
  const int r = blockIdx.x, chunk = blockIdx.y;
  if (active && !active[r]) return;
  const int n_keys = pos[r] + 1;
  const int nb = (n_keys + KV_BLOCK - 1) / KV_BLOCK;
  cb = decode_row_chunk(nb, cb);  // this row's own chunking: batch-invariant
  const int n_chunks = (nb + cb - 1) / cb;
  if (chunk >= n_chunks) return;
  const int b0 = chunk * cb, nblk = min(nb, b0 + cb) - b0;
  const int *btr = bt + (size_t)r * bt_stride + b0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto issue = [&](int i) {  // block i of the chunk -> stage i % 3 (thread 0 only)
    const int s = i % D3_STAGES, row0 = btr[i] * KV_BLOCK;
    const uint32_t bar = full0 + 8 * s, kb = sKV + s * D3_STAGE_BYTES, vb = kb + 4 * D3_SUB;
    d3_expect_tx(bar, D3_STAGE_BYTES);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      d3_tma(&kmap, bar, kb + j * D3_SUB, 64 * j, row0);
      d3_tma(&vmap, bar, vb + j * D3_SUB, 64 * j, row0);
    }
  };
  int pre = 0;  // blocks issued before the wait: all but the block holding pos[r]
  if (threadIdx.x == 0)
    for (; pre < min(nblk, D3_STAGES) && b0 + pre < nb - 1; ++pre) issue(pre);
  pdl_wait();
  if (threadIdx.x == 0)
    for (int i = pre; i < min(nblk, D3_STAGES); ++i) issue(i);
  // Q: the 8 heads as MMA rows 0..7 (rows 8..15 zero)
  const bf16 *qr = q + (size_t)r * Q_HEADS * HEAD_DIM;
  for (int i = threadIdx.x; i < 16 * 32; i += 128) {
    const int row = i >> 5, c = i & 31;
    const uint32_t dst = tile16(sQ, 16, row, c);
    if (row < Q_HEADS) cp_async16(dst, qr + (size_t)row * HEAD_DIM + c * 8);
    else asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0));
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();

  float o[32][4];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const int krow = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
  const int vrow = warp * 16 + (lane & 15);
  for (int i = 0; i < nblk; ++i) {
    const int s = i % D3_STAGES;
    d3_wait(full0 + 8 * s, (i / D3_STAGES) & 1);
    const uint32_t kb = sKV + s * D3_STAGE_BYTES, vb = kb + 4 * D3_SUB;
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < HEAD_DIM / 16; ++kk) {
      uint32_t a0, a1, a2, a3, k0, k1, k2, k3;
      ldsm_x4(tile16(sQ, 16, lane & 15, kk * 2 + (lane >> 4)), a0, a1, a2, a3);
      ldsm_x4(tile16(kb, 64, krow, kk * 2 + ((lane >> 3) & 1)), k0, k1, k2, k3);
      mma16816(sc[0], a0, a1, a2, a3, k0, k1);
      mma16816(sc[1], a0, a1, a2, a3, k2, k3);
    }
    const int kbase = (b0 + i) * KV_BLOCK + warp * 16 + (lane & 3) * 2;
    float mx = m_run;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float v = sc[nt][e] * scale_log2;
        if (kbase + nt * 8 + e >= n_keys) v = -INFINITY;
        sc[nt][e] = v;
        mx = fmaxf(mx, v);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float corr = (mx == -INFINITY) ? 1.f : exp2f(m_run - mx);
    float ls = 0.f;
    const float mxs = mx == -INFINITY ? 0.f : mx;  // all keys masked: every score is -inf
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float p = exp2_approx(sc[nt][e] - mxs);
        sc[nt][e] = p;
        ls += p;
      }
    ls += __shfl_xor_sync(0xffffffffu, ls, 1);
    ls += __shfl_xor_sync(0xffffffffu, ls, 2);
    l_run = l_run * corr + ls;
    m_run = mx;
#pragma unroll
    for (int nt = 0; nt < 32; ++nt) {
      o[nt][0] *= corr;
      o[nt][1] *= corr;
    }
    // P rows 8..15 (padding) are zero
    const uint32_t pa0 = pack_bf16(sc[0][0], sc[0][1]), pa2 = pack_bf16(sc[1][0], sc[1][1]);
#pragma unroll
    for (int np = 0; np < 16; ++np) {
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(tile16(vb, 64, vrow, np * 2 + (lane >> 4)), v0, v1, v2, v3);
      mma16816(o[2 * np], pa0, 0u, pa2, 0u, v0, v1);
      mma16816(o[2 * np + 1], pa0, 0u, pa2, 0u, v2, v3);
    }
    __syncthreads();  // stage s fully consumed
    if (threadIdx.x == 0 && i + D3_STAGES < nblk) issue(i + D3_STAGES);
  }
  // ---- merge the 4 warps (stage memory reused) -> chunk result
  float *sO = reinterpret_cast<float *>(smem + 4 * 16 * 128);   // [4][8][256]
  float *sM = sO + 4 * 8 * HEAD_DIM;                             // [4][8] m, [4][8] l
  const int g = lane >> 2;
#pragma unroll
  for (int nt = 0; nt < 32; ++nt)
    *reinterpret_cast<float2 *>(sO + (warp * 8 + g) * HEAD_DIM + nt * 8 + (lane & 3) * 2) =
        make_float2(o[nt][0], o[nt][1]);
  if ((lane & 3) == 0) {
    sM[warp * 8 + g] = m_run;
    sM[32 + warp * 8 + g] = l_run;
  }
  __syncthreads();
  bf16 *orow = out + (size_t)r * Q_HEADS * HEAD_DIM;
  float *part = ws + ((size_t)r * max_chunks + chunk) * DA_PART;
  for (int i = threadIdx.x; i < Q_HEADS * HEAD_DIM; i += 128) {
    const int h = i >> 8, d = i & 255;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sM[w * 8 + h]);
    float acc = 0.f, L = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = sM[w * 8 + h];
      if (mw == -INFINITY) continue;
      const float e = exp2f(mw - M);
      acc += sO[(w * 8 + h) * HEAD_DIM + d] * e;
      L += sM[32 + w * 8 + h] * e;
    }
    if (n_chunks == 1) {
      orow[i] = __float2bfloat16(acc / L);
    } else {
      part[h * (HEAD_DIM + 2) + d] = acc;
      if (d == 0) {
        part[h * (HEAD_DIM + 2) + HEAD_DIM] = M;
        part[h * (HEAD_DIM + 2) + HEAD_DIM + 1] = L;
      }
    }
  }
}

// chunk merge: CTA = (row, head), thread = output dim; chunk order fixed
__global__ void decode_merge3_kernel(const float *ws, bf16 *out, const int *pos, const int *active, int cb,
                                     int max_chunks) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  if (active && !active[r]) return;
  const int nb = (pos[r] + KV_BLOCK) / KV_BLOCK;
  cb = decode_row_chunk(nb, cb);
  const int n_chunks = (nb + cb - 1) / cb;
  if (n_chunks == 1) return;  // written directly by the attention kernel
  const float *base = ws + (size_t)r * max_chunks * DA_PART + h * (HEAD_DIM + 2);
  __shared__ float wsh[64];
  __shared__ float s_inv;
  if (threadIdx.x < 32) {  // warp 0: chunk weights once (chunks <= 64)
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const int c0 = threadIdx.x, c1 = threadIdx.x + 32;
    if (c0 < n_chunks) { m0 = base[(size_t)c0 * DA_PART + HEAD_DIM]; l0 = base[(size_t)c0 * DA_PART + HEAD_DIM + 1]; }
    if (c1 < n_chunks) { m1 = base[(size_t)c1 * DA_PART + HEAD_DIM]; l1 = base[(size_t)c1 * DA_PART + HEAD_DIM + 1]; }
    const float M = warp_max(fmaxf(m0, m1));
    const float w0 = c0 < n_chunks ? exp2f(m0 - M) : 0.f, w1 = c1 < n_chunks ? exp2f(m1 - M) : 0.f;
    const float L = warp_sum(l0 * w0 + l1 * w1);
    wsh[c0] = w0;
    wsh[c1] = w1;
    if (threadIdx.x == 0) s_inv = 1.f / L;
  }
  __syncthreads();
  float acc = 0.f;
#pragma unroll 8
  for (int c = 0; c < n_chunks; ++c) acc += base[(size_t)c * DA_PART + d] * wsh[c];  // chunk order
  out[(size_t)r * Q_HEADS * HEAD_DIM + h * HEAD_DIM + d] = __float2bfloat16(acc * s_inv);
}

void decode_attention_v3(const CUtensorMap &kmap, const CUtensorMap &vmap, const bf16 *q, bf16 *out, const int *bt,
                         int bt_stride, const int *pos, const int *active, int rows, int max_blocks, float scale,
                         float *ws, int sms, cudaStream_t st) {
  if (rows <= 0) return;
  static bool attr = false;
  if (!attr) {
    OXY_CUDA(cudaFuncSetAttribute(decode_attn_v3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)D3_SMEM));
    attr = true;
  }
  (void)sms;
  const int cb = DECODE_CHUNK_BLOCKS;
  const int max_chunks = std::min(64, (max_blocks + cb - 1) / cb);
  launch_pdl(decode_attn_v3_kernel, dim3(rows, max_chunks), dim3(128), D3_SMEM, st, kmap, vmap, q, bt, bt_stride,
             pos, active, cb, max_chunks, scale * 1.4426950408889634f, ws, out);
  if (max_chunks > 1)
    launch_pdl(decode_merge3_kernel, dim3(rows, Q_HEADS), dim3(HEAD_DIM), 0, st, ws, out, pos, active, cb,
               max_chunks);
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
  OXY_REQUIRE(rows >= 1 && max_blocks >= 1 && bt_stride >= max_blocks && num_blocks >= 1,
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
