// F1: the reference toy transformer (kvweaver/backend.py:235-420) on the GPU.
//
// Verification mode: fp32 (or fp64) on CUDA-core FMA — no TF32, no tensor
// cores — so greedy tokens match the reference's float64 CPU path.  Every
// kernel computes one output from one row in a fixed reduction order, so
// results do not depend on batch composition, split points or which other
// rows are active (batch invariance: kvweaver/verify.py:121-222 routes agree
// bit-for-bit, which is stricter than the reference itself, README.md:201).
//
// KV lives in the unified paged pool: per layer K and V of
// [num_blocks, block_size, d_model]; a position p of a handle lives at slot
// blocks[p / B] * B + p % B.
#include <cmath>
#include <vector>

#include "cuda_util.cuh"

namespace oxy {
namespace toy {

// ---------------------------------------------------------------- kernels

template <typename T>
__global__ void init_uniform_kernel(T *out, int64_t n, uint64_t seed, int64_t offset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // -0.1 + 0.2 * u without FMA contraction (kvweaver/backend.py:252)
    double u = splitmix_uniform(seed, (uint64_t)(offset + i));
    out[i] = (T)__dadd_rn(-0.1, __dmul_rn(0.2, u));
  }
}

// x[r, :] = embed[tok[r], :] + PE(pos[r])   (kvweaver/backend.py:208-215, 271-274)
template <typename T>
__global__ void embed_kernel(T *x, const T *embed, const int *tok, const int *pos,
                             const int *active, int d) {
  const int r = blockIdx.x;
  if (active && !active[r]) return;
  const int t = tok[r];
  const double p = (double)pos[r];
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const int i = j >> 1;
    const double inv = pow(10000.0, -((double)i * 2.0) / (double)d);
    const double ang = p * inv;
    const double pe = (j & 1) ? cos(ang) : sin(ang);
    x[(size_t)r * d + j] = embed[(size_t)t * d + j] + (T)pe;
  }
}

// y[r, n] = (res ? res[r, n] : 0) + act(sum_k x[r, k] * W[k, n]); W row-major [K, N].
// blockIdx.z picks one of up to three (W, y) pairs (fused Q/K/V projection).
template <typename T>
struct LinearArgs {
  const T *w[3];
  T *y[3];
};

template <typename T>
__global__ void linear_kernel(LinearArgs<T> a, const T *x, const T *res, const int *active,
                              int K, int N, int relu) {
  extern __shared__ unsigned char smem_raw[];
  T *xs = reinterpret_cast<T *>(smem_raw);
  const int r = blockIdx.y;
  if (active && !active[r]) return;
  const T *W = a.w[blockIdx.z];
  T *Y = a.y[blockIdx.z];
  for (int k = threadIdx.x; k < K; k += blockDim.x) xs[k] = x[(size_t)r * K + k];
  __syncthreads();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  T acc = T(0);
  for (int k = 0; k < K; ++k) acc = fma(xs[k], W[(size_t)k * N + n], acc);
  if (relu) acc = acc > T(0) ? acc : T(0);
  if (res) acc = res[(size_t)r * N + n] + acc;
  Y[(size_t)r * N + n] = acc;
}

// K/V rows -> pool slots for one layer.  slot[r] < 0 skips the row.
template <typename T>
__global__ void kv_append_kernel(T *kpool, T *vpool, const T *k, const T *v, const int *slot,
                                 const int *active, int d) {
  const int r = blockIdx.x;
  if (active && !active[r]) return;
  const int s = slot[r];
  if (s < 0) return;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    kpool[(size_t)s * d + j] = k[(size_t)r * d + j];
    vpool[(size_t)s * d + j] = v[(size_t)r * d + j];
  }
}

// Row r, head h: softmax(q k^T * scale) v over this row's visible keys.
// Dense causal mode (kbase != null): keys 0..r of a [T, d] buffer.
// Paged mode: keys 0..pos[r] of the row's block table.  (backend.py:287-295, 365-384)
template <typename T>
__global__ void attention_kernel(T *ctx, const T *q, const T *kdense, const T *vdense,
                                 const T *kpool, const T *vpool, const int *block_tables,
                                 int bt_stride, int block_size, const int *pos,
                                 const int *active, int d, int dh, T scale) {
  extern __shared__ unsigned char smem_raw[];
  T *red = reinterpret_cast<T *>(smem_raw);  // 32 entries
  T *qs = red + 32;                           // dh
  T *p = qs + dh;                             // n_keys
  const int r = blockIdx.x, h = blockIdx.y;
  if (active && !active[r]) return;
  const bool dense = kdense != nullptr;
  const int n_keys = (dense ? r : pos[r]) + 1;
  const int *bt = dense ? nullptr : block_tables + (size_t)r * bt_stride;
  for (int j = threadIdx.x; j < dh; j += blockDim.x) qs[j] = q[(size_t)r * d + h * dh + j];
  __syncthreads();
  T mx = -INFINITY;
  for (int j = threadIdx.x; j < n_keys; j += blockDim.x) {
    const T *kr = dense ? kdense + (size_t)j * d
                        : kpool + ((size_t)bt[j / block_size] * block_size + j % block_size) * d;
    kr += h * dh;
    T s = T(0);
    for (int e = 0; e < dh; ++e) s = fma(qs[e], kr[e], s);
    s *= scale;
    p[j] = s;
    mx = max(mx, s);
  }
  mx = block_max(mx, red);
  T sum = T(0);
  for (int j = threadIdx.x; j < n_keys; j += blockDim.x) {
    T e = exp(p[j] - mx);
    p[j] = e;
    sum += e;
  }
  sum = block_sum(sum, red);
  __syncthreads();
  for (int j = threadIdx.x; j < n_keys; j += blockDim.x) p[j] = p[j] / sum;
  __syncthreads();
  for (int e = threadIdx.x; e < dh; e += blockDim.x) {
    T acc = T(0);
    for (int j = 0; j < n_keys; ++j) {
      const T *vr = dense ? vdense + (size_t)j * d
                          : vpool + ((size_t)bt[j / block_size] * block_size + j % block_size) * d;
      acc = fma(p[j], vr[h * dh + e], acc);
    }
    ctx[(size_t)r * d + h * dh + e] = acc;
  }
}

// Greedy pick with lowest-id tie-break (np.argmax, backend.py:388) and the
// per-row termination update (backend.py:389-397), all on device.
template <typename T>
__global__ void argmax_update_kernel(const T *logits, int V, int step, int k, int eos,
                                     int *active, int *tok, int *pos, int *count,
                                     const int *budget, int *out_tokens) {
  __shared__ T bv[32];
  __shared__ int bi[32];
  const int r = blockIdx.x;
  if (!active[r]) return;
  const T *lg = logits + (size_t)r * V;
  T best = -INFINITY;
  int idx = 0x7fffffff;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    T v = lg[j];
    if (v > best) { best = v; idx = j; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    T ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { bv[w] = best; bi[w] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (bv[i] > best || (bv[i] == best && bi[i] < idx)) { best = bv[i]; idx = bi[i]; }
    if (idx == 0x7fffffff) idx = 0;  // all-NaN row: deterministic fallback
    out_tokens[(size_t)r * k + step] = idx;
    tok[r] = idx;
    pos[r] += 1;
    int c = ++count[r];
    if (idx == eos || c == budget[r]) active[r] = 0;
  }
}

// Slot of the next position of each active row, from its block table.
__global__ void slot_kernel(int *slot, const int *pos, const int *active, const int *bt,
                            int bt_stride, int block_size, int rows) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (!active[r]) { slot[r] = -1; return; }
  int p = pos[r];
  slot[r] = bt[(size_t)r * bt_stride + p / block_size] * block_size + p % block_size;
}

// Copy-on-write of a shared tail block: slots [0, n) of src -> dst, all layers.
template <typename T>
__global__ void cow_kernel(T *pool, const int *cow, int rows, int L, size_t layer_stride,
                           size_t kv_stride, int block_size, int d) {
  const int r = blockIdx.x, l = blockIdx.y;
  const int src = cow[r * 3], dst = cow[r * 3 + 1], n = cow[r * 3 + 2];
  if (src < 0) return;
  for (int kv = 0; kv < 2; ++kv) {
    T *base = pool + l * layer_stride + kv * kv_stride;
    for (int i = threadIdx.x; i < n * d; i += blockDim.x)
      base[(size_t)dst * block_size * d + i] = base[(size_t)src * block_size * d + i];
  }
}

// ctx = mean_t V_last[t]; target = head @ ctx; S Euler steps (backend.py:316-332).
template <typename T>
__global__ void denoise_kernel(T *out, const T *vpool, const int *blocks, int seq_len,
                               int block_size, const T *head, int d, int HA, int S) {
  extern __shared__ unsigned char smem_raw[];
  T *ctx = reinterpret_cast<T *>(smem_raw);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    T s = T(0);
    for (int t = 0; t < seq_len; ++t)
      s += vpool[((size_t)blocks[t / block_size] * block_size + t % block_size) * d + j];
    ctx[j] = s / (T)seq_len;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HA; i += blockDim.x) {
    T tgt = T(0);
    for (int j = 0; j < d; ++j) tgt = fma(head[(size_t)i * d + j], ctx[j], tgt);
    T a = T(0);
    for (int s = 0; s < S; ++s) {
      T delta = (tgt - a) / (T)(S - s);
      a = a + delta;
    }
    out[i] = a;
  }
}

template <typename T>
__global__ void gather_kv_kernel(T *kout, T *vout, const T *kpool, const T *vpool,
                                 const int *blocks, int seq_len, int block_size, int d) {
  const int t = blockIdx.x;
  const size_t s = (size_t)blocks[t / block_size] * block_size + t % block_size;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    kout[(size_t)t * d + j] = kpool[s * d + j];
    vout[(size_t)t * d + j] = vpool[s * d + j];
  }
}

template <typename T>
__global__ void scatter_kv_kernel(T *kpool, T *vpool, const double *kin, const double *vin,
                                  const int *blocks, int seq_len, int block_size, int d) {
  const int t = blockIdx.x;
  const size_t s = (size_t)blocks[t / block_size] * block_size + t % block_size;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    kpool[s * d + j] = (T)kin[(size_t)t * d + j];
    vpool[s * d + j] = (T)vin[(size_t)t * d + j];
  }
}

template <typename T>
__global__ void cast_kernel(double *out, const T *in, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

template <typename T>
__global__ void uncast_kernel(T *out, const double *in, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)in[i];
}

// ---------------------------------------------------------------- model

struct Base {
  virtual ~Base() = default;
};

template <typename T>
struct Model : Base {
  oxy_toy_config c{};
  int d = 0, ff = 0, nh = 0, dh = 0, B = 0, NB = 0;
  T scale{};
  T *weights = nullptr;               // one allocation, reference draw order
  T *embed, *unembed, *head;
  std::vector<T *> wq, wk, wv, wo, w1, w2;
  T *pool = nullptr;                  // [L][2][NB][B][d]
  size_t layer_stride = 0, kv_stride = 0;
  DevBuf x, q, kk, vv, ctx, hid, logits, ints, staging, cast;

  T *kpool(int l) { return pool + l * layer_stride; }
  T *vpool(int l) { return pool + l * layer_stride + kv_stride; }

  ~Model() override {
    cudaFree(weights);
    cudaFree(pool);
    for (DevBuf *b : {&x, &q, &kk, &vv, &ctx, &hid, &logits, &ints, &staging, &cast}) b->release();
  }

  void create(const oxy_toy_config &cfg, int nb, int bs, cudaStream_t st) {
    c = cfg;
    d = c.d_model;
    ff = 4 * d;
    nh = c.n_heads;
    dh = d / nh;
    B = bs;
    NB = nb;
    scale = (T)(1.0 / std::sqrt((double)dh));
    const int64_t V = c.vocab, HA = (int64_t)c.H * c.action_dim;
    const int64_t per_layer = 4LL * d * d + 2LL * d * ff;
    const int64_t total = V * d + c.L * per_layer + d * V + HA * d;
    OXY_CUDA(cudaMalloc(&weights, total * sizeof(T)));
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    init_uniform_kernel<T><<<blocks, 256, 0, st>>>(weights, total, c.seed, 0);
    OXY_LAUNCH_CHECK();
    T *p = weights;
    auto take = [&](int64_t n) { T *r = p; p += n; return r; };
    embed = take(V * d);
    for (int l = 0; l < c.L; ++l) {
      wq.push_back(take((int64_t)d * d));
      wk.push_back(take((int64_t)d * d));
      wv.push_back(take((int64_t)d * d));
      wo.push_back(take((int64_t)d * d));
      w1.push_back(take((int64_t)d * ff));
      w2.push_back(take((int64_t)ff * d));
    }
    unembed = take((int64_t)d * V);
    head = take(HA * d);
    kv_stride = (size_t)NB * B * d;
    layer_stride = 2 * kv_stride;
    OXY_CUDA(cudaMalloc(&pool, c.L * layer_stride * sizeof(T)));
    OXY_CUDA(cudaMemsetAsync(pool, 0, c.L * layer_stride * sizeof(T), st));
  }

  T *weight_ptr(int which, int layer, int64_t *n) {
    const int64_t V = c.vocab, HA = (int64_t)c.H * c.action_dim;
    OXY_REQUIRE(which >= 0 && which <= 8, "unknown weight id %d", which);
    if (which >= 1 && which <= 6) OXY_REQUIRE(layer >= 0 && layer < c.L, "layer %d out of range", layer);
    switch (which) {
      case 0: *n = V * d; return embed;
      case 1: *n = (int64_t)d * d; return wq[layer];
      case 2: *n = (int64_t)d * d; return wk[layer];
      case 3: *n = (int64_t)d * d; return wv[layer];
      case 4: *n = (int64_t)d * d; return wo[layer];
      case 5: *n = (int64_t)d * ff; return w1[layer];
      case 6: *n = (int64_t)ff * d; return w2[layer];
      case 7: *n = (int64_t)d * V; return unembed;
      default: *n = HA * d; return head;
    }
  }

  void linear(cudaStream_t st, int rows, const T *xin, int K, int N, const T *w0, T *y0,
              const T *res = nullptr, bool relu = false, const int *active = nullptr,
              const T *w1p = nullptr, T *y1 = nullptr, const T *w2p = nullptr, T *y2 = nullptr) {
    LinearArgs<T> a{{w0, w1p, w2p}, {y0, y1, y2}};
    int nz = w2p ? 3 : (w1p ? 2 : 1);
    dim3 grid((N + 127) / 128, rows, nz);
    linear_kernel<T><<<grid, 128, K * sizeof(T), st>>>(a, xin, res, active, K, N, relu ? 1 : 0);
    OXY_LAUNCH_CHECK();
  }

  void attention(cudaStream_t st, int rows, const T *qin, T *out, const T *kd, const T *vd,
                 int l, const int *bt, int bt_stride, const int *pos, const int *active,
                 int max_keys) {
    size_t sm = (32 + dh + (size_t)max_keys) * sizeof(T);
    if (sm > 48 * 1024) {
      OXY_CUDA(cudaFuncSetAttribute(attention_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)std::min<size_t>(sm, 227 * 1024)));
    }
    OXY_REQUIRE(sm <= 227 * 1024, "sequence of %d positions exceeds the toy attention limit", max_keys);
    attention_kernel<T><<<dim3(rows, nh), 128, sm, st>>>(
        out, qin, kd, vd, kd ? nullptr : kpool(l), kd ? nullptr : vpool(l), bt, bt_stride, B,
        pos, active, d, dh, scale);
    OXY_LAUNCH_CHECK();
  }

  // Causal pass over T tokens.  slots != null: write K/V to the pool.
  // want_logits: final hidden of the last row -> logits (recompute route).
  void dense_forward(cudaStream_t st, const int *tokens_h, int T_, const int *slots_h,
                     T *logits_out) {
    int *ints_d = ints.as<int>(3 * (size_t)T_);
    std::vector<int> host(3 * (size_t)T_);
    for (int i = 0; i < T_; ++i) {
      host[i] = tokens_h[i];
      host[T_ + i] = i;
      host[2 * T_ + i] = slots_h ? slots_h[i] : -1;
    }
    OXY_CUDA(cudaMemcpyAsync(ints_d, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    T *X = x.as<T>((size_t)T_ * d), *Q = q.as<T>((size_t)T_ * d), *K = kk.as<T>((size_t)T_ * d),
      *Vv = vv.as<T>((size_t)T_ * d), *C = ctx.as<T>((size_t)T_ * d), *Hh = hid.as<T>((size_t)T_ * ff);
    embed_kernel<T><<<T_, 128, 0, st>>>(X, embed, ints_d, ints_d + T_, nullptr, d);
    OXY_LAUNCH_CHECK();
    for (int l = 0; l < c.L; ++l) {
      linear(st, T_, X, d, d, wq[l], Q, nullptr, false, nullptr, wk[l], K, wv[l], Vv);
      if (slots_h) {
        kv_append_kernel<T><<<T_, 128, 0, st>>>(kpool(l), vpool(l), K, Vv, ints_d + 2 * T_, nullptr, d);
        OXY_LAUNCH_CHECK();
        if (l == c.L - 1 && !logits_out) break;  // the last block's output is not cached
      }
      attention(st, T_, Q, C, K, Vv, l, nullptr, 0, nullptr, nullptr, T_);
      linear(st, T_, C, d, d, wo[l], X, X);
      linear(st, T_, X, d, ff, w1[l], Hh, nullptr, true);
      linear(st, T_, Hh, ff, d, w2[l], X, X);
    }
    if (logits_out) linear(st, 1, X + (size_t)(T_ - 1) * d, d, c.vocab, unembed, logits_out);
  }

  void to_host_f64(cudaStream_t st, const T *src, double *dst, int64_t n) {
    double *tmp = cast.as<double>(n);
    cast_kernel<T><<<(int)std::min<int64_t>((n + 255) / 256, 2048), 256, 0, st>>>(tmp, src, n);
    OXY_LAUNCH_CHECK();
    OXY_CUDA(cudaMemcpyAsync(dst, tmp, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    OXY_CUDA(cudaStreamSynchronize(st));
  }

  void decode(cudaStream_t st, int rows, int k, const int32_t *bt_h, int maxb, const int32_t *seq_h,
              const int32_t *last_h, const int32_t *budget_h, const int32_t *cow_h,
              int32_t *out_tok_h, int32_t *out_cnt_h) {
    // device int state: bt | cow | active | tok | pos | count | budget | slot | out
    const size_t n_bt = (size_t)rows * maxb, n_out = (size_t)rows * k;
    const size_t total = n_bt + 3 * (size_t)rows + 6 * (size_t)rows + n_out;
    std::vector<int> h(total, 0);
    int *hp = h.data();
    std::copy(bt_h, bt_h + n_bt, hp);
    std::copy(cow_h, cow_h + 3 * rows, hp + n_bt);
    int *h_active = hp + n_bt + 3 * rows, *h_tok = h_active + rows, *h_pos = h_tok + rows,
        *h_cnt = h_pos + rows, *h_bud = h_cnt + rows;
    int max_pos = 0;
    for (int r = 0; r < rows; ++r) {
      h_active[r] = 1;
      h_tok[r] = last_h[r];
      h_pos[r] = seq_h[r];
      h_bud[r] = budget_h[r];
      OXY_REQUIRE(seq_h[r] >= 1 && budget_h[r] >= 1, "row %d: seq_len and budget must be >= 1", r);
      OXY_REQUIRE(last_h[r] >= 0 && last_h[r] < c.vocab, "token %d outside vocab", last_h[r]);
      max_pos = std::max(max_pos, seq_h[r] + std::min(k, budget_h[r]));
    }
    OXY_REQUIRE(maxb >= 1 && (max_pos + B - 1) / B <= maxb, "block table too short for %d positions", max_pos);
    check_block_ids(bt_h, (int64_t)n_bt, NB, "decode");
    check_cow(cow_h, rows, NB, B);
    int *dv = ints.as<int>(total);
    OXY_CUDA(cudaMemcpyAsync(dv, hp, total * sizeof(int), cudaMemcpyHostToDevice, st));
    int *d_bt = dv, *d_cow = dv + n_bt, *d_active = d_cow + 3 * rows, *d_tok = d_active + rows,
        *d_pos = d_tok + rows, *d_cnt = d_pos + rows, *d_bud = d_cnt + rows, *d_slot = d_bud + rows,
        *d_out = d_slot + rows;
    cow_kernel<T><<<dim3(rows, c.L), 128, 0, st>>>(pool, d_cow, rows, c.L, layer_stride, kv_stride, B, d);
    OXY_LAUNCH_CHECK();
    T *X = x.as<T>((size_t)rows * d), *Q = q.as<T>((size_t)rows * d), *K = kk.as<T>((size_t)rows * d),
      *Vv = vv.as<T>((size_t)rows * d), *C = ctx.as<T>((size_t)rows * d),
      *Hh = hid.as<T>((size_t)rows * ff), *LG = logits.as<T>((size_t)rows * c.vocab);
    for (int s = 0; s < k; ++s) {
      embed_kernel<T><<<rows, 128, 0, st>>>(X, embed, d_tok, d_pos, d_active, d);
      slot_kernel<<<(rows + 127) / 128, 128, 0, st>>>(d_slot, d_pos, d_active, d_bt, maxb, B, rows);
      OXY_LAUNCH_CHECK();
      for (int l = 0; l < c.L; ++l) {
        linear(st, rows, X, d, d, wq[l], Q, nullptr, false, d_active, wk[l], K, wv[l], Vv);
        kv_append_kernel<T><<<rows, 128, 0, st>>>(kpool(l), vpool(l), K, Vv, d_slot, d_active, d);
        OXY_LAUNCH_CHECK();
        attention(st, rows, Q, C, nullptr, nullptr, l, d_bt, maxb, d_pos, d_active, max_pos + 1);
        linear(st, rows, C, d, d, wo[l], X, X, false, d_active);
        linear(st, rows, X, d, ff, w1[l], Hh, nullptr, true, d_active);
        linear(st, rows, Hh, ff, d, w2[l], X, X, false, d_active);
      }
      linear(st, rows, X, d, c.vocab, unembed, LG, nullptr, false, d_active);
      argmax_update_kernel<T><<<rows, 256, 0, st>>>(LG, c.vocab, s, k, c.eos_token, d_active, d_tok,
                                                    d_pos, d_cnt, d_bud, d_out);
      OXY_LAUNCH_CHECK();
    }
    OXY_CUDA(cudaMemcpyAsync(out_tok_h, d_out, n_out * sizeof(int), cudaMemcpyDeviceToHost, st));
    OXY_CUDA(cudaMemcpyAsync(out_cnt_h, d_cnt, rows * sizeof(int), cudaMemcpyDeviceToHost, st));
    OXY_CUDA(cudaStreamSynchronize(st));
  }
};

}  // namespace toy
}  // namespace oxy

struct oxy_toy {
  int dtype = 0;
  oxy::toy::Base *impl = nullptr;
  ~oxy_toy() { delete impl; }
};

namespace {
template <typename F>
void dispatch(oxy_toy *m, F &&f) {
  OXY_REQUIRE(m && m->impl, "null toy model");
  if (m->dtype == 0) f(*static_cast<oxy::toy::Model<float> *>(m->impl));
  else f(*static_cast<oxy::toy::Model<double> *>(m->impl));
}
std::vector<int32_t> slots_for(const int32_t *blocks, int B, int n) {
  std::vector<int32_t> s(n);
  for (int p = 0; p < n; ++p) s[p] = blocks[p / B] * B + p % B;
  return s;
}
}  // namespace

extern "C" {

int oxy_toy_create(const oxy_toy_config *cfg, int32_t dtype, int32_t num_blocks, int32_t block_size,
                   void *stream, oxy_toy **out) {
  OXY_API_BEGIN
  OXY_REQUIRE(cfg && cfg->L >= 1 && cfg->d_model >= 2 && cfg->n_heads >= 1 &&
                  cfg->d_model % cfg->n_heads == 0 && cfg->vocab >= 2,
              "invalid toy config");
  OXY_REQUIRE(dtype == 0 || dtype == 1, "dtype must be 0 (f32) or 1 (f64)");
  auto *m = new oxy_toy;
  m->dtype = dtype;
  try {
    if (dtype == 0) {
      auto *impl = new oxy::toy::Model<float>;
      m->impl = impl;
      impl->create(*cfg, num_blocks, block_size, oxy::as_stream(stream));
    } else {
      auto *impl = new oxy::toy::Model<double>;
      m->impl = impl;
      impl->create(*cfg, num_blocks, block_size, oxy::as_stream(stream));
    }
    OXY_CUDA(cudaStreamSynchronize(oxy::as_stream(stream)));
  } catch (...) {
    delete m;
    throw;
  }
  *out = m;
  OXY_API_END
}

int oxy_toy_destroy(oxy_toy *m) {
  delete m;
  return OXY_OK;
}

int oxy_toy_weight(oxy_toy *m, int32_t which, int32_t layer, double *host, int64_t n, int32_t write,
                   void *stream) {
  OXY_API_BEGIN
  auto st = oxy::as_stream(stream);
  dispatch(m, [&](auto &M) {
    using T = std::remove_reference_t<decltype(*M.embed)>;
    int64_t cnt = 0;
    T *w = M.weight_ptr(which, layer, &cnt);
    OXY_REQUIRE(n == cnt, "weight %d has %lld elements, got %lld", which, (long long)cnt, (long long)n);
    if (!write) {
      M.to_host_f64(st, w, host, n);
    } else {
      double *tmp = M.cast.template as<double>(n);
      OXY_CUDA(cudaMemcpyAsync(tmp, host, n * sizeof(double), cudaMemcpyHostToDevice, st));
      oxy::toy::uncast_kernel<T><<<(int)std::min<int64_t>((n + 255) / 256, 2048), 256, 0, st>>>(w, tmp, n);
      OXY_LAUNCH_CHECK();
      OXY_CUDA(cudaStreamSynchronize(st));
    }
  });
  OXY_API_END
}

int oxy_toy_prefill(oxy_toy *m, const int32_t *tokens_h, int32_t T, const int32_t *blocks_h, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(T >= 1, "prefill needs at least one token");
  dispatch(m, [&](auto &M) {
    for (int i = 0; i < T; ++i)
      OXY_REQUIRE(tokens_h[i] >= 0 && tokens_h[i] < M.c.vocab, "observation token %d outside vocab of %d",
                  tokens_h[i], M.c.vocab);
    oxy::check_block_ids(blocks_h, (T + M.B - 1) / M.B, M.NB, "prefill");
    auto slots = slots_for(blocks_h, M.B, T);
    M.dense_forward(oxy::as_stream(stream), tokens_h, T, slots.data(), nullptr);
  });
  OXY_API_END
}

int oxy_toy_recompute_logits(oxy_toy *m, const int32_t *tokens_h, int32_t T, double *logits_h,
                             void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(T >= 1, "recompute needs at least one token");
  auto st = oxy::as_stream(stream);
  dispatch(m, [&](auto &M) {
    using Tp = std::remove_reference_t<decltype(*M.embed)>;
    Tp *lg = M.logits.template as<Tp>(M.c.vocab);
    M.dense_forward(st, tokens_h, T, nullptr, lg);
    M.to_host_f64(st, lg, logits_h, M.c.vocab);
  });
  OXY_API_END
}

int oxy_toy_denoise(oxy_toy *m, const int32_t *blocks_h, int32_t seq_len, int32_t S, double *actions_h,
                    void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(S >= 1, "denoise step count must be >= 1, got %d", S);
  OXY_REQUIRE(seq_len >= 1, "denoise needs a non-empty cache");
  auto st = oxy::as_stream(stream);
  dispatch(m, [&](auto &M) {
    using Tp = std::remove_reference_t<decltype(*M.embed)>;
    const int nb = (seq_len + M.B - 1) / M.B, HA = M.c.H * M.c.action_dim;
    oxy::check_block_ids(blocks_h, nb, M.NB, "denoise");
    int *bd = M.ints.template as<int>(nb);
    OXY_CUDA(cudaMemcpyAsync(bd, blocks_h, nb * sizeof(int), cudaMemcpyHostToDevice, st));
    Tp *out = M.q.template as<Tp>(HA);
    oxy::toy::denoise_kernel<Tp><<<1, 256, M.d * sizeof(Tp), st>>>(out, M.vpool(M.c.L - 1), bd, seq_len,
                                                                   M.B, M.head, M.d, HA, S);
    OXY_LAUNCH_CHECK();
    M.to_host_f64(st, out, actions_h, HA);
  });
  OXY_API_END
}

int oxy_toy_decode(oxy_toy *m, int32_t rows, int32_t k, const int32_t *block_tables_h, int32_t max_blocks,
                   const int32_t *seq_lens_h, const int32_t *last_tokens_h, const int32_t *budgets_h,
                   const int32_t *cow_h, int32_t *out_tokens_h, int32_t *out_count_h, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(rows >= 1, "decode needs at least one row");
  OXY_REQUIRE(k >= 1, "decode step count must be >= 1, got %d", k);
  dispatch(m, [&](auto &M) {
    M.decode(oxy::as_stream(stream), rows, k, block_tables_h, max_blocks, seq_lens_h, last_tokens_h,
             budgets_h, cow_h, out_tokens_h, out_count_h);
  });
  OXY_API_END
}

int oxy_toy_read_kv(oxy_toy *m, const int32_t *blocks_h, int32_t seq_len, int32_t layer, double *keys_h,
                    double *values_h, void *stream) {
  OXY_API_BEGIN
  auto st = oxy::as_stream(stream);
  dispatch(m, [&](auto &M) {
    using Tp = std::remove_reference_t<decltype(*M.embed)>;
    OXY_REQUIRE(layer >= 0 && layer < M.c.L, "layer %d out of range", layer);
    if (seq_len == 0) return;
    OXY_REQUIRE(seq_len > 0, "negative sequence length");
    const int nb = (seq_len + M.B - 1) / M.B;
    oxy::check_block_ids(blocks_h, nb, M.NB, "kv access");
    int *bd = M.ints.template as<int>(nb);
    OXY_CUDA(cudaMemcpyAsync(bd, blocks_h, nb * sizeof(int), cudaMemcpyHostToDevice, st));
    Tp *ko = M.kk.template as<Tp>((size_t)seq_len * M.d), *vo = M.vv.template as<Tp>((size_t)seq_len * M.d);
    oxy::toy::gather_kv_kernel<Tp><<<seq_len, 128, 0, st>>>(ko, vo, M.kpool(layer), M.vpool(layer), bd,
                                                            seq_len, M.B, M.d);
    OXY_LAUNCH_CHECK();
    M.to_host_f64(st, ko, keys_h, (int64_t)seq_len * M.d);
    M.to_host_f64(st, vo, values_h, (int64_t)seq_len * M.d);
  });
  OXY_API_END
}

int oxy_toy_write_kv(oxy_toy *m, const int32_t *blocks_h, int32_t seq_len, int32_t layer,
                     const double *keys_h, const double *values_h, void *stream) {
  OXY_API_BEGIN
  auto st = oxy::as_stream(stream);
  dispatch(m, [&](auto &M) {
    using Tp = std::remove_reference_t<decltype(*M.embed)>;
    OXY_REQUIRE(layer >= 0 && layer < M.c.L, "layer %d out of range", layer);
    if (seq_len == 0) return;
    OXY_REQUIRE(seq_len > 0, "negative sequence length");
    const int nb = (seq_len + M.B - 1) / M.B;
    oxy::check_block_ids(blocks_h, nb, M.NB, "kv access");
    const size_t n = (size_t)seq_len * M.d;
    int *bd = M.ints.template as<int>(nb);
    double *tmp = M.cast.template as<double>(2 * n);
    OXY_CUDA(cudaMemcpyAsync(bd, blocks_h, nb * sizeof(int), cudaMemcpyHostToDevice, st));
    OXY_CUDA(cudaMemcpyAsync(tmp, keys_h, n * sizeof(double), cudaMemcpyHostToDevice, st));
    OXY_CUDA(cudaMemcpyAsync(tmp + n, values_h, n * sizeof(double), cudaMemcpyHostToDevice, st));
    oxy::toy::scatter_kv_kernel<Tp><<<seq_len, 128, 0, st>>>(M.kpool(layer), M.vpool(layer), tmp,
                                                             tmp + n, bd, seq_len, M.B, M.d);
    OXY_LAUNCH_CHECK();
    OXY_CUDA(cudaStreamSynchronize(st));
  });
  OXY_API_END
}

}  // extern "C"
