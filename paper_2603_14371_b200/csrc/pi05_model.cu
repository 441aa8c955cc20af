// F2: pi0.5-shaped Mixture-of-Transformers VLA on the B200 (bf16, tcgen05).
//
// The reference models the action and language experts as one toy backbone
// (kvweaver/backend.py:21-33); the paper's system is openpi pi0.5 (PAPER.md
// 85-87).  This runtime implements the pi0.5 shape:
//   * SigLIP So400m/14 vision tower, per camera, then a linear projection;
//   * Gemma-2B prefix (RMSNorm(1+w), MQA 8q/1kv heads of 256, RoPE, GeGLU),
//     prefix-LM bidirectional attention, K/V written ONCE into the unified
//     paged pool through the block table (shared prefix prefill);
//   * Gemma-300M action expert: flow-matching Euler from noise, adaRMS
//     time conditioning with gated residuals, suffix queries attending to
//     [paged prefix K/V of the same layer || suffix K/V] (cross-task sharing);
//   * greedy language decode continuously batched over rows, K/V appended to
//     the same pool, LM head + lowest-id argmax, per-row stop on device.
// Weight values are the builder's choice (random init, stated in DESIGN.md):
// splitmix64 counter draws, U(+-sqrt(3/fan_in)) for matrices.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "cuda_util.cuh"
#include "gemm_sm100.cuh"
#include "pi05_kernels.cuh"


namespace oxy {
namespace pi05 {

using gemm::EpiParams;

struct Tensor {
  std::string name;
  int64_t rows, cols;
  int dtype;  // 0 bf16, 1 f32
  float bound, center;
  uint64_t offset;
  void *ptr;
  int64_t numel() const { return rows * cols; }
};

struct LayerW {
  float *ln1, *ln2;
  bf16 *wqkv, *wo, *wgu, *wd;
};
struct ExpertW {
  bf16 *wqkv, *wo, *wgu, *wd;
};
struct VitW {
  float *ln1w, *ln1b, *ln2w, *ln2b, *bqkv, *bo, *b1, *b2;
  bf16 *wqkv, *wo, *w1, *w2;
};

constexpr int PATCH_K = 640;  // 14*14*3 = 588 padded to a multiple of 64
constexpr int QDIM = Q_HEADS * HEAD_DIM;
constexpr int QKV = (Q_HEADS + 2) * HEAD_DIM;
constexpr int MAX_DECODE_ROWS = 8192;

struct Model {
  oxy_pi05_config c{};
  int sms = 148;
  std::vector<Tensor> tensors;
  void *wmem = nullptr;
  // handles into wmem
  bf16 *embed = nullptr, *lm_head = nullptr;
  float *final_norm = nullptr;
  std::vector<LayerW> L;
  std::vector<ExpertW> E;
  std::vector<VitW> V;
  bf16 *e_in, *e_out, *t1, *t2, *wmod, *vpatch, *vproj;
  float *e_in_b, *e_out_b, *t1_b, *t2_b, *bmod, *vpatch_b, *vpos, *vln_w, *vln_b, *vproj_b;
  int n_mod = 0;
  // pool
  bf16 *pool = nullptr;
  std::vector<CUtensorMap> kv_maps;  // per layer: K, V
  int NB = 0;
  size_t kv_stride = 0, layer_stride = 0;
  // denoise constants
  float *noise = nullptr;           // [H, A]
  int mod_S = -1;
  DevBuf mod;                        // [S, n_mod] f32
  // scratch
  DevBuf x, y, qkv, q, o, hmid, ws, ints, kd, vd, attn_groups, attn_ws, attn_ml, logits, amv, ami,
      vit_h, vit_y, vit_qkv, vit_o, vit_m, patches, act, act_bf, vel, xe, dec_ws, kvread_i, kvread_f;
  cudaEvent_t ev = nullptr;

  bf16 *kpool(int l) { return pool + l * layer_stride; }
  bf16 *vpool(int l) { return pool + l * layer_stride + kv_stride; }

  ~Model() {
    if (pf_start) cudaEventDestroy(pf_start);
    for (cudaEvent_t e : pf_layer) cudaEventDestroy(e);
    destroy_exec();
    cudaFree(wmem);
    cudaFree(pool);
    cudaFree(noise);
    cudaFree(rope_inv);
    cudaFree(rope_cs);
    for (DevBuf *b : {&mod, &x, &y, &qkv, &q, &o, &hmid, &ws, &ints, &kd, &vd, &attn_groups, &attn_ws,
                      &attn_ml, &logits, &amv, &ami, &vit_h, &vit_y, &vit_qkv, &vit_o, &vit_m, &patches,
                      &act, &act_bf, &vel, &xe, &dec_ws, &kvread_i, &kvread_f})
      b->release();
  }

  // ------------------------------------------------------------ weights
  uint64_t next_offset = 0;
  void add(const std::string &name, int64_t rows, int64_t cols, int dtype, float bound, float center = 0.f) {
    Tensor t{name, rows, cols, dtype, bound, center, next_offset, nullptr};
    next_offset += (uint64_t)(rows * cols);
    tensors.push_back(t);
  }
  static float mat_bound(int64_t fan_in) { return (float)std::sqrt(3.0 / (double)fan_in); }
  // Gemma/expert QKV weights are stored with rotary pairs interleaved (gemm::qkv_rope_row)
  static bool is_rope_qkv(const std::string &n) {
    return (n.rfind("llm.", 0) == 0 || n.rfind("expert.", 0) == 0) && n.size() > 5 &&
           n.compare(n.size() - 5, 5, ".wqkv") == 0;
  }
  float *rope_inv = nullptr;
  float2 *rope_cs = nullptr;  // [ROPE_TABLE_POS][128] (cos, sin), gemm::QkvRope::cs
  // action vectors are padded to 8 lanes so the in-projection's K stride is 16-byte aligned
  int apad() const { return (c.action_dim + 7) / 8 * 8; }

  void declare() {
    const int W = c.width, We = c.expert_width, Dv = c.vit_width;
    add("embed", c.vocab, W, 0, mat_bound(W));
    for (int l = 0; l < c.depth; ++l) {
      std::string p = "llm." + std::to_string(l) + ".";
      add(p + "ln1", 1, W, 1, 0.1f);
      add(p + "wqkv", QKV, W, 0, mat_bound(W));
      add(p + "wo", W, QDIM, 0, mat_bound(QDIM));
      add(p + "ln2", 1, W, 1, 0.1f);
      add(p + "wgu", 2 * c.mlp, W, 0, mat_bound(W));
      add(p + "wd", W, c.mlp, 0, mat_bound(c.mlp));
    }
    add("final_norm", 1, W, 1, 0.1f);
    // untied LM head: with random weights a tied head echoes its input, so
    // EOS-as-BOS (kvweaver/backend.py:30-32) would end every request at once
    add("lm_head", c.vocab, W, 0, mat_bound(W));
    for (int l = 0; l < c.depth; ++l) {
      std::string p = "expert." + std::to_string(l) + ".";
      add(p + "wqkv", QKV, We, 0, mat_bound(We));
      add(p + "wo", We, QDIM, 0, mat_bound(QDIM));
      add(p + "wgu", 2 * c.expert_mlp, We, 0, mat_bound(We));
      add(p + "wd", We, c.expert_mlp, 0, mat_bound(c.expert_mlp));
    }
    n_mod = c.depth * 6 * We + 2 * We;
    add("action_in", We, apad(), 0, mat_bound(c.action_dim));
    add("action_in.b", 1, We, 1, 0.02f);
    add("action_out", c.action_dim, We, 0, mat_bound(We));
    add("action_out.b", 1, c.action_dim, 1, 0.02f);
    add("time1", We, We, 0, mat_bound(We));
    add("time1.b", 1, We, 1, 0.02f);
    add("time2", We, We, 0, mat_bound(We));
    add("time2.b", 1, We, 1, 0.02f);
    add("mod", n_mod, We, 0, 0.1f * mat_bound(We));
    add("mod.b", 1, n_mod, 1, 0.02f);
    if (c.vit_depth > 0) {
      add("vit.patch", Dv, PATCH_K, 0, mat_bound(588));
      add("vit.patch.b", 1, Dv, 1, 0.02f);
      add("vit.pos", 256, Dv, 1, 0.02f);
      for (int l = 0; l < c.vit_depth; ++l) {
        std::string p = "vit." + std::to_string(l) + ".";
        add(p + "ln1.w", 1, Dv, 1, 0.1f, 1.f);
        add(p + "ln1.b", 1, Dv, 1, 0.02f);
        add(p + "wqkv", 3 * Dv, Dv, 0, mat_bound(Dv));
        add(p + "bqkv", 1, 3 * Dv, 1, 0.02f);
        add(p + "wo", Dv, Dv, 0, mat_bound(Dv));
        add(p + "bo", 1, Dv, 1, 0.02f);
        add(p + "ln2.w", 1, Dv, 1, 0.1f, 1.f);
        add(p + "ln2.b", 1, Dv, 1, 0.02f);
        add(p + "w1", c.vit_mlp, Dv, 0, mat_bound(Dv));
        add(p + "b1", 1, c.vit_mlp, 1, 0.02f);
        add(p + "w2", Dv, c.vit_mlp, 0, mat_bound(c.vit_mlp));
        add(p + "b2", 1, Dv, 1, 0.02f);
      }
      add("vit.ln.w", 1, Dv, 1, 0.1f, 1.f);
      add("vit.ln.b", 1, Dv, 1, 0.02f);
      add("vit.proj", W, Dv, 0, mat_bound(Dv));
      add("vit.proj.b", 1, W, 1, 0.02f);
    }
  }

  void materialise(cudaStream_t st) {
    size_t bytes = 0;
    for (auto &t : tensors) {
      bytes = (bytes + 255) / 256 * 256;
      t.ptr = reinterpret_cast<void *>(bytes);
      bytes += t.numel() * (t.dtype == 0 ? 2 : 4);
    }
    OXY_CUDA(cudaMalloc(&wmem, bytes));
    for (auto &t : tensors) {
      t.ptr = static_cast<char *>(wmem) + reinterpret_cast<size_t>(t.ptr);
      if (t.dtype == 0)
        init_uniform_bf16(static_cast<bf16 *>(t.ptr), t.numel(), c.seed, t.offset, t.bound, st);
      else
        init_uniform_f32(static_cast<float *>(t.ptr), t.numel(), c.seed, t.offset, t.bound, t.center, st);
    }
    {
      Tensor &ai = find("action_in");
      if (apad() > c.action_dim)
        OXY_CUDA(cudaMemset2DAsync(static_cast<bf16 *>(ai.ptr) + c.action_dim, apad() * 2, 0,
                                   (apad() - c.action_dim) * 2, ai.rows, st));
    }
    if (c.vit_depth > 0) {  // patch columns 588..639 multiply zero padding; keep them zero
      Tensor &pt = find("vit.patch");
      OXY_CUDA(cudaMemset2DAsync(static_cast<bf16 *>(pt.ptr) + 588, PATCH_K * 2, 0, (PATCH_K - 588) * 2,
                                 pt.rows, st));
    }
    size_t i = 0;
    auto nb = [&]() { return static_cast<bf16 *>(tensors[i++].ptr); };
    auto nf = [&]() { return static_cast<float *>(tensors[i++].ptr); };
    embed = nb();
    for (int l = 0; l < c.depth; ++l) {
      LayerW w;
      w.ln1 = nf(); w.wqkv = nb(); w.wo = nb(); w.ln2 = nf(); w.wgu = nb(); w.wd = nb();
      L.push_back(w);
    }
    final_norm = nf();
    lm_head = nb();
    for (int l = 0; l < c.depth; ++l) {
      ExpertW w;
      w.wqkv = nb(); w.wo = nb(); w.wgu = nb(); w.wd = nb();
      E.push_back(w);
    }
    e_in = nb(); e_in_b = nf(); e_out = nb(); e_out_b = nf();
    t1 = nb(); t1_b = nf(); t2 = nb(); t2_b = nf(); wmod = nb(); bmod = nf();
    if (c.vit_depth > 0) {
      vpatch = nb(); vpatch_b = nf(); vpos = nf();
      for (int l = 0; l < c.vit_depth; ++l) {
        VitW w;
        w.ln1w = nf(); w.ln1b = nf(); w.wqkv = nb(); w.bqkv = nf(); w.wo = nb(); w.bo = nf();
        w.ln2w = nf(); w.ln2b = nf(); w.w1 = nb(); w.b1 = nf(); w.w2 = nb(); w.b2 = nf();
        V.push_back(w);
      }
      vln_w = nf(); vln_b = nf(); vproj = nb(); vproj_b = nf();
    }
  }

  Tensor &find(const std::string &n) {
    for (auto &t : tensors)
      if (t.name == n) return t;
    fail(OXY_EINVAL, "no tensor %s", n.c_str());
  }

  void create(const oxy_pi05_config &cfg, int num_blocks, cudaStream_t st) {
    c = cfg;
    int dev = 0;
    OXY_CUDA(cudaGetDevice(&dev));
    OXY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    declare();
    materialise(st);
    {  // device RoPE table for the fused QKV epilogue, and the rotary-pair row order
      float inv[128];
      for (int i = 0; i < 128; ++i) inv[i] = (float)std::pow(10000.0, -2.0 * i / 256.0);
      OXY_CUDA(cudaMalloc(&rope_inv, sizeof(inv)));
      OXY_CUDA(cudaMemcpyAsync(rope_inv, inv, sizeof(inv), cudaMemcpyHostToDevice, st));
      OXY_CUDA(cudaMalloc(&rope_cs, (size_t)gemm::ROPE_TABLE_POS * 128 * sizeof(float2)));
      rope_table(rope_cs, rope_inv, gemm::ROPE_TABLE_POS, st);
      bf16 *tmp = nullptr;
      const int kmax = std::max(c.width, c.expert_width);
      OXY_CUDA(cudaMalloc(&tmp, (size_t)QKV * kmax * sizeof(bf16)));
      for (auto &t : tensors)
        if (is_rope_qkv(t.name)) {
          OXY_CUDA(cudaMemcpyAsync(tmp, t.ptr, t.numel() * 2, cudaMemcpyDeviceToDevice, st));
          permute_rows(static_cast<bf16 *>(t.ptr), tmp, (int)t.rows, (int)t.cols, st);
        }
      OXY_CUDA(cudaStreamSynchronize(st));
      cudaFree(tmp);
    }
    NB = num_blocks;
    kv_stride = (size_t)NB * KV_BLOCK * HEAD_DIM;
    layer_stride = 2 * kv_stride;
    OXY_CUDA(cudaMalloc(&pool, (size_t)c.depth * layer_stride * sizeof(bf16)));
    for (int l = 0; l < c.depth; ++l) {  // TMA views of each layer's K and V pool: [NB*64, 256]
      kv_maps.push_back(gemm::make_map(kpool(l), NB * KV_BLOCK, HEAD_DIM, KV_BLOCK));
      kv_maps.push_back(gemm::make_map(vpool(l), NB * KV_BLOCK, HEAD_DIM, KV_BLOCK));
    }
    OXY_CUDA(cudaMemsetAsync(pool, 0, (size_t)c.depth * layer_stride * sizeof(bf16), st));
    // noise [H, apad] (pad lanes zero) from H*A standard normals
    OXY_CUDA(cudaMalloc(&noise, (size_t)c.H * apad() * sizeof(float)));
    OXY_CUDA(cudaMemsetAsync(noise, 0, (size_t)c.H * apad() * sizeof(float), st));
    float *tmp = vel.as<float>((size_t)c.H * c.action_dim);
    normal_noise(tmp, (int64_t)c.H * c.action_dim, c.seed ^ 0x6E6F697365ull, st);  // "noise"
    OXY_CUDA(cudaMemcpy2DAsync(noise, apad() * sizeof(float), tmp, c.action_dim * sizeof(float),
                               c.action_dim * sizeof(float), c.H, cudaMemcpyDeviceToDevice, st));
    OXY_CUDA(cudaStreamSynchronize(st));
    init_exec();
  }

  // ------------------------------------------------------------ execution
  // Every call = host planning (all per-call integers and attention
  // descriptors packed into one stable device arena, uploaded with a single
  // H2D copy) + a kernel-only body.  The body runs eagerly the first time a
  // shape is seen (sizing the grow-only scratch), is captured into a CUDA
  // graph the second time and replayed from then on.  Any scratch regrowth
  // bumps a generation counter that invalidates captured graphs.
  cudaStream_t mst = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  uint8_t *arena_d = nullptr;
  std::vector<uint8_t> arena_h;
  size_t arena_cap = 0, arena_used = 0;
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    unsigned long long gen = 0;
    int seen = 0;
    unsigned long long kernels = 0;  // kernel nodes, counted per replay
  };
  std::map<std::string, Graph> graphs;
  bool use_graphs = [] {  // OXY_GRAPHS=0: every call eager (sanitizer runs, debugging)
    const char *e = getenv("OXY_GRAPHS");
    return !e || atoi(e) != 0;
  }();

  int *gemm_counters = nullptr;
  // profiling only: OXY_DBG_SKIP bitmask drops kernels from the denoise chain
  // (results are garbage; used to measure each kernel's marginal cost in-graph)
  int dbg_skip = [] {
    const char *e = getenv("OXY_DBG_SKIP");
    return e ? atoi(e) : 0;
  }();

  // ---- execution lanes.  The members above (stream, events, arena, graph
  // cache, split-K counters) and the per-call scratch describe the ACTIVE lane.
  // Lane 0 runs prefill and language decode; lane 1 (`alt`) runs the action
  // expert, so a frame's denoise can overlap its decode (they share no
  // writable memory: denoise reads prefix slots [0, P), decode appends >= P).
  // LaneSwap exchanges the two sets around an enqueue (host calls are serial).
  struct LaneState {
    cudaStream_t mst = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, t0 = nullptr, t1 = nullptr;
    uint8_t *arena_d = nullptr;
    std::vector<uint8_t> arena_h;
    size_t arena_cap = 0, arena_used = 0;
    std::map<std::string, Graph> graphs;
    int *gemm_counters = nullptr;
    DevBuf y, q, o, hmid, ws, kd, vd, attn_ws, attn_ml;
  } alt;
  // Layer-pipelined overlapped denoise (OXY_PIPE_PREFILL=0: off): the prefill records
  // one event per Gemma layer once that layer's prefix K/V are in the pool; an
  // overlapped denoise on the expert partition of exactly those prefixes waits on them
  // layer by layer in its first Euler step (expert layer l reads only Gemma layer l's
  // K/V) instead of on the whole prefill, so that step runs under the prefill.  Same
  // kernels and plans: results are unchanged (the cross-variant tests compare it with
  // stage-serial frames bit for bit).  1 stream: 15.08 -> 14.90 ms per frame.
  bool pipe_prefill = [] {
    const char *e = getenv("OXY_PIPE_PREFILL");
    return !e || atoi(e) != 0;
  }();
  cudaEvent_t pf_start = nullptr;
  std::vector<cudaEvent_t> pf_layer;
  std::vector<int> pf_blocks;  // the last prefill's block ids (empty: nothing to pipeline behind)
  // external event record / wait nodes when capturing a graph, plain calls when eager
  unsigned capture_flag(unsigned ext) const {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    OXY_CUDA(cudaStreamIsCapturing(mst, &cs));
    return cs == cudaStreamCaptureStatusActive ? ext : 0u;
  }
  void pf_events() {
    if (!pf_start) OXY_CUDA(cudaEventCreateWithFlags(&pf_start, cudaEventDisableTiming));
    while ((int)pf_layer.size() < c.depth) {
      cudaEvent_t e;
      OXY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      pf_layer.push_back(e);
    }
  }
  void swap_lane(LaneState &s) {
    std::swap(mst, s.mst);
    std::swap(ev_in, s.ev_in);
    std::swap(ev_out, s.ev_out);
    std::swap(arena_d, s.arena_d);
    std::swap(arena_h, s.arena_h);
    std::swap(arena_cap, s.arena_cap);
    std::swap(arena_used, s.arena_used);
    std::swap(graphs, s.graphs);
    std::swap(gemm_counters, s.gemm_counters);
    for (auto [a, b] : {std::pair<DevBuf *, DevBuf *>{&y, &s.y}, {&q, &s.q}, {&o, &s.o}, {&hmid, &s.hmid},
                        {&ws, &s.ws}, {&kd, &s.kd}, {&vd, &s.vd}, {&attn_ws, &s.attn_ws}, {&attn_ml, &s.attn_ml}})
      std::swap(*a, *b);
  }
  struct LaneSwap {
    Model &m;
    explicit LaneSwap(Model &mm) : m(mm) { m.swap_lane(m.alt); }
    ~LaneSwap() { m.swap_lane(m.alt); }
  };

  void init_lane(int priority) {
    OXY_CUDA(cudaMalloc(&gemm_counters, gemm::MAX_TILES * sizeof(int)));
    OXY_CUDA(cudaMemset(gemm_counters, 0, gemm::MAX_TILES * sizeof(int)));
    OXY_CUDA(cudaStreamCreateWithPriority(&mst, cudaStreamNonBlocking, priority));
    OXY_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    OXY_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
    arena_cap = 8u << 20;
    OXY_CUDA(cudaMalloc(&arena_d, arena_cap));
    arena_h.resize(arena_cap);
  }
  void destroy_lane() {
    for (auto &kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (mst) cudaStreamDestroy(mst);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    cudaFree(arena_d);
    cudaFree(gemm_counters);
  }
  void init_exec() {

    // The action-expert lane gets the highest stream priority: its denoise is a
    // latency-bound chain of small kernels, the concurrent language decode is
    // bandwidth-bound and fills whatever SMs the chain leaves (OXY_LANE_PRIO=0: equal)
    int lo = 0, hi = 0;
    OXY_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char *e = getenv("OXY_LANE_PRIO");
    const bool prio = !e || atoi(e) != 0;
    // A/B knob OXY_LANE0_PRIO=1: lane 0 (prefill, decode) at the highest priority too
    const char *e0 = getenv("OXY_LANE0_PRIO");
    init_lane(e0 && atoi(e0) != 0 ? hi : lo);
    {
      LaneSwap g(*this);
      init_lane(prio ? hi : lo);
    }
    OXY_CUDA(cudaEventCreate(&alt.t0));
    OXY_CUDA(cudaEventCreate(&alt.t1));
    init_green();
  }
  void destroy_exec() {
    destroy_lane();
    {
      LaneSwap g(*this);
      destroy_lane();
    }
    destroy_green();  // after the graphs captured on its streams
    if (alt.t0) cudaEventDestroy(alt.t0);
    if (alt.t1) cudaEventDestroy(alt.t1);
    for (DevBuf *b : {&alt.y, &alt.q, &alt.o, &alt.hmid, &alt.ws, &alt.kd, &alt.vd, &alt.attn_ws, &alt.attn_ml})
      b->release();
  }
  // ---- SM partition of the overlapped section (OXY_GREEN=<expert SMs>, 0 = off).
  // While a frame's denoise overlaps its decode, the two chains otherwise fight
  // for SM slots: the decode's long weight-streaming CTAs hold the slots the
  // expert chain's next kernel needs, and the 209 KB tcgen05 attention needs a
  // whole SM.  Two green contexts split the SMs; an overlapped denoise of up to
  // OXY_GREEN_MAX_STREAMS streams runs on one partition and the decode it overlaps
  // on the other.  Stand-alone calls (prefill, a denoise or decode with nothing
  // overlapping, multi-stream denoise) keep every SM.  Plans do not change
  // (split-K partitions depend on (phase, N, K) only), so results are bit-identical
  // either way.  Measured (profiles/r02/green_ab*.txt): 1 stream 16.6 -> 15.8 ms per
  // frame with 80 expert SMs (64: 16.2, 72: 15.9, 88: 16.8); 2-8 streams slower with
  // any split (the expert chain needs the whole GPU), hence the stream cap.
  struct Green {
    int dn_sms = 0, dec_sms = 0;
    cudaStream_t dn = nullptr, dec = nullptr;
    void *g_dn = nullptr, *g_dec = nullptr;  // CUgreenCtx
  } green;
  bool denoise_pending = false;  // an overlapped denoise on the partition was enqueued, not joined yet
  bool on_partition = false;     // the call being enqueued runs on a green-context partition
  int green_max_streams = [] {
    const char *e = getenv("OXY_GREEN_MAX_STREAMS");
    return e ? atoi(e) : 1;
  }();
  void init_green() {
    const char *e = getenv("OXY_GREEN");
    // with the layer-pipelined first Euler step: 136 expert SMs and an 88-SM decode
    // partition sharing 76 of them (14.56 ms/frame with disjoint 72 / 76, 14.43 at 96 / 80,
    // 14.23 at 136 / 88, profiles/r02/overlap_ab*.txt); else disjoint 80 / 68
    const int want = e ? atoi(e) : pipe_prefill ? 136 : 80;
    if (want <= 0 || want >= sms) return;
    try {
      make_green(want);
    } catch (const std::exception &) {  // no green contexts on this driver: one shared SM pool
      green = Green{};
    }
  }
  void make_green(int want) {
    typedef CUresult (*GetRes)(CUdevice, CUdevResource *, CUdevResourceType);
    typedef CUresult (*Split)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *, unsigned, unsigned);
    typedef CUresult (*GenDesc)(CUdevResourceDesc *, CUdevResource *, unsigned);
    typedef CUresult (*Create)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned);
    typedef CUresult (*StreamCreate)(CUstream *, CUgreenCtx, unsigned, int);
    auto sym = [](const char *name) {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      OXY_CUDA(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess) fail(OXY_ECUDA, "%s unavailable", name);
      return fn;
    };
    int dev = 0;
    OXY_CUDA(cudaGetDevice(&dev));
    CUdevResource all{}, part[2]{}, rest{};
    unsigned n = 1;
    auto chk = [](CUresult r, const char *what) {
      if (r != CUDA_SUCCESS) fail(OXY_ECUDA, "%s failed (%d)", what, (int)r);
    };
    chk(reinterpret_cast<GetRes>(sym("cuDeviceGetDevResource"))((CUdevice)dev, &all, CU_DEV_RESOURCE_TYPE_SM),
        "cuDeviceGetDevResource");
    chk(reinterpret_cast<Split>(sym("cuDevSmResourceSplitByCount"))(part, &n, &all, &rest, 0, (unsigned)want),
        "cuDevSmResourceSplitByCount");
    // OXY_GREEN_DEC=<SMs> (default 88 with the pipelined first step, else 0 = the
    // complement): the decode partition from a second split of all SMs (the complement
    // of its first sms - <SMs>), so it shares SMs with the expert's.  Green contexts may
    // overlap; plans do not depend on the partition, so results are unchanged.
    const char *edec = getenv("OXY_GREEN_DEC");
    const int want_dec = edec ? atoi(edec) : pipe_prefill ? 88 : 0;
    if (want_dec > 0 && want_dec < sms && want_dec + want > sms) {
      CUdevResource part2[1]{};
      unsigned n2 = 1;
      chk(reinterpret_cast<Split>(sym("cuDevSmResourceSplitByCount"))(part2, &n2, &all, &rest, 0,
                                                                       (unsigned)(sms - want_dec)),
          "cuDevSmResourceSplitByCount (decode)");
    }
    CUdevResourceDesc d_dn, d_dec;
    auto gen = reinterpret_cast<GenDesc>(sym("cuDevResourceGenerateDesc"));
    chk(gen(&d_dn, &part[0], 1), "cuDevResourceGenerateDesc");
    chk(gen(&d_dec, &rest, 1), "cuDevResourceGenerateDesc");
    auto create = reinterpret_cast<Create>(sym("cuGreenCtxCreate"));
    CUgreenCtx g_dn, g_dec;
    chk(create(&g_dn, d_dn, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    chk(create(&g_dec, d_dec, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    int lo = 0, hi = 0;
    OXY_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    auto screate = reinterpret_cast<StreamCreate>(sym("cuGreenCtxStreamCreate"));
    CUstream s_dn, s_dec;
    // the expert partition's stream at the prefill's (low) priority: the decode runs on
    // other SMs, and the pipelined first Euler step then does not take freed SM slots
    // ahead of the prefill it runs under (14.69 -> 14.56 ms/frame, profiles/r02/prio_ab.txt;
    // OXY_GREEN_DN_PRIO=1: highest)
    const char *edp = getenv("OXY_GREEN_DN_PRIO");
    const int dn_prio = !edp || atoi(edp) == 0 ? lo : atoi(edp) == 2 ? (lo + hi) / 2 : hi;  // 2: between (A/B)
    chk(screate(&s_dn, g_dn, CU_STREAM_NON_BLOCKING, dn_prio), "cuGreenCtxStreamCreate");
    chk(screate(&s_dec, g_dec, CU_STREAM_NON_BLOCKING, lo), "cuGreenCtxStreamCreate");
    green.dn = reinterpret_cast<cudaStream_t>(s_dn);
    green.dec = reinterpret_cast<cudaStream_t>(s_dec);
    green.g_dn = g_dn;
    green.g_dec = g_dec;
    green.dn_sms = (int)part[0].sm.smCount;
    green.dec_sms = (int)rest.sm.smCount;
  }
  void destroy_green() {
    if (!green.g_dn) return;
    typedef CUresult (*Destroy)(CUgreenCtx);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuGreenCtxDestroy", &fn, cudaEnableDefault, &q) == cudaSuccess && fn) {
      cudaStreamDestroy(green.dn);
      cudaStreamDestroy(green.dec);
      reinterpret_cast<Destroy>(fn)(static_cast<CUgreenCtx>(green.g_dn));
      reinterpret_cast<Destroy>(fn)(static_cast<CUgreenCtx>(green.g_dec));
    }
    green = Green{};
  }
  // run one call of the active lane on a partition stream (graph keys get a suffix:
  // a graph captured on a partition stream keeps running on that partition)
  struct StreamScope {
    Model &m;
    cudaStream_t prev;
    bool on;
    StreamScope(Model &mm, cudaStream_t s) : m(mm), prev(mm.mst), on(s != nullptr) {
      if (on) {
        m.mst = s;
        m.on_partition = true;
      }
    }
    ~StreamScope() {
      if (on) {
        m.mst = prev;
        m.on_partition = false;
      }
    }
  };

  // the action-expert lane's last denoise: make `caller` wait for it
  void join_alt(cudaStream_t caller) {
    OXY_CUDA(cudaStreamWaitEvent(caller, alt.ev_out, 0));
    denoise_pending = false;
  }
  float alt_elapsed_ms() {
    OXY_CUDA(cudaEventSynchronize(alt.t1));
    float ms = 0.f;
    OXY_CUDA(cudaEventElapsedTime(&ms, alt.t0, alt.t1));
    return ms;
  }
  void enter(cudaStream_t caller) {
    OXY_CUDA(cudaEventRecord(ev_in, caller));
    OXY_CUDA(cudaStreamWaitEvent(mst, ev_in, 0));
  }
  void leave(cudaStream_t caller) {
    OXY_CUDA(cudaEventRecord(ev_out, mst));
    OXY_CUDA(cudaStreamWaitEvent(caller, ev_out, 0));
  }
  template <typename T>
  T *arena_put(const T *src, size_t n) {
    const size_t off = (arena_used + 15) & ~static_cast<size_t>(15);
    const size_t bytes = n * sizeof(T);
    if (off + bytes > arena_cap) fail(OXY_EINVAL, "call too large for the planning arena (%zu bytes)", off + bytes);
    if (src) std::memcpy(arena_h.data() + off, src, bytes);
    else std::memset(arena_h.data() + off, 0, bytes);
    arena_used = off + bytes;
    return reinterpret_cast<T *>(arena_d + off);
  }
  void arena_upload() {
    if (arena_used)
      OXY_CUDA(cudaMemcpyAsync(arena_d, arena_h.data(), arena_used, cudaMemcpyHostToDevice, mst));
  }

  template <typename F>
  void run_body(const std::string &key, bool allow_graph, F &&body) {
    if (!use_graphs || !allow_graph) {
      body();
      return;
    }
    Graph &g = graphs[key];
    if (g.exec && g.gen == g_devbuf_reallocs) {
      OXY_CUDA(cudaGraphLaunch(g.exec, mst));
      __atomic_fetch_add(&g_launches, g.kernels, __ATOMIC_RELAXED);
      return;
    }
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    if (g.seen++ == 0) {
      body();
      return;
    }
    const unsigned long long gen0 = g_devbuf_reallocs;
    cudaGraph_t graph = nullptr;
    const unsigned long long k0 = g_launches;
    OXY_CUDA(cudaStreamBeginCapture(mst, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(mst, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    OXY_CUDA(cudaStreamEndCapture(mst, &graph));
    if (g_devbuf_reallocs != gen0) fail(OXY_ESTATE, "scratch reallocated during graph capture");
    OXY_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
    g.gen = g_devbuf_reallocs;
    g.kernels = g_launches - k0;  // counted once here for the launch just below
    OXY_CUDA(cudaGraphLaunch(g.exec, mst));
  }

  // SMs the GEMM / attention split policies may fill.  A/B knob OXY_LANE_SMS=dn,dec
  // caps the action-expert denoise and the language decode separately (0 = all),
  // so two concurrent chains can be sized to share the SMs instead of each
  // splitting for the whole GPU.
  int plan_sms = 0;
  int psms() const { return plan_sms > 0 ? std::min(plan_sms, sms) : sms; }
  std::pair<int, int> lane_sms = [] {
    std::pair<int, int> v{0, 0};
    if (const char *e = getenv("OXY_LANE_SMS")) sscanf(e, "%d,%d", &v.first, &v.second);
    return v;
  }();
  struct PlanSms {
    Model &m;
    int prev;
    PlanSms(Model &mm, int v) : m(mm), prev(mm.plan_sms) { m.plan_sms = v; }
    ~PlanSms() { m.plan_sms = prev; }
  };

  // Batch invariance: every projection's K partition comes from the phase policy
  // (gemm::policy_splits: a function of phase, N_out and K only), so a row's
  // result never depends on the token count of the call — the rows of a decode
  // batch, the streams of a batched prefill / denoise — nor on the lane's SM cap.
  int phase = gemm::PH_CHAIN;
  struct PhaseScope {
    Model &m;
    int prev;
    PhaseScope(Model &mm, int ph) : m(mm), prev(mm.phase) { m.phase = ph; }
    ~PhaseScope() { m.phase = prev; }
  };
  // Cluster split-K (gemm_sm100.cu) for the decode / denoise chains: the split
  // reduction (and a residual projection's RMSNorm) run inside the GEMM instead of
  // a reduce launch.  Bit-identical to the reduce kernels, so the choice may vary.
  // Off by default: measured slower in the chain (denoise 10.1 -> 17.1 ms per
  // frame; the in-kernel slice reduce + epilogue costs ~4.5 us of dependent L2
  // round trips after the cluster barrier, against ~2-3 us for the PDL-overlapped
  // reduce launch; profiles/r02_csk.md).  OXY_CSK=1 turns it on (A/B).
  bool use_csk = [] {
    const char *e = getenv("OXY_CSK");
    return e && atoi(e) != 0;
  }();
  gemm::Plan plan_for(int n_out, int k, int t) const {
    const int sp = gemm::policy_splits(phase, n_out, k, sms);
    gemm::Plan p = phase == gemm::PH_CHAIN ? gemm::make_chain_plan(n_out, k, t, psms(), sp)
                                           : gemm::make_prefill_plan(n_out, k, t, psms(), sp);
    p.csk = use_csk && !p.kmulti && phase == gemm::PH_CHAIN && p.cg == 0 && p.splits >= 2 &&
            p.splits <= gemm::CSK_MAX;
    return p;
  }
  // split-K workspace is reserved by plan_gemm(); gemm() only fetches it
  size_t ws_need = 0;
  void plan_gemm(int n_out, int k, int t) {
    if (t <= 0) return;
    gemm::Plan p = plan_for(n_out, k, t);
    if (p.splits > 1) ws_need = std::max(ws_need, (size_t)p.splits * t * n_out);
  }
  void gemm(const bf16 *w, const bf16 *xin, int n_out, int k, int t, int mode, void *out, int ldo,
            const float *bias = nullptr, const float *gate = nullptr) {
    if (t <= 0) return;
    gemm::Plan plan = plan_for(n_out, k, t);
    float *wsp = plan.splits > 1 ? ws.as<float>((size_t)plan.splits * t * n_out) : nullptr;
    EpiParams e{mode, out, ldo, bias, nullptr, 0, gate, {}};
    gemm::launch(w, xin, n_out, k, t, e, plan, wsp, gemm_counters, mst);
  }
  // residual projection (x += [gate *] W h) followed by the next RMSNorm/adaRMS (-> y).
  // Split-K: partials + one fused reduce/residual/norm kernel; else GEMM epilogue + norm.
  void gemm_res_norm(const bf16 *w, const bf16 *xin, int n_out, int k, int t, const float *gate, float *X, bf16 *Y,
                     const float *norm_w, const float *mod_scale, const float *mod_shift) {
    if (t <= 0) return;
    gemm::Plan plan = plan_for(n_out, k, t);
    if (plan.csk && n_out % 128 == 0 && n_out <= 2048) {
      // chain phase: residual add in the cluster split-K epilogue, then the row norm —
      // fused into the GEMM's last cluster for up to NORM_FUSE_MAX_T rows, else one
      // bit-identical row-norm launch (so a row's result never depends on the batch)
      float *wsp = ws.as<float>((size_t)plan.splits * t * n_out);
      gemm::NormFuse nf;
      nf.y = Y;
      nf.ldy = n_out;
      nf.w = norm_w;
      nf.ms = mod_scale;
      nf.mb = mod_shift;
      nf.eps = 1e-6f;
      const bool fuse = t <= gemm::NORM_FUSE_MAX_T;
      EpiParams e{gate ? gemm::EPI_ADD_GATED_F32 : gemm::EPI_ADD_F32, X, n_out, nullptr, nullptr, 0, gate, {}};
      if (fuse) e.norm = nf;
      gemm::launch(w, xin, n_out, k, t, e, plan, wsp, gemm_counters, mst);
      if (!fuse && !(dbg_skip & 128)) gemm::rownorm(X, n_out, t, n_out, nf, mst);
      return;
    }
    if (plan.splits > 1 && n_out <= 2048) {
      float *wsp = ws.as<float>((size_t)plan.splits * t * n_out);
      EpiParams e{gemm::EPI_PARTIALS, nullptr, 0, nullptr, nullptr, 0, nullptr, {}};
      gemm::launch(w, xin, n_out, k, t, e, plan, wsp, gemm_counters, mst);
      if (!(dbg_skip & 128))
        gemm::splitk_residual_norm(wsp, plan.partials(), t, n_out, gate, X, n_out, Y, n_out, norm_w, mod_scale,
                                   mod_shift, 1e-6f, mst);
      return;
    }
    gemm(w, xin, n_out, k, t, gate ? gemm::EPI_ADD_GATED_F32 : gemm::EPI_ADD_F32, X, n_out, nullptr, gate);
    rmsnorm(X, n_out, Y, n_out, norm_w, mod_scale, mod_shift, t, n_out, 1e-6f, mst);
  }
  // fused QKV projection + RoPE + K/V append (slot == null: dense k/v rows)
  void gemm_qkv(const bf16 *w, const bf16 *xin, int k, int t, const int *pos, const int *slot, bf16 *q_out,
                bf16 *k_dst, bf16 *v_dst) {
    if (t <= 0) return;
    gemm::Plan plan = plan_for(QKV, k, t);
    float *wsp = plan.splits > 1 ? ws.as<float>((size_t)plan.splits * t * QKV) : nullptr;
    EpiParams e{gemm::EPI_QKV_ROPE, nullptr, 0, nullptr, nullptr, 0, nullptr,
                gemm::QkvRope{rope_inv, rope_cs, pos, slot, q_out, k_dst, v_dst}};
    gemm::launch(w, xin, QKV, k, t, e, plan, wsp, gemm_counters, mst);
  }

  struct AttnPlan {
    AttnGroup *groups = nullptr;
    int n = 0, q_tiles = 0, splits = 1, hd = 256, rows = 0, max_tiles = 0, tps = 0;
  };
  size_t attn_ws_need = 0, attn_ml_need = 0;
  // pass 1: shapes only (reserve workspace); pass 2 (after scratch is final): upload descriptors
  AttnPlan shape_attention(std::vector<AttnGroup> &groups, int head_dim) {
    AttnPlan p;
    p.n = (int)groups.size();
    p.hd = head_dim;
    int max_nq = 0;
    for (auto &g : groups) {
      g.wrow0 = p.rows;
      p.rows += g.nq;
      max_nq = std::max(max_nq, g.nq);
      p.max_tiles = std::max(p.max_tiles, (g.nka + 63) / 64 + (g.nkb + 63) / 64);
    }
    p.q_tiles = (max_nq + 63) / 64;
    const int ctas = p.n * p.q_tiles;
    // SigLIP (head dim 72, 256 keys): one split, so an image's output never depends on
    // how many images share the call.  Head dim 256 here is only the OXY_ATTN_TC=0
    // A/B path (split-KV to fill the SMs; not batch-invariant).
    if (head_dim == 256 && ctas < sms && p.max_tiles > 1)
      p.splits = std::min({p.max_tiles, 32, std::max(1, (2 * sms) / ctas)});
    if (p.splits > 1) {
      const int hdp = head_dim == 256 ? 256 : 80;
      attn_ws_need = std::max(attn_ws_need, (size_t)p.splits * p.rows * hdp);
      attn_ml_need = std::max(attn_ml_need, (size_t)p.splits * p.rows * 2);
    }
    return p;
  }
  void attend(const AttnPlan &p, const bf16 *kp, const bf16 *vp) {
    if (!p.n) return;
    float *wo = nullptr, *wml = nullptr;
    if (p.splits > 1) {
      const int hdp = p.hd == 256 ? 256 : 80;
      wo = attn_ws.as<float>((size_t)p.splits * p.rows * hdp);
      wml = attn_ml.as<float>((size_t)p.splits * p.rows * 2);
    }
    flash_attention(p.groups, p.n, p.q_tiles, p.hd, kp, vp, 1.f / std::sqrt((float)p.hd), p.splits, p.max_tiles,
                    wo, wml, p.rows, mst);
  }
  // tcgen05 attention (attn_tc.cu) for head dim 256: OXY_ATTN_TC=0 falls back to the mma.sync kernel
  bool use_attn_tc = [] {
    const char *e = getenv("OXY_ATTN_TC");
    return !e || atoi(e) != 0;
  }();
  // SigLIP attention on tcgen05 (vit_attn_tc_kernel); OXY_VIT_TC=0: the mma.sync kernel (A/B)
  bool use_vit_tc = [] {
    const char *e = getenv("OXY_VIT_TC");
    return !e || atoi(e) != 0;
  }();
  // tps: key tiles (of 64) per split, per phase (batch invariance: a group's split
  // count is attn_group_splits(its key tiles, tps) whatever else shares the call)
  AttnPlan shape_attention_tc(std::vector<AttnGroup> &groups, int tps) {
    AttnPlan p;
    p.n = (int)groups.size();
    p.hd = HEAD_DIM;
    p.tps = tps;
    int max_nq = 0;
    for (auto &g : groups) {  // workspace rows padded to whole 128-row tiles (TMA-stored partials)
      g.wrow0 = p.rows;
      p.rows += (g.nq + 127) / 128 * 128;
      max_nq = std::max(max_nq, g.nq);
      const int tiles = (g.nka + 63) / 64 + (g.nkb + 63) / 64;
      int per;
      p.max_tiles = std::max(p.max_tiles, tiles);
      p.splits = std::max(p.splits, attn_group_splits(tiles, tps, per));
    }
    p.q_tiles = (max_nq + 127) / 128;
    if (p.splits > 1) {
      attn_ws_need = std::max(attn_ws_need, (size_t)p.splits * p.rows * 256);
      attn_ml_need = std::max(attn_ml_need, (size_t)p.splits * p.rows * 2);
    }
    return p;
  }
  // key tiles per split: prefill 7 (P = 800: 13 tiles -> 2 splits, 100 CTAs per layer at
  // 1 stream), expert suffix 2 (P + 50 = 850 keys: 7 two-tile splits merged over a
  // 7-CTA cluster).  A group's split count may not depend on how many streams share
  // the call (batch invariance), so one value serves every stream count: 2 tiles per
  // split costs 1 stream 0.07 ms per frame against 1 tile and saves 8 streams 3.5 ms
  // (profiles/r02/policy_ab.txt).  OXY_ATTN_TPS=prefill,denoise (A/B)
  std::pair<int, int> attn_tps = [] {
    std::pair<int, int> v{7, 2};
    if (const char *e = getenv("OXY_ATTN_TPS")) sscanf(e, "%d,%d", &v.first, &v.second);
    return v;
  }();
  void attend_tc(const AttnPlan &p, int layer, const bf16 *q_base, int q_rows, const bf16 *kd, const bf16 *vd,
                 int kd_rows, bool kv_ready) {
    if (!p.n) return;
    float *wo = nullptr, *wml = nullptr;
    if (p.splits > 1) {
      wo = attn_ws.as<float>((size_t)p.splits * p.rows * 256);
      wml = attn_ml.as<float>((size_t)p.splits * p.rows * 2);
    }
    // inside an SM partition (green context) only portable clusters (<= 8 CTAs) are sure
    // to be schedulable; larger split counts merge through the workspace (same arithmetic)
    const int cmax = on_partition ? std::min(8, attn_cluster_merge_max()) : attn_cluster_merge_max();
    const bool cm = p.splits > 1 && p.splits <= cmax;
    flash_attention_tc(p.groups, p.n, p.q_tiles, p.splits, p.tps, q_base, q_rows, kv_maps[2 * layer],
                       kv_maps[2 * layer + 1], kd, vd, kd_rows, 1.f / 16.f, wo, wml, p.rows, kv_ready, cm, mst,
                       psms());
    if (p.splits > 1 && !cm && !(dbg_skip & 4))
      flash_merge(p.groups, p.n, p.q_tiles * 128, p.splits, p.tps, reinterpret_cast<const bf16 *>(wo), wml, p.rows,
                  mst);
  }

  void reserve_common() {
    if (ws_need) ws.as<float>(ws_need);
    if (attn_ws_need) attn_ws.as<float>(attn_ws_need);
    if (attn_ml_need) attn_ml.as<float>(attn_ml_need);
    ws_need = attn_ws_need = attn_ml_need = 0;
  }

  // ------------------------------------------------------------ prefill
  // n_obs observations; obs i has n_img[i] images (in images_d order) and
  // n_txt[i] text tokens (concatenated in tokens_h); prefix = [images; text].
  // blocks_h: per obs ceil(P_i/64) block ids, concatenated.
  void prefill(cudaStream_t caller, int n_obs, const int *n_img, const int *n_txt, const int *tokens_h,
               const uint8_t *images_d, const int *blocks_h) {
    // K >= 2048 projections (Gemma qkv / o / down, ViT fc2) take 128-token tiles with
    // split-K 2 (gemm::policy_splits): half the weight re-reads through L2, both CTA
    // slots busy, and the o / down residual + RMSNorm fused into the split reduce;
    // 1024 <= K < 2048 (the ViT qkv / o / fc1) take 96-token tiles (OXY_PREFILL_DEEPK=0:
    // off; OXY_PREFILL_MIDK=kmin,bn,splits A/B).  Token tiles never change results.
    struct BandScope {
      explicit BandScope(bool deepk) {
        if (deepk) {
          const int band[6] = {2048, 128, 2, 1024, 96, 1};
          for (int i = 0; i < 6; ++i) gemm::g_deepk[i] = band[i];
        }
        if (const char *e = getenv("OXY_PREFILL_MIDK"))
          sscanf(e, "%d,%d,%d", &gemm::g_deepk[3], &gemm::g_deepk[4], &gemm::g_deepk[5]);
      }
      ~BandScope() {
        for (int &v : gemm::g_deepk) v = 0;
      }
    } band_scope(prefill_deepk);
    PhaseScope phase_scope(*this, gemm::PH_PREFILL);
    const int W = c.width, Dv = c.vit_width, nh = c.vit_heads, hd = nh ? Dv / nh : 72;
    std::vector<int> P(n_obs), off(n_obs), boff(n_obs);
    int T = 0, nb = 0, n_images = 0, n_tok = 0;
    std::string key = "prefill";
    for (int i = 0; i < n_obs; ++i) {
      OXY_REQUIRE(n_img[i] >= 0 && n_txt[i] >= 0, "negative prefix part");
      OXY_REQUIRE(n_img[i] == 0 || c.vit_depth > 0, "this model has no vision tower");
      P[i] = n_img[i] * 256 + n_txt[i];
      OXY_REQUIRE(P[i] >= 1, "observation needs at least one token");
      off[i] = T;
      boff[i] = nb;
      T += P[i];
      nb += (P[i] + KV_BLOCK - 1) / KV_BLOCK;
      n_images += n_img[i];
      n_tok += n_txt[i];
      key += "/" + std::to_string(n_img[i]) + "," + std::to_string(n_txt[i]);
    }
    for (int i = 0; i < n_tok; ++i)
      OXY_REQUIRE(tokens_h[i] >= 0 && tokens_h[i] < c.vocab, "observation token %d outside vocab of %d",
                  tokens_h[i], c.vocab);
    check_block_ids(blocks_h, nb, NB, "prefill");
    const int Tv = n_images * 256;
    // ---- plan pass 1: reserve scratch
    x.as<float>((size_t)T * W);
    y.as<bf16>((size_t)T * W);
    qkv.as<float>((size_t)T * QKV);
    q.as<bf16>((size_t)T * QDIM);
    o.as<bf16>((size_t)T * QDIM);
    hmid.as<bf16>((size_t)T * c.mlp);
    arena_used = 0;
    plan_gemm(QKV, W, T);
    plan_gemm(W, QDIM, T);
    plan_gemm(2 * c.mlp, W, T);
    plan_gemm(W, c.mlp, T);
    std::vector<AttnGroup> g_llm(n_obs), g_vit;
    for (int i = 0; i < n_obs; ++i) {
      g_llm[i] = AttnGroup{};
      g_llm[i].nq = P[i] * Q_HEADS;
      g_llm[i].nka = P[i];
    }
    AttnPlan a_llm = use_attn_tc ? shape_attention_tc(g_llm, attn_tps.first) : shape_attention(g_llm, HEAD_DIM), a_vit;
    if (Tv) {
      patches.as<bf16>((size_t)Tv * PATCH_K);
      vit_h.as<float>((size_t)Tv * Dv);
      vit_y.as<bf16>((size_t)Tv * Dv);
      vit_qkv.as<bf16>((size_t)Tv * 3 * Dv);
      vit_o.as<bf16>((size_t)Tv * Dv);
      vit_m.as<bf16>((size_t)Tv * c.vit_mlp);
      plan_gemm(Dv, PATCH_K, Tv);
      plan_gemm(3 * Dv, Dv, Tv);
      plan_gemm(Dv, Dv, Tv);
      plan_gemm(c.vit_mlp, Dv, Tv);
      plan_gemm(Dv, c.vit_mlp, Tv);
      for (int i = 0; i < n_obs; ++i) plan_gemm(W, Dv, n_img[i] * 256);
      g_vit.resize((size_t)n_images * nh);
      for (auto &g : g_vit) {
        g = AttnGroup{};
        g.nq = 256;
        g.nkb = 256;
      }
      a_vit = shape_attention(g_vit, hd);
    }
    reserve_common();
    // ---- plan pass 2: pointers are final; build the arena
    float *X = x.as<float>(0);
    bf16 *Y = y.as<bf16>(0), *Qb = q.as<bf16>(0), *Ob = o.as<bf16>(0), *Hm = hmid.as<bf16>(0);
    float *QKVf = qkv.as<float>(0);
    std::vector<int> tok(T), pos(T), slot(T);
    int ti = 0;
    for (int i = 0; i < n_obs; ++i)
      for (int p = 0; p < P[i]; ++p) {
        const int r = off[i] + p;
        tok[r] = p < n_img[i] * 256 ? 0 : tokens_h[ti++];
        pos[r] = p;
        slot[r] = blocks_h[boff[i] + p / KV_BLOCK] * KV_BLOCK + p % KV_BLOCK;
      }
    int *d_tok = arena_put(tok.data(), T), *d_pos = arena_put(pos.data(), T), *d_slot = arena_put(slot.data(), T);
    int *d_bt = arena_put(blocks_h, nb);
    for (int i = 0; i < n_obs; ++i) {
      AttnGroup &g = g_llm[i];
      g.q = Qb + (size_t)off[i] * QDIM;
      g.ldq = HEAD_DIM;
      g.o = Ob + (size_t)off[i] * QDIM;
      g.ldo = HEAD_DIM;
      g.bt = d_bt + boff[i];
    }
    a_llm.groups = arena_put(g_llm.data(), g_llm.size());
    bf16 *pt = nullptr, *yv = nullptr, *qkvv = nullptr, *ov = nullptr, *mv = nullptr;
    float *hv = nullptr;
    if (Tv) {
      pt = patches.as<bf16>(0);
      hv = vit_h.as<float>(0);
      yv = vit_y.as<bf16>(0);
      qkvv = vit_qkv.as<bf16>(0);
      ov = vit_o.as<bf16>(0);
      mv = vit_m.as<bf16>(0);
      for (int im = 0, gi = 0; im < n_images; ++im)
        for (int hh = 0; hh < nh; ++hh, ++gi) {
          AttnGroup &g = g_vit[gi];
          g.q = qkvv + (size_t)im * 256 * 3 * Dv + hh * hd;
          g.ldq = 3 * Dv;
          g.o = ov + (size_t)im * 256 * Dv + hh * hd;
          g.ldo = Dv;
          g.kb = g.q + Dv;
          g.vb = g.q + 2 * Dv;
          g.ldkv = 3 * Dv;
        }
      a_vit.groups = arena_put(g_vit.data(), g_vit.size());
    }
    if (pipe_prefill) {
      pf_events();
      OXY_CUDA(cudaEventRecord(pf_start, caller));
      pf_blocks.assign(blocks_h, blocks_h + nb);
    }
    enter(caller);
    arena_upload();
    if (Tv) patchify(images_d, n_images, pt, PATCH_K, mst);  // caller's buffer: outside the graph
    auto body = [&]() {
      for (int i = 0; i < n_obs; ++i) {
        const int r0 = off[i] + n_img[i] * 256;
        embed_rows(X + (size_t)r0 * W, W, embed, d_tok + r0, nullptr, n_txt[i], W, std::sqrt((float)W), mst);
      }
      if (Tv) {
        tile_rows(hv, Dv, vpos, Dv, Tv, 256, Dv, mst);
        gemm(vpatch, pt, Dv, PATCH_K, Tv, gemm::EPI_ADD_F32, hv, Dv, vpatch_b);
        for (int l = 0; l < c.vit_depth; ++l) {
          const VitW &w = V[l];
          layernorm(hv, Dv, yv, Dv, w.ln1w, w.ln1b, Tv, Dv, 1e-6f, mst);
          gemm(w.wqkv, yv, 3 * Dv, Dv, Tv, gemm::EPI_BF16, qkvv, 3 * Dv, w.bqkv);
          if (use_vit_tc) vit_attention_tc(qkvv, ov, n_images, nh, mst);
          else attend(a_vit, nullptr, nullptr);
          gemm(w.wo, ov, Dv, Dv, Tv, gemm::EPI_ADD_F32, hv, Dv, w.bo);
          layernorm(hv, Dv, yv, Dv, w.ln2w, w.ln2b, Tv, Dv, 1e-6f, mst);
          gemm(w.w1, yv, c.vit_mlp, Dv, Tv, gemm::EPI_GELU_BF16, mv, c.vit_mlp, w.b1);
          gemm(w.w2, mv, Dv, c.vit_mlp, Tv, gemm::EPI_ADD_F32, hv, Dv, w.b2);
        }
        layernorm(hv, Dv, yv, Dv, vln_w, vln_b, Tv, Dv, 1e-6f, mst);
        for (int i = 0, img0 = 0; i < n_obs; img0 += n_img[i], ++i)
          if (n_img[i] > 0)
            gemm(vproj, yv + (size_t)img0 * 256 * Dv, W, Dv, n_img[i] * 256, gemm::EPI_F32,
                 X + (size_t)off[i] * W, W, vproj_b);
      }
      // residual projections go through gemm_res_norm: with the prefill's split-K
      // plans the split reduce, the residual add and the next RMSNorm are one kernel
      rmsnorm(X, W, Y, W, L[0].ln1, nullptr, nullptr, T, W, 1e-6f, mst);
      for (int l = 0; l < c.depth; ++l) {
        const LayerW &w = L[l];
        gemm_qkv(w.wqkv, Y, W, T, d_pos, d_slot, Qb, kpool(l), vpool(l));
        if (pipe_prefill) OXY_CUDA(cudaEventRecordWithFlags(pf_layer[l], mst, capture_flag(cudaEventRecordExternal)));
        if (l == c.depth - 1) break;  // the last block's output is not cached
        if (use_attn_tc) attend_tc(a_llm, l, Qb, T * Q_HEADS, nullptr, nullptr, 0, false);
        else attend(a_llm, kpool(l), vpool(l));
        gemm_res_norm(w.wo, Ob, W, QDIM, T, nullptr, X, Y, w.ln2, nullptr, nullptr);
        gemm(w.wgu, Y, 2 * c.mlp, W, T, gemm::EPI_GEGLU_BF16, Hm, c.mlp);
        gemm_res_norm(w.wd, Hm, W, c.mlp, T, nullptr, X, Y, L[l + 1].ln1, nullptr, nullptr);
      }
    };
    run_body(key, true, body);
    leave(caller);
  }

  // ------------------------------------------------------------ action expert
  void ensure_mod(int S) {
    if (mod_S == S) return;
    const int We = c.expert_width;
    // time embedding of t_s = 1 - s/S (openpi posemb_sincos: periods 4e-3 .. 4)
    std::vector<float> temb((size_t)S * We);
    const int half = We / 2;
    for (int s = 0; s < S; ++s) {
      const double t = 1.0 - (double)s / S;
      for (int i = 0; i < half; ++i) {
        const double frac = half > 1 ? (double)i / (half - 1) : 0.0;
        const double period = 4e-3 * std::pow(4.0 / 4e-3, frac);
        const double ang = t / period * 2.0 * M_PI;
        temb[(size_t)s * We + i] = (float)std::sin(ang);
        temb[(size_t)s * We + half + i] = (float)std::cos(ang);
      }
    }
    plan_gemm(We, We, S);
    plan_gemm(n_mod, We, S);
    reserve_common();
    float *tf = xe.as<float>((size_t)S * We * 2);
    bf16 *tb = act_bf.as<bf16>((size_t)S * We * 3);
    float *m = mod.as<float>((size_t)S * n_mod);
    bf16 *h1 = tb + (size_t)S * We, *h2 = h1 + (size_t)S * We;
    OXY_CUDA(cudaMemcpyAsync(tf, temb.data(), temb.size() * sizeof(float), cudaMemcpyHostToDevice, mst));
    f32_to_bf16(tf, tb, (int64_t)S * We, mst);
    gemm(t1, tb, We, We, S, gemm::EPI_SWISH_BF16, h1, We, t1_b);
    gemm(t2, h1, We, We, S, gemm::EPI_SWISH_BF16, h2, We, t2_b);
    gemm(wmod, h2, n_mod, We, S, gemm::EPI_F32, m, n_mod, bmod);
    OXY_CUDA(cudaStreamSynchronize(mst));
    mod_S = S;
  }

  // n streams; stream i's prefix has P[i] positions in blocks (concatenated).
  // Runs on the action-expert lane.  join = false leaves the caller stream
  // free (decode may be enqueued behind it and overlap); join_alt() syncs.
  void denoise(cudaStream_t caller, int n, const int *P, const int *blocks_h, int S, float *actions_out_d,
               bool join = true) {
    OXY_REQUIRE(S >= 1, "denoise step count must be >= 1, got %d", S);
    LaneSwap lane(*this);
    static const bool force_part = getenv("OXY_GREEN_FORCE") && atoi(getenv("OXY_GREEN_FORCE")) != 0;  // measurement
    const bool part = (!join || force_part) && green.dn && n <= green_max_streams;  // overlapped: expert partition
    PlanSms plan_scope(*this, part ? green.dn_sms : lane_sms.first);
    const int We = c.expert_width, H = c.H, A = c.action_dim, T = n * H, AP = apad();
    ensure_mod(S);
    StreamScope stream_scope(*this, part ? green.dn : nullptr);
    std::string key = std::string(part ? "denoise-g/" : "denoise/") + std::to_string(S);
    int nb = 0;
    for (int i = 0; i < n; ++i) {
      OXY_REQUIRE(P[i] >= 1, "denoise needs a non-empty prefix");
      nb += (P[i] + KV_BLOCK - 1) / KV_BLOCK;
      key += "," + std::to_string(P[i]);
    }
    check_block_ids(blocks_h, nb, NB, "denoise");
    // multi-stream overlapped frames (all SMs, no partition) pipeline their first step
    // too: 8 streams 51.1-51.4 -> 50.6-51.0 ms/frame (profiles/r02/ms_pipe_ab.txt;
    // OXY_PIPE_ALL=0: partitioned frames only)
    static const bool pipe_all = !getenv("OXY_PIPE_ALL") || atoi(getenv("OXY_PIPE_ALL")) != 0;
    const bool pipe = pipe_prefill && (part || pipe_all) && !join && (int)pf_blocks.size() == nb &&
                      std::equal(pf_blocks.begin(), pf_blocks.end(), blocks_h);
    pf_blocks.clear();
    if (pipe) key += "/pipe";
    // ---- plan pass 1
    arena_used = 0;
    act.as<float>((size_t)T * AP);
    act_bf.as<bf16>((size_t)T * AP);
    xe.as<float>((size_t)T * We);
    y.as<bf16>((size_t)T * std::max(We, QDIM));
    q.as<bf16>((size_t)T * QDIM);
    o.as<bf16>((size_t)T * QDIM);
    kd.as<bf16>((size_t)T * HEAD_DIM);
    vd.as<bf16>((size_t)T * HEAD_DIM);
    hmid.as<bf16>((size_t)T * c.expert_mlp);
    vel.as<float>((size_t)T * AP);
    plan_gemm(We, AP, T);
    plan_gemm(QKV, We, T);
    plan_gemm(We, QDIM, T);
    plan_gemm(2 * c.expert_mlp, We, T);
    plan_gemm(We, c.expert_mlp, T);
    plan_gemm(A, We, T);
    std::vector<AttnGroup> groups(n);
    for (int i = 0; i < n; ++i) {
      groups[i] = AttnGroup{};
      groups[i].nq = H * Q_HEADS;
      groups[i].nka = P[i];
      groups[i].nkb = H;
    }
    AttnPlan ap = use_attn_tc ? shape_attention_tc(groups, attn_tps.second) : shape_attention(groups, HEAD_DIM);
    reserve_common();
    // ---- plan pass 2
    float *a = act.as<float>(0), *X = xe.as<float>(0), *vel_d = vel.as<float>(0);
    bf16 *ab = act_bf.as<bf16>(0), *Y = y.as<bf16>(0), *Qb = q.as<bf16>(0), *Ob = o.as<bf16>(0),
         *Kd = kd.as<bf16>(0), *Vd = vd.as<bf16>(0), *Hm = hmid.as<bf16>(0);
    const float *modp = mod.as<float>(0);
    std::vector<int> pos(T);
    std::vector<int> boff(n);
    for (int i = 0, b = 0; i < n; ++i) {
      boff[i] = b;
      b += (P[i] + KV_BLOCK - 1) / KV_BLOCK;
      for (int j = 0; j < H; ++j) pos[i * H + j] = P[i] + j;
    }
    int *d_pos = arena_put(pos.data(), T);
    int *d_bt = arena_put(blocks_h, nb);
    for (int i = 0; i < n; ++i) {
      AttnGroup &g = groups[i];
      g.q = Qb + (size_t)i * H * QDIM;
      g.ldq = HEAD_DIM;
      g.o = Ob + (size_t)i * H * QDIM;
      g.ldo = HEAD_DIM;
      g.bt = d_bt + boff[i];
      g.kb = Kd + (size_t)i * H * HEAD_DIM;
      g.vb = Vd + (size_t)i * H * HEAD_DIM;
      g.ldkv = HEAD_DIM;
    }
    ap.groups = arena_put(groups.data(), groups.size());
    if (pipe) OXY_CUDA(cudaStreamWaitEvent(mst, pf_start, 0));  // + per-layer waits in step 0
    else enter(caller);
    OXY_CUDA(cudaEventRecord(alt.t0, mst));
    arena_upload();
    auto body = [&]() {
      for (int i = 0; i < n; ++i)
        OXY_CUDA(cudaMemcpyAsync(a + (size_t)i * H * AP, noise, (size_t)H * AP * sizeof(float),
                                 cudaMemcpyDeviceToDevice, mst));
      OXY_CUDA(cudaMemsetAsync(vel_d, 0, (size_t)T * AP * sizeof(float), mst));
      f32_to_bf16(a, ab, (int64_t)T * AP, mst);
      const float dt = -1.f / (float)S;
      for (int s = 0; s < S; ++s) {
        const float *ms = modp + (size_t)s * n_mod;
        gemm(e_in, ab, We, AP, T, gemm::EPI_F32, X, We, e_in_b);
        rmsnorm(X, We, Y, We, nullptr, ms, ms + We, T, We, 1e-6f, mst);
        const float *mf = ms + (size_t)c.depth * 6 * We;
        for (int l = 0; l < c.depth; ++l) {
          const ExpertW &w = E[l];
          const float *m = ms + (size_t)l * 6 * We;
          const float *mn = l + 1 < c.depth ? m + 6 * We : mf;  // the norm that follows this layer
          if (!(dbg_skip & 1)) gemm_qkv(w.wqkv, Y, We, T, d_pos, nullptr, Qb, Kd, Vd);
          if (pipe && s == 0) OXY_CUDA(cudaStreamWaitEvent(mst, pf_layer[l], capture_flag(cudaEventWaitExternal)));
          if (!(dbg_skip & 2)) {
            if (use_attn_tc) attend_tc(ap, l, Qb, T * Q_HEADS, Kd, Vd, T, true);
            else attend(ap, kpool(l), vpool(l));
          }
          if (!(dbg_skip & 8)) gemm_res_norm(w.wo, Ob, We, QDIM, T, m + 2 * We, X, Y, nullptr, m + 3 * We, m + 4 * We);
          if (!(dbg_skip & 16)) gemm(w.wgu, Y, 2 * c.expert_mlp, We, T, gemm::EPI_GEGLU_BF16, Hm, c.expert_mlp);
          if (!(dbg_skip & 32))
            gemm_res_norm(w.wd, Hm, We, c.expert_mlp, T, m + 5 * We, X, Y, nullptr, mn, mn + We);
        }
        gemm(e_out, Y, A, We, T, gemm::EPI_F32, vel_d, AP, e_out_b);
        euler_step(a, vel_d, ab, (int64_t)T * AP, dt, mst);
      }
    };
    run_body(key, true, body);
    OXY_CUDA(cudaMemcpy2DAsync(actions_out_d, A * sizeof(float), a, AP * sizeof(float), A * sizeof(float), T,
                               cudaMemcpyDeviceToDevice, mst));
    OXY_CUDA(cudaEventRecord(alt.t1, mst));
    if (join) leave(caller);
    else OXY_CUDA(cudaEventRecord(ev_out, mst));
    denoise_pending = part;
  }

  // ------------------------------------------------------------ no-cache recompute
  // recompute_logits (kvweaver/backend.py:301-304): logits of the last of T tokens
  // from one dense forward over the whole sequence — prefix [0, P) bidirectional,
  // positions >= P causal — through the prefill GEMM plans and a plain fp32
  // attention kernel; no pool, no block tables, no decode kernels.  The oracle
  // route suite_reference compares cached decode against.
  void recompute(cudaStream_t caller, const int *tok_h, int T, int P, float *logits_h) {
    OXY_REQUIRE(T >= 1 && P >= 0 && P <= T, "recompute needs T >= 1 and 0 <= P <= T");
    for (int i = 0; i < T; ++i)
      OXY_REQUIRE(tok_h[i] >= 0 && tok_h[i] < c.vocab, "token %d outside vocab of %d", tok_h[i], c.vocab);
    PhaseScope phase_scope(*this, gemm::PH_PREFILL);
    const int W = c.width;
    arena_used = 0;
    x.as<float>((size_t)T * W);
    y.as<bf16>((size_t)T * W);
    q.as<bf16>((size_t)T * QDIM);
    o.as<bf16>((size_t)T * QDIM);
    kd.as<bf16>((size_t)T * HEAD_DIM);
    vd.as<bf16>((size_t)T * HEAD_DIM);
    hmid.as<bf16>((size_t)T * c.mlp);
    logits.as<float>((size_t)c.vocab);
    plan_gemm(QKV, W, T);
    plan_gemm(W, QDIM, T);
    plan_gemm(2 * c.mlp, W, T);
    plan_gemm(W, c.mlp, T);
    plan_gemm(c.vocab, W, 1);
    reserve_common();
    float *X = x.as<float>(0), *LG = logits.as<float>(0);
    bf16 *Y = y.as<bf16>(0), *Qb = q.as<bf16>(0), *Ob = o.as<bf16>(0), *Kd = kd.as<bf16>(0), *Vd = vd.as<bf16>(0),
         *Hm = hmid.as<bf16>(0);
    std::vector<int> pos(T);
    for (int i = 0; i < T; ++i) pos[i] = i;
    int *d_tok = arena_put(tok_h, T), *d_pos = arena_put(pos.data(), T);
    enter(caller);
    arena_upload();
    embed_rows(X, W, embed, d_tok, nullptr, T, W, std::sqrt((float)W), mst);
    rmsnorm(X, W, Y, W, L[0].ln1, nullptr, nullptr, T, W, 1e-6f, mst);
    for (int l = 0; l < c.depth; ++l) {
      const LayerW &w = L[l];
      const float *next_norm = l + 1 < c.depth ? L[l + 1].ln1 : final_norm;
      gemm_qkv(w.wqkv, Y, W, T, d_pos, nullptr, Qb, Kd, Vd);
      prefix_lm_attention_ref(Qb, Kd, Vd, Ob, T, P, 1.f / 16.f, mst);
      gemm_res_norm(w.wo, Ob, W, QDIM, T, nullptr, X, Y, w.ln2, nullptr, nullptr);
      gemm(w.wgu, Y, 2 * c.mlp, W, T, gemm::EPI_GEGLU_BF16, Hm, c.mlp);
      gemm_res_norm(w.wd, Hm, W, c.mlp, T, nullptr, X, Y, next_norm, nullptr, nullptr);
    }
    gemm(lm_head, Y + (size_t)(T - 1) * W, c.vocab, W, 1, gemm::EPI_F32, LG, c.vocab);
    OXY_CUDA(cudaMemcpyAsync(logits_h, LG, (size_t)c.vocab * sizeof(float), cudaMemcpyDeviceToHost, mst));
    OXY_CUDA(cudaStreamSynchronize(mst));
    leave(caller);
  }

  // ------------------------------------------------------------ decode
  // A/B: OXY_DECODE_EARLY=0 turns off early PDL for the decode lane's skinny
  // GEMMs (their waiting CTAs then do not hold SMs the concurrent denoise needs)
  bool prefill_deepk = [] {
    const char *e = getenv("OXY_PREFILL_DEEPK");
    return !e || atoi(e) != 0;
  }();
  // OXY_FUSED_ARGMAX=0: materialise the logits and argmax them in two kernels (A/B)
  bool fused_argmax = [] {
    const char *e = getenv("OXY_FUSED_ARGMAX");
    return !e || atoi(e) != 0;
  }();
  int decode_early = [] {
    const char *e = getenv("OXY_DECODE_EARLY");
    return e ? atoi(e) : -1;
  }();
  void decode(cudaStream_t caller, int rows, int k, const int *bt_h, int maxb, const int *seq_h, const int *last_h,
              const int *budget_h, const int *cow_h, int *out_tok_h, int *out_cnt_h, float *logits_h) {
    struct EarlyScope {
      explicit EarlyScope(int v) { gemm::g_early_override = v; }
      ~EarlyScope() { gemm::g_early_override = -1; }
    } early_scope(decode_early);
    static const bool force_part = getenv("OXY_GREEN_FORCE") && atoi(getenv("OXY_GREEN_FORCE")) != 0;  // measurement
    const bool part = green.dec && (denoise_pending || force_part);  // overlapping the expert: decode partition
    PlanSms plan_scope(*this, part ? green.dec_sms : lane_sms.second);
    StreamScope stream_scope(*this, part ? green.dec : nullptr);
    const int W = c.width;
    // a row appends at most min(k, budget) positions (argmax_update stops it at its
    // budget), so its table only has to cover seq + min(k, budget)
    int max_pos = 0;
    for (int r = 0; r < rows; ++r) {
      OXY_REQUIRE(last_h[r] >= 0 && last_h[r] < c.vocab, "token %d outside vocab", last_h[r]);
      OXY_REQUIRE(seq_h[r] >= 1 && budget_h[r] >= 1, "row %d: seq_len and budget must be >= 1", r);
      max_pos = std::max(max_pos, seq_h[r] + std::min(k, budget_h[r]));
    }
    OXY_REQUIRE(maxb >= 1 && (max_pos + KV_BLOCK - 1) / KV_BLOCK <= maxb, "block table too short for %d positions",
                max_pos);
    check_block_ids(bt_h, (int64_t)rows * maxb, NB, "decode");
    check_cow(cow_h, rows, NB, KV_BLOCK);
    // ---- plan pass 1
    arena_used = 0;
    x.as<float>((size_t)rows * W);
    y.as<bf16>((size_t)rows * W);
    qkv.as<float>((size_t)rows * QKV);
    q.as<bf16>((size_t)rows * QDIM);
    o.as<bf16>((size_t)rows * QDIM);
    hmid.as<bf16>((size_t)rows * c.mlp);
    logits.as<float>((size_t)rows * c.vocab);
    const int head_tiles = (c.vocab + gemm::BM - 1) / gemm::BM;
    amv.as<float>((size_t)rows * std::max(64, head_tiles));
    ami.as<int>((size_t)rows * std::max(64, head_tiles));
    dec_ws.as<float>((size_t)rows * maxb * Q_HEADS * (HEAD_DIM + 2));
    plan_gemm(QKV, W, rows);
    plan_gemm(W, QDIM, rows);
    plan_gemm(2 * c.mlp, W, rows);
    plan_gemm(W, c.mlp, rows);
    plan_gemm(c.vocab, W, rows);
    reserve_common();
    // ---- plan pass 2
    float *X = x.as<float>(0), *QKVf = qkv.as<float>(0), *LG = logits.as<float>(0), *pv = amv.as<float>(0),
          *dws = dec_ws.as<float>(0);
    bf16 *Y = y.as<bf16>(0), *Qb = q.as<bf16>(0), *Ob = o.as<bf16>(0), *Hm = hmid.as<bf16>(0);
    int *pi = ami.as<int>(0);
    std::vector<int> ones(rows, 1), zeros((size_t)rows * k, 0);
    int *d_bt = arena_put(bt_h, (size_t)rows * maxb);
    int *d_cow = arena_put(cow_h, (size_t)rows * 3);
    int *d_active = arena_put(ones.data(), rows);
    int *d_tok = arena_put(last_h, rows);
    int *d_pos = arena_put(seq_h, rows);
    int *d_cnt = arena_put(zeros.data(), rows);
    int *d_bud = arena_put(budget_h, rows);
    int *d_slot = arena_put(zeros.data(), rows);
    int *d_out = arena_put(zeros.data(), (size_t)rows * k);
    const float scale = 1.f / 16.f;  // 1/sqrt(256)
    // the argmax epilogue needs the unsplit one-tile-per-CTA LM-head plan (always the
    // case for decode rows <= 64); logits requested -> the materialising path
    const gemm::Plan head_plan = plan_for(c.vocab, W, rows);
    const bool fused_head = fused_argmax && !logits_h && head_plan.cg == 0 && head_plan.splits == 1;
    enter(caller);
    arena_upload();
    auto body = [&]() {
      cow_blocks(pool, d_cow, rows, c.depth, layer_stride, kv_stride, mst);
      for (int s = 0; s < k; ++s) {
        embed_rows(X, W, embed, d_tok, nullptr, rows, W, std::sqrt((float)W), mst);
        next_slots(d_slot, d_pos, d_active, d_bt, maxb, rows, mst);
        rmsnorm(X, W, Y, W, L[0].ln1, nullptr, nullptr, rows, W, 1e-6f, mst);
        for (int l = 0; l < c.depth; ++l) {
          const LayerW &w = L[l];
          const float *next_norm = l + 1 < c.depth ? L[l + 1].ln1 : final_norm;
          if (!(dbg_skip & 256)) gemm_qkv(w.wqkv, Y, W, rows, d_pos, d_slot, Qb, kpool(l), vpool(l));
          if (!(dbg_skip & 512))
            decode_attention_v3(kv_maps[2 * l], kv_maps[2 * l + 1], Qb, Ob, d_bt, maxb, d_pos, d_active, rows, maxb,
                                scale, dws, psms(), mst);
          if (!(dbg_skip & 2048)) gemm_res_norm(w.wo, Ob, W, QDIM, rows, nullptr, X, Y, w.ln2, nullptr, nullptr);
          if (!(dbg_skip & 4096)) gemm(w.wgu, Y, 2 * c.mlp, W, rows, gemm::EPI_GEGLU_BF16, Hm, c.mlp);
          if (!(dbg_skip & 8192)) gemm_res_norm(w.wd, Hm, W, c.mlp, rows, nullptr, X, Y, next_norm, nullptr, nullptr);
        }
        if (fused_head) {
          // greedy LM head: per-(row, weight tile) (max, id) straight from the
          // accumulators, no logits in HBM
          const gemm::Plan hp = plan_for(c.vocab, W, rows);
          EpiParams e{gemm::EPI_ARGMAX, pv, head_tiles, nullptr, nullptr, 0, nullptr, {}};
          e.amax_idx = pi;
          if (!(dbg_skip & 16384)) gemm::launch(lm_head, Y, c.vocab, W, rows, e, hp, nullptr, gemm_counters, mst);
          argmax_tiles_update(rows, head_tiles, pv, pi, s, k, c.eos_token, d_active, d_tok, d_pos, d_cnt, d_bud,
                              d_out, mst);
          continue;
        }
        if (!(dbg_skip & 16384)) gemm(lm_head, Y, c.vocab, W, rows, gemm::EPI_F32, LG, c.vocab);
        if (logits_h)
          OXY_CUDA(cudaMemcpyAsync(logits_h + (size_t)s * rows * c.vocab, LG, (size_t)rows * c.vocab * sizeof(float),
                                   cudaMemcpyDeviceToHost, mst));
        argmax_update(LG, rows, c.vocab, s, k, c.eos_token, d_active, d_tok, d_pos, d_cnt, d_bud, d_out, pv, pi,
                      mst);
      }
    };
    const std::string key = std::string(part ? "decode-g/" : "decode/") + std::to_string(rows) + "," +
                            std::to_string(k) + "," + std::to_string(maxb);
    run_body(key, logits_h == nullptr, body);
    OXY_CUDA(cudaMemcpyAsync(out_tok_h, d_out, (size_t)rows * k * sizeof(int), cudaMemcpyDeviceToHost, mst));
    OXY_CUDA(cudaMemcpyAsync(out_cnt_h, d_cnt, rows * sizeof(int), cudaMemcpyDeviceToHost, mst));
    OXY_CUDA(cudaStreamSynchronize(mst));
    leave(caller);
  }
};

__global__ void gather_kv_f32(float *kout, float *vout, const bf16 *kp, const bf16 *vp, const int *blocks,
                              int seq_len) {
  const int t = blockIdx.x;
  const size_t s = (size_t)blocks[t / KV_BLOCK] * KV_BLOCK + t % KV_BLOCK;
  for (int j = threadIdx.x; j < HEAD_DIM; j += blockDim.x) {
    kout[(size_t)t * HEAD_DIM + j] = __bfloat162float(kp[s * HEAD_DIM + j]);
    vout[(size_t)t * HEAD_DIM + j] = __bfloat162float(vp[s * HEAD_DIM + j]);
  }
}

}  // namespace pi05
}  // namespace oxy

struct oxy_pi05 {
  oxy::pi05::Model m;
};

extern "C" {

int oxy_pi05_create(const oxy_pi05_config *cfg, int32_t num_blocks, void *stream, oxy_pi05 **out) {
  OXY_API_BEGIN
  OXY_REQUIRE(cfg && cfg->width % 64 == 0 && cfg->expert_width % 64 == 0 && cfg->mlp % 64 == 0 &&
                  cfg->expert_mlp % 64 == 0 && cfg->depth >= 1 && cfg->vocab >= 2,
              "invalid pi05 config (widths must be multiples of 64)");
  OXY_REQUIRE(cfg->vit_depth == 0 || (cfg->vit_heads > 0 && cfg->vit_width == 72 * cfg->vit_heads &&
                                      cfg->vit_mlp % 8 == 0),
              "vision tower needs head dim 72 and vit_mlp % 8 == 0");
  OXY_REQUIRE(cfg->eos_token >= 0 && cfg->eos_token < cfg->vocab, "eos outside vocab");
  OXY_REQUIRE(num_blocks > 0, "pool needs blocks");
  auto *p = new oxy_pi05;
  try {
    p->m.create(*cfg, num_blocks, oxy::as_stream(stream));
    OXY_CUDA(cudaStreamSynchronize(oxy::as_stream(stream)));
  } catch (...) {
    delete p;
    throw;
  }
  *out = p;
  OXY_API_END
}

int oxy_pi05_destroy(oxy_pi05 *p) {
  delete p;
  return OXY_OK;
}

int oxy_pi05_num_tensors(oxy_pi05 *p, int32_t *n) {
  *n = (int32_t)p->m.tensors.size();
  return OXY_OK;
}

int oxy_pi05_tensor_info(oxy_pi05 *p, int32_t i, char *name64, int64_t *shape2, int32_t *dtype,
                         uint64_t *offset, float *bound, float *center) {
  OXY_API_BEGIN
  OXY_REQUIRE(i >= 0 && i < (int32_t)p->m.tensors.size(), "tensor index out of range");
  const auto &t = p->m.tensors[i];
  std::snprintf(name64, 64, "%s", t.name.c_str());
  shape2[0] = t.rows;
  shape2[1] = t.cols;
  *dtype = t.dtype;
  *offset = t.offset;
  *bound = t.bound;
  *center = t.center;
  OXY_API_END
}

int oxy_pi05_tensor_read(oxy_pi05 *p, int32_t i, void *host, int64_t nbytes, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(i >= 0 && i < (int32_t)p->m.tensors.size(), "tensor index out of range");
  const auto &t = p->m.tensors[i];
  OXY_REQUIRE(nbytes == t.numel() * (t.dtype == 0 ? 2 : 4), "tensor %s byte count mismatch", t.name.c_str());
  auto st = oxy::as_stream(stream);
  OXY_CUDA(cudaMemcpyAsync(host, t.ptr, nbytes, cudaMemcpyDeviceToHost, st));
  OXY_CUDA(cudaStreamSynchronize(st));
  if (oxy::pi05::Model::is_rope_qkv(t.name)) {  // return the canonical row order
    std::vector<uint16_t> dev(static_cast<uint16_t *>(host), static_cast<uint16_t *>(host) + t.numel());
    uint16_t *out = static_cast<uint16_t *>(host);
    for (int64_t f = 0; f < t.rows; ++f)
      std::memcpy(out + (size_t)oxy::gemm::qkv_rope_row((int)f) * t.cols, dev.data() + (size_t)f * t.cols,
                  t.cols * 2);
  }
  OXY_API_END
}

int oxy_pi05_prefill(oxy_pi05 *p, int32_t n_obs, const int32_t *n_img_h, const int32_t *n_txt_h,
                     const int32_t *tokens_h, const uint8_t *images_d, const int32_t *blocks_h, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(n_obs >= 1, "prefill needs at least one observation");
  p->m.prefill(oxy::as_stream(stream), n_obs, n_img_h, n_txt_h, tokens_h, images_d, blocks_h);
  OXY_API_END
}

int oxy_pi05_denoise(oxy_pi05 *p, int32_t n, const int32_t *prefix_lens_h, const int32_t *blocks_h, int32_t S,
                     float *actions_d, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(n >= 1, "denoise needs at least one stream");
  p->m.denoise(oxy::as_stream(stream), n, prefix_lens_h, blocks_h, S, actions_d);
  OXY_API_END
}

int oxy_pi05_denoise_async(oxy_pi05 *p, int32_t n, const int32_t *prefix_lens_h, const int32_t *blocks_h,
                           int32_t S, float *actions_d, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(n >= 1, "denoise needs at least one stream");
  p->m.denoise(oxy::as_stream(stream), n, prefix_lens_h, blocks_h, S, actions_d, false);
  OXY_API_END
}

int oxy_pi05_join(oxy_pi05 *p, void *stream) {
  OXY_API_BEGIN
  p->m.join_alt(oxy::as_stream(stream));
  OXY_API_END
}

int oxy_pi05_denoise_elapsed_us(oxy_pi05 *p, double *us) {
  OXY_API_BEGIN
  OXY_REQUIRE(us != nullptr, "null output pointer");
  *us = 1e3 * (double)p->m.alt_elapsed_ms();
  OXY_API_END
}

int oxy_pi05_decode(oxy_pi05 *p, int32_t rows, int32_t k, const int32_t *block_tables_h, int32_t max_blocks,
                    const int32_t *seq_lens_h, const int32_t *last_tokens_h, const int32_t *budgets_h,
                    const int32_t *cow_h, int32_t *out_tokens_h, int32_t *out_count_h, float *logits_h,
                    void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(rows >= 1, "decode needs at least one row");
  OXY_REQUIRE(rows <= oxy::pi05::MAX_DECODE_ROWS, "at most %d decode rows per call",
              oxy::pi05::MAX_DECODE_ROWS);
  OXY_REQUIRE(k >= 1, "decode step count must be >= 1, got %d", k);
  p->m.decode(oxy::as_stream(stream), rows, k, block_tables_h, max_blocks, seq_lens_h, last_tokens_h, budgets_h,
              cow_h, out_tokens_h, out_count_h, logits_h);
  OXY_API_END
}

int oxy_pi05_recompute_logits(oxy_pi05 *p, const int32_t *tokens_h, int32_t n, int32_t prefix_len, float *logits_h,
                              void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(tokens_h && logits_h && n >= 1, "recompute needs at least one token");
  p->m.recompute(oxy::as_stream(stream), tokens_h, n, prefix_len, logits_h);
  OXY_API_END
}

int oxy_pi05_read_kv(oxy_pi05 *p, const int32_t *blocks_h, int32_t seq_len, int32_t layer, float *keys_h,
                     float *values_h, void *stream) {
  OXY_API_BEGIN
  auto &m = p->m;
  OXY_REQUIRE(layer >= 0 && layer < m.c.depth, "layer %d out of range", layer);
  if (seq_len == 0) return OXY_OK;
  auto st = oxy::as_stream(stream);
  OXY_REQUIRE(seq_len > 0, "negative sequence length");
  const int nb = (seq_len + 63) / 64;
  oxy::check_block_ids(blocks_h, nb, m.NB, "read_kv");
  int *bd = m.kvread_i.as<int>(nb);
  OXY_CUDA(cudaMemcpyAsync(bd, blocks_h, nb * sizeof(int), cudaMemcpyHostToDevice, st));
  float *ko = m.kvread_f.as<float>((size_t)2 * seq_len * 256);
  oxy::pi05::gather_kv_f32<<<seq_len, 256, 0, st>>>(ko, ko + (size_t)seq_len * 256, m.kpool(layer), m.vpool(layer),
                                                    bd, seq_len);
  OXY_LAUNCH_CHECK();
  OXY_CUDA(cudaMemcpyAsync(keys_h, ko, (size_t)seq_len * 256 * 4, cudaMemcpyDeviceToHost, st));
  OXY_CUDA(cudaMemcpyAsync(values_h, ko + (size_t)seq_len * 256, (size_t)seq_len * 256 * 4, cudaMemcpyDeviceToHost, st));
  OXY_CUDA(cudaStreamSynchronize(st));
  OXY_API_END
}

}  // extern "C"
