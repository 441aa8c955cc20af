// Persistent layer-program kernel ("megakernel") for the skinny token counts of
// the action expert's denoise loop (T = 50 per stream) and language decode
// (T = rows): one cooperative launch runs a whole program of phases — tcgen05
// GEMM tiles, split-K reductions fused with RoPE / residual / (ada)RMSNorm,
// flash-attention tiles and their split merge, Euler updates — with a grid
// barrier between dependent phases.  It replaces ~10 kernel launches per layer
// (each paying launch + prologue + pipeline-fill latency at a few us of work)
// by phases whose cost is their data movement plus one ~1 us barrier.
//
// Work inside a phase is split into items distributed round-robin over the
// CTAs (one per SM).  GEMM phases keep the warp-specialised tcgen05 structure
// (warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 TMEM epilogue) with the
// smem ring, the two TMEM accumulators and their mbarrier phases carried
// across phases.  Split-K reductions are done in a fixed split order, so the
// program is deterministic and batch-invariant like the multi-kernel path.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "gemm_sm100.cuh"
#include "pi05_kernels.cuh"

namespace oxy {
namespace mk {

using bf16 = __nv_bfloat16;

enum PhaseType : int {
  PH_GEMM = 0,        // Y (op)= W X over (m-tile, token-tile, k-split) items
  PH_REDUCE_EPI = 1,  // fixed-order sum of split-K partials + a GEMM epilogue (RoPE, GeGLU, ...)
  PH_RES_NORM = 2,    // x += gate * sum(partials); y = RMSNorm / adaRMS(x)   (one row per item)
  PH_ATTN = 3,        // flash-attention (group, q-tile, key-split) items
  PH_ATTN_MERGE = 4,  // merge key-split partials in split order (one query row per item)
  PH_EULER = 5,       // a += dt * v; a_bf16 = bf16(a)
};

struct GemmPh {
  int map_a, map_b;  // indices into the program's tensor-map table (A: weights, B: activations)
  int n_out, k, t, bn, m_tiles, n_tiles, splits, kb_per_split, kb_total;
  gemm::EpiParams epi;  // splits == 1
  float *ws;            // splits > 1: partials [splits][t][n_out]
};
struct ReducePh {
  const float *ws;
  int splits, t, n;
  gemm::EpiParams epi;
};
struct NormPh {
  const float *ws;  // null: no residual update, normalise x only
  int splits, t, n;
  const float *gate;  // per-feature residual gate or null
  float *x;
  int ldx;
  bf16 *y;
  int ldy;
  const float *w, *ms, *mb;  // RMSNorm (1 + w) or adaRMS (1 + ms, + mb)
  float eps;
};
struct AttnPh {
  const pi05::AttnGroup *groups;
  int n_groups, q_tiles, splits, ws_rows, max_nq;
  const bf16 *kpool, *vpool;
  float scale_log2;
  float *ws_o, *ws_ml;
};
struct EulerPh {
  float *a;
  const float *v;
  bf16 *ab;
  int n;
  float dt;
};

struct Phase {
  int type, items;
  union {
    GemmPh g;
    ReducePh r;
    NormPh nm;
    AttnPh at;
    EulerPh eu;
  };
};

constexpr int MK_THREADS = 192;
constexpr int MK_STAGES = 6;
constexpr int MK_MAX_BN = 128;  // two TMEM accumulators of up to 128 columns

// Host-side program: phases + tensor maps, uploaded once and replayed.
struct Program {
  std::vector<Phase> phases;
  std::vector<CUtensorMap> maps;
  std::vector<const void *> map_keys;  // (ptr) dedupe, with rows/k/box below
  std::vector<int> map_meta;
  Phase *d_phases = nullptr;
  CUtensorMap *d_maps = nullptr;
  unsigned *d_sync = nullptr;
  unsigned long long *d_times = nullptr;  // per-phase end timestamps (profile != 0)
  int profile = 0;
  size_t cap_phases = 0, cap_maps = 0;
  int grid = 0;
  unsigned long long gen = ~0ull;  // scratch generation the pointers were taken at

  ~Program();
  void clear() {
    phases.clear();
    maps.clear();
    map_keys.clear();
    map_meta.clear();
  }
  int map(const void *ptr, int rows, int k, int box_rows);
  // Y[t, f] (op)= sum_k W[f, k] X[t, k]; splits from the skinny GEMM planner.
  // Returns the split count (> 1: partials in ws, reduce with reduce_epi / res_norm).
  int gemm(const bf16 *w, const bf16 *x, int n_out, int k, int t, const gemm::EpiParams &epi, float *ws,
           int sms, int force_splits = 0);
  void reduce_epi(const float *ws, int splits, int t, int n, const gemm::EpiParams &epi);
  void res_norm(const float *ws, int splits, int t, int n, const float *gate, float *x, int ldx, bf16 *y, int ldy,
                const float *w, const float *ms, const float *mb, float eps);
  void attention(const pi05::AttnGroup *groups_d, int n_groups, int q_tiles, int max_nq, int splits, int ws_rows,
                 const bf16 *kpool, const bf16 *vpool, float scale, float *ws_o, float *ws_ml);
  void euler(float *a, const float *v, bf16 *ab, int n, float dt);
  void upload(cudaStream_t st);
  void launch(cudaStream_t st);
};

size_t mk_smem_bytes();
// split-K count Program::gemm will pick for (n_out, k, t) on `sms` SMs
int gemm_splits(int n_out, int k, int t, int sms);

}  // namespace mk
}  // namespace oxy
