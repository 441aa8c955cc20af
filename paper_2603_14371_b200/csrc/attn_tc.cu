// tcgen05 flash attention for head dim 256 (prefix-LM prefill over the paged
// pool; action-expert suffix over [paged prefix || dense suffix]).
//
// CTA = one 128-row query tile x one key split; 6 warps:
//   warp 0     TMA producer: the Q tile once (4 boxes of 128 rows x 64 dims),
//              then K and V tiles of 64 keys (one pool block: 4 boxes each)
//              into a 2-slot ring; paged tiles by block id, dense by row;
//   warp 1     MMA issuer (one thread): S = Q K^T (M 128, N 64, K 256) into one
//              of two TMEM S buffers, then O += P V (M 128, N 256, K 64; V read
//              MN-major straight from its TMA layout) into the TMEM O tile;
//   warps 2-5  softmax: thread = query row (TMEM lane), 64 scores per tile in
//              registers, online softmax in the log2 domain with a lazy
//              reference max (O and l are rescaled only when the row max grows
//              by more than 2^8), P written bf16 to smem in the 128B-swizzled
//              K-major layout the PV MMA reads; final O / l to bf16 rows, or
//              bf16 partials (unnormalised O) + fp32 (m, l) for the split merge.
// Split merge, two ways: (a) cluster merge — the splits of a query tile are one
// thread-block cluster (<= 16 CTAs); each keeps its fp32 partial and (m, l) in
// its own smem, and after a cluster barrier CTA k merges rows
// [128k/splits, 128(k+1)/splits) of the tile by reading every peer's rows over
// DSMEM, in split order, and writes the bf16 output (no workspace round trip,
// no merge launch); (b) bf16 partials TMA-stored to a workspace, merged by
// fa_merge (splits > 16, or OXY_ATTN_CMERGE=0).  The two measure the same in the
// frame: the DSMEM reads run at ~15-25 GB/s per SM when all 14 CTAs of a
// cluster exchange rows (a push variant with bulk copies into the owners' freed
// K/V smem was slower still: 2.7 us to move 64 KB per CTA), so the cluster
// merge only saves the launch and the L2 round trip.
// Invariant relied on: pool slots past a sequence's length hold finite values
// (the pool is zeroed at creation and only ever written with finite K/V), so
// masked keys contribute p = 0 exactly.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "cuda_util.cuh"
#include "gemm_device.cuh"
#include "pi05_kernels.cuh"

namespace oxy {
namespace pi05 {

using namespace gemm;

namespace tc {
constexpr int TQ = 128, TK = 64, HD = 256;
constexpr int Q_BOX = TQ * 128;          // 16 KB: 128 rows x 64 dims
constexpr int KV_BOX = TK * 128;         // 8 KB: 64 keys x 64 dims
constexpr int Q_BYTES = 4 * Q_BOX;       // 64 KB
constexpr int KV_BYTES = 4 * KV_BOX;     // 32 KB (K or V tile)
constexpr int P_BYTES = TQ * 128;        // 16 KB: 128 rows x 64 keys bf16
constexpr int OFF_K = Q_BYTES, OFF_V = OFF_K + 2 * KV_BYTES, OFF_P = OFF_V + 2 * KV_BYTES;
constexpr int OFF_BAR = OFF_P + P_BYTES;  // 208 KB
// barriers: q_full, kv_full[2], kv_empty[2], s_full[2], s_empty[2], p_full, o_done
constexpr int N_BARS = 11;
constexpr size_t SMEM = 1024 + OFF_BAR + N_BARS * 8 + 16;
constexpr uint32_t TMEM_COLS = 512;  // O: 0..255, S buffers: 256.., 320..
constexpr float LAZY = 8.f;          // rescale when the row max grows by > 2^8
constexpr int MAX_CLUSTER = 16;      // cluster merge: splits per cluster (non-portable above 8)
}  // namespace tc

// MN-major, 128B-swizzled operand (V as the B operand: dims contiguous):
// 8-key atoms of 1024 B (SBO), 64-dim groups one TMA box apart (LBO).
__device__ __forceinline__ uint64_t make_sdesc_mn(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

#ifdef OXY_WATCHDOG
// debug builds: a wait that exceeds ~2 s reports who waits on what, then traps
__device__ __forceinline__ void wd_wait(uint32_t bar, uint32_t parity, int tag) {
  const long long t0 = clock64();
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (!ok && clock64() - t0 > 4000000000ll) {
      printf("flash_tc hang: cta (%d,%d) thread %d tag %d parity %u\n", blockIdx.x, blockIdx.y, threadIdx.x, tag,
             parity);
      asm volatile("trap;");
    }
  }
}
#define MBW(bar, par, tag) wd_wait(bar, par, tag)
#else
#define MBW(bar, par, tag) mbar_wait(bar, par)
#endif

#ifdef OXY_ATTN_PROF
// timing builds: %globaltimer at pipeline events of query tile 0, splits < 32
// (the last launch wins), read back by oxy_debug_attn_prof()
__device__ unsigned long long g_attn_prof[32][24];
#define APROF(ev)                                                                  \
  do {                                                                             \
    if (blockIdx.x == 0 && blockIdx.y < 32) {                                      \
      unsigned long long t_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
      g_attn_prof[blockIdx.y][ev] = t_;                                            \
    }                                                                              \
  } while (0)
// stamp taken after `dep` is computed (the timer read takes it as an operand)
#define APROF_DEP(ev, dep)                                                         \
  do {                                                                             \
    if (blockIdx.x == 0 && blockIdx.y < 32) {                                      \
      unsigned long long t_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "f"(dep));           \
      g_attn_prof[blockIdx.y][ev] = t_;                                            \
    }                                                                              \
  } while (0)
#else
#define APROF_DEP(ev, dep) \
  do {                     \
  } while (0)
#define APROF(ev) \
  do {            \
  } while (0)
#endif

// Cluster-merge output rows [rb, rb + nr) of a query tile: the gs bf16 partials of
// each (row, 8 columns) item read over DSMEM from the cluster's staged tiles (4 boxes
// of 128 rows x 64 bf16, 128B-swizzled), weighted in split order.  GS >= gs; 16 / GS
// items per thread are loaded before any is combined.
template <int GS>
__device__ __forceinline__ void merge_rows(const AttnGroup &g, int q0, int rb, int nr, int gs, uint32_t st_s,
                                           const float *wgt, int ndb, int db0) {
  constexpr int IT = 16 / GS, TQ = tc::TQ;
  const int cpr = ndb * 8;  // 8-column chunks per row of this CTA's dim range
  const int total = nr * cpr;
  for (int base = threadIdx.x; base < total; base += blockDim.x * IT) {
    uint4 v[IT][GS];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int idx = base + u * blockDim.x;
      const int i = idx / cpr, c8 = idx % cpr, row = rb + i;
      // 8 bf16 c8 of the row: box c8/8 (64 columns), 16-byte chunk (c8%8) ^ (row%8)
      const uint32_t off = (c8 >> 3) * (TQ * 128) + row * 128 + (((c8 & 7) ^ (row & 7)) << 4);
#pragma unroll
      for (int j = 0; j < GS; ++j)
        if (idx < total && j < gs)
          asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v[u][j].x), "=r"(v[u][j].y), "=r"(v[u][j].z), "=r"(v[u][j].w)
                       : "r"(map_to_rank(st_s + off, j)));
    }
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int idx = base + u * blockDim.x;
      if (idx >= total) continue;
      const int i = idx / cpr, c8 = idx % cpr, row = rb + i;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < GS; ++j)
        if (j < gs) {  // split order
          const float w = wgt[i * 16 + j];
          const uint32_t uu[4] = {v[u][j].x, v[u][j].y, v[u][j].z, v[u][j].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&uu[e]));
            acc[2 * e] += w * f.x;
            acc[2 * e + 1] += w * f.y;
          }
        }
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
        o[e] = *reinterpret_cast<uint32_t *>(&h);
      }
      *reinterpret_cast<uint4 *>(g.o + (size_t)(q0 + row) * g.ldo + db0 * 64 + c8 * 8) =
          make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

struct TcAttnArgs {
  const AttnGroup *groups;
  int q_tiles, splits, ws_rows;  // splits = grid y = the largest group's split count
  int tps;                       // key tiles per split (attn_group_splits)
  const bf16 *q_base, *kd_base;  // row offsets of the groups' q / dense k,v pointers
  int kv_ready;  // 1: the paged K/V were not written by the previous kernel (prefetch before the PDL wait)
  int cmerge;    // 1: launched as clusters of `splits` CTAs along y, merge over DSMEM
  int dsplit;    // 1, 2 or 4: grid z = head-dim parts of V / O (each CTA: full S, PV over its part)
  float scale_log2;
  float *ws_o, *ws_ml;
};

__global__ void __launch_bounds__(192, 1)
    flash_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kpmap,
                    const __grid_constant__ CUtensorMap vpmap, const __grid_constant__ CUtensorMap kdmap,
                    const __grid_constant__ CUtensorMap vdmap, const __grid_constant__ CUtensorMap wsmap,
                    TcAttnArgs a) {
  using namespace tc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~static_cast<uintptr_t>(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  const uint32_t b_q = smem_u32(bars), b_kvf = b_q + 8, b_kve = b_q + 24, b_sf = b_q + 40, b_se = b_q + 56,
                 b_pf = b_q + 72, b_od = b_q + 80;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) APROF(0);

  const AttnGroup g = a.groups[blockIdx.x / a.q_tiles];
  const int qt = blockIdx.x % a.q_tiles, q0 = qt * TQ;
  if (q0 >= g.nq) return;  // uniform per CTA, before any barrier or TMEM use
  const int split = blockIdx.y;
  // dim split: this CTA computes S and the softmax over all 256 dims but P.V (and the
  // merge / output) only for V-dim boxes [db0, db0 + ndb): half the V ingest and half the
  // merge volume per CTA, twice the CTAs; every output element's arithmetic is unchanged
  const int ndb = 4 / a.dsplit, db0 = blockIdx.z * ndb, dw = ndb * 64;
  const int ta = (g.nka + TK - 1) / TK, tb = (g.nkb + TK - 1) / TK, tiles = ta + tb;
  // this group's own key partition (a function of its key count only: batch-invariant);
  // CTAs past it (split >= gs) idle, or only help with the cluster merge
  int per;
  const int gs = attn_group_splits(tiles, a.tps, per);
  const int t0 = min(tiles, split * per), t1 = min(tiles, t0 + per), n = split < gs ? t1 - t0 : 0;

  if (threadIdx.x == 0) {
    mbar_init(b_q, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(b_kvf + 8 * s, 1);
      mbar_init(b_kve + 8 * s, 1);
      mbar_init(b_sf + 8 * s, 1);
      mbar_init(b_se + 8 * s, 4);
    }
    mbar_init(b_pf, 4);
    mbar_init(b_od, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kpmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vpmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // let the next kernel (split merge / o-projection) be scheduled now: it waits
  // in griddepcontrol.wait for our outputs and meanwhile streams its weights
  if (threadIdx.x == 0) {
    pdl_trigger();
    APROF(1);
  }

  if (warp == 0) {
    if (n > 0) {  // the whole warp walks the loads (uniform registers); the elected lane issues
      const int drow0 = g.kb ? (int)((g.kb - a.kd_base) / HD) : 0;
      auto issue = [&](int i) {
        const int j = t0 + i, s = i & 1;
        MBW(b_kve + 8 * s, ((i >> 1) & 1) ^ 1, 1);
        const bool paged = j < ta;
        const int row = paged ? g.bt[j] * TK : drow0 + (j - ta) * TK;
        const CUtensorMap *km = paged ? &kpmap : &kdmap, *vm = paged ? &vpmap : &vdmap;
        if (elect_one()) {
          mbar_expect_tx(b_kvf + 8 * s, KV_BYTES + ndb * KV_BOX);
          for (int b = 0; b < 4; ++b) {
            tma_load_2d(km, b_kvf + 8 * s, smem_u32(sm + OFF_K + s * KV_BYTES + b * KV_BOX), b * 64, row);
            if (b < ndb)
              tma_load_2d(vm, b_kvf + 8 * s, smem_u32(sm + OFF_V + s * KV_BYTES + b * KV_BOX), (db0 + b) * 64, row);
          }
        }
        __syncwarp();
      };
      int i = 0;
      // paged prefix K/V written long before this kernel (the expert suffix case):
      // fill the ring while the previous kernel drains
      if (a.kv_ready)
        for (; i < n && i < 2 && t0 + i < ta; ++i) issue(i);
      pdl_wait();  // Q (and dense K/V) come from the previous kernel
      if (lane == 0) APROF(2);
      const int qrow = (int)((g.q - a.q_base) / HD) + q0;
      if (elect_one()) {
        mbar_expect_tx(b_q, Q_BYTES);
        for (int b = 0; b < 4; ++b) tma_load_2d(&qmap, b_q, smem_u32(sm + b * Q_BOX), b * 64, qrow);
      }
      __syncwarp();
      for (; i < n; ++i) issue(i);
    }
  } else if (warp == 1) {
    if (n > 0) {  // the whole warp walks the loop (uniform registers); the elected lane issues
      // kind::f16, bf16 in, f32 accumulate; S: K-major A and B, N = 64; O: B (V) MN-major, N = 256
      const uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TK >> 3) << 17) |
                               ((uint32_t)(TQ >> 4) << 24);
      const uint32_t idesc_o = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(dw >> 3) << 17) |
                               ((uint32_t)(TQ >> 4) << 24);
      const uint32_t q_s = smem_u32(sm), p_s = smem_u32(sm + OFF_P);
      MBW(b_q, 0, 2);
      if (lane == 0) APROF(3);
      auto issue_pv = [&](int i) {
        MBW(b_pf, i & 1, 3);
        tc_fence_after();
        const uint32_t v_s = smem_u32(sm + OFF_V + (i & 1) * KV_BYTES);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < TK / 16; ++kk)
            mma_bf16(tmem, make_sdesc(p_s + kk * 32), make_sdesc_mn(v_s + kk * 2048, KV_BOX), idesc_o,
                     (i | kk) != 0 ? 1u : 0u);
          mma_commit(b_kve + 8 * (i & 1));
          mma_commit(b_od);
        }
        __syncwarp();
      };
      for (int i = 0; i < n; ++i) {
        const int s = i & 1;
        MBW(b_kvf + 8 * s, (i >> 1) & 1, 4);
        MBW(b_se + 8 * s, ((i >> 1) & 1) ^ 1, 5);
        tc_fence_after();
        const uint32_t k_s = smem_u32(sm + OFF_K + s * KV_BYTES);
        const uint32_t d_s = tmem + 256 + s * TK;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16(d_s, make_sdesc(q_s + (kk >> 2) * Q_BOX + (kk & 3) * 32),
                     make_sdesc(k_s + (kk >> 2) * KV_BOX + (kk & 3) * 32), idesc_s, kk != 0 ? 1u : 0u);
          mma_commit(b_sf + 8 * s);
        }
        __syncwarp();
        if (i > 0) issue_pv(i - 1);
      }
      issue_pv(n - 1);
    }
    __syncwarp();
  } else {
    // softmax / epilogue: thread = query row
    pdl_wait();  // outputs / workspace may still be read by earlier kernels
    if (threadIdx.x == 64) APROF(4);
    const int quad = warp & 3, row = quad * 32 + lane;
    const uint32_t lanes = (uint32_t)(quad * 32) << 16;
    const int r = q0 + row;
    float m_ref = -INFINITY, l = 0.f;
    uint8_t *prow = sm + OFF_P + row * 128;
    for (int i = 0; i < n; ++i) {
      const int j = t0 + i, s = i & 1;
      const int nvalid = j < ta ? min(TK, g.nka - j * TK) : min(TK, g.nkb - (j - ta) * TK);
      MBW(b_sf + 8 * s, (i >> 1) & 1, 6);
      tc_fence_after();
      if (threadIdx.x == 64 && i < 2) APROF(i == 0 ? 5 : 16);
      // Rolled 16-score chunks re-read from TMEM: this code runs once or a few
      // times per CTA, so it is instruction-fetch bound when cold; a fully
      // unrolled 64-score body measured 2-3x slower on its first pass.
      const uint32_t s_t = tmem + 256 + s * TK + lanes;
      float mx = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < TK / 16; ++c) {
        uint32_t v[16];
        tmem_ld16_nowait(s_t + c * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (c * 16 + e < nvalid) mx = fmaxf(mx, __uint_as_float(v[e]));
      }
      mx *= a.scale_log2;  // scale > 0: max commutes with it
      if (threadIdx.x == 64 && i < 2) APROF_DEP(i == 0 ? 14 : 17, mx);
      float corr = 1.f;
      if (mx > m_ref + LAZY || (m_ref == -INFINITY && mx > -INFINITY)) {
        corr = m_ref == -INFINITY ? 0.f : exp2f(m_ref - mx);
        m_ref = mx;
      }
      // PV(i-1) must be complete before O is rescaled and before P is overwritten
      // (a second P buffer, letting this tile's exp overlap PV(i-1), measured no
      // faster: the tile pace is K/V ingest, profiles/r02_attn.md)
      if (i > 0) {
        MBW(b_od, (i - 1) & 1, 7);
        tc_fence_after();
        // tcgen05.ld/st are warp-collective: rescale the warp's 32 rows together
        // whenever any of them needs it (rows that do not multiply by 1)
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < dw; c += 16) {
            uint32_t v[16];
            tmem_ld16_nowait(tmem + lanes + c, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * corr);
            tmem_st16(tmem + lanes + c, v);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      const float mref = m_ref == -INFINITY ? 0.f : m_ref;  // fully masked so far: every score is -inf
      float rs = 0.f;
#pragma unroll 1
      for (int c = 0; c < TK / 16; ++c) {
        uint32_t v[16];
        tmem_ld16_nowait(s_t + c * 16, v);
        tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float x0 = c * 16 + e < nvalid ? __uint_as_float(v[e]) * a.scale_log2 : -INFINITY;
          const float x1 = c * 16 + e + 1 < nvalid ? __uint_as_float(v[e + 1]) * a.scale_log2 : -INFINITY;
          const float p0 = exp2_approx(x0 - mref), p1 = exp2_approx(x1 - mref);
          rs += p0 + p1;
          __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
          pk[e / 2] = *reinterpret_cast<uint32_t *>(&h);
        }
        // 128B swizzle: 16-byte chunk ch of row r lives at ch ^ (r & 7)
        *reinterpret_cast<uint4 *>(prow + (((2 * c) ^ (row & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4 *>(prow + (((2 * c + 1) ^ (row & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      l = l * corr + rs;
      if (threadIdx.x == 64 && i < 2) APROF_DEP(i == 0 ? 15 : 18, l);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(b_se + 8 * s);  // S buffer may be overwritten
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(b_pf);
      if (threadIdx.x == 64) APROF(6);
      if (threadIdx.x == 64 && i >= 2 && i < 6) APROF(18 + i);  // P of tile i written (tiles 2..5)
    }
    // epilogue
    if (n > 0) {
      MBW(b_od, (n - 1) & 1, 8);
      tc_fence_after();
    }
    if (threadIdx.x == 64) APROF(7);
    const bool ok = r < g.nq && split == 0;
    if (gs == 1) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      bf16 *orow = g.o + (size_t)r * g.ldo + db0 * 64;
#pragma unroll 1
      for (int c = 0; c < dw; c += 16) {
        uint32_t v[16];
        if (n > 0) {
          tmem_ld16_nowait(tmem + lanes + c, v);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0u;
        }
        uint32_t o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          __nv_bfloat162 h =
              __floats2bfloat162_rn(__uint_as_float(v[2 * e]) * inv, __uint_as_float(v[2 * e + 1]) * inv);
          o[e] = *reinterpret_cast<uint32_t *>(&h);
        }
        if (ok) {
          *reinterpret_cast<uint4 *>(orow + c) = make_uint4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<uint4 *>(orow + c + 8) = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
    } else if (split < gs) {
      // bf16 partials through TMA stores: rows staged in smem as 4 boxes of
      // 128 rows x 64 bf16 in the 128B-swizzled box layout (conflict-free: the
      // 8 rows of an smem phase hit 8 different 16-byte slots), then one thread
      // stores the whole 128-row tile.  Workspace rows are padded per group to
      // multiples of 128, so rows past nq land in that group's padding.
      uint8_t *stage = sm;  // Q slot: free once the last PV retired
#pragma unroll 1
      for (int b = 0; b < ndb; ++b) {  // partials in bf16 (unnormalised O; m, l stay fp32)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t v[32];
          if (n > 0) {
            tmem_ld16_nowait(tmem + lanes + b * 64 + hh * 32, *reinterpret_cast<uint32_t(*)[16]>(v));
            tmem_ld16_nowait(tmem + lanes + b * 64 + hh * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0u;
          }
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
            pk[e] = *reinterpret_cast<uint32_t *>(&h);
          }
          uint8_t *rowp = stage + b * (TQ * 128) + row * 128;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int ch = hh * 4 + q;
            *reinterpret_cast<uint4 *>(rowp + ((ch ^ (row & 7)) << 4)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
      }
      // the (m, l) staging below reuses the P tile's bytes: every P row is dead once
      // the last PV MMA retired (b_od), but order the softmax threads explicitly so the
      // reuse does not rest on the tensor-core commit alone (compute-sanitizer racecheck)
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (a.cmerge) {  // (m, l) next to the partial; peers read both after the cluster barrier
        reinterpret_cast<float2 *>(sm + OFF_P)[row] = make_float2(m_ref, l);
      } else {
        if (r < g.nq && blockIdx.z == 0) {  // (m, l) are the same in every dim half
          const size_t wr = (size_t)split * a.ws_rows + g.wrow0 + r;
          a.ws_ml[wr * 2] = m_ref;
          a.ws_ml[wr * 2 + 1] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (threadIdx.x == 64) APROF(8);
      if (threadIdx.x == 64 && !a.cmerge) {
        const int row0 = split * a.ws_rows + g.wrow0 + q0;
        for (int b = 0; b < ndb; ++b)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                           reinterpret_cast<uint64_t>(&wsmap)),
                       "r"((db0 + b) * 64), "r"(row0), "r"(smem_u32(stage + b * (TQ * 128)))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // smem may be released once the copies have READ it; the global writes
        // complete before the grid does (what the merge waits for)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        APROF(9);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) APROF(10);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
  if (a.cmerge && gs > 1) {  // gs is uniform over the cluster (one query tile)
    cluster_sync_all();  // every split's partial and (m, l) are staged
    if (threadIdx.x == 0) APROF(11);
    const int cs = a.splits;  // cluster size: rows of the tile are shared out over it
    const int rb = split * TQ / cs, re = min((split + 1) * TQ / cs, g.nq - q0);
    const int nr = max(0, re - rb);
    float *wgt = reinterpret_cast<float *>(sm + OFF_V);  // [nr][16]: split weight / L per row
    const uint32_t ml_s = smem_u32(sm + OFF_P), st_s = smem_u32(sm);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
      const int row = rb + i;
      float m[16], lv[16], M = -INFINITY;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < gs) {
          asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];"
                       : "=f"(m[j]), "=f"(lv[j])
                       : "r"(map_to_rank(ml_s + row * 8, j))
                       : "memory");
          M = fmaxf(M, m[j]);
        }
      float L = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < gs) {
          m[j] = m[j] == -INFINITY ? 0.f : exp2f(m[j] - M);
          L += lv[j] * m[j];
        }
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < gs) wgt[i * 16 + j] = m[j] * inv;
    }
    __syncthreads();
    // the DSMEM loads of several (row, 8-column) items are in flight before any is
    // used (a plain loop waited one DSMEM round trip per item: 8 us for the 2-split
    // prefill tile, profiles/r02_attn.md)
    if (gs <= 2) merge_rows<2>(g, q0, rb, nr, gs, st_s, wgt, ndb, db0);
    else if (gs <= 4) merge_rows<4>(g, q0, rb, nr, gs, st_s, wgt, ndb, db0);
    else if (gs <= 8) merge_rows<8>(g, q0, rb, nr, gs, st_s, wgt, ndb, db0);
    else merge_rows<16>(g, q0, rb, nr, gs, st_s, wgt, ndb, db0);
    if (threadIdx.x == 0) APROF(12);
    cluster_sync_all();  // peers may still be reading this CTA's smem
    if (threadIdx.x == 0) APROF(13);
  }
}

// ------------------------------------------------------------------ SigLIP attention
//
// SigLIP So400m/14 self-attention on tcgen05: 16 heads of dim 72 over the 256
// patch tokens of one image (no mask).  CTA = (image, head, 128-query tile);
// all 256 keys fit at once, so no online softmax:
//   warp 0     TMA: Q (128 x [64 | 64] dims), K and V (256 x [64 | 64] dims) of the
//              head straight out of the fused qkv rows [T, 3 * 1152]; the second
//              64-dim box of a head also covers the next head's first dims;
//   warps 2-5  zero Q's dims 72..127 in smem (so S only sums the head's 72 dims:
//              the MMAs run K = 80), then softmax with thread = query row: max and
//              exp2 over the row's 256 TMEM scores, P bf16 into the (now free) K
//              smem in the 128B-swizzled K-major layout, O / l to bf16;
//   warp 1     S = Q K^T (M 128, N 256, K 80) into TMEM; O = P V (M 128, N 80,
//              K 256; V read MN-major from its TMA layout; O dims >= 72 dropped).
namespace vt {
constexpr int TQ = 128, NK = 256, HD = 72;
constexpr int Q_ATOM = TQ * 128;    // 16 KB: 128 rows x 64 dims
constexpr int KV_ATOM = NK * 128;   // 32 KB: 256 keys x 64 dims
constexpr int OFF_K = 2 * Q_ATOM;   // P (4 atoms of 128 rows x 64 keys) reuses K's 64 KB
constexpr int OFF_V = OFF_K + 2 * KV_ATOM;
constexpr int OFF_BAR = OFF_V + 2 * KV_ATOM;  // 160 KB
// barriers: q_full, k_full, v_full, q_ready (4 warps), s_full, p_full (4 warps), o_full
constexpr int N_BARS = 7;
constexpr size_t SMEM = 1024 + OFF_BAR + N_BARS * 8 + 16;
constexpr uint32_t TMEM_COLS = 512;  // S: 0..255, O: 256..335
}  // namespace vt

__global__ void __launch_bounds__(192, 1)
    vit_attn_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kvmap, bf16 *out,
                       int heads, float scale_log2) {
  using namespace vt;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~static_cast<uintptr_t>(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + N_BARS);
  const uint32_t b_q = smem_u32(bars), b_k = b_q + 8, b_v = b_q + 16, b_qr = b_q + 24, b_s = b_q + 32,
                 b_p = b_q + 40, b_o = b_q + 48;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int img = blockIdx.x / heads, h = blockIdx.x % heads, q0 = blockIdx.y * TQ;
  const int D = heads * HD;  // 1152
  const int row_img = img * NK;
  if (threadIdx.x == 0) {
    mbar_init(b_q, 1);
    mbar_init(b_k, 1);
    mbar_init(b_v, 1);
    mbar_init(b_qr, 4);
    mbar_init(b_s, 1);
    mbar_init(b_p, 4);
    mbar_init(b_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kvmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) pdl_trigger();  // the o-projection may start streaming its weights
  pdl_wait();                           // q/k/v rows come from the qkv projection
  if (warp == 0) {
    if (lane == 0) {
      const int cq = h * HD, ck = D + h * HD, cv = 2 * D + h * HD;
      mbar_expect_tx(b_q, 2 * Q_ATOM);
      mbar_expect_tx(b_k, 2 * KV_ATOM);
      mbar_expect_tx(b_v, 2 * KV_ATOM);
      for (int b = 0; b < 2; ++b) tma_load_2d(&qmap, b_q, smem_u32(sm + b * Q_ATOM), cq + 64 * b, row_img + q0);
      for (int b = 0; b < 2; ++b) tma_load_2d(&kvmap, b_k, smem_u32(sm + OFF_K + b * KV_ATOM), ck + 64 * b, row_img);
      for (int b = 0; b < 2; ++b) tma_load_2d(&kvmap, b_v, smem_u32(sm + OFF_V + b * KV_ATOM), cv + 64 * b, row_img);
    }
  } else if (warp == 1) {
    {  // the whole warp waits; the elected lane issues
      const uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NK >> 3) << 17) |
                               ((uint32_t)(TQ >> 4) << 24);
      const uint32_t idesc_o = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(80 >> 3) << 17) |
                               ((uint32_t)(TQ >> 4) << 24);
      const uint32_t q_s = smem_u32(sm), k_s = smem_u32(sm + OFF_K), v_s = smem_u32(sm + OFF_V);
      mbar_wait(b_k, 0);
      mbar_wait(b_qr, 0);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 5; ++kk)  // K = 80: dims 0..63 (atom 0), 64..79 (atom 1; Q zero past 71)
          mma_bf16(tmem, make_sdesc(q_s + (kk >> 2) * Q_ATOM + (kk & 3) * 32),
                   make_sdesc(k_s + (kk >> 2) * KV_ATOM + (kk & 3) * 32), idesc_s, kk != 0 ? 1u : 0u);
        mma_commit(b_s);
      }
      __syncwarp();
      mbar_wait(b_v, 0);
      mbar_wait(b_p, 0);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < NK / 16; ++kk)  // P atoms of 64 keys at OFF_K + 16 KB each
          mma_bf16(tmem + 256, make_sdesc(k_s + (kk >> 2) * Q_ATOM + (kk & 3) * 32),
                   make_sdesc_mn(v_s + kk * 2048, KV_ATOM), idesc_o, kk != 0 ? 1u : 0u);
        mma_commit(b_o);
      }
    }
    __syncwarp();
  } else {
    const int quad = warp & 3, row = quad * 32 + lane;
    const uint32_t lanes = (uint32_t)(quad * 32) << 16;
    // Q dims 72..127 (atom 1, logical 16-byte chunks 1..7 of the row) -> 0
    mbar_wait(b_q, 0);
    uint8_t *qrow = sm + Q_ATOM + row * 128;
#pragma unroll
    for (int ch = 1; ch < 8; ++ch) *reinterpret_cast<uint4 *>(qrow + ((ch ^ (row & 7)) << 4)) = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive_local(b_qr);
    // softmax over the row's 256 scores
    mbar_wait(b_s, 0);
    tc_fence_after();
    float mx = -INFINITY;
#pragma unroll 1
    for (int c = 0; c < NK / 16; ++c) {
      uint32_t v[16];
      tmem_ld16_nowait(tmem + lanes + c * 16, v);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 16; ++e) mx = fmaxf(mx, __uint_as_float(v[e]));
    }
    const float mref = mx * scale_log2;
    float l = 0.f;
#pragma unroll 1
    for (int c = 0; c < NK / 16; ++c) {
      uint32_t v[16];
      tmem_ld16_nowait(tmem + lanes + c * 16, v);
      tmem_ld_wait();
      uint32_t pk[8];
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        const float p0 = exp2_approx(__uint_as_float(v[e]) * scale_log2 - mref);
        const float p1 = exp2_approx(__uint_as_float(v[e + 1]) * scale_log2 - mref);
        l += p0 + p1;
        __nv_bfloat162 hh = __floats2bfloat162_rn(p0, p1);
        pk[e / 2] = *reinterpret_cast<uint32_t *>(&hh);
      }
      // P atom c / 4 (keys 64 (c/4) ..), 16-byte chunks 2 (c % 4), +1 of the row, 128B swizzle
      uint8_t *prow = sm + OFF_K + (c >> 2) * Q_ATOM + row * 128;
      const int ch = 2 * (c & 3);
      *reinterpret_cast<uint4 *>(prow + ((ch ^ (row & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      *reinterpret_cast<uint4 *>(prow + (((ch + 1) ^ (row & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_local(b_p);
    mbar_wait(b_o, 0);
    tc_fence_after();
    const float inv = 1.f / l;
    uint32_t o[40];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      uint32_t v[16];
      tmem_ld16_nowait(tmem + lanes + 256 + c * 16, v);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        __nv_bfloat162 hh =
            __floats2bfloat162_rn(__uint_as_float(v[2 * e]) * inv, __uint_as_float(v[2 * e + 1]) * inv);
        o[c * 8 + e] = *reinterpret_cast<uint32_t *>(&hh);
      }
    }
    uint4 *orow = reinterpret_cast<uint4 *>(out + (size_t)(row_img + q0 + row) * D + h * HD);  // 144 B, 16-aligned
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) orow[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

void vit_attention_tc(const bf16 *qkv, bf16 *out, int n_images, int heads, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    OXY_CUDA(cudaFuncSetAttribute(vit_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vt::SMEM));
    attr = true;
  }
  if (n_images <= 0) return;
  if (heads < 1 || (reinterpret_cast<uintptr_t>(qkv) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    fail(OXY_EINVAL, "SigLIP attention: heads >= 1 and 16-byte aligned q/k/v and output rows");
  const int D = heads * vt::HD;
  // boxes of 64 dims over the fused [n_images * 256, 3 D] qkv rows: 128 query rows, 256 key rows
  const CUtensorMap qm = gemm::make_map(qkv, n_images * vt::NK, 3 * D, vt::TQ);
  const CUtensorMap kvm = gemm::make_map(qkv, n_images * vt::NK, 3 * D, vt::NK);
  ++gemm::g_plan_counts[gemm::PC_VIT_TC];
  launch_pdl(vit_attn_tc_kernel, dim3(n_images * heads, vt::NK / vt::TQ), dim3(192), vt::SMEM, st, qm, kvm, out,
             heads, 1.4426950408889634f / std::sqrt((float)vt::HD));
}

int attn_cluster_merge_max() {
  static const int v = [] {
    const char *e = getenv("OXY_ATTN_CMERGE");
    return std::min(tc::MAX_CLUSTER, e ? atoi(e) : tc::MAX_CLUSTER);
  }();
  return v;
}

void flash_attention_tc(const AttnGroup *groups_d, int n_groups, int q_tiles, int splits, int tps, const bf16 *q_base,
                        int q_rows, const CUtensorMap &kpool_map, const CUtensorMap &vpool_map, const bf16 *kd_base,
                        const bf16 *vd_base, int kd_rows, float scale, float *ws_o, float *ws_ml, int ws_rows,
                        bool kv_ready, bool cmerge, cudaStream_t st, int lane_sms) {
  static bool attr = false;
  if (!attr) {
    OXY_CUDA(cudaFuncSetAttribute(flash_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM));
    OXY_CUDA(cudaFuncSetAttribute(flash_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cmerge = cmerge && splits > 1;
  if (cmerge && splits > tc::MAX_CLUSTER) fail(OXY_EINVAL, "cluster merge needs splits <= %d", tc::MAX_CLUSTER);
  if (n_groups <= 0 || q_tiles <= 0) return;
  const CUtensorMap qm = gemm::make_map(q_base, q_rows, tc::HD, tc::TQ);
  // dense suffix K/V (or the pool maps again when there is none)
  const CUtensorMap kdm = kd_base ? gemm::make_map(kd_base, kd_rows, tc::HD, tc::TK) : kpool_map;
  const CUtensorMap vdm = vd_base ? gemm::make_map(vd_base, kd_rows, tc::HD, tc::TK) : vpool_map;
  if (kd_base && vd_base - kd_base != 0 && (vd_base - kd_base) % tc::HD != 0)
    fail(OXY_EINVAL, "dense K/V buffers must be row-aligned");
  if (splits > 1 && !cmerge && ws_rows % tc::TQ != 0) fail(OXY_EINVAL, "attention workspace rows must be padded to 128");
  // bf16 partial rows [splits * ws_rows, 256], box 64 x 128 (128-byte rows), 128B swizzle
  const CUtensorMap wsm =
      splits > 1 && !cmerge ? gemm::make_map(reinterpret_cast<const bf16 *>(ws_o), splits * ws_rows, tc::HD, tc::TQ)
                            : qm;
  ++gemm::g_plan_counts[splits == 1 ? gemm::PC_ATTN_ONE : cmerge ? gemm::PC_ATTN_CMERGE : gemm::PC_ATTN_WSMERGE];
  // head-dim halves when twice the (query tile, key split) CTAs still fit one wave (the
  // expert suffix: 28 -> 56 CTAs; not the 1-stream prefill, 100 CTAs, where 200 made two
  // waves): half the V ingest and merge volume per CTA, same arithmetic per element
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  static const int knob = [] {
    const char *e = getenv("OXY_ATTN_DSPLIT");  // 0: off, 1: auto (default), 2 / 4: always that many
    return e ? atoi(e) : 1;
  }();
  static const int auto_max = [] {
    const char *e = getenv("OXY_ATTN_DSPLIT_MAX");  // largest automatic split (A/B)
    return e ? atoi(e) : 2;
  }();
  const int ctas = n_groups * q_tiles * splits;
  const int avail = lane_sms > 0 ? std::min(lane_sms, sms) : sms;  // the caller's SM partition
  int dsplit = knob >= 2 ? knob : 1;
  if (knob == 1)
    for (int d = auto_max; d >= 2; d /= 2)
      if (d * ctas <= avail) {
        dsplit = d;
        break;
      }
  if (dsplit != 1 && dsplit != 2 && dsplit != 4) fail(OXY_EINVAL, "attention head-dim split must be 1, 2 or 4");
  TcAttnArgs a{groups_d, q_tiles, splits, ws_rows, tps, q_base, kd_base, kv_ready ? 1 : 0, cmerge ? 1 : 0,
               dsplit, scale * 1.4426950408889634f, ws_o, ws_ml};
  launch_pdl_cluster(flash_tc_kernel, dim3(n_groups * q_tiles, splits, dsplit), dim3(192), tc::SMEM, st,
                     dim3(1, cmerge ? splits : 1, 1), qm, kpool_map, vpool_map, kdm, vdm, wsm, a);
}

}  // namespace pi05
}  // namespace oxy

extern "C" int oxy_prefix_attention(const void *q_d, void *out_d, const void *kpool_d, const void *vpool_d,
                                    int32_t num_blocks, const int32_t *bt_d, int32_t nka, const void *kd_d,
                                    const void *vd_d, int32_t nkb, int32_t nq, int32_t splits, float *ws_o,
                                    float *ws_ml, void *stream) {
  OXY_API_BEGIN
  using oxy::pi05::bf16;
  OXY_REQUIRE(nq >= 1 && nka >= 0 && nkb >= 0 && nka + nkb >= 1 && num_blocks >= 1, "bad attention shape");
  OXY_REQUIRE(nkb == 0 || (kd_d && vd_d), "dense keys need kd/vd");
  const int tiles = (nka + 63) / 64 + (nkb + 63) / 64;
  OXY_REQUIRE(splits >= 1 && splits <= 32 && splits <= tiles, "splits must be in [1, min(32, key tiles)]");
  auto st = oxy::as_stream(stream);
  oxy::pi05::AttnGroup g{};
  g.q = static_cast<const bf16 *>(q_d);
  g.o = static_cast<bf16 *>(out_d);
  g.ldq = g.ldo = 256;
  g.nq = nq;
  g.bt = bt_d;
  g.nka = nka;
  g.kb = static_cast<const bf16 *>(kd_d);
  g.vb = static_cast<const bf16 *>(vd_d);
  g.ldkv = 256;
  g.nkb = nkb;
  g.wrow0 = 0;
  oxy::pi05::AttnGroup *gd = nullptr;
  OXY_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&gd), sizeof(g), st));
  OXY_CUDA(cudaMemcpyAsync(gd, &g, sizeof(g), cudaMemcpyHostToDevice, st));
  const CUtensorMap km = oxy::gemm::make_map(kpool_d, num_blocks * 64, 256, 64);
  const CUtensorMap vm = oxy::gemm::make_map(vpool_d, num_blocks * 64, 256, 64);
  const int q_tiles = (nq + 127) / 128, ws_rows = q_tiles * 128;
  const int tps = (tiles + splits - 1) / splits;  // the key partition `splits` asks for
  int per = 0;
  splits = oxy::pi05::attn_group_splits(tiles, tps, per);  // e.g. 9 tiles / 4 splits -> 3 x 3
  const bool cm = splits > 1 && splits <= oxy::pi05::attn_cluster_merge_max();
  if (splits > 1 && !cm && !(ws_o && ws_ml)) {
    cudaFreeAsync(gd, st);
    oxy::fail(OXY_EINVAL, "split attention needs a workspace");
  }
  oxy::pi05::flash_attention_tc(gd, 1, q_tiles, splits, tps, g.q, nq, km, vm, g.kb, g.vb, std::max(nkb, 1),
                                1.f / 16.f, ws_o, ws_ml, ws_rows, false, cm, st);
  if (splits > 1 && !cm)
    oxy::pi05::flash_merge(gd, 1, ws_rows, splits, tps, reinterpret_cast<const bf16 *>(ws_o), ws_ml, ws_rows, st);
  OXY_CUDA(cudaFreeAsync(gd, st));
  OXY_API_END
}

extern "C" int oxy_vit_attention(const void *qkv_d, void *out_d, int32_t n_images, int32_t heads, void *stream) {
  OXY_API_BEGIN
  OXY_REQUIRE(n_images >= 1 && heads >= 1 && heads <= 64, "bad SigLIP attention shape");
  oxy::pi05::vit_attention_tc(static_cast<const oxy::pi05::bf16 *>(qkv_d), static_cast<oxy::pi05::bf16 *>(out_d),
                              n_images, heads, oxy::as_stream(stream));
  OXY_API_END
}

#ifdef OXY_ATTN_PROF
extern "C" int oxy_debug_attn_prof(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, oxy::pi05::g_attn_prof, sizeof(oxy::pi05::g_attn_prof)) == cudaSuccess ? 0 : -1;
}
#endif
