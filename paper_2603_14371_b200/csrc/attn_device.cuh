// Flash-attention tile body (mma.sync bf16, online softmax) shared by the
// stand-alone kernel (pi05_kernels.cu) and the persistent layer kernel
// (megakernel.cu), plus the ldmatrix / cp.async / mma wrappers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "cuda_util.cuh"
#include "pi05_kernels.cuh"

namespace oxy {
namespace pi05 {

// ============================================================ flash attention

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

constexpr int FA_BQ = 64;  // query rows per CTA (4 warps x 16)
constexpr int FA_BK = 64;  // keys per tile (= KV_BLOCK)
constexpr int FA_THREADS = 128;
// the 4 attention warps synchronise on named barrier 2 (the persistent layer
// kernel runs them next to warps doing other work)
__device__ __forceinline__ void fa_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

template <int HD>
struct FaCfg {
  static constexpr int HDP = (HD + 15) / 16 * 16;  // padded to the MMA K step
  static constexpr int LDS = HDP + 8;               // +16 B: conflict-free ldmatrix
  static constexpr int CHUNKS = HD / 8;             // 16-byte chunks holding data
  static constexpr int PCHUNKS = HDP / 8;
  static constexpr int TILE = FA_BQ * LDS;          // elements per smem tile
  static constexpr size_t SMEM = (size_t)5 * TILE * sizeof(bf16);
};

// Stage one 64-row tile (rows from `row_ptr(r)` or zero) into smem via cp.async.
template <int HD>
__device__ __forceinline__ void load_tile(int tid, bf16 *dst, const bf16 *base, int ld, int nrows_valid,
                                          const int *map_block, int key0) {
  using C = FaCfg<HD>;
  for (int idx = tid; idx < FA_BQ * C::PCHUNKS; idx += FA_THREADS) {
    const int r = idx / C::PCHUNKS, ch = idx % C::PCHUNKS;
    bf16 *d = dst + r * C::LDS + ch * 8;
    if (r < nrows_valid && ch < C::CHUNKS) {
      const bf16 *src;
      if (map_block) src = base + ((size_t)map_block[0] * KV_BLOCK + r) * HD + ch * 8;
      else src = base + (size_t)(key0 + r) * ld + ch * 8;
      cp_async16(smem_addr(d), src);
    } else {
      *reinterpret_cast<int4 *>(d) = make_int4(0, 0, 0, 0);
    }
  }
}

// One (query tile, key split) work item of 64 query rows x the split's key
// tiles, run by threads tid = 0..127 (4 warps).  smem: 5 tiles (Q, K x2, V x2).
// splits == 1: normalised bf16 rows to g.o; else fp32 partial O and (m, l) rows
// to ws_o / ws_ml (merged in split order by fa_merge).
template <int HD>
__device__ __forceinline__ void flash_item(const AttnGroup &g, int qt, int split, int splits, const bf16 *kpool,
                                           const bf16 *vpool, float scale_log2, float *ws_o, float *ws_ml,
                                           int ws_rows, bf16 *smem, int tid) {
  using C = FaCfg<HD>;
  constexpr int NT = C::HDP / 8;  // output n-tiles per warp
  bf16 *sQ = smem;
  bf16 *sK[2] = {sQ + C::TILE, sQ + 2 * C::TILE};
  bf16 *sV[2] = {sQ + 3 * C::TILE, sQ + 4 * C::TILE};

  const int q0 = qt * FA_BQ;
  if (q0 >= g.nq) return;
  const int ta = (g.nka + FA_BK - 1) / FA_BK, tb = (g.nkb + FA_BK - 1) / FA_BK;
  const int tiles = ta + tb;
  const int per = (tiles + splits - 1) / splits;
  const int t_begin = split * per, t_end = min(tiles, t_begin + per);
  const int warp = tid >> 5, lane = tid & 31;

  auto issue_tile = [&](int ti, int buf) {
    if (ti < ta) {
      const int nvalid = min(FA_BK, g.nka - ti * FA_BK);
      load_tile<HD>(tid, sK[buf], kpool, HD, nvalid, g.bt + ti, 0);
      load_tile<HD>(tid, sV[buf], vpool, HD, nvalid, g.bt + ti, 0);
    } else {
      const int j0 = (ti - ta) * FA_BK;
      const int nvalid = min(FA_BK, g.nkb - j0);
      load_tile<HD>(tid, sK[buf], g.kb, g.ldkv, nvalid, nullptr, j0);
      load_tile<HD>(tid, sV[buf], g.vb, g.ldkv, nvalid, nullptr, j0);
    }
    cp_commit();
  };

  // Q tile
  load_tile<HD>(tid, sQ, g.q, g.ldq, min(FA_BQ, g.nq - q0), nullptr, q0);
  cp_commit();
  if (t_begin < t_end) issue_tile(t_begin, 0);

  float o[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const uint32_t q_base = smem_addr(sQ + (warp * 16 + (lane & 15)) * C::LDS + (lane >> 4) * 8);

  for (int ti = t_begin; ti < t_end; ++ti) {
    const int buf = (ti - t_begin) & 1;
    if (ti + 1 < t_end) {
      issue_tile(ti + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    fa_bar();
    const int nvalid = ti < ta ? min(FA_BK, g.nka - ti * FA_BK) : min(FA_BK, g.nkb - (ti - ta) * FA_BK);

    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
    const bf16 *kt = sK[buf];
#pragma unroll
    for (int kk = 0; kk < C::HDP / 16; ++kk) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(q_base + kk * 32, a0, a1, a2, a3);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int col = kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_addr(kt + key * C::LDS + col), b0, b1, b2, b3);
        mma16816(s[2 * np], a0, a1, a2, a3, b0, b1);
        mma16816(s[2 * np + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // mask + online softmax (rows g and g+8 of this warp)
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = nt * 8 + (lane & 3) * 2 + (e & 1);
        float v = s[nt][e] * scale_log2;
        if (key >= nvalid) v = -INFINITY;
        s[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int h = 0; h < 2; ++h) corr[h] = (mx[h] == -INFINITY) ? 1.f : exp2f(m_r[h] - mx[h]);
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mref = mx[e >> 1] == -INFINITY ? 0.f : mx[e >> 1];  // fully masked row: scores are -inf
        const float p = exp2_approx(s[nt][e] - mref);
        s[nt][e] = p;
        rs[e >> 1] += p;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pa[j][0] = pack_bf16(s[2 * j][0], s[2 * j][1]);
      pa[j][1] = pack_bf16(s[2 * j][2], s[2 * j][3]);
      pa[j][2] = pack_bf16(s[2 * j + 1][0], s[2 * j + 1][1]);
      pa[j][3] = pack_bf16(s[2 * j + 1][2], s[2 * j + 1][3]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 1);
      rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 2);
      l_r[h] = l_r[h] * corr[h] + rs[h];
      m_r[h] = mx[h];
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      o[nt][0] *= corr[0];
      o[nt][1] *= corr[0];
      o[nt][2] *= corr[1];
      o[nt][3] *= corr[1];
    }
    // O += P V
    const bf16 *vt = sV[buf];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        const int key = j * 16 + (lane & 15);
        const int col = np * 16 + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_addr(vt + key * C::LDS + col), b0, b1, b2, b3);
        mma16816(o[2 * np], pa[j][0], pa[j][1], pa[j][2], pa[j][3], b0, b1);
        mma16816(o[2 * np + 1], pa[j][0], pa[j][1], pa[j][2], pa[j][3], b2, b3);
      }
    }
    fa_bar();
  }

  cp_wait<0>();  // no cp.async may still target smem when the item returns (empty splits)
  // epilogue
  const int rbase = q0 + warp * 16 + (lane >> 2);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = rbase + h * 8;
    if (r >= g.nq) continue;
    if (splits == 1) {
      const float inv = l_r[h] > 0.f ? 1.f / l_r[h] : 0.f;
      bf16 *orow = g.o + (size_t)r * g.ldo;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + (lane & 3) * 2;
        if (c < HD)
          *reinterpret_cast<__nv_bfloat162 *>(orow + c) =
              __floats2bfloat162_rn(o[nt][2 * h] * inv, o[nt][2 * h + 1] * inv);
      }
    } else {
      const size_t wr = (size_t)split * ws_rows + g.wrow0 + r;
      float *orow = ws_o + wr * C::HDP;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + (lane & 3) * 2;
        orow[c] = o[nt][2 * h];
        orow[c + 1] = o[nt][2 * h + 1];
      }
      if ((lane & 3) == 0) {
        ws_ml[wr * 2] = m_r[h];
        ws_ml[wr * 2 + 1] = l_r[h];
      }
    }
  }
}


}  // namespace pi05
}  // namespace oxy
