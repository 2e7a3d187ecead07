// Epilogue pieces shared by the streamed score kernels (score_st.cu: 3xTF32 on
// fp32 rows; score_sh.cu: fp16 rows for the Gram path): accumulator read-back,
// the Gram path's corrected argmax and its exact near-tie re-check.
#pragma once

#include "common.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {
namespace epi {

using namespace sm100;

// Accumulator read-back: with two MMA chains (hi.hi in one accumulator, the
// small hi.lo + lo.hi in a second one `off2` columns further) the two are summed.
__device__ __forceinline__ void acc_ld32(uint32_t taddr, uint32_t off2, float (&v)[32]) {
  tmem_ld32(taddr, v);
  if (off2) {
    float w[32];
    tmem_ld32(taddr + off2, w);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += w[j];
  }
}

// Half-precision rows (score_sh.cu): the accumulator holds kPieces column groups,
// x16 . p0 | x16 . p1 (| x16 . p2) with the centroid c = p0 + 2^-11 p1 (+ 2^-22 p2)
// in fp16 pieces (table_h_kernel) and x16 = fp16(s x) for the patch's
// power-of-two scale s; `scale` = 1 / s.  Two pieces carry 22 significant bits
// of c: a score error below 2^-23 ||x||, far inside the re-check window.
constexpr int kPieces = 2;
constexpr float kPieceStep = 1.f / 2048.f;
__device__ __forceinline__ void acc_ld32h(uint32_t taddr, uint32_t off2, float scale, float (&v)[32]) {
  float w[32];
  if (kPieces == 3) {
    tmem_ld32(taddr + 2 * off2, w);
    tmem_ld32(taddr + off2, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaf(kPieceStep, w[j], v[j]);
  } else {
    tmem_ld32(taddr + off2, v);
  }
  tmem_ld32(taddr, w);
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = scale * fmaf(kPieceStep, v[j], w[j]);
}
// the same for 16 columns (two pieces): the epilogue of score_sh works in 16-column
// steps to stay inside its register budget
__device__ __forceinline__ void acc_ld16h(uint32_t taddr, uint32_t off2, float scale, float (&v)[16]) {
  float w[16];
  tmem_ld16(taddr + off2, v);
  tmem_ld16(taddr, w);
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = scale * fmaf(kPieceStep, v[j], w[j]);
}
// rows of either kind: `scale` > 0 selects the three-piece half-precision read-back
__device__ __forceinline__ void acc_ld32x(uint32_t taddr, uint32_t off2, float scale, float (&v)[32]) {
  if (scale > 0.f)
    acc_ld32h(taddr, off2, scale, v);
  else
    acc_ld32(taddr, off2, v);
}

// first max of |score| over the node's children (ties to the lowest child
// position, pursuit.py:151), two passes as tmem_abs_argmax (sm100.cuh)
__device__ __forceinline__ void acc_abs_argmax(uint32_t taddr, uint32_t off2, int ncols, int nvalid, float& bestv,
                                               int& best) {
  float m = -1.f;
  int bc = 0;
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    float v[32];
    acc_ld32(taddr + (uint32_t)c0, off2, v);
    if (c0 + 32 > nvalid) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = c0 + j < nvalid ? v[j] : 0.f;
    }
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
      for (int j = 0; j < w; ++j) v[j] = fmaxf(fabsf(v[j]), fabsf(v[j + w]));
    const float t = fabsf(v[0]);
    if (t > m) {
      m = t;
      bc = c0;
    }
  }
  // the TMEM address of tcgen05.ld must be warp-uniform: every lane walks every
  // chunk and resolves the column inside its own winning chunk
  int idx = 0;
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    float v[32];
    acc_ld32(taddr + (uint32_t)c0, off2, v);
    if (c0 == bc) {
      idx = 31;
#pragma unroll
      for (int j = 31; j >= 0; --j) idx = (c0 + j < nvalid && fabsf(v[j]) == m) ? j : idx;
    }
  }
  bestv = m;
  best = bc + idx;
}

// Epilogue of the Gram path (gram_path.cu): the accumulator holds c_v . x for
// the node's cc children; subtract the support's contribution
// sum_k c_k P[S_k][colbase + v] (the patch's current OMP support and
// coefficients), then the first max of |score| in child order
// (pursuit.py:151); `second` is the runner-up's |score| (the near-tie test).
// Iteration 0's root pass also stores every raw score (raw_out) for the later
// root choices.  p < 0: no patch row.
__device__ __forceinline__ void corr_abs_argmax(uint32_t taddr, uint32_t off2, int cc, const ScoreArgs& a, int p,
                                                int colbase, float& bestv, int& best, float& second,
                                                float scale = 0.f) {
  const int T = p >= 0 && a.corr ? a.sup_t : 0;
  const bool vec = ((colbase | (int)a.corr_w) & 3) == 0;
  for (int c0 = 0; c0 < cc; c0 += 32) {
    float v[32];
    acc_ld32x(taddr + (uint32_t)c0, off2, scale, v);   // every lane of the warp takes part
    if (p < 0) continue;
    const int nc = min(32, cc - c0);
    if (a.raw_out) {
      float* dst = a.raw_out + (int64_t)p * a.raw_w + c0;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nc && c0 + j < a.raw_w) dst[j] = v[j];
    }
    if (a.corr_pre != nullptr && T > 0) {   // one precomputed row (gram_corr_kernel)
      const float* row = a.corr_pre + (int64_t)p * a.corr_pre_ld + c0;
      if (nc == 32 && (a.corr_pre_ld & 3) == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 t4 = __ldg(reinterpret_cast<const float4*>(row) + q);
          v[4 * q] -= t4.x;
          v[4 * q + 1] -= t4.y;
          v[4 * q + 2] -= t4.z;
          v[4 * q + 3] -= t4.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nc) v[j] -= __ldg(row + j);
      }
    }
    for (int k = 0; k < (a.corr_pre != nullptr ? 0 : T); ++k) {
      const int sk = __ldg(a.sup + (int64_t)p * a.sup_ld + k);
      const float ck = __ldg(a.supc + (int64_t)p * a.sup_ld + k);
      const float* row = a.corr + (int64_t)sk * a.corr_w + colbase + c0;
      if (vec && nc == 32) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 t4 = __ldg(reinterpret_cast<const float4*>(row) + q);
          v[4 * q] = fmaf(-ck, t4.x, v[4 * q]);
          v[4 * q + 1] = fmaf(-ck, t4.y, v[4 * q + 1]);
          v[4 * q + 2] = fmaf(-ck, t4.z, v[4 * q + 2]);
          v[4 * q + 3] = fmaf(-ck, t4.w, v[4 * q + 3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nc) v[j] = fmaf(-ck, __ldg(row + j), v[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nc) {
        const float m = fabsf(v[j]);
        if (m > bestv) {
          second = bestv;
          bestv = m;
          best = c0 + j;
        } else {
          second = fmaxf(second, m);
        }
      }
  }
}

// Exact FFMA dot of patch row x (ld floats, the padding is zero) with centroid row c, by one warp.
__device__ __forceinline__ float warp_dot(const float* __restrict__ x, const float* __restrict__ c, int ld) {
  float s = 0.f;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* c4 = reinterpret_cast<const float4*>(c);
  // four float4 of each row in flight per lane (a serial loop pays one memory
  // round trip per 128 columns: ~13 us for a 1600-float row, which made the
  // re-checks the bottleneck of the whole pass); per-lane summation order is the
  // plain loop's, so the result is bit-identical
  const int nq = ld / 4;
  int i = (int)(threadIdx.x & 31);
  for (; i < nq; i += 4 * 32) {
    float4 u[4], v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool on = i + 32 * q < nq;
      u[q] = on ? __ldg(x4 + i + 32 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[q] = on ? __ldg(c4 + i + 32 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i + 32 * q < nq) {
        s = fmaf(u[q].x, v[q].x, s);
        s = fmaf(u[q].y, v[q].y, s);
        s = fmaf(u[q].z, v[q].z, s);
        s = fmaf(u[q].w, v[q].w, s);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

// Gram-path near-tie re-check, warp-cooperative (all 32 lanes of a stager warp
// call it).  The tensor cores' fp32 accumulation truncates, leaving ~1e-6 ||x||
// of error on c . x; a row whose two best corrected scores are closer than
// delta = recheck_rel * ||x|| is re-scored exactly (FFMA dots) for every child
// whose approximate score lies within 2 delta of the best -- the others cannot
// win -- and the first maximum in child order is kept (pursuit.py:151).
__device__ __forceinline__ void recheck_near_ties(uint32_t taddr, uint32_t off2, int cc, int cb, const ScoreArgs& a,
                                                  int p, float second, float& bestv, int& best, float scale = 0.f) {
  const int lane = (int)(threadIdx.x & 31);
  // half-precision rows add their quantisation noise to the window: recheck_q * ||x - x16 / s||
  const float delta = p >= 0 ? a.recheck_rel * (float)sqrt(a.xn2[p]) + (a.qerr ? a.recheck_q * a.qerr[p] : 0.f) : 0.f;
  unsigned todo = __ballot_sync(kFull, p >= 0 && bestv - second < delta);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int q = __shfl_sync(kFull, p, src);
    const float lo = __shfl_sync(kFull, bestv, src) - 2.f * __shfl_sync(kFull, delta, src);
    const float* xrow = a.R + (int64_t)q * a.ld;
    float nbv = -1.f;
    int nbest = 0;
    for (int c0 = 0; c0 < cc; c0 += 32) {
      float v[32];
      acc_ld32x(taddr + (uint32_t)c0, off2, scale, v);
      float mine = 0.f;   // row q's raw score of child c0 + lane
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float t = __shfl_sync(kFull, v[j], src);
        if (j == lane) mine = t;
      }
      const int col = c0 + lane;
      float corr = 0.f;
      if (col < cc && a.corr_pre != nullptr)
        corr = a.sup_t > 0 ? __ldg(a.corr_pre + (int64_t)q * a.corr_pre_ld + col) : 0.f;
      else if (col < cc)
        for (int k = 0; k < a.sup_t; ++k) {
          const int sk = __ldg(a.sup + (int64_t)q * a.sup_ld + k);
          corr = fmaf(__ldg(a.supc + (int64_t)q * a.sup_ld + k),
                      __ldg(a.corr + (int64_t)sk * a.corr_w + (cb - a.corr_off) + col), corr);
        }
      unsigned cand = __ballot_sync(kFull, col < cc && fabsf(mine - corr) >= lo);
      while (cand) {
        const int j = __ffs(cand) - 1;
        cand &= cand - 1;
        const float raw = warp_dot(xrow, a.cent + (int64_t)(cb + c0 + j) * a.ld, a.ld);
        const float sj = fabsf(raw - __shfl_sync(kFull, corr, j));
        if (sj > nbv) {   // columns visited in increasing order: strict > keeps the first max
          nbv = sj;
          nbest = c0 + j;
        }
      }
    }
    if (lane == src) {
      bestv = nbv;
      best = nbest;
    }
  }
}

}  // namespace epi
}  // namespace stmp
