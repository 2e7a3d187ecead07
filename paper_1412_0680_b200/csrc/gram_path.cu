// Gram path of the staged OMP encoder: no residual in HBM.
//
// The residual-based pipeline reads and writes r = x - A_S c every iteration
// and rebuilds it from the T support rows: for 1600-dim light-field atoms
// (config 4) that is ~6.4 KB x (T + 3) per patch and iteration, 60 % of the
// step.  With 180 GB of HBM the products every score needs can instead be
// tabulated once per tree: for each level l, P_l[a][v] = c_v . a_a over the
// depth-(l+1) nodes v and all atoms a (config 4: 64 + 4096 + 131072 columns,
// 71 GB; the last level's nodes are single atoms, so P_{L-1} is the Gram matrix
// in leaf order).  Then
//   * a child's score is c_v . r = c_v . x - sum_k c_k P_l[S_k][v]: the score
//     passes multiply the patches x (not r) on the tensor cores and subtract the
//     support's contribution in the epilogue (score_st.cu);
//   * the root scores c_v . x never change: iteration 0 stores them, later
//     iterations only subtract the correction (this file, fused into the update);
//   * the OMP refit needs the Gram column g_k = a . a_{S_k} = P_{L-1}[S_k][pos(a)]
//     and b = a . x (the winner's raw score from the last pass); the inverse
//     Cholesky factor update is the one of the lockstep kernel (encode_update.cu);
//   * ||r||^2 = ||x||^2 - sum_j y_j^2 (y = M A_S^T x), accumulated in f64.  When
//     it falls below rho ||x||^2 the cancellation is large, so the update
//     computes the residual norm explicitly from x and the support rows.
// Semantics are the OMP restatement of SURVEY §8c over pursuit.py:112-162 and
// omp_refit (pursuit.py:235-250); scores differ from the residual form only by
// rounding (c . x and the table products are fp32-accurate), so decisions can
// differ only at near ties.
#include <cublas_v2.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

int g_gram_path = 1;

namespace {

constexpr int kMaxGramK = 16;

// every depth-L node has one leaf whose atom equals the node's centroid bitwise
__global__ void leaf_atom_check_kernel(const float* __restrict__ cent, const float* __restrict__ atoms, int ld,
                                       const int* child_begin, const int* leaf_atom, int64_t v0, int64_t nv,
                                       int* ok) {
  const int64_t v = v0 + blockIdx.x;
  if (blockIdx.x >= nv) return;
  const int a = leaf_atom[child_begin[v]];
  const float* c = cent + v * (int64_t)ld;
  const float* r = atoms + (int64_t)a * ld;
  for (int i = threadIdx.x; i < ld; i += blockDim.x)
    if (__float_as_uint(c[i]) != __float_as_uint(r[i])) atomicExch(ok, 0);
}

__global__ void leaf_pos_kernel(const int* child_begin, const int* leaf_atom, int64_t v0, int64_t nv, int* pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nv) pos[leaf_atom[child_begin[v0 + i]]] = (int)i;
}

// Exact FFMA dot of two zero-padded rows of ld floats (16-byte aligned), one warp.
__device__ __forceinline__ float warp_dot_rows(const float* __restrict__ x, const float* __restrict__ c, int ld) {
  float s = 0.f;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* c4 = reinterpret_cast<const float4*>(c);
  const int lane = (int)(threadIdx.x & 31);
  const int nq = ld / 4;
  // eight float4 of each row in flight per lane before the first FMA (a 1600-float
  // row is 12.5 float4 per lane): the dot is latency-bound otherwise
  int i = lane;
  for (; i + 7 * 32 < nq; i += 8 * 32) {
    float4 u[8], v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      u[q] = __ldg(x4 + i + 32 * q);
      v[q] = __ldg(c4 + i + 32 * q);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s = fmaf(u[q].x, v[q].x, s);
      s = fmaf(u[q].y, v[q].y, s);
      s = fmaf(u[q].z, v[q].z, s);
      s = fmaf(u[q].w, v[q].w, s);
    }
  }
  for (; i < nq; i += 32) {
    const float4 u = __ldg(x4 + i), v = __ldg(c4 + i);
    s = fmaf(u.x, v.x, s);
    s = fmaf(u.y, v.y, s);
    s = fmaf(u.z, v.z, s);
    s = fmaf(u.w, v.w, s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// One warp per patch.  Iteration T (= support size of every active patch):
//   * b = a . x of the atom the last score pass chose, as an exact FFMA dot (the
//     tensor cores' truncating fp32 accumulation leaves ~1e-5 relative error on a
//     1600-term dot: enough for the argmax with the near-tie re-check, not for
//     the refit's right-hand side);
//   * refit on Gram entries: g_k = P_{L-1}[S_k][pos(a)], lane j owning row j of
//     the inverse Cholesky factor M = L^{-1} (as the lockstep kernel in
//     encode_update.cu); ||r||^2 = ||x||^2 - sum_j y_j^2, or the explicit norm
//     when that falls below rho ||x||^2;
//   * if the patch goes on, the next iteration's root choice from the cached
//     root scores s0, with the near-tie re-check (exact dots; the re-scored s0
//     entries are written back).
// Solver state is laid out per patch: S, c, y [N][K], M [N][K(K+1)/2].
// four CTAs per SM (64 registers, ~80 B of spills) for root nodes of <= 64 children: left to
// itself ptxas takes 72-74 registers at T = 5, 9, 10, 11 and those launches run 7-13 % slower
#ifndef STMP_GRAM_MINB
#define STMP_GRAM_MINB 4
#endif
template <int T, int kMaxPer>   // kMaxPer: root children per lane (root_w <= 32 kMaxPer)
__global__ void __launch_bounds__(256, (STMP_GRAM_MINB > 1 && kMaxPer == 2) ? STMP_GRAM_MINB : 1) update_gram_kernel(GramArgs a) {
  pdl_enter();
  __shared__ int hist[256];
  for (int i = threadIdx.x; i < a.root_w; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const bool act = p < a.N && a.active[p] != 0;   // warp-uniform
  if (act) {
    const int K = a.K;
    const int64_t KM = (int64_t)K * (K + 1) / 2;
    const float* xr = a.xr + p * a.ld;
    // every load that does not depend on the solve is issued before the dot, so
    // the patch pays one memory round trip for its state instead of one per use
    // (ld_now: the compiler may not sink them below the dot)
    const int atom = ld_now(a.leaf_sel + p);
    int Sk = 0;
    float ck = 0.f, yk = 0.f;
    if (lane < T) {
      Sk = ld_now(a.S_ws + p * K + lane);
      ck = ld_now(a.c_ws + p * K + lane);
      yk = ld_now(a.yv + p * K + lane);
    }
    float mrow[T + 1];
#pragma unroll
    for (int k = 0; k < T; ++k)
      mrow[k] = (lane < T && k <= lane) ? ld_now(a.Lf + p * KM + lane * (lane + 1) / 2 + k) : 0.f;
    const int pa = __ldg(a.leaf_pos + atom);
    const float gk = lane < T ? ld_now(a.gram + (int64_t)Sk * a.gram_w + pa) : 0.f;   // a . a_{S_k}
    const float gtt = ld_now(a.gram + (int64_t)atom * a.gram_w + pa);
    const double e_prev = ld_now(a.e_ws + p), xn2 = ld_now(a.xn2 + p);
    const float tolp = ld_now(a.tol + p);
    float* s0 = a.s0 + p * a.root_w;
    float s0v[kMaxPer];
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q)
      s0v[q] = (T + 1 < K && lane + 32 * q < a.root_w) ? ld_now(s0 + lane + 32 * q) : 0.f;
    const float b = warp_dot_rows(xr, a.atoms + (int64_t)atom * a.ld, a.ld);
    const bool dup = __any_sync(kFull, lane < T && Sk == atom);
    float w = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k) w = fmaf(mrow[k], __shfl_sync(kFull, gk, k), w);
    const float gc = warp_sum_f(gk * ck);
    const float wsum = warp_sum_f(w * w);
    const float wy = warp_sum_f(w * yk);
    const float score = b - gc;   // a . r (pursuit.py:217 zero-score stop)
    const bool ok = !dup && score != 0.f;
    const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
    const float inv_d = 1.f / dg;
    const float yy = (b - wy) * inv_d;
    // column sums colw_k = sum_j w_j M[j][k] -> lane k; new row T of M and c_new
    float colw = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const float v = warp_sum_f(w * mrow[k]);
      if (lane == k) colw = v;
    }
    const float mt = lane < T ? -inv_d * colw : (lane == T ? inv_d : 0.f);
    const float cn = lane < T ? fmaf(mt, yy, ck) : (lane == T ? inv_d * yy : 0.f);
    const int Sn = lane < T ? Sk : (lane == T ? atom : 0);
    bool act_next = false;
    if (ok) {
      double e = e_prev - (double)yy * yy;
      if (e < (double)a.rho * xn2) {
        // cancellation: the explicit residual norm, lanes over the row
        double s2 = 0.0;
        for (int i = lane; i < a.ld; i += 32) {
          float r = xr[i];
#pragma unroll
          for (int k = 0; k <= T; ++k)
            r = fmaf(-__shfl_sync(kFull, cn, k), __ldg(a.atoms + (int64_t)__shfl_sync(kFull, Sn, k) * a.ld + i), r);
          s2 += (double)r * r;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(kFull, s2, o);
        e = s2;
      }
      const float rn = (float)sqrt(fmax(e, 0.0));
      act_next = (T + 1 < K) && rn > tolp;
      if (lane == 0) {
        a.count[p] = T + 1;
        a.resnorm[p] = rn;
      }
      if (act_next) {
        if (lane <= T) {
          a.Lf[p * KM + T * (T + 1) / 2 + lane] = mt;
          a.c_ws[p * K + lane] = cn;
        }
        if (lane == 0) {
          a.yv[p * K + T] = yy;
          a.S_ws[p * K + T] = atom;
          a.e_ws[p] = e;
        }
      }
    }
    const float cf = ok ? cn : ck;
    if (!act_next) {
      // final rows of the caller's idx / coef (T or T + 1 entries; the rest stay -1 / 0 from init)
      if (lane < (ok ? T + 1 : T)) {
        a.idx[p * K + lane] = Sn;
        a.coef[p * K + lane] = cf;
      }
    }
    if (lane == 0) a.active[p] = act_next ? 1 : 0;
    if (act_next) {
      // next iteration's root choice: s_j = (c_j . x) - sum_k c_k P_0[S_k][j],
      // first max of |s| in child order (pursuit.py:151)
      float sv[kMaxPer], corr[kMaxPer];
      float bestv = -1.f;
      int best = 0;
#pragma unroll
      for (int q = 0; q < kMaxPer; ++q) {
        const int j = lane + 32 * q;
        corr[q] = 0.f;
        sv[q] = 0.f;
        if (32 * q < a.root_w) {
#pragma unroll
          for (int k = 0; k <= T; ++k) {
            const float c_k = __shfl_sync(kFull, cn, k);
            const int s_k = __shfl_sync(kFull, Sn, k);
            if (j < a.root_w) corr[q] = fmaf(c_k, __ldg(a.root_tab + (int64_t)s_k * a.root_w + j), corr[q]);
          }
          if (j < a.root_w) {
            sv[q] = s0v[q] - corr[q];
            if (fabsf(sv[q]) > bestv) {
              bestv = fabsf(sv[q]);
              best = j;
            }
          }
        }
      }
      // warp argmax, ties to the lowest child index
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(kFull, bestv, o);
        const int oj = __shfl_xor_sync(kFull, best, o);
        if (ov > bestv || (ov == bestv && oj < best)) {
          bestv = ov;
          best = oj;
        }
      }
      float second = -1.f;
#pragma unroll
      for (int q = 0; q < kMaxPer; ++q) {
        const int j = lane + 32 * q;
        if (j < a.root_w && j != best) second = fmaxf(second, fabsf(sv[q]));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) second = fmaxf(second, __shfl_xor_sync(kFull, second, o));
      const float delta = a.recheck_rel * (float)sqrt(xn2);
      if (bestv - second < delta) {
        // near tie: exact c_j . x for every child within 2 delta of the best
        const float lo = bestv - 2.f * delta;
        float nbv = -1.f;
        int nbest = 0;
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
          const int j = lane + 32 * q;
          unsigned cand = __ballot_sync(kFull, j < a.root_w && fabsf(sv[q]) >= lo);
          while (cand) {
            const int l = __ffs(cand) - 1;
            cand &= cand - 1;
            const int jj = l + 32 * q;
            const float raw = warp_dot_rows(xr, a.cent + (int64_t)(a.root_cb + jj) * a.ld, a.ld);
            const float sj = fabsf(raw - __shfl_sync(kFull, corr[q], l));
            if (lane == 0) s0[jj] = raw;   // the cache keeps the exact value
            if (sj > nbv) {
              nbv = sj;
              nbest = jj;
            }
          }
        }
        best = nbest;
      }
      if (lane == 0) {
        const int child = a.root_cb + best;
        a.path_ws[p * a.L] = child;
        if (a.path_out) a.path_out[(p * K + (T + 1)) * a.L] = child;
        if (a.ip) add_ip(a.ip, p, a.root_w, a.root_w);
        atomicAdd(&hist[best], 1);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.root_w; i += blockDim.x)
    if (hist[i]) atomicAdd(&a.root_counts[i], hist[i]);
}

#ifndef STMP_CORR_MINB
#define STMP_CORR_MINB 8
#endif
__global__ void __launch_bounds__(256, STMP_CORR_MINB) gram_corr_kernel(int64_t N, const int* active, const int* path_ws, int L,
                                                        int level, const int* child_begin, const int* child_count,
                                                        int col_off, const float* __restrict__ tab, int64_t tab_w,
                                                        const int* S_ws, const float* c_ws, int K, int T,
                                                        float* out, int ld) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= N) return;
  // one round trip for the patch's state (ld_now: issued here, before anything
  // waits), one for its node's child range, then the table rows
  const int act = ld_now(active + p);
  const int node = ld_now(path_ws + p * L + level - 1);
  const int Sk = lane < T ? ld_now(S_ws + p * K + lane) : 0;
  const float ck = lane < T ? ld_now(c_ws + p * K + lane) : 0.f;
  if (!act) return;
  const int cb = __ldg(child_begin + node), cc = __ldg(child_count + node);
  const float* base = tab + (cb - col_off);
  // support rows loaded before the first FMA.  Measured on config 4 (22 launches
  // per encode): 1 row 301 us per launch, 4 rows 274, 6 rows 270, 8 rows 345 (spills
  // at the 32-register bound), 8 / 12 rows at 40 / 48 registers 314 / 397: beyond a
  // few rows in flight the random table rows (TLB reach, DRAM pages), not the load
  // latency, set the pace, and occupancy matters more.
#ifndef STMP_CORR_BATCH
#define STMP_CORR_BATCH 6
#endif
  constexpr int kB = STMP_CORR_BATCH;
  for (int j0 = 0; j0 < cc; j0 += 32) {
    const int j = j0 + lane;
    float acc = 0.f;
    for (int k0 = 0; k0 < T; k0 += kB) {
      float v[kB], c_k[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int k = min(k0 + q, T - 1);
        const int s_k = __shfl_sync(kFull, Sk, k);
        c_k[q] = __shfl_sync(kFull, ck, k);
        v[q] = j < cc ? __ldg(base + (int64_t)s_k * tab_w + j) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (k0 + q < T) acc = fmaf(c_k[q], v[q], acc);
    }
    if (j < cc) out[p * ld + j] = acc;
  }
}

}  // namespace

cudaError_t launch_gram_corr(int64_t N, const int* active, const int* path_ws, int L, int level,
                             const int* child_begin, const int* child_count, int col_off, const float* tab,
                             int64_t tab_w, const int* S_ws, const float* c_ws, int K, int T, float* out, int ld,
                             cudaStream_t st) {
  return launch_kernel(gram_corr_kernel, (unsigned)((N + 7) / 8), 256, 0, st, true, N, active, path_ws, L, level,
                       child_begin, child_count, col_off, tab, tab_w, S_ws, c_ws, K, T, out, ld);
}

namespace {

cublasHandle_t blas_handle() {
  static cublasHandle_t h = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) h = nullptr;
    // plain fp32 FFMA GEMMs: the tables must be fp32-accurate (no TF32)
    if (h) cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);
  });
  return h;
}

}  // namespace

bool gram_path_supported(const DictHandle* d, const TreeHandle* t, int K, int method) {
  if (t == nullptr || method != kMethodOMP || K > kMaxGramK || g_gram_path == 0 || t->levels < 2) return false;
  if (t->max_leaf_children != 1 || t->num_leaves != d->m || t->leaf_pos == nullptr) return false;
  if (t->root_children > 256) return false;
  if (g_gram_path == 2) return true;
  // auto: rows much wider than the nodes, where the residual traffic dominates
  int maxk = 0;
  for (int k : t->branching) maxk = std::max(maxk, k);
  return d->n >= 256 && d->n >= 8 * maxk;
}

bool ensure_pair_tables(TreeHandle* t, const DictHandle* d, cudaStream_t st) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (t->pair_tried) return !t->pair_tables.empty();
  t->pair_tried = true;
  const int L = t->levels;
  const int64_t m = d->m;
  // the last level's centroids must be the atoms themselves
  {
    int* ok = nullptr;
    if (cudaMalloc(&ok, sizeof(int)) != cudaSuccess) return false;
    const int one = 1;
    cudaMemcpyAsync(ok, &one, sizeof(int), cudaMemcpyHostToDevice, st);
    const int64_t v0 = t->level_offsets[L], nv = t->level_offsets[L + 1] - v0;
    leaf_atom_check_kernel<<<(unsigned)nv, 128, 0, st>>>(t->cent, d->atoms, d->ld, t->child_begin, t->leaf_atom, v0,
                                                         nv, ok);
    note_launch();
    int h = 0;
    cudaMemcpyAsync(&h, ok, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(ok);
    t->leaf_is_atom = (e == cudaSuccess && h) ? 1 : 0;
    if (!t->leaf_is_atom) return false;
  }
  std::vector<int64_t> width(L);
  size_t total = 0;
  for (int l = 0; l < L; ++l) {
    width[l] = t->level_offsets[l + 2] - t->level_offsets[l + 1];
    total += (size_t)m * width[l] * sizeof(float);
  }
  size_t free_b = 0, tot_b = 0;
  if (cudaMemGetInfo(&free_b, &tot_b) != cudaSuccess || total + (4ull << 30) > free_b) return false;
  cublasHandle_t h = blas_handle();
  if (h == nullptr || cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return false;
  std::vector<float*> tabs(L, nullptr);
  bool good = true;
  for (int l = 0; l < L && good; ++l) {
    if (cudaMalloc(&tabs[l], (size_t)m * width[l] * sizeof(float)) != cudaSuccess) {
      good = false;
      break;
    }
    // P_l [m][W] row-major = (C_l A^T) column-major W x m: cent rows of depth l + 1
    const float* cent = t->cent + t->level_offsets[l + 1] * (int64_t)d->ld;
    const float one = 1.f, zero = 0.f;
    const int64_t blk = 8192;
    for (int64_t a0 = 0; a0 < m && good; a0 += blk) {
      const int mb = (int)std::min(blk, m - a0);
      good = cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)width[l], mb, d->n, &one, cent, d->ld,
                         d->atoms + a0 * d->ld, d->ld, &zero, tabs[l] + a0 * width[l], (int)width[l]) ==
             CUBLAS_STATUS_SUCCESS;
    }
  }
  if (good) good = cudaStreamSynchronize(st) == cudaSuccess;
  if (!good) {
    for (float* p : tabs) cudaFree(p);
    cudaGetLastError();
    return false;
  }
  t->pair_tables = tabs;
  t->pair_width = width;
  // fp16 piece tables of the levels >= 1 for the half-precision passes (score_sh.cu);
  // without them (shape or memory) the passes stay on fp32 rows
  bool fits = true;
  for (int l = 1; l < L; ++l) fits = fits && score_sh_fits(t->ld, t->staged_levels[l].npad);
  if (fits) {
    std::vector<uint8_t*> ht(L, nullptr);
    for (int l = 1; l < L && fits; ++l) fits = (ht[l] = build_half_table(t, l, st)) != nullptr;
    if (fits)
      t->half_tables = ht;
    else
      for (uint8_t* p : ht) cudaFree(p);
  }
  return true;
}

// leaf_pos (host-side at tree creation would need the leaf order; done here on the device)
bool build_leaf_pos(TreeHandle* t, int64_t m, cudaStream_t st) {
  const int L = t->levels;
  const int64_t v0 = t->level_offsets[L], nv = t->level_offsets[L + 1] - v0;
  if (t->max_leaf_children != 1 || nv != m || t->num_leaves != m) return false;
  if (cudaMalloc(&t->leaf_pos, m * sizeof(int)) != cudaSuccess) {
    t->leaf_pos = nullptr;
    return false;
  }
  leaf_pos_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(t->child_begin, t->leaf_atom, v0, nv, t->leaf_pos);
  note_launch();
  return cudaGetLastError() == cudaSuccess;
}

void free_pair_tables(TreeHandle* t) {
  for (float* p : t->pair_tables) cudaFree(p);
  t->pair_tables.clear();
  for (uint8_t* p : t->half_tables) cudaFree(p);
  t->half_tables.clear();
  cudaFree(t->leaf_pos);
  t->leaf_pos = nullptr;
}

cudaError_t launch_update_gram(const GramArgs& a, cudaStream_t st) {
  const unsigned blocks = (unsigned)((a.N + 7) / 8);
  switch (a.iter) {
#define STMP_GRAM_CASE(t)                                                                    \
  case t:                                                                                    \
    return a.root_w <= 64 ? launch_kernel(update_gram_kernel<t, 2>, blocks, 256, 0, st, true, a) \
                          : launch_kernel(update_gram_kernel<t, 8>, blocks, 256, 0, st, true, a);
    STMP_GRAM_CASE(0) STMP_GRAM_CASE(1) STMP_GRAM_CASE(2) STMP_GRAM_CASE(3) STMP_GRAM_CASE(4) STMP_GRAM_CASE(5)
    STMP_GRAM_CASE(6) STMP_GRAM_CASE(7) STMP_GRAM_CASE(8) STMP_GRAM_CASE(9) STMP_GRAM_CASE(10) STMP_GRAM_CASE(11)
    STMP_GRAM_CASE(12) STMP_GRAM_CASE(13) STMP_GRAM_CASE(14) STMP_GRAM_CASE(15)
#undef STMP_GRAM_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace stmp
