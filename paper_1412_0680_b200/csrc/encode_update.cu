// Per-patch kernels of the staged encoder: init (padded residual copy,
// tolerance, root bin count) and update (leaf choice + MP step or OMP refit).
//
// A group of G = 8 (or 32 for wide rows) lanes owns one patch.  Rows are
// read in an interleaved layout -- lane gl touches the 16-B chunks gl, gl+G,
// gl+2G, ... -- so one warp load instruction covers whole 128-B lines of a
// few rows (the L1 wavefront count per row is minimal).  Dot products are
// group reductions; the small triangular solves of the OMP refit are
// column sweeps in which lane j owns rows j, j+G, ... of the Cholesky factor.
// Semantics: pkg/src/stmp/pursuit.py:207-221 (MP) and the SURVEY §8c OMP
// restatement over omp_refit (pursuit.py:235-250).
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

namespace {

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  return G >= 32 ? kFull : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
}

// Sum over the G lanes of this patch group.  The mask names only the group's
// own lanes: groups of one warp diverge (different patches stop at different
// iterations), so a full-warp mask would wait for lanes that never arrive.
template <int G>
__device__ __forceinline__ float group_sum(float v) {
  const unsigned mask = group_mask<G>();
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// Count the patches that stay active into the root bin: one fire-and-forget
// atomic per warp (called by every lane; `act` true on at most one lane per
// patch group), spread over kRootStripes counters so the adds of a whole grid
// do not serialise on one L2 address.  scan_kernel folds the stripes.
__device__ __forceinline__ void count_root(bool act, int* stripes) {
  if (stripes == nullptr) return;   // root pass runs over the batch in patch order
  const unsigned m = __ballot_sync(kFull, act);
  if (m && (int)(threadIdx.x & 31) == __ffs(m) - 1)
    atomicAdd(&stripes[(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) & (kRootStripes - 1)], __popc(m));
}

// Row slice of this lane: chunks gl + G*i (i < CPL) of F 16-byte chunks.
template <int G, int CPL>
struct Slice {
  float v[CPL * 4];

  __device__ __forceinline__ void load(const float* __restrict__ row, int gl, int F) {
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = gl + G * i;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < F) q = __ldg(reinterpret_cast<const float4*>(row) + c);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
  }
  __device__ __forceinline__ void store(float* row, int gl, int F) const {
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = gl + G * i;
      if (c < F) reinterpret_cast<float4*>(row)[c] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
  __device__ __forceinline__ float dot(const Slice& o) const {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CPL * 4; ++i) s = fmaf(v[i], o.v[i], s);
    return s;
  }
};

// ------------------------------------------------------------------ init
template <int G, int CPL>
__global__ void __launch_bounds__(128) init_kernel(UpdateArgs a) {
  pdl_enter();
  const int gpb = blockDim.x / G;
  const int64_t p = (int64_t)blockIdx.x * gpb + threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int F = a.ld >> 2;
  const bool inb = p < a.N;
  Slice<G, CPL> x;
  float ss = 0.f;
  // rows already padded and 16-byte aligned: vector loads
  const bool vec = a.n == a.ld && (a.ldx & 3) == 0 && ((uintptr_t)a.X & 15) == 0;
  if (inb) {
    const float* xp = a.X + p * a.ldx;
    if (vec) {
      x.load(xp, gl, F);
    } else {
#pragma unroll
      for (int i = 0; i < CPL; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int d = 4 * (gl + G * i) + k;
          x.v[4 * i + k] = d < a.n ? __ldg(xp + d) : 0.f;
        }
    }
#pragma unroll
    for (int i = 0; i < CPL * 4; ++i) ss = fmaf(x.v[i], x.v[i], ss);
    if (a.xn2) {   // Gram path: ||x||^2 in f64 (gram_path.cu)
      double ds = 0.0;
#pragma unroll
      for (int i = 0; i < CPL * 4; ++i) ds += (double)x.v[i] * x.v[i];
#pragma unroll
      for (int o = G >> 1; o; o >>= 1) ds += __shfl_xor_sync(group_mask<G>(), ds, o);
      if (gl == 0) {
        a.xn2[p] = ds;
        a.e_ws[p] = ds;
      }
    }
    if (a.R) x.store(a.R + p * a.ld, gl, F);
    if (a.X2) x.store(const_cast<float*>(a.X2) + p * a.ld2, gl, F);
    if (a.x16) {
      // fp16 row copy for the Gram path's level passes (score_sh.cu): s = 2^(15 - e)
      // with max |x| = f 2^e, f in [0.5, 1), so the largest element lands in
      // [2^14, 2^15) and elements down to 2^-28 of it stay normal halfs
      float mx = 0.f;
#pragma unroll
      for (int i = 0; i < CPL * 4; ++i) mx = fmaxf(mx, fabsf(x.v[i]));
#pragma unroll
      for (int o = G >> 1; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(group_mask<G>(), mx, o));
      int e = 0;
      if (mx > 0.f && mx < 3.0e38f) frexpf(mx, &e);
      const int sh = max(-100, min(100, 15 - e));
      const float s = ldexpf(1.f, sh), is = ldexpf(1.f, -sh);
      uint2* out = reinterpret_cast<uint2*>(a.x16 + p * a.ld);
      float err2 = 0.f;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        const int c = gl + G * i;
        if (c < F) {
          unsigned short h[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __half hv = __float2half_rn(x.v[4 * i + k] * s);
            const float d = x.v[4 * i + k] - __half2float(hv) * is;
            err2 = fmaf(d, d, err2);
            h[k] = __half_as_ushort(hv);
          }
          out[c] = make_uint2((unsigned)h[0] | ((unsigned)h[1] << 16), (unsigned)h[2] | ((unsigned)h[3] << 16));
        }
      }
#pragma unroll
      for (int o = G >> 1; o; o >>= 1) err2 += __shfl_xor_sync(group_mask<G>(), err2, o);
      if (gl == 0) {
        a.inv_scale[p] = is;
        a.qerr[p] = sqrtf(err2);
      }
    }
  }
  ss = group_sum<G>(ss);
  const float xn = sqrtf(ss);
  bool act = false;
  if (inb) {
    const float tol = a.tol_abs >= 0.f ? a.tol_abs : kRelTol * xn;
    act = xn > tol;   // pursuit.py:214 on the first iteration
    if (gl == 0) {
      a.tol[p] = tol;
      a.resnorm[p] = xn;
      a.count[p] = 0;
      a.active[p] = act ? 1 : 0;
      if (a.ip) { a.ip[2 * p] = 0; a.ip[2 * p + 1] = 0; }
    }
    for (int j = gl; j < a.K; j += G) { a.idx[p * a.K + j] = -1; a.coef[p * a.K + j] = 0.f; }
    if (a.path_out)
      for (int j = gl; j < a.K * a.L; j += G) a.path_out[p * a.K * a.L + j] = -1;
  }
  count_root(act && gl == 0, a.root_count);
}

// ------------------------------------------------------------------ update
// Shared scratch per patch group (floats): S[K] | c[K] | y[K] | M[K(K+1)/2] | g[K] | w[K] | cn[K]
__host__ __device__ inline int upd_scalar_floats(int K) { return (6 * K + K * (K + 1) / 2 + 3) & ~3; }

// (no minimum-blocks bound: an explicit one, even 1, makes ptxas spend more
// registers -- 88 instead of 60 for <8, 2> -- and costs config 1 MP 0.5 ms)
template <int G, int CPL>
__global__ void __launch_bounds__(128) update_kernel(UpdateArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) float upd_smem[];
  const int gpb = blockDim.x / G;
  const int grp = threadIdx.x / G;
  const int64_t p = (int64_t)blockIdx.x * gpb + grp;
  const int gl = threadIdx.x % G;
  const unsigned gmask = group_mask<G>();
  const int K = a.K;
  const int F = a.ld >> 2;
  float* gs = upd_smem + grp * upd_scalar_floats(K);
  int* S_s = reinterpret_cast<int*>(gs);
  float* c_s = gs + K;       // previous coefficients
  float* y_s = c_s + K;      // L y = A_S x (forward-substituted rhs); reused as the back-sweep rhs
  float* L_s = y_s + K;      // packed inverse Cholesky factor M = L^{-1}, rows 0..t-1
  float* g_s = L_s + K * (K + 1) / 2;  // Gram column of the new atom
  float* w_s = g_s + K;      // w = M g
  float* cn_s = w_s + K;     // new coefficients
  const bool inb = p < a.N;
  bool act = inb && a.active[p];
  using Sl = Slice<G, CPL>;
  // every independent load of the patch is issued before the active test
  // (one round trip instead of two); out-of-range groups read patch 0
  const int64_t pc = inb ? p : 0;
  const int t = a.count[pc];
  const int lsel = a.leaf_sel[pc];
  const bool omp = a.method == kMethodOMP;
  Sl r, x;
  if (omp) {
    x.load(a.X2 + pc * a.ld2, gl, F);
    // the patch's solver state -> shared (bounded by K, not t, so the loads
    // do not wait for the count)
    for (int i = gl; i < K; i += G) {
      S_s[i] = a.idx[pc * K + i];
      c_s[i] = a.coef[pc * K + i];
      y_s[i] = a.yv[pc * K + i];
    }
    const float* Lp = a.Lf + pc * (int64_t)(K * (K + 1) / 2);
    for (int i = gl; i < K * (K + 1) / 2; i += G) L_s[i] = Lp[i];
  }
  if (act) {
    if (!omp || lsel < 0) r.load(a.R_in + p * a.ld, gl, F);
    // leaf choice: single-atom leaves were resolved by the last score pass;
    // otherwise max |a . r| over the node's atoms, ties to the lowest atom index
    int atom = lsel;
    if (lsel < 0) {
      const int node = -1 - lsel;
      const int cb = __ldg(a.child_begin + node), cc = __ldg(a.child_count + node);
      float bestv = -1.f;
      atom = __ldg(a.leaf_atom + cb);
      for (int j = 0; j < cc; ++j) {
        const int aj = __ldg(a.leaf_atom + cb + j);
        Sl v;
        v.load(a.atoms + (int64_t)aj * a.ld, gl, F);
        const float m = fabsf(group_sum<G>(v.dot(r)));
        if (m > bestv || (m == bestv && aj < atom)) { bestv = m; atom = aj; }
      }
    }
    Sl av;
    av.load(a.atoms + (int64_t)atom * a.ld, gl, F);
    int32_t* S = a.idx + p * K;
    if (!omp) {
      const float s = group_sum<G>(av.dot(r));
      if (s == 0.f) {
        act = false;   // pursuit.py:217
      } else {
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < CPL * 4; ++i) { r.v[i] = fmaf(-s, av.v[i], r.v[i]); s2 = fmaf(r.v[i], r.v[i], s2); }
        r.store(a.R + p * a.ld, gl, F);
        const float rn = sqrtf(group_sum<G>(s2));
        if (gl == 0) {
          S[t] = atom;
          a.coef[p * K + t] = s;
          a.count[p] = t + 1;
          a.resnorm[p] = rn;
        }
        act = (t + 1 < K) && rn > a.tol[p];
      }
    } else {
      __syncwarp(gmask);
      bool dup = false;
      for (int j = 0; j < t; ++j) dup |= (S_s[j] == atom);
      const float bt = group_sum<G>(av.dot(x));
      const float gtt = group_sum<G>(av.dot(av));
      // Gram column of the new atom against the support: independent dots,
      // several rows' loads in flight at once
#pragma unroll 4
      for (int j = 0; j < t; ++j) {
        Sl sv;
        sv.load(a.atoms + (int64_t)S_s[j] * a.ld, gl, F);
        const float g = group_sum<G>(sv.dot(av));
        if (gl == (j % G)) g_s[j] = g;
      }
      __syncwarp(gmask);
      float gc = 0.f;
      for (int j = gl; j < t; j += G) gc = fmaf(g_s[j], c_s[j], gc);
      gc = group_sum<G>(gc);         // a . (A_S c_prev)
      const float score = bt - gc;   // a . r for r = x - A_S c_prev (pursuit.py:217 check)
      if (dup || score == 0.f) {
        act = false;   // re-selection (or a zero score) ends the loop
      } else {
        // Inverse-Cholesky refit: M = L^{-1} is kept per patch (G_S^{-1} = M^T M),
        // so every step is a small mat-vec that the G lanes share instead of a
        // sequential triangular sweep.
        //   w = M g,  d = sqrt(a.a + ridge - w.w),  y_t = (b_t - w.y) / d,
        //   new row of M: (-(1/d) w^T M, 1/d),  c = M^T y.
        for (int j = gl; j < t; j += G) {
          const float* Mj = L_s + j * (j + 1) / 2;
          float acc = 0.f;
          for (int k = 0; k <= j; ++k) acc = fmaf(Mj[k], g_s[k], acc);
          w_s[j] = acc;
        }
        __syncwarp(gmask);
        float wsum = 0.f, wy = 0.f;
        for (int j = gl; j < t; j += G) {
          wsum = fmaf(w_s[j], w_s[j], wsum);
          wy = fmaf(w_s[j], y_s[j], wy);
        }
        wsum = group_sum<G>(wsum);
        wy = group_sum<G>(wy);
        const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
        const float inv_d = 1.f / dg;
        const float yy = (bt - wy) * inv_d;
        float* Mt = a.Lf + p * (int64_t)(K * (K + 1) / 2) + t * (t + 1) / 2;
        for (int k = gl; k <= t; k += G) {
          float mk = inv_d, ck = 0.f;
          if (k < t) {
            float s1 = 0.f;
            for (int j = k; j < t; ++j) {
              const float Mjk = L_s[j * (j + 1) / 2 + k];
              s1 = fmaf(w_s[j], Mjk, s1);
              ck = fmaf(Mjk, y_s[j], ck);
            }
            mk = -inv_d * s1;
          }
          ck = fmaf(mk, yy, ck);
          Mt[k] = mk;
          cn_s[k] = ck;
          a.coef[p * K + k] = ck;
        }
        __syncwarp(gmask);
        // residual r = x - A_S c with the new atom
        const float ct = cn_s[t];
#pragma unroll
        for (int i = 0; i < CPL * 4; ++i) r.v[i] = fmaf(-ct, av.v[i], x.v[i]);
#pragma unroll 4
        for (int j = 0; j < t; ++j) {
          Sl sv;
          sv.load(a.atoms + (int64_t)S_s[j] * a.ld, gl, F);
          const float cj = cn_s[j];
#pragma unroll
          for (int i = 0; i < CPL * 4; ++i) r.v[i] = fmaf(-cj, sv.v[i], r.v[i]);
        }
        r.store(a.R + p * a.ld, gl, F);
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < CPL * 4; ++i) s2 = fmaf(r.v[i], r.v[i], s2);
        const float rn = sqrtf(group_sum<G>(s2));
        if (gl == 0) {
          a.yv[p * (int64_t)K + t] = yy;
          S[t] = atom;
          a.count[p] = t + 1;
          a.resnorm[p] = rn;
        }
        act = (t + 1 < K) && rn > a.tol[p];
      }
    }
    if (gl == 0) a.active[p] = act ? 1 : 0;
  }
  count_root(act && gl == 0, a.root_count);
}

// ------------------------------------------------------------------ OMP update, wide rows
// One CTA of 128 threads per patch for rows too wide for a lane group to hold
// (config 4: 1600 floats): each thread keeps CPT 16-byte chunks of a row, so a
// row slice is 4*CPT registers instead of 52 and 12-20 warps stay resident per
// SM (the 32-lane version ran at 8).  Every dot product is one warp butterfly
// plus a 4-entry shared-memory sum; the small solve (t <= K) runs redundantly
// in every thread from shared memory, so it needs no further communication.
// Same state layout and semantics as update_kernel's OMP branch.
template <int CPT>
__global__ void __launch_bounds__(128) update_wide_kernel(UpdateArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) float wsm[];
  const int K = a.K;
  const int64_t p = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int F = a.ld >> 2;
  int* S_s = reinterpret_cast<int*>(wsm);           // [K]
  float* c_s = wsm + K;                             // [K] current coefficients
  float* y_s = c_s + K;                             // [K]
  float* M_s = y_s + K;                             // [K(K+1)/2] packed M = L^{-1}
  float* g_s = M_s + K * (K + 1) / 2;               // [K + 2] Gram column, a.a, a.x
  float* red = g_s + K + 2;                         // [4][K + 2] per-warp partial sums
  float* cn_s = red + 4 * (K + 2);                  // [K] new coefficients
  __shared__ int s_atom;
  if (!a.active[p]) return;   // CTA-uniform
  const int t = a.count[p];
  const int lsel = a.leaf_sel[p];
  for (int i = tid; i < K; i += 128) {
    S_s[i] = a.idx[p * K + i];
    c_s[i] = a.coef[p * K + i];
    y_s[i] = a.yv[p * K + i];
  }
  for (int i = tid; i < K * (K + 1) / 2; i += 128) M_s[i] = a.Lf[p * (int64_t)(K * (K + 1) / 2) + i];
  auto load = [&](const float* row, float4 (&v)[CPT]) {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = tid + 128 * i;
      v[i] = c < F ? __ldg(reinterpret_cast<const float4*>(row) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto dot = [&](const float4 (&u)[CPT], const float4 (&v)[CPT]) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      s = fmaf(u[i].x, v[i].x, s);
      s = fmaf(u[i].y, v[i].y, s);
      s = fmaf(u[i].z, v[i].z, s);
      s = fmaf(u[i].w, v[i].w, s);
    }
    return s;
  };
  // warp butterfly, lane 0 stores the warp's partial of value j
  auto part = [&](float s, int j) {
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) red[warp * (K + 2) + j] = s;
  };
  float4 x[CPT], av[CPT];
  load(a.X2 + p * a.ld2, x);
  int atom = lsel;
  if (lsel < 0) {   // multi-atom leaf: max |a . r|, ties to the lowest atom index
    float4 r[CPT];
    load(a.R_in + p * a.ld, r);
    const int node = -1 - lsel;
    const int cb = __ldg(a.child_begin + node), cc = __ldg(a.child_count + node);
    float bestv = -1.f;
    atom = __ldg(a.leaf_atom + cb);
    for (int j = 0; j < cc; ++j) {
      const int aj = __ldg(a.leaf_atom + cb + j);
      float4 v[CPT];
      load(a.atoms + (int64_t)aj * a.ld, v);
      __syncthreads();   // red is reused
      part(dot(v, r), 0);
      __syncthreads();
      const float mv = fabsf(red[0] + red[K + 2] + red[2 * (K + 2)] + red[3 * (K + 2)]);
      if (mv > bestv || (mv == bestv && aj < atom)) { bestv = mv; atom = aj; }
    }
  }
  load(a.atoms + (int64_t)atom * a.ld, av);
  __syncthreads();   // state in shared memory
  // Gram column against the support, a.a and a.x: one partial per value and warp
  for (int k = 0; k < t; ++k) {
    float4 sv[CPT];
    load(a.atoms + (int64_t)S_s[k] * a.ld, sv);
    part(dot(sv, av), k);
  }
  part(dot(av, av), t);
  part(dot(av, x), t + 1);
  __syncthreads();
  for (int j = tid; j < t + 2; j += 128)
    g_s[j] = red[j] + red[(K + 2) + j] + red[2 * (K + 2) + j] + red[3 * (K + 2) + j];
  __syncthreads();
  bool dup = false;
  for (int k = 0; k < t; ++k) dup |= S_s[k] == atom;
  float gc = 0.f;
  for (int k = 0; k < t; ++k) gc = fmaf(g_s[k], c_s[k], gc);
  const float gtt = g_s[t], bt = g_s[t + 1];
  const float score = bt - gc;   // a . r for r = x - A_S c_prev (pursuit.py:217 check)
  bool act = true;
  if (dup || score == 0.f) {
    act = false;   // re-selection (or a zero score) ends the loop
  } else {
    // inverse-Cholesky refit (same algebra as update_kernel), every thread redundantly:
    //   w = M g, d = sqrt(a.a + ridge - w.w), y_t = (b_t - w.y) / d,
    //   new row of M: (-(1/d) w^T M, 1/d), c_new = c_prev + m_t y_t
    float wsum = 0.f, wy = 0.f;
    for (int j = 0; j < t; ++j) {
      const float* Mj = M_s + j * (j + 1) / 2;
      float w = 0.f;
      for (int k = 0; k <= j; ++k) w = fmaf(Mj[k], g_s[k], w);
      red[j] = w;   // (all warps' partial sums were consumed above)
      wsum = fmaf(w, w, wsum);
      wy = fmaf(w, y_s[j], wy);
    }
    const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
    const float inv_d = 1.f / dg;
    const float yy = (bt - wy) * inv_d;
    __syncthreads();   // w (red) written identically by every thread
    float* Mt = a.Lf + p * (int64_t)(K * (K + 1) / 2) + t * (t + 1) / 2;
    for (int k = tid; k <= t; k += 128) {
      float mk = inv_d;
      if (k < t) {
        float s1 = 0.f;
        for (int j = k; j < t; ++j) s1 = fmaf(red[j], M_s[j * (j + 1) / 2 + k], s1);
        mk = -inv_d * s1;
      }
      const float ck = k < t ? fmaf(mk, yy, c_s[k]) : inv_d * yy;
      Mt[k] = mk;
      cn_s[k] = ck;
      a.coef[p * K + k] = ck;
    }
    if (tid == 0) s_atom = atom;
    __syncthreads();
    // residual r = x - A_S c - c_t a (support rows again, now from L2)
    float4 r[CPT];
    const float ct = cn_s[t];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      r[i].x = fmaf(-ct, av[i].x, x[i].x);
      r[i].y = fmaf(-ct, av[i].y, x[i].y);
      r[i].z = fmaf(-ct, av[i].z, x[i].z);
      r[i].w = fmaf(-ct, av[i].w, x[i].w);
    }
    for (int k = 0; k < t; ++k) {
      float4 sv[CPT];
      load(a.atoms + (int64_t)S_s[k] * a.ld, sv);
      const float ck = cn_s[k];
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        r[i].x = fmaf(-ck, sv[i].x, r[i].x);
        r[i].y = fmaf(-ck, sv[i].y, r[i].y);
        r[i].z = fmaf(-ck, sv[i].z, r[i].z);
        r[i].w = fmaf(-ck, sv[i].w, r[i].w);
      }
    }
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = tid + 128 * i;
      if (c < F) reinterpret_cast<float4*>(a.R + p * a.ld)[c] = r[i];
    }
    part(dot(r, r), 0);
    __syncthreads();
    const float rn = sqrtf(red[0] + red[K + 2] + red[2 * (K + 2)] + red[3 * (K + 2)]);
    act = (t + 1 < K) && rn > a.tol[p];
    if (tid == 0) {
      a.yv[p * (int64_t)K + t] = yy;
      a.idx[p * K + t] = s_atom;
      a.count[p] = t + 1;
      a.resnorm[p] = rn;
    }
  }
  if (tid == 0) a.active[p] = act ? 1 : 0;
  if (tid == 0 && act && a.root_count)
    atomicAdd(&a.root_count[blockIdx.x & (kRootStripes - 1)], 1);
}

// ------------------------------------------------------------------ OMP update, K <= 8
// Lockstep specialisation for the common small-K case with an atom Gram table.
// In the staged pipeline every patch still active at iteration T holds exactly
// T atoms, so T is a template parameter: every loop over the support is fully
// unrolled with no support-size predicates.  The 8 lanes of a patch group own
// one row each of the inverse Cholesky factor M (and the matching y_j, c_j),
// every lane holds the Gram column, and the column sums of the refit are
// butterfly all-reductions.  Solver state is laid out [entry][patch] (S_ws,
// c_ws, yv, Lf), so one entry of the 4 patches of a warp is one sector; the
// caller-visible idx / coef rows are written once, when the patch stops.
#ifndef STMP_OMP8_MINB
#define STMP_OMP8_MINB 8
#endif
#ifndef STMP_OMP8_MINB0
#define STMP_OMP8_MINB0 10
#endif
#ifndef STMP_OMP8_MINBW
#define STMP_OMP8_MINBW 5   // rows of 96-160 floats
#endif
// The Gram column is T group dot products against the support rows, which the residual rebuild
// reads again (from L1 / L2).
// G = 16 lanes per patch (rows of <= 128 floats) lifts the support limit to 16.
//
// The solve runs warp-uniformly: a warp whose patches are all inactive returns,
// otherwise every lane executes the refit (results of inactive patches are
// never stored), so every shuffle is a plain full-warp SHFL with no divergence
// handling.  The reductions are shaped to the refit's data flow:
//   * the T + 2 dot products (g_k, a.a, a.x) are one reduce-scatter over the
//     group (lane k receives value k) followed by broadcasts of g;
//   * w_j = sum_k M[j][k] g_k is lane-local (lane j owns row j of M);
//   * the column sums sum_j w_j M[j][k] of the new row are one reduce-scatter
//     (lane k receives column k, which is exactly the entry it stores);
//   * c_new = c_prev + m_T y_T reuses the stored c_prev (c_prev = M^T y over
//     the previous rows), so no M^T y sweep is needed.
template <int G>
__device__ __forceinline__ float gsum_full(float v) {
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Reduce-scatter over the G lanes of a group (all 32 lanes call): on return
// lane gl holds the group sum of p[gl].
template <int G>
__device__ __forceinline__ float group_reduce_scatter(float (&p)[G], int gl) {
#pragma unroll
  for (int o = G >> 1; o >= 1; o >>= 1) {
    const bool upper = (gl & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const float send = upper ? p[j] : p[j + o];
      const float keep = upper ? p[j + o] : p[j];
      p[j] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
  return p[0];
}

template <int G>
__device__ __forceinline__ float group_bcast(float v, int k) { return __shfl_sync(kFull, v, k, G); }

// Reduce-scatter of NR * G values over the G lanes of a group: on return r[i]
// on lane gl holds the group sum of p[gl + G * i].
template <int G, int NR>
__device__ __forceinline__ void group_reduce_scatter_n(float (&p)[NR * G], int gl, float (&r)[NR]) {
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    float q[G];
#pragma unroll
    for (int k = 0; k < G; ++k) q[k] = p[G * i + k];
    r[i] = group_reduce_scatter<G>(q, gl);
  }
}

// Lane gl owns rows gl + G * i (i < NR) of the inverse Cholesky factor M (and the
// matching y_j, c_j): NR = 1 while the support fits the group, 2 up to 2G atoms.
template <int G, int CPL, int T>
__global__ void __launch_bounds__(128, CPL <= 2 ? (T == 0 ? STMP_OMP8_MINB0 : (T < G ? STMP_OMP8_MINB : 5))
                                                : STMP_OMP8_MINBW)
    update_omp8_kernel(UpdateArgs a) {
  constexpr int NR = T < G ? 1 : 2;     // Cholesky rows per lane
  constexpr int NV = NR * G;            // reduce-scatter width
  static_assert(T < 2 * G, "lockstep support index must fit two rows per lane");
  pdl_enter();
  const int64_t N = a.N;
  const int64_t p = (int64_t)blockIdx.x * (128 / G) + threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const int K = a.K;
  constexpr int F = G * CPL;   // 16-byte chunks per row: ld is a multiple of 32, so F == G * CPL exactly
  using Sl = Slice<G, CPL>;
  const bool inb = p < N;
  const int64_t pc = inb ? p : 0;
  // ---- every independent load of the patch, issued together and before the
  // activity test (volatile loads: the compiler may not sink them into the
  // branch, which would add a dependent round trip)
  const int act_in = inb ? sm100::ld_now(a.active + pc) : 0;
  const int lsel = sm100::ld_now(a.leaf_sel + pc);
  const float tol_p = sm100::ld_now(a.tol + pc);   // needed last: issued with the first loads
  Sl x;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int ch = gl + G * i;
    const float4 q = ch < F ? sm100::ld_now(reinterpret_cast<const float4*>(a.X2 + pc * a.ld2) + ch)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    x.v[4 * i] = q.x; x.v[4 * i + 1] = q.y; x.v[4 * i + 2] = q.z; x.v[4 * i + 3] = q.w;
  }
  int S[T + 1];
#pragma unroll
  for (int k = 0; k < T; ++k) S[k] = sm100::ld_now(a.S_ws + k * N + pc);
  float cj[NR], yj[NR], mrow[NR][T + 1];
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const int j = gl + G * i;
    const bool live = j < T;
    cj[i] = live ? sm100::ld_now(a.c_ws + j * N + pc) : 0.f;
    yj[i] = live ? sm100::ld_now(a.yv + j * N + pc) : 0.f;
    const float* Mrow = a.Lf + (int64_t)(j * (j + 1) / 2) * N + pc;
#pragma unroll
    for (int k = 0; k < T; ++k) mrow[i][k] = (live && k <= j) ? sm100::ld_now(Mrow + k * N) : 0.f;
  }
  const bool act = act_in != 0;
  if (!__any_sync(kFull, act)) return;   // warp-uniform: nothing to do, nothing to count
  // inactive patches run along on valid (atom 0) addresses; nothing of theirs is stored
#pragma unroll
  for (int k = 0; k < T; ++k) S[k] = act ? S[k] : 0;
  int atom = act && lsel >= 0 ? lsel : 0;
  const bool multi = act && lsel < 0;
  if (__any_sync(kFull, multi)) {  // multi-atom leaf: max |a . r|, ties to the lowest atom index
    Sl r;
    r.load(a.R_in + pc * a.ld, gl, F);
    const int node = multi ? -1 - lsel : 0;
    const int cb = multi ? __ldg(a.child_begin + node) : 0;
    const int cc = multi ? __ldg(a.child_count + node) : 0;
    int ccmax = cc;
#pragma unroll
    for (int o = 16; o; o >>= 1) ccmax = max(ccmax, __shfl_xor_sync(kFull, ccmax, o));
    float bestv = -1.f;
    if (multi) atom = __ldg(a.leaf_atom + cb);
    for (int j = 0; j < ccmax; ++j) {
      const bool in = j < cc;
      const int aj = in ? __ldg(a.leaf_atom + cb + j) : 0;
      Sl v;
      v.load(a.atoms + (int64_t)aj * a.ld, gl, F);
      const float mv = fabsf(gsum_full<G>(v.dot(r)));
      if (in && (mv > bestv || (mv == bestv && aj < atom))) { bestv = mv; atom = aj; }
    }
  }
  Sl av;
  av.load(a.atoms + (int64_t)atom * a.ld, gl, F);
  float g[T + 1];
  bool dup = false;
#pragma unroll
  for (int k = 0; k < T; ++k) dup |= S[k] == atom;
  float gtt, bt;
  {
    // value k < T: a . a_{S_k};  T: a . a;  T + 1: a . x (if it fits)
    float pv[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) pv[k] = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      Sl sv;
      sv.load(a.atoms + (int64_t)S[k] * a.ld, gl, F);
      pv[k] = sv.dot(av);
    }
    pv[T] = av.dot(av);
    constexpr bool kBtInRs = T + 1 < NV;
    const float bt_part = av.dot(x);
    if constexpr (kBtInRs) pv[T + 1] = bt_part;
    float mine[NR];
    group_reduce_scatter_n<G, NR>(pv, gl, mine);
#pragma unroll
    for (int k = 0; k < T; ++k) g[k] = group_bcast<G>(mine[k / G], k % G);
    gtt = group_bcast<G>(mine[T / G], T % G);
    if constexpr (kBtInRs) bt = group_bcast<G>(mine[(T + 1) / G], (T + 1) % G);
    else bt = gsum_full<G>(bt_part);
  }
  // w = M g (lane: its rows); one butterfly for a.(A_S c_prev), w.w, w.y
  float wj[NR];
  float gc = 0.f, wsum = 0.f, wy = 0.f;
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    float gm = 0.f;   // g[gl + G i] without dynamic indexing
    float w = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k) {
      gm = k == gl + G * i ? g[k] : gm;
      w = fmaf(mrow[i][k], g[k], w);
    }
    wj[i] = w;
    gc = fmaf(gm, cj[i], gc);
    wsum = fmaf(w, w, wsum);
    wy = fmaf(w, yj[i], wy);
  }
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) {
    gc += __shfl_xor_sync(kFull, gc, o);
    wsum += __shfl_xor_sync(kFull, wsum, o);
    wy += __shfl_xor_sync(kFull, wy, o);
  }
  const float score = bt - gc;   // a . r for r = x - A_S c_prev (pursuit.py:217 check)
  const bool ok = act && !dup && score != 0.f;   // re-selection or a zero score ends the loop
  const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
  const float inv_d = 1.f / dg;
  const float yy = (bt - wy) * inv_d;
  // column sums colw_k = sum_j w_j M[j][k]: lane gl receives columns gl + G i
  float pcol[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    float v = 0.f;
    if (k < T) {
#pragma unroll
      for (int i = 0; i < NR; ++i) v = fmaf(wj[i], mrow[i][k < T ? k : 0], v);
    }
    pcol[k] = v;
  }
  float colw[NR];
  group_reduce_scatter_n<G, NR>(pcol, gl, colw);
  // new row T of M: (-(1/d) w^T M, 1/d);  c_new = c_prev + m_T y_T
  float mt[NR], cn[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const int j = gl + G * i;
    mt[i] = j < T ? -inv_d * colw[i] : (j == T ? inv_d : 0.f);
    cn[i] = j < T ? fmaf(mt[i], yy, cj[i]) : (j == T ? inv_d * yy : 0.f);
  }
  S[T] = atom;
  bool act_next = false;
  float c[T + 1];
#pragma unroll
  for (int k = 0; k <= T; ++k) c[k] = group_bcast<G>(ok ? cn[k / G] : cj[k / G], k % G);
  if (__any_sync(kFull, ok)) {
    // residual r = x - A_S c (support rows from L1 / L2 / shared memory) - c_T a
    Sl r;
#pragma unroll
    for (int i = 0; i < CPL * 4; ++i) r.v[i] = fmaf(-c[T], av.v[i], x.v[i]);
#pragma unroll
    for (int k = 0; k < T; ++k)
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        const int ch = gl + G * i;
        if (ch < F) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(a.atoms + (int64_t)S[k] * a.ld) + ch);
          r.v[4 * i] = fmaf(-c[k], q.x, r.v[4 * i]);
          r.v[4 * i + 1] = fmaf(-c[k], q.y, r.v[4 * i + 1]);
          r.v[4 * i + 2] = fmaf(-c[k], q.z, r.v[4 * i + 2]);
          r.v[4 * i + 3] = fmaf(-c[k], q.w, r.v[4 * i + 3]);
        }
      }
    float s2 = 0.f;
#pragma unroll
    for (int i = 0; i < CPL * 4; ++i) s2 = fmaf(r.v[i], r.v[i], s2);
    const float rn = sqrtf(gsum_full<G>(s2));
    if (ok) {
      r.store(a.R + p * a.ld, gl, F);
      act_next = (T + 1 < K) && rn > tol_p;
      if (act_next) {
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const int j = gl + G * i;
          if (j <= T) {
            a.Lf[(int64_t)(T * (T + 1) / 2 + j) * N + p] = mt[i];
            a.c_ws[j * N + p] = cn[i];
          }
        }
        if (gl == 0) {
          a.yv[T * N + p] = yy;
          a.S_ws[T * N + p] = atom;
        }
      }
      if (gl == 0) {
        a.count[p] = T + 1;
        a.resnorm[p] = rn;
      }
    }
  }
  if (act && !act_next) {
    // final rows of the caller's idx / coef (T or T + 1 entries; the rest stay -1 / 0 from init)
    const int n_out = ok ? T + 1 : T;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int j = gl + G * i;
      if (j < n_out) {
        int s_mine = S[0];
#pragma unroll
        for (int k = 1; k <= T; ++k) s_mine = k == j ? S[k] : s_mine;
        a.idx[p * K + j] = s_mine;
        a.coef[p * K + j] = ok ? cn[i] : cj[i];
      }
    }
  }
  if (act && gl == 0) a.active[p] = act_next ? 1 : 0;
  count_root(act_next && gl == 0, a.root_count);
}

}  // namespace

int lockstep_lanes(int ld, int K) {
  // 8 lanes per patch; each lane owns one Cholesky row up to 8 atoms, two up to 16
  if (K <= 8 && ld <= 160) return 8;
  if (K <= 16 && ld <= 64) return 8;
  return 0;
}

cudaError_t launch_update_omp8(const UpdateArgs& a, cudaStream_t st) {
  const int G = lockstep_lanes(a.ld, a.K);
  if (G == 0 || a.method != kMethodOMP || a.S_ws == nullptr) return cudaErrorNotSupported;
  const int blocks = (int)((a.N + (128 / G) - 1) / (128 / G));
  const int cpl = (a.ld / 4 + G - 1) / G;
  switch ((G * 8 + cpl) * 16 + a.iter) {
#define STMP_OMP8_CASE(g, cp, t) \
  case (g * 8 + cp) * 16 + t: return launch_kernel(update_omp8_kernel<g, cp, t>, blocks, 128, 0, st, true, a);
#define STMP_OMP8_ITERS(g, cp)                                                                          \
  STMP_OMP8_CASE(g, cp, 0) STMP_OMP8_CASE(g, cp, 1) STMP_OMP8_CASE(g, cp, 2) STMP_OMP8_CASE(g, cp, 3) \
  STMP_OMP8_CASE(g, cp, 4) STMP_OMP8_CASE(g, cp, 5) STMP_OMP8_CASE(g, cp, 6) STMP_OMP8_CASE(g, cp, 7)
#define STMP_OMP16_ITERS(cp)                                                                            \
  STMP_OMP8_CASE(8, cp, 8) STMP_OMP8_CASE(8, cp, 9) STMP_OMP8_CASE(8, cp, 10) STMP_OMP8_CASE(8, cp, 11) \
  STMP_OMP8_CASE(8, cp, 12) STMP_OMP8_CASE(8, cp, 13) STMP_OMP8_CASE(8, cp, 14) STMP_OMP8_CASE(8, cp, 15)
    STMP_OMP8_ITERS(8, 1) STMP_OMP8_ITERS(8, 2) STMP_OMP8_ITERS(8, 3) STMP_OMP8_ITERS(8, 4) STMP_OMP8_ITERS(8, 5)
    STMP_OMP16_ITERS(1) STMP_OMP16_ITERS(2)
#undef STMP_OMP16_ITERS
#undef STMP_OMP8_ITERS
#undef STMP_OMP8_CASE
    default: return cudaErrorNotSupported;
  }
}

bool update_config(int ld, int K, UpdateCfg& c) {
  (void)K;
  const int F = ld / 4;
  if (ld % 32 != 0 || ld > 2048) return false;
  c.G = F <= 64 ? 8 : 32;
  c.E = (F + c.G - 1) / c.G;   // chunks per lane (CPL)
  c.KC = 0;
  switch (c.G * 100 + c.E) {
    case 801: case 802: case 803: case 804: case 805: case 806: case 807: case 808:
    case 3203: case 3204: case 3205: case 3206: case 3207: case 3208: case 3209: case 3210: case 3211:
    case 3212: case 3213: case 3214: case 3215: case 3216:
      return true;
    default:
      return false;
  }
}

#define STMP_UPD_CASES(X)                                                                              \
  X(8, 1) X(8, 2) X(8, 3) X(8, 4) X(8, 5) X(8, 6) X(8, 7) X(8, 8) X(32, 3) X(32, 4) X(32, 5) X(32, 6) \
  X(32, 7) X(32, 8) X(32, 9) X(32, 10) X(32, 11) X(32, 12) X(32, 13) X(32, 14) X(32, 15) X(32, 16)

cudaError_t launch_init(const UpdateCfg& c, const UpdateArgs& a, int blocks, cudaStream_t st) {
  switch (c.G * 100 + c.E) {
#define STMP_INIT_CASE(g, e) \
  case g * 100 + e: return launch_kernel(init_kernel<g, e>, blocks, 128, 0, st, false, a);
    STMP_UPD_CASES(STMP_INIT_CASE)
#undef STMP_INIT_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_update(const UpdateCfg& c, const UpdateArgs& a, int blocks, size_t smem, cudaStream_t st) {
  switch (c.G * 100 + c.E) {
#define STMP_UPD_CASE(g, e)                                                         \
  case g * 100 + e: {                                                               \
    cudaError_t err = cudaFuncSetAttribute(update_kernel<g, e>,                     \
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                    \
    if (err != cudaSuccess) return err;                                             \
    return launch_kernel(update_kernel<g, e>, blocks, 128, smem, st, true, a);     \
  }
    STMP_UPD_CASES(STMP_UPD_CASE)
#undef STMP_UPD_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// wide-row OMP update: one CTA per patch (ld > 160 floats, OMP)
int wide_update_cpt(int ld) { return ld > 160 && ld <= 2048 ? (ld / 4 + 127) / 128 : 0; }

cudaError_t launch_update_wide(const UpdateArgs& a, cudaStream_t st) {
  const int cpt = wide_update_cpt(a.ld);
  const int K = a.K;
  const size_t smem = (size_t)(3 * K + K * (K + 1) / 2 + 5 * (K + 2) + K) * 4;
  switch (cpt) {
#define STMP_WIDE_CASE(c)                                                                     \
  case c: {                                                                                   \
    if (smem > 48 * 1024) {                                                                   \
      cudaError_t err = cudaFuncSetAttribute(update_wide_kernel<c>,                           \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (err != cudaSuccess) return err;                                                     \
    }                                                                                         \
    return launch_kernel(update_wide_kernel<c>, (unsigned)a.N, 128, smem, st, true, a);       \
  }
    STMP_WIDE_CASE(1) STMP_WIDE_CASE(2) STMP_WIDE_CASE(3) STMP_WIDE_CASE(4)
#undef STMP_WIDE_CASE
    default: return cudaErrorNotSupported;
  }
}

size_t update_smem_bytes(const UpdateCfg& c, int K, int ld, bool cache_atoms) {
  (void)ld;
  (void)cache_atoms;
  return (size_t)(128 / c.G) * upd_scalar_floats(K) * 4;
}

}  // namespace stmp
