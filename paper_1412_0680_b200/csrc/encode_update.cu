// Per-patch kernels of the staged encoder: init (padded residual copy,
// tolerance, root bucketing) and update (leaf choice + MP step or OMP refit).
//
// A group of G lanes owns one patch; lane gl holds elements [gl*E, gl*E+E) of
// the padded row.  For OMP the support atoms are loaded once per iteration as
// one batch into registers (KC-entry cache) and reused by both the Gram
// column and the residual rebuild, so an iteration costs two dependent
// global round trips instead of 2t.  The small triangular solves run
// redundantly on the G lanes (no shuffles); dot products are group
// reductions.  Semantics: pkg/src/stmp/pursuit.py:207-221 (MP) and the
// SURVEY §8c OMP restatement over omp_refit (pursuit.py:235-250).
#include "common.cuh"
#include "kernels.cuh"
#include "staged.cuh"

namespace stmp {

namespace {

template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// warp-aggregated rank in the single root bin (called by every lane; `act`
// must be true on at most one lane per patch group)
__device__ __forceinline__ int root_rank(bool act, int* counter) {
  const unsigned m = __ballot_sync(kFull, act);
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (m) {
    const int leader = __ffs(m) - 1;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(kFull, base, leader);
  }
  return base + __popc(m & ((1u << lane) - 1u));
}

template <int E>
__device__ __forceinline__ void load_vec(const float* __restrict__ src, float (&v)[E]) {
  if constexpr (E % 4 == 0) {
#pragma unroll
    for (int i = 0; i < E / 4; ++i) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(src) + i);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
  } else if constexpr (E % 2 == 0) {
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(src) + i);
      v[2 * i] = q.x; v[2 * i + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = __ldg(src + i);
  }
}

template <int E>
__device__ __forceinline__ void store_vec(float* dst, const float (&v)[E]) {
  if constexpr (E % 4 == 0) {
#pragma unroll
    for (int i = 0; i < E / 4; ++i)
      reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else if constexpr (E % 2 == 0) {
#pragma unroll
    for (int i = 0; i < E / 2; ++i) reinterpret_cast<float2*>(dst)[i] = make_float2(v[2 * i], v[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) dst[i] = v[i];
  }
}

template <int E>
__device__ __forceinline__ float dot_vec(const float (&a)[E], const float (&b)[E]) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < E; ++i) s = fmaf(a[i], b[i], s);
  return s;
}

// ------------------------------------------------------------------ init
template <int G, int E>
__global__ void __launch_bounds__(128) init_kernel(UpdateArgs a) {
  const int gpb = blockDim.x / G;
  const int64_t p = (int64_t)blockIdx.x * gpb + threadIdx.x / G;
  const int gl = threadIdx.x % G;
  const bool inb = p < a.N;
  float x[E];
  float ss = 0.f;
  if (inb) {
    const float* xp = a.X + p * a.ldx;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int d = gl * E + i;
      x[i] = d < a.n ? __ldg(xp + d) : 0.f;
      ss = fmaf(x[i], x[i], ss);
    }
    store_vec<E>(a.R + p * a.ld + gl * E, x);
    if (a.X2) store_vec<E>(const_cast<float*>(a.X2) + p * a.ld2 + gl * E, x);
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
  const int r = root_rank(act && gl == 0, a.root_count);
  if (inb && gl == 0) a.rank[p] = act ? r : -1;
}

// ------------------------------------------------------------------ update
template <int G, int E, int KC>
__global__ void __launch_bounds__(128) update_kernel(UpdateArgs a) {
  extern __shared__ float upd_smem[];
  const int gpb = blockDim.x / G;
  const int grp = threadIdx.x / G;
  const int64_t p = (int64_t)blockIdx.x * gpb + grp;
  const int gl = threadIdx.x % G;
  const int K = a.K;
  float* wv = upd_smem + grp * 2 * K;   // new Cholesky row w (identical on the G lanes)
  float* cv = wv + K;                    // refit coefficients
  const bool inb = p < a.N;
  bool act = inb && a.active[p];
  const int64_t off = (int64_t)gl * E;
  if (act) {
    const int t = a.count[p];
    const int* pw = a.path_ws + p * a.L;
    const int nodeL = pw[a.L - 1];
    const int cb = __ldg(a.child_begin + nodeL);
    const int cc = __ldg(a.child_count + nodeL);
    int ipc = __ldg(a.child_count + 0);
    for (int l = 1; l < a.L; ++l) ipc += __ldg(a.child_count + pw[l - 1]);
    if (gl == 0 && a.ip) { a.ip[2 * p] += ipc + cc; a.ip[2 * p + 1] += ipc; }
    int32_t* S = a.idx + p * K;

    float r[E];
    const bool need_r = a.method == kMethodMP || cc > 1;
    if (need_r) load_vec<E>(a.R + p * a.ld + off, r);
    // ---- leaf choice: max |a . r| over the node's atoms, ties to the lowest atom index
    int atom = __ldg(a.leaf_atom + cb);
    if (cc > 1) {
      float bestv = -1.f;
      for (int j = 0; j < cc; ++j) {
        const int aj = __ldg(a.leaf_atom + cb + j);
        float av[E];
        load_vec<E>(a.atoms + (int64_t)aj * a.ld + off, av);
        const float m = fabsf(group_sum<G>(dot_vec<E>(av, r)));
        if (m > bestv || (m == bestv && aj < atom)) { bestv = m; atom = aj; }
      }
    }
    float av[E];
    load_vec<E>(a.atoms + (int64_t)atom * a.ld + off, av);
    if (a.method == kMethodMP) {
      const float s = group_sum<G>(dot_vec<E>(av, r));
      if (s == 0.f) {
        act = false;   // pursuit.py:217
      } else {
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < E; ++i) { r[i] = fmaf(-s, av[i], r[i]); s2 = fmaf(r[i], r[i], s2); }
        store_vec<E>(a.R + p * a.ld + off, r);
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
      // support indices and (when cached) the support atoms, all loads issued together
      int sidx[KC > 0 ? KC : 1];
      float sat[KC > 0 ? KC : 1][E];
      bool dup = false;
      if constexpr (KC > 0) {
#pragma unroll
        for (int j = 0; j < KC; ++j) sidx[j] = j < t ? S[j] : -1;
#pragma unroll
        for (int j = 0; j < KC; ++j)
          if (j < t) load_vec<E>(a.atoms + (int64_t)sidx[j] * a.ld + off, sat[j]);
#pragma unroll
        for (int j = 0; j < KC; ++j) dup |= (sidx[j] == atom);
      } else {
        for (int j = 0; j < t; ++j) dup |= (S[j] == atom);
      }
      float x[E];
      load_vec<E>(a.X2 + p * a.ld2 + off, x);
      const float bt = group_sum<G>(dot_vec<E>(av, x));
      const float gtt = group_sum<G>(dot_vec<E>(av, av));
      const float* Lp = a.Lf + p * (int64_t)(K * (K + 1) / 2);
      const float* yp = a.yv + p * (int64_t)K;
      // Gram column of the new atom against the support, forward substitution
      float wsum = 0.f, gc = 0.f;
      for (int j = 0; j < t; ++j) {
        float g;
        if constexpr (KC > 0) {
          float part = 0.f;
#pragma unroll
          for (int q = 0; q < KC; ++q)
            if (q == j) part = dot_vec<E>(sat[q], av);
          g = group_sum<G>(part);
        } else {
          float sj[E];
          load_vec<E>(a.atoms + (int64_t)S[j] * a.ld + off, sj);
          g = group_sum<G>(dot_vec<E>(sj, av));
        }
        gc = fmaf(g, a.coef[p * K + j], gc);   // a . (A_S c_prev)
        const float* Lj = Lp + j * (j + 1) / 2;
        float v = g;
        for (int k = 0; k < j; ++k) v = fmaf(-Lj[k], wv[k], v);
        v /= Lj[j];
        wv[j] = v;
        wsum = fmaf(v, v, wsum);
      }
      const float score = bt - gc;   // a . r for r = x - A_S c_prev (pursuit.py:217 check)
      if (dup || score == 0.f) {
        act = false;   // re-selection (or a zero score) ends the loop
      } else {
        const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
        float yy = bt;
        for (int j = 0; j < t; ++j) yy = fmaf(-wv[j], yp[j], yy);
        yy /= dg;
        // back substitution L^T c = y; row t of L is (w, dg)
        for (int j = t; j >= 0; --j) {
          float v = j == t ? yy : yp[j];
          for (int k = j + 1; k <= t; ++k) {
            const float Lkj = k == t ? wv[j] : Lp[k * (k + 1) / 2 + j];
            v = fmaf(-Lkj, cv[k], v);
          }
          cv[j] = v / (j == t ? dg : Lp[j * (j + 1) / 2 + j]);
        }
        // residual r = x - A_S c with the new atom
#pragma unroll
        for (int i = 0; i < E; ++i) r[i] = fmaf(-cv[t], av[i], x[i]);
        if constexpr (KC > 0) {
#pragma unroll
          for (int j = 0; j < KC; ++j) {
            if (j < t) {
              const float cj = cv[j];
#pragma unroll
              for (int i = 0; i < E; ++i) r[i] = fmaf(-cj, sat[j][i], r[i]);
            }
          }
        } else {
          for (int j = 0; j < t; ++j) {
            float sj[E];
            load_vec<E>(a.atoms + (int64_t)S[j] * a.ld + off, sj);
            const float cj = cv[j];
#pragma unroll
            for (int i = 0; i < E; ++i) r[i] = fmaf(-cj, sj[i], r[i]);
          }
        }
        store_vec<E>(a.R + p * a.ld + off, r);
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < E; ++i) s2 = fmaf(r[i], r[i], s2);
        const float rn = sqrtf(group_sum<G>(s2));
        if (gl == 0) {
          float* Lt = a.Lf + p * (int64_t)(K * (K + 1) / 2) + t * (t + 1) / 2;
          for (int j = 0; j < t; ++j) Lt[j] = wv[j];
          Lt[t] = dg;
          a.yv[p * (int64_t)K + t] = yy;
          S[t] = atom;
          for (int j = 0; j <= t; ++j) a.coef[p * K + j] = cv[j];
          a.count[p] = t + 1;
          a.resnorm[p] = rn;
        }
        act = (t + 1 < K) && rn > a.tol[p];
      }
    }
    if (gl == 0) a.active[p] = act ? 1 : 0;
  }
  const int rr = root_rank(act && gl == 0, a.root_count);
  if (inb && gl == 0) a.rank[p] = act ? rr : -1;
}

}  // namespace

bool update_config(int ld, int K, UpdateCfg& c) {
  static const int kLd[] = {32, 64, 96, 128, 160, 192, 256, 512, 1024, 1600, 2048};
  bool ok = false;
  for (int v : kLd) ok |= (v == ld);
  if (!ok) return false;
  int G = 1;
  while (G < 32 && ld / G > 8) G <<= 1;
  c.G = G;
  c.E = ld / G;
  c.KC = 0;
  if (c.E <= 8 && K <= 16) c.KC = K <= 8 ? 8 : 16;
  else if (c.E <= 16 && K <= 8) c.KC = 8;
  return true;
}

#define STMP_UPD_CASES(X) \
  X(4, 8) X(8, 8) X(16, 6) X(16, 8) X(32, 5) X(32, 6) X(32, 8) X(32, 16) X(32, 32) X(32, 50) X(32, 64)

cudaError_t launch_init(const UpdateCfg& c, const UpdateArgs& a, int blocks, cudaStream_t st) {
  switch (c.G * 1000 + c.E) {
#define STMP_INIT_CASE(g, e) \
  case g * 1000 + e: init_kernel<g, e><<<blocks, 128, 0, st>>>(a); break;
    STMP_UPD_CASES(STMP_INIT_CASE)
#undef STMP_INIT_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_update(const UpdateCfg& c, const UpdateArgs& a, int blocks, size_t smem, cudaStream_t st) {
  switch ((c.G * 1000 + c.E) * 100 + c.KC) {
#define STMP_UPD_CASE(g, e)                                                                     \
  case (g * 1000 + e) * 100 + 0: update_kernel<g, e, 0><<<blocks, 128, smem, st>>>(a); break;  \
  case (g * 1000 + e) * 100 + 8: update_kernel<g, e, (e <= 16 ? 8 : 0)><<<blocks, 128, smem, st>>>(a); break; \
  case (g * 1000 + e) * 100 + 16: update_kernel<g, e, (e <= 8 ? 16 : 0)><<<blocks, 128, smem, st>>>(a); break;
    STMP_UPD_CASES(STMP_UPD_CASE)
#undef STMP_UPD_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace stmp
