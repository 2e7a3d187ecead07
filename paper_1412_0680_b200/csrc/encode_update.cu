// Per-patch kernels of the staged encoder: init (padded residual copy,
// tolerance, root bucketing) and update (leaf choice + MP step or OMP refit).
//
// A group of G lanes owns one patch; lane gl holds elements [gl*E, gl*E+E) of
// the padded row.  For OMP the patch's solver state and its support atoms are
// pulled into shared memory as one batch of independent (async) loads and
// reused by both the Gram column and the residual rebuild, so an iteration
// costs a few dependent global round trips instead of 2t.  The small
// triangular solves run redundantly on the G lanes (no shuffles); dot
// products are group reductions.  Semantics: pkg/src/stmp/pursuit.py:207-221 (MP) and the
// SURVEY §8c OMP restatement over omp_refit (pursuit.py:235-250).
#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

namespace {

// Sum over the G lanes of this patch group.  The mask names only the group's
// own lanes: groups of one warp diverge (different patches stop at different
// iterations), so a full-warp mask would wait for lanes that never arrive.
template <int G>
__device__ __forceinline__ float group_sum(float v) {
  const unsigned mask = G >= 32 ? kFull : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// Count the patches that stay active into the single root bin: one
// fire-and-forget atomic per warp (called by every lane; `act` true on at
// most one lane per patch group).  Slots are assigned later by the scatter.
__device__ __forceinline__ void count_root(bool act, int* counter) {
  const unsigned m = __ballot_sync(kFull, act);
  if (m && (int)(threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(counter, __popc(m));
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
  count_root(act && gl == 0, a.root_count);
}

// ------------------------------------------------------------------ update
// Shared scratch per patch group (floats):
//   S[K] | c[K] | y[K] | L[K(K+1)/2] | w[K] | cn[K] | support atoms [K][ld] (optional)
__host__ __device__ inline int upd_scalar_floats(int K) { return (5 * K + K * (K + 1) / 2 + 3) & ~3; }

template <int E>
__device__ __forceinline__ void load_gen(const float* src, float (&v)[E]) {
  if constexpr (E % 4 == 0) {
#pragma unroll
    for (int i = 0; i < E / 4; ++i) {
      const float4 q = reinterpret_cast<const float4*>(src)[i];
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = src[i];
  }
}

template <int G, int E>
__global__ void __launch_bounds__(128) update_kernel(UpdateArgs a) {
  extern __shared__ __align__(16) float upd_smem[];
  const int gpb = blockDim.x / G;
  const int grp = threadIdx.x / G;
  const int64_t p = (int64_t)blockIdx.x * gpb + grp;
  const int gl = threadIdx.x % G;
  const unsigned gmask = G >= 32 ? kFull : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int K = a.K;
  const int sfl = upd_scalar_floats(K);
  float* gs = upd_smem + grp * (sfl + (a.cache_atoms ? K * a.ld : 0));
  int* S_s = reinterpret_cast<int*>(gs);
  float* c_s = gs + K;
  float* y_s = c_s + K;
  float* L_s = y_s + K;
  float* w_s = L_s + K * (K + 1) / 2;
  float* cn_s = w_s + K;
  float* A_s = gs + sfl;
  const bool inb = p < a.N;
  bool act = inb && a.active[p];
  const int64_t off = (int64_t)gl * E;
  if (act) {
    const int t = a.count[p];
    const int lsel = a.leaf_sel[p];
    const bool omp = a.method == kMethodOMP;
    float r[E], x[E];
    if (!omp || lsel < 0) load_vec<E>(a.R + p * a.ld + off, r);
    if (omp) {
      load_vec<E>(a.X2 + p * a.ld2 + off, x);
      // the patch's solver state -> shared, as one batch of independent loads
      // (bounded by K, not t, so they do not wait for the count load)
      for (int i = gl; i < K; i += G) {
        S_s[i] = a.idx[p * K + i];
        c_s[i] = a.coef[p * K + i];
        y_s[i] = a.yv[p * K + i];
      }
      const float* Lp = a.Lf + p * (int64_t)(K * (K + 1) / 2);
      for (int i = gl; i < K * (K + 1) / 2; i += G) L_s[i] = Lp[i];
      __syncwarp(gmask);
      if (a.cache_atoms) {  // support atoms -> shared with async copies, all in flight at once
        const int F = a.ld >> 2;
        for (int e = gl; e < t * F; e += G) {
          const int j = e / F, q = e - j * F;
          sm100::cp_async16(sm100::smem_u32(A_s + j * a.ld + 4 * q), a.atoms + (int64_t)S_s[j] * a.ld + 4 * q, 16u);
        }
      }
    }
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
        float v[E];
        load_vec<E>(a.atoms + (int64_t)aj * a.ld + off, v);
        const float m = fabsf(group_sum<G>(dot_vec<E>(v, r)));
        if (m > bestv || (m == bestv && aj < atom)) { bestv = m; atom = aj; }
      }
    }
    float av[E];
    load_vec<E>(a.atoms + (int64_t)atom * a.ld + off, av);
    int32_t* S = a.idx + p * K;
    if (!omp) {
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
      if (a.cache_atoms) sm100::cp_async_wait_all();
      __syncwarp(gmask);
      bool dup = false;
      for (int j = 0; j < t; ++j) dup |= (S_s[j] == atom);
      const float bt = group_sum<G>(dot_vec<E>(av, x));
      const float gtt = group_sum<G>(dot_vec<E>(av, av));
      // Gram column of the new atom against the support (independent dots, the
      // row loads of several j in flight at once), then forward substitution
      float* g_s = cn_s;  // cn is produced only after the Gram column is consumed
#pragma unroll 4
      for (int j = 0; j < t; ++j) {
        float sv[E];
        if (a.cache_atoms) load_gen<E>(A_s + j * a.ld + off, sv);
        else load_vec<E>(a.atoms + (int64_t)S_s[j] * a.ld + off, sv);
        const float g = group_sum<G>(dot_vec<E>(sv, av));
        if (gl == 0) g_s[j] = g;
      }
      __syncwarp(gmask);
      float wsum = 0.f, gc = 0.f;
      for (int j = 0; j < t; ++j) {
        const float g = g_s[j];
        gc = fmaf(g, c_s[j], gc);   // a . (A_S c_prev)
        const float* Lj = L_s + j * (j + 1) / 2;
        float v = g;
        for (int k = 0; k < j; ++k) v = fmaf(-Lj[k], w_s[k], v);
        v /= Lj[j];
        w_s[j] = v;
        wsum = fmaf(v, v, wsum);
      }
      const float score = bt - gc;   // a . r for r = x - A_S c_prev (pursuit.py:217 check)
      __syncwarp(gmask);  // every lane has read g_s before cn_s is overwritten
      if (dup || score == 0.f) {
        act = false;   // re-selection (or a zero score) ends the loop
      } else {
        const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
        float yy = bt;
        for (int j = 0; j < t; ++j) yy = fmaf(-w_s[j], y_s[j], yy);
        yy /= dg;
        // back substitution L^T c = y; row t of L is (w, dg)
        for (int j = t; j >= 0; --j) {
          float v = j == t ? yy : y_s[j];
          for (int k = j + 1; k <= t; ++k) {
            const float Lkj = k == t ? w_s[j] : L_s[k * (k + 1) / 2 + j];
            v = fmaf(-Lkj, cn_s[k], v);
          }
          cn_s[j] = v / (j == t ? dg : L_s[j * (j + 1) / 2 + j]);
        }
        // residual r = x - A_S c with the new atom
        const float ct = cn_s[t];
#pragma unroll
        for (int i = 0; i < E; ++i) r[i] = fmaf(-ct, av[i], x[i]);
#pragma unroll 4
        for (int j = 0; j < t; ++j) {
          float sv[E];
          if (a.cache_atoms) load_gen<E>(A_s + j * a.ld + off, sv);
          else load_vec<E>(a.atoms + (int64_t)S_s[j] * a.ld + off, sv);
          const float cj = cn_s[j];
#pragma unroll
          for (int i = 0; i < E; ++i) r[i] = fmaf(-cj, sv[i], r[i]);
        }
        store_vec<E>(a.R + p * a.ld + off, r);
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < E; ++i) s2 = fmaf(r[i], r[i], s2);
        const float rn = sqrtf(group_sum<G>(s2));
        float* Lt = a.Lf + p * (int64_t)(K * (K + 1) / 2) + t * (t + 1) / 2;
        for (int i = gl; i <= t; i += G) {
          Lt[i] = i < t ? w_s[i] : dg;
          a.coef[p * K + i] = cn_s[i];
        }
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

}  // namespace

bool update_config(int ld, int K, UpdateCfg& c) {
  static const int kLd[] = {32, 64, 96, 128, 160, 192, 256, 512, 1024, 1600, 2048};
  bool ok = false;
  for (int v : kLd) ok |= (v == ld);
  if (!ok) return false;
  // few lanes per patch: the scalar triangular solves run once per G lanes, so
  // small groups keep the warp instruction count per patch low
  int G = 1;
  while (G < 32 && ld / G > 32) G <<= 1;
  c.G = G;
  c.E = ld / G;
  c.KC = 0;
  return true;
}

#define STMP_UPD_CASES(X) \
  X(1, 32) X(2, 32) X(4, 24) X(4, 32) X(8, 20) X(8, 24) X(8, 32) X(16, 32) X(32, 32) X(32, 50) X(32, 64)

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
  switch (c.G * 1000 + c.E) {
#define STMP_UPD_CASE(g, e)                                                         \
  case g * 1000 + e: {                                                              \
    cudaError_t err = cudaFuncSetAttribute(update_kernel<g, e>,                     \
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                    \
    if (err != cudaSuccess) return err;                                             \
    update_kernel<g, e><<<blocks, 128, smem, st>>>(a);                              \
    break;                                                                          \
  }
    STMP_UPD_CASES(STMP_UPD_CASE)
#undef STMP_UPD_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

size_t update_smem_bytes(const UpdateCfg& c, int K, int ld, bool cache_atoms) {
  const int groups = 128 / c.G;
  return (size_t)groups * (upd_scalar_floats(K) + (cache_atoms ? K * ld : 0)) * 4;
}

}  // namespace stmp
