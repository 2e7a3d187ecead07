// Fused warp-per-patch encoder: greedy tree descent (or exhaustive scan),
// leaf scoring and the MP / OMP update for one patch per warp, residual kept
// in registers for all K iterations.  Used for small batches (config 0 is
// launch-bound, SURVEY §7 "hard parts") and as the general path for any
// (n, K, tree shape), including ragged trees.
//
// Reference semantics reproduced:
//   internal level: argmax |child_matrix @ r|, ties to the lowest child
//     position (pkg/src/stmp/pursuit.py:141-153 with keep == 1);
//   leaf: max |score| over the node's atoms, ties to the lowest ATOM index,
//     signed score returned (pursuit.py:155-162);
//   exhaustive: argmax |A r|, lowest index (pursuit.py:102-109);
//   MP: tolerance check before selecting, stop on score == 0,
//     r -= s * a_i (pursuit.py:207-220);
//   OMP: the SURVEY §8c restatement -- refit over the growing support with
//     the ridge-1e-8 normal equations of omp_refit (pursuit.py:235-250),
//     solved here by an incremental Cholesky factor, r = x - A_S^T c; stop
//     when an atom is re-selected.
#include "common.cuh"
#include "kernels.cuh"

namespace stmp {

namespace {

// Score `cnt` rows of `tab` (row stride ld) against the lane-strided residual
// r and fold the winner into (bk, bs).  GATHER=false: rows base..base+cnt-1,
// tie id = position; GATHER=true: rows rowmap[j], tie id = rowmap[j] (atom).
template <int VPL, bool GATHER>
__device__ __forceinline__ void score_rows(const float* __restrict__ tab, int ld, int64_t base,
                                           const int* __restrict__ rowmap, int cnt,
                                           const float (&r)[VPL], int lane,
                                           unsigned long long& bk, float& bs) {
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const int nr = min(32, cnt - c0);
    int myrow = 0;
    if (GATHER) myrow = lane < nr ? __ldg(rowmap + c0 + lane) : 0;
    float p[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) p[j] = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < nr) {
        const int64_t row = GATHER ? (int64_t)__shfl_sync(kFull, myrow, j) : base + c0 + j;
        const float* rp = tab + row * ld + lane;
#pragma unroll
        for (int i = 0; i < VPL; ++i) p[j] = fmaf(rp[32 * i], r[i], p[j]);
      }
    }
    const float s = reduce_scatter32(p, lane);
    const bool valid = lane < nr;
    const unsigned id = GATHER ? (unsigned)myrow : (unsigned)(c0 + lane);
    const unsigned long long key = valid ? score_key(s, id) : 0ull;
    const unsigned long long wm = warp_max_u64(key);
    if (wm > bk) {
      const int src = __ffs(__ballot_sync(kFull, key == wm)) - 1;
      bs = __shfl_sync(kFull, s, src);
      bk = wm;
    }
  }
}

__device__ __forceinline__ int key_id(unsigned long long k) {
  return (int)(0xFFFFFFFFu - (unsigned)(k & 0xFFFFFFFFull));
}

// Beam descent (pursuit.py:134-162 for retained_count > 1): every frontier node
// keeps its `keep` best children by |score| (a stable sort on -|score|: ties to
// the lower position), in child order; the next frontier is the concatenation
// over the frontier in order.  Then the leaf atoms of all surviving depth-L
// nodes are scored, max |score|, ties to the lowest atom index.  One warp per
// patch; frontiers and a node's child scores live in the warp's global scratch.
// Returns the leaf winner in (bk, bs); writes the first survivor per level to
// `path_row` (the oracle's path) when given.
template <int VPL>
__device__ void beam_select(const FusedArgs& a, const float (&r)[VPL], int lane, int* scr, int* path_row,
                            unsigned long long& bk, float& bs, int& ipc, int& ipa) {
  const int ld = a.ld;
  const int L = a.tree.levels;
  int* fr = scr;
  int* fn = scr + a.max_frontier;
  float* sc = reinterpret_cast<float*>(scr + 2 * a.max_frontier);
  if (lane == 0) fr[0] = 0;
  int nf = 1;
  __syncwarp();
  for (int lvl = 0; lvl < L; ++lvl) {
    const int keep = a.keep[lvl];
    int nn = 0;
    for (int f = 0; f < nf; ++f) {
      const int node = fr[f];
      const int b = __ldg(a.tree.child_begin + node);
      const int c = __ldg(a.tree.child_count + node);
      ipc += c;
      if (keep >= c) {
        for (int j = lane; j < c; j += 32) fn[nn + j] = b + j;
        nn += c;
        continue;
      }
      // |score| of every child
      for (int c0 = 0; c0 < c; c0 += 32) {
        const int nr = min(32, c - c0);
        float p[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) p[j] = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nr) {
            const float* rp = a.tree.cent + (int64_t)(b + c0 + j) * ld + lane;
#pragma unroll
            for (int i = 0; i < VPL; ++i) p[j] = fmaf(rp[32 * i], r[i], p[j]);
          }
        const float s = reduce_scatter32(p, lane);
        if (lane < nr) sc[c0 + lane] = fabsf(s);
      }
      __syncwarp();
      // the keep best, ties to the lower position (a stable argsort of -|s|)
      for (int q = 0; q < keep; ++q) {
        unsigned long long best = 0ull;
        for (int j = lane; j < c; j += 32) {
          const float v = sc[j];
          const unsigned long long k = v >= 0.f ? score_key(v, (unsigned)j) : 0ull;
          best = k > best ? k : best;
        }
        best = warp_max_u64(best);
        if (lane == 0) sc[key_id(best)] = -1.f;   // taken
        __syncwarp();
      }
      // survivors in child order
      for (int c0 = 0; c0 < c; c0 += 32) {
        const bool taken = c0 + lane < c && sc[c0 + lane] < 0.f;
        const unsigned m = __ballot_sync(kFull, taken);
        if (taken) fn[nn + __popc(m & ((1u << lane) - 1u))] = b + c0 + lane;
        nn += __popc(m);
      }
      __syncwarp();
    }
    if (path_row != nullptr && lane == 0) path_row[lvl] = fn[0];
    int* tmp = fr;
    fr = fn;
    fn = tmp;
    nf = nn;
    __syncwarp();
  }
  bk = 0ull;
  for (int f = 0; f < nf; ++f) {
    const int node = fr[f];
    const int b = __ldg(a.tree.child_begin + node);
    const int c = __ldg(a.tree.child_count + node);
    score_rows<VPL, true>(a.atoms, ld, 0, a.tree.leaf_atom + b, c, r, lane, bk, bs);
    ipa += c;
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) encode_fused_kernel(FusedArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int ld = a.ld;
  const int K = a.K;
  const int L = a.tree.levels;

  float* root_tab = smem;
  const int root_floats = a.root_smem_rows * ld;
  if (a.root_smem_rows > 0) {
    const float4* src = reinterpret_cast<const float4*>(a.tree.cent + (int64_t)a.root_begin * ld);
    float4* dst = reinterpret_cast<float4*>(root_tab);
    for (int i = threadIdx.x; i < root_floats / 4; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();

  float* ws = smem + root_floats + warp * a.warp_smem_floats;
  float* Lm = ws;                                  // packed lower-triangular Cholesky factor
  float* gv = Lm + K * (K + 1) / 2;                // Gram column of the new atom
  float* yv = gv + K;                              // L y = A_S x
  float* cv = yv + K;                              // coefficients
  int* sidx = reinterpret_cast<int*>(cv + K);      // support in selection order
  float* acache = reinterpret_cast<float*>(sidx + K);  // cached support atoms (optional)

  const int64_t wstride = (int64_t)gridDim.x * wpb;
  for (int64_t p = (int64_t)blockIdx.x * wpb + warp; p < a.N; p += wstride) {
    float x[VPL], r[VPL];
    const float* xp = a.X + p * a.ldx;
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int d = lane + 32 * i;
      x[i] = d < a.n ? __ldg(xp + d) : 0.f;
      r[i] = x[i];
      ss = fmaf(x[i], x[i], ss);
    }
    float rnorm = sqrtf(warp_sum(ss));
    const float tol = a.tol_abs >= 0.f ? a.tol_abs : kRelTol * rnorm;
    int t = 0, ipc = 0, ipa = 0;

    for (int it = 0; it < K; ++it) {
      if (a.method != kMethodSelect && rnorm <= tol) break;
      // ---------------- selection ----------------
      unsigned long long bk = 0ull;
      float bs = 0.f;
      if (a.has_tree && a.beam) {
        const int64_t gw = (int64_t)blockIdx.x * wpb + warp;
        beam_select<VPL>(a, r, lane, a.scratch + gw * beam_scratch_ints(a.max_frontier),
                         a.path != nullptr ? a.path + (p * K + t) * L : nullptr, bk, bs, ipc, ipa);
      } else if (a.has_tree) {
        int node = 0;
        for (int lvl = 0; lvl < L; ++lvl) {
          const int b = __ldg(a.tree.child_begin + node);
          const int c = __ldg(a.tree.child_count + node);
          const bool in_smem = (lvl == 0) && a.root_smem_rows > 0;
          bk = 0ull;
          score_rows<VPL, false>(in_smem ? root_tab : a.tree.cent, ld, in_smem ? 0 : b, nullptr,
                                 c, r, lane, bk, bs);
          ipc += c;
          node = b + key_id(bk);
          if (a.path != nullptr && lane == 0) a.path[(p * K + t) * L + lvl] = node;
        }
        const int b = __ldg(a.tree.child_begin + node);
        const int c = __ldg(a.tree.child_count + node);
        bk = 0ull;
        score_rows<VPL, true>(a.atoms, ld, 0, a.tree.leaf_atom + b, c, r, lane, bk, bs);
        ipa += c;
      } else {
        score_rows<VPL, false>(a.atoms, ld, 0, nullptr, (int)a.m, r, lane, bk, bs);
        ipa += (int)a.m;
      }
      const int atom = key_id(bk);

      if (a.method == kMethodSelect) {
        if (lane == 0) {
          a.idx[p * K] = atom;
          a.coef[p * K] = bs;
        }
        t = 1;
        break;
      }
      if (bs == 0.f) break;  // pursuit.py:217
      if (a.method == kMethodOMP) {
        bool dup = false;
        for (int j = 0; j < t; ++j) dup |= (sidx[j] == atom);
        if (dup) break;  // re-selection ends the OMP loop
      }
      if (lane == 0) a.idx[p * K + t] = atom;
      const float* arow = a.atoms + (int64_t)atom * ld + lane;

      if (a.method == kMethodMP) {
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          r[i] = fmaf(-bs, __ldg(arow + 32 * i), r[i]);
          s2 = fmaf(r[i], r[i], s2);
        }
        rnorm = sqrtf(warp_sum(s2));
        if (lane == 0) a.coef[p * K + t] = bs;
        ++t;
        continue;
      }

      // ---------------- OMP: incremental Cholesky of the support Gram ----------------
      float av[VPL];
      float gtt = 0.f, bt = 0.f;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        av[i] = __ldg(arow + 32 * i);
        gtt = fmaf(av[i], av[i], gtt);
        bt = fmaf(av[i], x[i], bt);
        if (a.cache_atoms) acache[t * ld + lane + 32 * i] = av[i];
      }
      if (lane == 0) sidx[t] = atom;
      __syncwarp();
      for (int j = 0; j < t; ++j) {
        const float* sj = (a.cache_atoms ? acache + (int64_t)j * ld
                                         : a.atoms + (int64_t)sidx[j] * ld) + lane;
        float part = 0.f;
#pragma unroll
        for (int i = 0; i < VPL; ++i) part = fmaf(sj[32 * i], av[i], part);
        part = warp_sum(part);
        if (lane == 0) gv[j] = part;
      }
      gtt = warp_sum(gtt);
      bt = warp_sum(bt);
      if (lane == 0) {
        float* Lt = Lm + t * (t + 1) / 2;
        float wsum = 0.f;
        for (int j = 0; j < t; ++j) {
          const float* Lj = Lm + j * (j + 1) / 2;
          float v = gv[j];
          for (int k = 0; k < j; ++k) v = fmaf(-Lj[k], Lt[k], v);
          v /= Lj[j];
          Lt[j] = v;
          wsum = fmaf(v, v, wsum);
        }
        const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
        Lt[t] = dg;
        float yy = bt;
        for (int j = 0; j < t; ++j) yy = fmaf(-Lt[j], yv[j], yy);
        yv[t] = yy / dg;
        for (int j = t; j >= 0; --j) {
          float v = yv[j];
          for (int k = j + 1; k <= t; ++k) v = fmaf(-Lm[k * (k + 1) / 2 + j], cv[k], v);
          cv[j] = v / Lm[j * (j + 1) / 2 + j];
        }
      }
      __syncwarp();
      ++t;
#pragma unroll
      for (int i = 0; i < VPL; ++i) r[i] = x[i];
      for (int j = 0; j < t; ++j) {
        const float cj = cv[j];
        const float* sj = (a.cache_atoms ? acache + (int64_t)j * ld
                                         : a.atoms + (int64_t)sidx[j] * ld) + lane;
#pragma unroll
        for (int i = 0; i < VPL; ++i) r[i] = fmaf(-cj, sj[32 * i], r[i]);
      }
      float s2 = 0.f;
#pragma unroll
      for (int i = 0; i < VPL; ++i) s2 = fmaf(r[i], r[i], s2);
      rnorm = sqrtf(warp_sum(s2));
    }

    // ---------------- epilogue ----------------
    if (a.method == kMethodOMP)
      for (int j = lane; j < t; j += 32) a.coef[p * K + j] = cv[j];
    for (int j = t + lane; j < K; j += 32) {
      a.idx[p * K + j] = -1;
      a.coef[p * K + j] = 0.f;
    }
    if (a.path != nullptr)
      for (int j = t * L + lane; j < K * L; j += 32) a.path[p * K * L + j] = -1;
    if (lane == 0) {
      if (a.count) a.count[p] = t;
      if (a.resnorm) a.resnorm[p] = rnorm;
      if (a.ip) {
        a.ip[2 * p] = ipc + ipa;
        a.ip[2 * p + 1] = ipc;
      }
    }
    __syncwarp();
  }
}

template <int VPL>
cudaError_t launch_vpl(const FusedArgs& a, size_t smem, int grid, cudaStream_t s) {
  auto k = encode_fused_kernel<VPL>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel(k, grid, 256, smem, s, false, a);
}

}  // namespace

int fused_vpl_for(int n) {
  static const int kV[] = {1, 2, 3, 4, 5, 6, 8, 12, 16, 24, 32, 50, 64};
  const int need = (n + 31) / 32;
  for (int v : kV)
    if (v >= need) return v;
  return -1;
}

int64_t fused_warps(int64_t N) {
  const int wpb = 8;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
  }
  const int64_t want = (N + wpb - 1) / wpb;
  const int64_t cap = (int64_t)sms * 4;
  return (want < cap ? (want > 0 ? want : 1) : cap) * wpb;
}

cudaError_t launch_encode_fused(const FusedArgs& a, cudaStream_t stream) {
  const int wpb = 8;
  const size_t smem = sizeof(float) * ((size_t)a.root_smem_rows * a.ld + (size_t)wpb * a.warp_smem_floats);
  const int grid = (int)(fused_warps(a.N) / wpb);
  switch (a.vpl) {
#define STMP_CASE(V) \
  case V:            \
    return launch_vpl<V>(a, smem, grid, stream);
    STMP_CASE(1) STMP_CASE(2) STMP_CASE(3) STMP_CASE(4) STMP_CASE(5) STMP_CASE(6) STMP_CASE(8)
    STMP_CASE(12) STMP_CASE(16) STMP_CASE(24) STMP_CASE(32) STMP_CASE(50) STMP_CASE(64)
#undef STMP_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace stmp
