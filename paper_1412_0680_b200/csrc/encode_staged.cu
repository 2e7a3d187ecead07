// Staged (level-synchronous) encoder for large batches.
//
// One greedy-pursuit iteration over all active patches is L+1 passes:
//   for each tree level l:  scan(bins of depth-l nodes) -> scatter(perm) ->
//                           score_tc(l): per (node, 128-patch tile) work item,
//                           gather the tile's residual rows, multiply against
//                           the node's child-centroid table on the 5th-gen
//                           tensor cores (tcgen05.mma kind::tf32, 3xTF32 split
//                           for fp32 accuracy, accumulator in TMEM), argmax
//                           epilogue straight out of TMEM (one thread per
//                           patch row), bucket the winners for the next level;
//   update: leaf choice + MP step or OMP incremental-Cholesky refit, residual
//           rebuilt and written once.
// Reference semantics are the same as encode_fused.cu (see its header).
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

namespace {

constexpr int kTile = 128;          // patches per work item (= UMMA M)
constexpr int kScoreThreads = 128;  // 4 warps: warp w owns TMEM lanes 32w..32w+31

// ------------------------------------------------------------------ score (tcgen05)
__global__ void __launch_bounds__(kScoreThreads, 1) score_tc_kernel(ScoreArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int kch = a.kchunks;
  const int npad = a.npad;
  float* Ahi = reinterpret_cast<float*>(base);
  float* Alo = Ahi + kch * kTile * 32;
  float* Btab = Alo + kch * kTile * 32;
  const uint32_t tab_bytes = (uint32_t)kch * 2u * npad * 128u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(Btab) + tab_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  int* s_rows = reinterpret_cast<int*>(tmem_slot + 4);
  int* s_hist = s_rows + kTile;      // [npad] local counts of the winning child
  int* s_base = s_hist + 256;        // [npad] global base rank per child

  if (warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 256; i += kScoreThreads) s_hist[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int num_items = *a.num_items;
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int i1 = min(num_items, i0 + per);
  int loaded_bin = -1;
  uint32_t tab_phase = 0, mma_phase = 0;
  const int F = a.ld >> 2;  // float4 per residual row
  const uint32_t idesc = idesc_tf32(kTile, npad);
  const uint32_t a_hi_s = smem_u32(Ahi), a_lo_s = smem_u32(Alo), b_s = smem_u32(Btab);

  for (int item = i0; item < i1; ++item) {
    const int4 it = a.items[item];
    const int bin = it.x, start = it.y, rows = it.z;
    if (tid < rows) s_rows[tid] = a.perm[start + tid];
    const bool new_tab = bin != loaded_bin;
    if (new_tab && tid == 0) {
      mbar_arrive_expect_tx(&bars[0], tab_bytes);
      const uint8_t* src = reinterpret_cast<const uint8_t*>(a.table) + (size_t)bin * tab_bytes;
      // chunked bulk copies (each <= 64 KB)
      for (uint32_t off = 0; off < tab_bytes; off += 65536u) {
        const uint32_t sz = min(65536u, tab_bytes - off);
        bulk_g2s(reinterpret_cast<uint8_t*>(Btab) + off, src + off, sz, &bars[0]);
      }
    }
    loaded_bin = bin;
    __syncthreads();

    // gather the tile's residual rows into the SW128 K-major hi/lo planes
    for (int e = tid; e < kTile * F; e += kScoreThreads) {
      const int row = e / F;
      const int c = e - row * F;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < rows) v = __ldg(reinterpret_cast<const float4*>(a.R + (int64_t)s_rows[row] * a.ld) + c);
      float4 h, l;
      h.x = tf32_hi(v.x); h.y = tf32_hi(v.y); h.z = tf32_hi(v.z); h.w = tf32_hi(v.w);
      l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
      const uint32_t off = (uint32_t)(c >> 3) * (kTile * 128u) + sw128_offset(row, c & 7);
      *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(Ahi) + off) = h;
      *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(Alo) + off) = l;
    }
    fence_proxy_async_smem();
    __syncthreads();

    if (tid == 0) {
      if (new_tab) {
        mbar_wait(&bars[0], tab_phase);
        tab_phase ^= 1u;
      }
      tc_fence_after();
      for (int kc = 0; kc < kch; ++kc) {
        const uint32_t ah = a_hi_s + kc * (kTile * 128u);
        const uint32_t al = a_lo_s + kc * (kTile * 128u);
        const uint32_t bh = b_s + kc * (2u * npad * 128u);
        const uint32_t bl = bh + npad * 128u;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = ks * 32u;
          mma_tf32(tmem, sw128_kmajor_desc(ah + o), sw128_kmajor_desc(bh + o), idesc, (kc | ks) ? 1u : 0u);
          mma_tf32(tmem, sw128_kmajor_desc(ah + o), sw128_kmajor_desc(bl + o), idesc, 1u);
          mma_tf32(tmem, sw128_kmajor_desc(al + o), sw128_kmajor_desc(bh + o), idesc, 1u);
        }
      }
      mma_commit(&bars[1]);
    }
    __syncwarp();
    mbar_wait(&bars[1], mma_phase);
    mma_phase ^= 1u;
    tc_fence_after();

    // epilogue: thread = patch row, argmax |score| over the node's children
    const int gnode = a.level_base + bin;
    const int cb = __ldg(a.child_begin + gnode);
    const int cc = __ldg(a.child_count + gnode);
    int best = 0;
    float bestv = -1.f;
    for (int col0 = 0; col0 < npad; col0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)col0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float m = fabsf(v[j]);
        if (col0 + j < cc && m > bestv) {
          bestv = m;
          best = col0 + j;
        }
      }
    }
    const int row = tid;
    const bool valid = row < rows;
    const int p = valid ? s_rows[row] : 0;
    const int child = cb + best;
    int local = 0;
    if (valid) {
      a.path_ws[(int64_t)p * a.L + a.level] = child;
      if (a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = child;
      if (a.next_counts) local = atomicAdd(&s_hist[best], 1);
    }
    if (a.next_counts) {
      __syncthreads();
      for (int j = tid; j < cc; j += kScoreThreads) {
        const int h = s_hist[j];
        if (h) s_base[j] = atomicAdd(&a.next_counts[cb + j - a.next_base], h);
        s_hist[j] = 0;
      }
      __syncthreads();
      if (valid) a.rank[p] = s_base[best] + local;
    }
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

// ------------------------------------------------------------------ scan (one CTA)
constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads) scan_kernel(int* counts, int nbins, int* offsets,
                                                             int4* items, int* num_items,
                                                             int* tile_off) {
  using Scan = cub::BlockScan<int, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry[2];
  if (threadIdx.x == 0) carry[0] = carry[1] = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nbins; b0 += kScanThreads) {
    const int b = b0 + threadIdx.x;
    const int c = b < nbins ? counts[b] : 0;
    const int tiles = (c + kTile - 1) / kTile;
    int pre_c, pre_t, tot_c, tot_t;
    Scan(tmp).ExclusiveSum(c, pre_c, tot_c);
    __syncthreads();
    Scan(tmp).ExclusiveSum(tiles, pre_t, tot_t);
    if (b < nbins) {
      offsets[b] = carry[0] + pre_c;
      tile_off[b] = carry[1] + pre_t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] += tot_c;
      carry[1] += tot_t;
    }
    __syncthreads();
  }
  const int total_tiles = carry[1];
  // one item per tile: binary-search the bin owning tile i
  for (int i = threadIdx.x; i < total_tiles; i += kScanThreads) {
    int lo = 0, hi = nbins - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tile_off[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int k = i - tile_off[lo];
    const int c = counts[lo];
    items[i] = make_int4(lo, offsets[lo] + k * kTile, min(kTile, c - k * kTile), 0);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += kScanThreads) counts[b] = 0;
  if (threadIdx.x == 0) *num_items = total_tiles;
}

// ------------------------------------------------------------------ scatter
__global__ void scatter_kernel(int64_t N, const int* rank, const int* path_ws, int L, int level,
                               int level_base, const int* offsets, int* perm) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int r = rank[p];
  if (r < 0) return;
  const int bin = level == 0 ? 0 : path_ws[p * L + level - 1] - level_base;
  perm[offsets[bin] + r] = (int)p;
}

// ------------------------------------------------------------------ group helpers
template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// warp-aggregated rank in the single root bin for lanes with `act` (group leaders only)
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
  } else {
#pragma unroll
    for (int i = 0; i < E / 2; ++i) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(src) + i);
      v[2 * i] = q.x; v[2 * i + 1] = q.y;
    }
  }
}

template <int E>
__device__ __forceinline__ void store_vec(float* dst, const float (&v)[E]) {
  if constexpr (E % 4 == 0) {
#pragma unroll
    for (int i = 0; i < E / 4; ++i)
      reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < E / 2; ++i) reinterpret_cast<float2*>(dst)[i] = make_float2(v[2 * i], v[2 * i + 1]);
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
    act = xn > tol;
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
template <int G, int E>
__global__ void __launch_bounds__(128) update_kernel(UpdateArgs a) {
  extern __shared__ float upd_smem[];
  const int gpb = blockDim.x / G;
  const int grp = threadIdx.x / G;
  const int64_t p = (int64_t)blockIdx.x * gpb + grp;
  const int gl = threadIdx.x % G;
  const int K = a.K;
  float* wv = upd_smem + grp * 2 * K;   // new Cholesky row w (then reused)
  float* cv = wv + K;                    // coefficients
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
    int32_t* S = a.idx + p * K;
    if (a.method == kMethodMP) {
      const float s = group_sum<G>(dot_vec<E>(av, r));
      if (s == 0.f) {
        act = false;
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
      bool dup = false;
      for (int j = 0; j < t; ++j) dup |= (S[j] == atom);
      float x[E];
      load_vec<E>(a.X2 + p * a.ld2 + off, x);
      const float bt = group_sum<G>(dot_vec<E>(av, x));
      const float gtt = group_sum<G>(dot_vec<E>(av, av));
      float* Lp = a.Lf + p * (int64_t)(K * (K + 1) / 2);
      float* yp = a.yv + p * (int64_t)K;
      float* Lt = Lp + t * (t + 1) / 2;
      // Gram column against the current support; forward substitution row by row
      float wsum = 0.f, gc = 0.f;
      for (int j = 0; j < t; ++j) {
        float sj[E];
        load_vec<E>(a.atoms + (int64_t)S[j] * a.ld + off, sj);
        const float g = group_sum<G>(dot_vec<E>(sj, av));
        gc = fmaf(g, a.coef[p * K + j], gc);   // a . A_S c_prev  (score identity)
        const float* Lj = Lp + j * (j + 1) / 2;
        float v = g;
        for (int k = 0; k < j; ++k) v = fmaf(-Lj[k], wv[k], v);
        v /= Lj[j];
        wv[j] = v;
        wsum = fmaf(v, v, wsum);
      }
      const float score = bt - gc;   // a . r with r = x - A_S c (pursuit.py:217 check)
      if (dup || score == 0.f) {
        act = false;
      } else {
        const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
        float yy = bt;
        for (int j = 0; j < t; ++j) yy = fmaf(-wv[j], yp[j], yy);
        yy /= dg;
        // back substitution L^T c = y over the t+1 unknowns; row t of L is (w, dg)
        for (int j = t; j >= 0; --j) {
          float v = j == t ? yy : yp[j];
          for (int k = j + 1; k <= t; ++k) {
            const float Lkj = k == t ? wv[j] : Lp[k * (k + 1) / 2 + j];
            v = fmaf(-Lkj, cv[k], v);
          }
          cv[j] = v / (j == t ? dg : Lp[j * (j + 1) / 2 + j]);
        }
        // residual r = x - A_S c, rebuilt with the new atom
#pragma unroll
        for (int i = 0; i < E; ++i) r[i] = fmaf(-cv[t], av[i], x[i]);
        for (int j = 0; j < t; ++j) {
          float sj[E];
          load_vec<E>(a.atoms + (int64_t)S[j] * a.ld + off, sj);
          const float cj = cv[j];
#pragma unroll
          for (int i = 0; i < E; ++i) r[i] = fmaf(-cj, sj[i], r[i]);
        }
        store_vec<E>(a.R + p * a.ld + off, r);
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < E; ++i) s2 = fmaf(r[i], r[i], s2);
        const float rn = sqrtf(group_sum<G>(s2));
        if (gl == 0) {
          for (int j = 0; j < t; ++j) Lt[j] = wv[j];
          Lt[t] = dg;
          yp[t] = yy;
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

// ------------------------------------------------------------------ dispatch helpers
struct GE {
  int G, E;
};

bool pick_ge(int ld, GE& ge) {
  static const GE table[] = {{1, 32}, {2, 32}, {2, 48}, {4, 32}, {4, 40}, {4, 48}, {8, 32}, {8, 40},
                             {8, 48}, {16, 32}, {16, 40}, {16, 48}, {32, 32}, {32, 40}, {32, 48}, {32, 50}};
  for (const GE& g : table)
    if (g.G * g.E == ld) { ge = g; return true; }
  return false;
}

#define STMP_GE_SWITCH(ge, KERNEL, ...)                                                  \
  do {                                                                                   \
    switch (ge.G * 1000 + ge.E) {                                                        \
      case 1032: KERNEL<1, 32> __VA_ARGS__; break;                                       \
      case 2032: KERNEL<2, 32> __VA_ARGS__; break;                                       \
      case 2048: KERNEL<2, 48> __VA_ARGS__; break;                                       \
      case 4032: KERNEL<4, 32> __VA_ARGS__; break;                                       \
      case 4040: KERNEL<4, 40> __VA_ARGS__; break;                                       \
      case 4048: KERNEL<4, 48> __VA_ARGS__; break;                                       \
      case 8032: KERNEL<8, 32> __VA_ARGS__; break;                                       \
      case 8040: KERNEL<8, 40> __VA_ARGS__; break;                                       \
      case 8048: KERNEL<8, 48> __VA_ARGS__; break;                                       \
      case 16032: KERNEL<16, 32> __VA_ARGS__; break;                                     \
      case 16040: KERNEL<16, 40> __VA_ARGS__; break;                                     \
      case 16048: KERNEL<16, 48> __VA_ARGS__; break;                                     \
      case 32032: KERNEL<32, 32> __VA_ARGS__; break;                                     \
      case 32040: KERNEL<32, 40> __VA_ARGS__; break;                                     \
      case 32048: KERNEL<32, 48> __VA_ARGS__; break;                                     \
      case 32050: KERNEL<32, 50> __VA_ARGS__; break;                                     \
      default: return cudaErrorInvalidValue;                                             \
    }                                                                                    \
  } while (0)

}  // namespace

size_t score_smem_bytes(int kchunks, int npad) {
  return 1024 + (size_t)kchunks * kTile * 128 * 2 + (size_t)kchunks * 2 * npad * 128 + 16 + 16 +
         (kTile + 512) * 4;
}

bool staged_supported(const DictHandle* d, const TreeHandle* t, int K, int method) {
  if (t == nullptr || (method != kMethodMP && method != kMethodOMP)) return false;
  GE ge;
  if (!pick_ge(d->ld, ge)) return false;
  if (t->staged_tables.empty()) return false;
  if (K > 64) return false;
  return true;
}

bool build_staged_tables(TreeHandle* t, const int32_t* child_begin, const int32_t* child_count,
                         const float* centroids, cudaStream_t st, std::string* err) {
  GE ge;
  if (!pick_ge(t->ld, ge)) return false;
  const int L = t->levels;
  const int kch = t->ld / 32;
  std::vector<StagedLevel> levels(L);
  for (int l = 0; l < L; ++l) {
    int mx = 1;
    for (int64_t v = t->level_offsets[l]; v < t->level_offsets[l + 1]; ++v) mx = std::max(mx, child_count[v]);
    if (mx > 256) return false;
    levels[l].npad = std::max(16, (mx + 15) / 16 * 16);
    int cols = 32;
    while (cols < levels[l].npad) cols <<= 1;
    levels[l].tmem_cols = cols;
    if (score_smem_bytes(kch, levels[l].npad) > 227 * 1024) return false;
  }
  std::vector<float*> tables(L, nullptr);
  for (int l = 0; l < L; ++l) {
    const int npad = levels[l].npad;
    const int64_t nodes = t->level_offsets[l + 1] - t->level_offsets[l];
    const size_t per_node = (size_t)kch * 2 * npad * 32;  // floats
    std::vector<float> host(per_node * nodes, 0.f);
    for (int64_t i = 0; i < nodes; ++i) {
      const int64_t v = t->level_offsets[l] + i;
      const int cb = child_begin[v], cc = child_count[v];
      float* blk = host.data() + per_node * i;
      for (int j = 0; j < cc; ++j) {
        const float* row = centroids + (int64_t)(cb + j) * t->n;
        for (int col = 0; col < t->n; ++col) {
          const float val = row[col];
          const float hi = sm100::tf32_hi(val);
          const float lo = val - hi;
          const int kc = col / 32, e = col % 32;
          const uint32_t off = sm100::sw128_offset(j, e / 4) / 4 + (e % 4);
          float* plane = blk + (size_t)kc * 2 * npad * 32;
          plane[off] = hi;
          plane[npad * 32 + off] = lo;
        }
      }
    }
    cudaError_t e = cudaMalloc(&tables[l], host.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tables[l], host.data(), host.size() * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      for (float* p : tables) cudaFree(p);
      if (err) *err = cudaGetErrorString(e);
      return false;
    }
  }
  t->staged_levels = levels;
  t->staged_tables = tables;
  return true;
}

void free_staged_tables(TreeHandle* t) {
  for (float* p : t->staged_tables) cudaFree(p);
  t->staged_tables.clear();
  t->staged_levels.clear();
}

size_t staged_workspace_bytes(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method) {
  const int L = t->levels;
  int64_t maxbins = 1, sumbins = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t b = t->level_offsets[l + 1] - t->level_offsets[l];
    maxbins = b > maxbins ? b : maxbins;
    sumbins += b;
  }
  size_t s = 0;
  auto add = [&](size_t bytes) { s += (bytes + 255) & ~(size_t)255; };
  add((size_t)N * d->ld * 4);              // R
  if (method == kMethodOMP) add((size_t)N * d->ld * 4);  // padded copy of X
  add((size_t)N * 4);                      // tol
  add((size_t)N * 4);                      // active
  add((size_t)N * 4);                      // rank
  add((size_t)N * 4);                      // perm
  add((size_t)N * L * 4);                  // path_ws
  add((size_t)N * K * (K + 1) / 2 * 4);    // Cholesky factors
  add((size_t)N * K * 4);                  // y
  add((size_t)sumbins * 4);                // per-level bin counts
  add((size_t)(maxbins + 1) * 4);          // offsets
  add((size_t)(maxbins + 1) * 4);          // tile offsets
  add((size_t)(N / kTile + maxbins + 2) * 16);  // items
  add(16);                                 // num_items
  return s;
}

cudaError_t run_staged(const DictHandle* d, const TreeHandle* t, const float* X, int64_t N,
                       int64_t ldx, int K, int method, float tol_abs, int32_t* idx, float* coef,
                       int32_t* count, float* resnorm, int32_t* path, int32_t* ip, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  if (ws == nullptr || ws_bytes < staged_workspace_bytes(d, t, N, K, method)) return cudaErrorInvalidValue;
  const int L = t->levels;
  uint8_t* w = static_cast<uint8_t*>(ws);
  auto take = [&](size_t bytes) {
    void* p = w;
    w += (bytes + 255) & ~(size_t)255;
    return p;
  };
  int64_t maxbins = 1, sumbins = 0;
  std::vector<int64_t> bin_off(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    const int64_t b = t->level_offsets[l + 1] - t->level_offsets[l];
    maxbins = b > maxbins ? b : maxbins;
    bin_off[l + 1] = bin_off[l] + b;
  }
  sumbins = bin_off[L];
  float* R = (float*)take((size_t)N * d->ld * 4);
  float* Xpad = method == kMethodOMP ? (float*)take((size_t)N * d->ld * 4) : nullptr;
  float* tol = (float*)take((size_t)N * 4);
  int* active = (int*)take((size_t)N * 4);
  int* rank = (int*)take((size_t)N * 4);
  int* perm = (int*)take((size_t)N * 4);
  int* path_ws = (int*)take((size_t)N * L * 4);
  float* Lf = (float*)take((size_t)N * K * (K + 1) / 2 * 4);
  float* yv = (float*)take((size_t)N * K * 4);
  int* counts = (int*)take((size_t)sumbins * 4);
  int* offsets = (int*)take((size_t)(maxbins + 1) * 4);
  int* tile_off = (int*)take((size_t)(maxbins + 1) * 4);
  int4* items = (int4*)take((size_t)(N / kTile + maxbins + 2) * 16);
  int* num_items = (int*)take(16);

  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)sumbins * 4, st);
  if (e != cudaSuccess) return e;

  GE ge;
  pick_ge(d->ld, ge);
  UpdateArgs u{};
  u.X = X; u.ldx = ldx; u.n = d->n; u.R = R; u.ld = d->ld;
  u.X2 = Xpad; u.ld2 = d->ld;  // OMP rebuilds r from this padded copy of x
  u.atoms = d->atoms; u.child_begin = t->child_begin; u.child_count = t->child_count;
  u.leaf_atom = t->leaf_atom; u.L = L; u.path_ws = path_ws; u.K = K; u.method = method;
  u.tol_abs = tol_abs; u.idx = idx; u.coef = coef; u.count = count; u.resnorm = resnorm;
  u.ip = ip; u.path_out = path; u.Lf = Lf; u.yv = yv; u.tol = tol; u.active = active;
  u.rank = rank; u.root_count = counts; u.N = N;

  const int gpb = 128 / ge.G;
  const int ublocks = (int)((N + gpb - 1) / gpb);
  // init writes the padded x into R (and into Xpad for OMP, whose update
  // rebuilds r = x - A_S c every iteration)
  STMP_GE_SWITCH(ge, init_kernel, <<<ublocks, 128, 0, st>>>(u));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;

  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int scatter_blocks = (int)((N + 255) / 256);
  const size_t usmem = (size_t)gpb * 2 * K * 4;

  for (int it = 0; it < K; ++it) {
    for (int l = 0; l < L; ++l) {
      const StagedLevel& lv = t->staged_levels[l];
      const int nb = (int)(t->level_offsets[l + 1] - t->level_offsets[l]);
      scan_kernel<<<1, kScanThreads, 0, st>>>(counts + bin_off[l], nb, offsets, items, num_items, tile_off);
      scatter_kernel<<<scatter_blocks, 256, 0, st>>>(N, rank, path_ws, L, l, (int)t->level_offsets[l],
                                                    offsets, perm);
      ScoreArgs s{};
      s.R = R; s.ld = d->ld; s.perm = perm; s.items = items; s.num_items = num_items;
      s.table = t->staged_tables[l]; s.npad = lv.npad; s.kchunks = d->ld / 32; s.tmem_cols = lv.tmem_cols;
      s.level = l; s.level_base = (int)t->level_offsets[l]; s.child_begin = t->child_begin;
      s.child_count = t->child_count; s.path_ws = path_ws; s.path_out = path; s.count = count;
      s.K = K; s.L = L; s.rank = rank;
      if (l + 1 < L) {
        s.next_counts = counts + bin_off[l + 1];
        s.next_base = (int)t->level_offsets[l + 1];
      }
      const size_t smem = score_smem_bytes(s.kchunks, lv.npad);
      e = cudaFuncSetAttribute(score_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      const int per_sm = (int)((227 * 1024) / smem) > 0 ? (int)((227 * 1024) / smem) : 1;
      const int grid = sms * (per_sm > 2 ? 2 : per_sm);
      score_tc_kernel<<<grid, kScoreThreads, smem, st>>>(s);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    STMP_GE_SWITCH(ge, update_kernel, <<<ublocks, 128, usmem, st>>>(u));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace stmp
