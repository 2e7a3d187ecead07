// Tile-based OMP update fused with the next iteration's root scoring.
//
// One CTA owns 128 consecutive patches, one thread per patch:
//   * the patch's x row arrives with coalesced cp.async into a 128-byte
//     swizzled tile (each thread then reads its own row without bank
//     conflicts) and stays in registers as the residual accumulator;
//   * the solver state lives in workspace arrays laid out [entry][patch], so a
//     warp's loads of one entry are one 128-byte line; the Gram column comes
//     from the atom Gram table;
//   * the refit is the inverse-Cholesky update of encode_update.cu, entirely in
//     registers (K <= 8);
//   * r = x - A_S c is rebuilt with one cooperative, double-buffered gather per
//     support slot j (the 128 rows S_j of the tile, 32 KB, coalesced), so the
//     row loads of the whole tile are in flight together;
//   * the new residual is staged in TMEM as tf32 hi/lo (tcgen05.st) and scored
//     against the root's children on the tensor cores (tcgen05.mma, 3xTF32),
//     which replaces the next iteration's root scan / scatter / score passes.
// Semantics: SURVEY §8c OMP restatement over omp_refit (pursuit.py:235-250);
// root selection pursuit.py:141-153 (argmax |score|, lowest child position).
#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

namespace {

constexpr int kTT = 128;
constexpr int KM = 8;            // max support size of this kernel
constexpr uint32_t kColAcc = 64; // TMEM: A hi [0,32), A lo [32,64), accumulator [64, 64+npad)

struct UtLayout {
  uint32_t bufA, bufB, btab, rid, hist, bars, slot, total;
};

__host__ __device__ inline uint32_t ut_align(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }

__host__ __device__ inline UtLayout ut_layout(int kch, int npad) {
  UtLayout L{};
  uint32_t o = 0;
  L.bufA = o; o += (uint32_t)kch * kTT * 128u;
  L.bufB = o; o += (uint32_t)kch * kTT * 128u;
  L.btab = o; o += ut_align(table_bytes(kch, npad, false), 1024u);
  L.rid = o; o += 2 * kTT * 4;
  L.hist = o; o += 256 * 4;
  L.bars = ut_align(o, 8); o = L.bars + 2 * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

// cooperative gather of one row per tile patch (row id -1: zero fill)
template <int KCH>
__device__ __forceinline__ void tile_gather(const float* __restrict__ base, int ld, const int* rid, uint32_t dst,
                                            int tid) {
  constexpr int F = 8 * KCH;
#pragma unroll 4
  for (int e = tid; e < kTT * F; e += kTT) {
    const int row = e / F;
    const int c = e - row * F;
    const int r = rid[row];
    const uint32_t off = (uint32_t)(c >> 3) * (kTT * 128u) + sw128_offset(row, c & 7);
    cp_async16(dst + off, base + (r >= 0 ? (int64_t)r * ld + 4 * c : 0), r >= 0 ? 16u : 0u);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KCH>
__device__ __forceinline__ void own_row(const uint8_t* buf, int row, float (&v)[32 * KCH]) {
#pragma unroll
  for (int kc = 0; kc < KCH; ++kc)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 q = *reinterpret_cast<const float4*>(buf + kc * (kTT * 128u) + sw128_offset(row, c));
      v[32 * kc + 4 * c] = q.x; v[32 * kc + 4 * c + 1] = q.y;
      v[32 * kc + 4 * c + 2] = q.z; v[32 * kc + 4 * c + 3] = q.w;
    }
}

template <int KCH>
__global__ void __launch_bounds__(kTT, 2) update_tile_kernel(TileArgs a) {
  pdl_enter();
  constexpr int LD = 32 * KCH;
  constexpr int F = 8 * KCH;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const UtLayout Ly = ut_layout(KCH, a.root_npad);
  uint8_t* bufA = base + Ly.bufA;
  uint8_t* bufB = base + Ly.bufB;
  uint8_t* btab = base + Ly.btab;
  int* s_rid = reinterpret_cast<int*>(base + Ly.rid);   // [2][128]
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + Ly.bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.slot);
  const uint32_t bufA_s = smem_u32(bufA), bufB_s = smem_u32(bufB);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int64_t N = a.u.N;
  const int64_t p0 = (int64_t)blockIdx.x * kTT;
  const int64_t p = p0 + tid;
  const bool inb = p < N;
  const int64_t pc = inb ? p : N - 1;
  const int K = a.u.K;
  const bool do_root = a.do_root != 0;
  const uint32_t tb = table_bytes(KCH, a.root_npad, false);

  if (do_root && warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if (do_root) {
      mbar_arrive_expect_tx(&bars[0], tb);
      for (uint32_t off = 0; off < tb; off += 65536u)
        bulk_g2s(btab + off, reinterpret_cast<const uint8_t*>(a.root_table) + off, min(65536u, tb - off), &bars[0]);
    }
  }
  for (int i = tid; i < 256; i += kTT) s_hist[i] = 0;
  // x tile (contiguous rows of the padded x) -> bufA
  s_rid[tid] = inb ? (int)p : -1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = do_root ? *tmem_slot : 0u;
  tile_gather<KCH>(a.u.X2, LD, s_rid, bufA_s, tid);

  // patch state: coalesced [entry][patch] loads, all independent
  bool act = inb && a.u.active[pc];
  const int t = a.u.count[pc];
  const int atom = a.u.leaf_sel[pc];
  int S[KM];
  float cprev[KM], y[KM], M[KM * (KM + 1) / 2], g[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    S[k] = k < K ? a.S_ws[(int64_t)k * N + pc] : 0;
    cprev[k] = k < K ? a.c_ws[(int64_t)k * N + pc] : 0.f;
    y[k] = k < K ? a.u.yv[(int64_t)k * N + pc] : 0.f;
  }
#pragma unroll
  for (int q = 0; q < KM * (KM + 1) / 2; ++q) M[q] = q < K * (K + 1) / 2 ? a.u.Lf[(int64_t)q * N + pc] : 0.f;
  // entries beyond the current support are stale workspace: zero them (selects,
  // no extra round trip) so 0 * NaN cannot leak into the sums below
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    cprev[k] = k < t ? cprev[k] : 0.f;
    y[k] = k < t ? y[k] : 0.f;
  }
#pragma unroll
  for (int j = 0; j < KM; ++j)
#pragma unroll
    for (int k = 0; k <= j; ++k) M[j * (j + 1) / 2 + k] = j < t ? M[j * (j + 1) / 2 + k] : 0.f;
  const float* grow = a.u.gram + (int64_t)(atom >= 0 ? atom : 0) * a.u.m;
  bool dup = false;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const bool in = k < t;
    g[k] = in ? __ldg(grow + S[k]) : 0.f;
    dup |= in && S[k] == atom;
  }
  const float gtt = __ldg(grow + (atom >= 0 ? atom : 0));

  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  float r[LD];
  own_row<KCH>(bufA, tid, r);   // x
  __syncthreads();              // bufA free
  // gather the selected atoms' rows of the tile
  s_rid[tid] = act ? atom : -1;
  __syncthreads();
  tile_gather<KCH>(a.u.atoms, LD, s_rid, bufA_s, tid);

  // refit scalars that do not need a . x
  float gc = 0.f;
#pragma unroll
  for (int k = 0; k < KM; ++k) gc = fmaf(g[k], cprev[k], gc);   // g[k] = 0 for k >= t
  float w[KM];
  float wsum = 0.f, wy = 0.f;
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k <= j; ++k) acc = fmaf(M[j * (j + 1) / 2 + k], g[k], acc);
    w[j] = j < t ? acc : 0.f;
    wsum = fmaf(w[j], w[j], wsum);
    wy = fmaf(w[j], y[j], wy);
  }

  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  float av[LD];
  own_row<KCH>(bufA, tid, av);
  float bt = 0.f;
#pragma unroll
  for (int i = 0; i < LD; ++i) bt = fmaf(av[i], r[i], bt);
  const float score = bt - gc;   // a . r for r = x - A_S c_prev (pursuit.py:217 check)
  const bool ok = act && !dup && score != 0.f;
  const float dg = sqrtf(fmaxf(gtt + kRidge - wsum, 1e-30f));
  const float inv_d = 1.f / dg;
  const float yy = (bt - wy) * inv_d;
  float mt[KM + 1], cn[KM + 1];
#pragma unroll
  for (int k = 0; k <= KM; ++k) {
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (k <= j) {
        const float Mjk = M[j * (j + 1) / 2 + k];
        s1 = fmaf(w[j], Mjk, s1);    // w[j] = 0 for j >= t
        s2 = fmaf(j < t ? y[j] : 0.f, Mjk, s2);
      }
    }
    mt[k] = k < t ? -inv_d * s1 : (k == t ? inv_d : 0.f);
    cn[k] = k < t ? fmaf(mt[k], yy, s2) : (k == t ? inv_d * yy : 0.f);
  }
  // residual: r = x - c_t a_new - sum_j c_j a_{S_j}
  float ct = 0.f;
#pragma unroll
  for (int k = 0; k <= KM; ++k) ct = k == t ? cn[k] : ct;
  if (ok) {
#pragma unroll
    for (int i = 0; i < LD; ++i) r[i] = fmaf(-ct, av[i], r[i]);
  }
  const int T = a.iter;   // every active patch of this iteration holds t == iter atoms
  __syncthreads();        // bufA (a_new rows) consumed
  if (T > 0) {
    s_rid[tid] = ok && 0 < t ? S[0] : -1;
    __syncthreads();
    tile_gather<KCH>(a.u.atoms, LD, s_rid, bufB_s, tid);
  }
  for (int j = 0; j < T; ++j) {
    const bool has_next = j + 1 < T;
    if (has_next) {
      int nid = -1;
#pragma unroll
      for (int k = 0; k < KM; ++k) nid = (k == j + 1 && ok && k < t) ? S[k] : nid;
      s_rid[((j + 1) & 1) * kTT + tid] = nid;
    }
    __syncthreads();   // row ids visible; everyone is done with the buffer refilled below
    if (has_next) tile_gather<KCH>(a.u.atoms, LD, s_rid + ((j + 1) & 1) * kTT, (j & 1) ? bufB_s : bufA_s, tid);
    if (has_next) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const uint8_t* cur = (j & 1) ? bufA : bufB;
    if (ok && j < t) {
      float cj = 0.f;
#pragma unroll
      for (int k = 0; k < KM; ++k) cj = k == j ? cn[k] : cj;
      float v[LD];
      own_row<KCH>(cur, tid, v);
#pragma unroll
      for (int i = 0; i < LD; ++i) r[i] = fmaf(-cj, v[i], r[i]);
    }
  }
  float s2 = 0.f;
#pragma unroll
  for (int i = 0; i < LD; ++i) s2 = fmaf(r[i], r[i], s2);
  const float rn = sqrtf(s2);
  const bool act_next = ok && (t + 1 < K) && rn > a.u.tol[pc];

  // ---- outputs and state (writes of one entry are coalesced across the warp)
  if (ok) {
    const int KK = K * (K + 1) / 2;
#pragma unroll
    for (int k = 0; k <= KM; ++k) {
      if (k <= t && k < K) {
        a.u.Lf[(int64_t)(t * (t + 1) / 2 + k) * N + p] = mt[k];
        a.c_ws[(int64_t)k * N + p] = cn[k];
        a.u.coef[p * K + k] = cn[k];
      }
    }
    (void)KK;
    if (t < K) {
      a.u.yv[(int64_t)t * N + p] = yy;
      a.S_ws[(int64_t)t * N + p] = atom;
      a.u.idx[p * K + t] = atom;
    }
    a.u.count[p] = t + 1;
    a.u.resnorm[p] = rn;
  }
  if (inb && act) a.u.active[p] = act_next ? 1 : 0;

  // ---- new residual: coalesced write-out through the swizzled tile (bufA)
  __syncthreads();
#pragma unroll
  for (int kc = 0; kc < KCH; ++kc)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<float4*>(bufA + kc * (kTT * 128u) + sw128_offset(tid, c)) =
          make_float4(r[32 * kc + 4 * c], r[32 * kc + 4 * c + 1], r[32 * kc + 4 * c + 2], r[32 * kc + 4 * c + 3]);
  __syncthreads();
#pragma unroll 4
  for (int e = tid; e < kTT * F; e += kTT) {
    const int row = e / F;
    const int c = e - row * F;
    if (p0 + row < N) {
      const float4 v = *reinterpret_cast<const float4*>(bufA + (c >> 3) * (kTT * 128u) + sw128_offset(row, c & 7));
      reinterpret_cast<float4*>(a.u.R + (p0 + row) * LD)[c] = v;
    }
  }

  // ---- next iteration's root scoring on the tensor cores
  if (do_root) {
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int npad = a.root_npad;
    const uint32_t idesc = idesc_tf32(kTT, npad);
    const uint32_t b_s = smem_u32(btab);
    uint32_t phase = 0;
#pragma unroll
    for (int kc = 0; kc < KCH; ++kc) {
      float hi[32], lo[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        hi[q] = tf32_hi(r[32 * kc + q]);
        lo[q] = r[32 * kc + q] - hi[q];
      }
      if (kc > 0) {
        mbar_wait(&bars[1], phase);
        phase ^= 1u;
        tc_fence_after();
      }
      tmem_st32(tmem + lane_base, hi);
      tmem_st32(tmem + lane_base + 32, lo);
      tmem_wait_st();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        if (kc == 0) mbar_wait(&bars[0], 0);
        tc_fence_after();
        const uint32_t bh = b_s + kc * (2u * npad * 128u);
        const uint32_t bl = bh + npad * 128u;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = ks * 32u;
          mma_tf32_ts(tmem + kColAcc, tmem + ks * 8, sw128_kmajor_desc(bh + o), idesc, (kc | ks) ? 1u : 0u);
          mma_tf32_ts(tmem + kColAcc, tmem + ks * 8, sw128_kmajor_desc(bl + o), idesc, 1u);
          mma_tf32_ts(tmem + kColAcc, tmem + 32 + ks * 8, sw128_kmajor_desc(bh + o), idesc, 1u);
        }
        mma_commit(&bars[1]);
      }
    }
    __syncwarp();
    mbar_wait(&bars[1], phase);
    tc_fence_after();
    const int cc = a.root_cc;
    int best = 0;
    float bestv = -1.f;
    for (int col0 = 0; col0 < npad; col0 += 32) {
      float v[32];
      tmem_ld32(tmem + lane_base + kColAcc + (uint32_t)col0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float mv = fabsf(v[j]);
        if (col0 + j < cc && mv > bestv) {
          bestv = mv;
          best = col0 + j;
        }
      }
    }
    if (act_next) {
      const int child = a.root_cb + best;
      a.path_ws[p * a.L] = child;
      if (a.u.path_out) a.u.path_out[(p * K + (t + 1)) * a.L] = child;
      atomicAdd(&s_hist[best], 1);
      if (a.u.ip) {  // ScoreCounter: the root's children for the next selection
        add_ip(a.u.ip, p, cc, cc);
      }
    }
    __syncthreads();
    for (int j = tid; j < cc; j += kTT) {
      const int h = s_hist[j];
      if (h) atomicAdd(&a.next_counts[a.root_cb + j - a.next_base], h);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
  }
}

template <int KCH>
cudaError_t launch_tile(TileArgs a, cudaStream_t st) {
  const UtLayout Ly = ut_layout(KCH, a.root_npad);
  int cols = 32;
  while (cols < (int)kColAcc + a.root_npad) cols <<= 1;
  a.tmem_cols = cols;
  cudaError_t e = cudaFuncSetAttribute(update_tile_kernel<KCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Ly.total);
  if (e != cudaSuccess) return e;
  const int blocks = (int)((a.u.N + kTT - 1) / kTT);
  return launch_kernel(update_tile_kernel<KCH>, blocks, kTT, (size_t)Ly.total, st, true, a);
}

}  // namespace

bool update_tile_supported(const DictHandle* d, const TreeHandle* t, int K, int method) {
  if (method != kMethodOMP || K > KM || t == nullptr || t->levels < 2) return false;
  if (d->ld != 32 && d->ld != 64) return false;
  if (d->m > kGramMaxAtoms) return false;
  if (t->max_leaf_children != 1) return false;
  if (t->staged_levels.empty() || t->staged_levels[0].npad + (int)kColAcc > 128) return false;
  return ut_layout(d->ld / 32, t->staged_levels[0].npad).total <= 110 * 1024;
}

cudaError_t launch_update_tile(const TileArgs& a, cudaStream_t st) {
  switch (a.u.ld) {
    case 32: return launch_tile<1>(a, st);
    case 64: return launch_tile<2>(a, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace stmp
