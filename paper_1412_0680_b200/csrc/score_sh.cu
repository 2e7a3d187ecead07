// Level passes of the Gram path on half-precision patch rows.
//
// On the Gram path (gram_path.cu) the rows the level passes multiply are the
// patches x themselves, never a residual, so they can be prepared once per
// encode: x16 = fp16(s_p x) with a power-of-two scale s_p per patch (half the
// bytes of every pass), and the exact near-tie re-check of the epilogue
// (score_epi.cuh) widens its window by the rows' quantisation noise, so a
// decision is either unaffected by it or re-taken with exact fp32 FFMA dots.
// The child centroids keep 22 significant bits: c = p0 + 2^-11 p1 with fp16
// pieces (two adjacent row blocks of the node table; a score error below
// 2^-23 ||x||), so one tcgen05.mma.kind::f16 per 16-column k-step with
// N = 2 npad yields x16 . p0 | x16 . p1 in two accumulator column groups,
// summed with their weights and unscaled by 1 / s_p in the epilogue.
//
// Against score_st.cu (3xTF32 on fp32 rows): half the row bytes, half the
// table bytes, a third of the tensor work, and no register staging at all -- both
// operands are read from shared memory (the gathered rows land directly in the
// UMMA K-major 128-byte-swizzle layout), so the stager warps only issue
// cp.async copies.  Roles per CTA (two CTAs per SM), 320 threads:
//   * warps 0-3: row gather (thread = patch row), NA landing slots of 128 rows
//     x 64 halfs, released by the MMA commits;
//   * warp 4: MMA issuer; warp 5: table producer (one bulk copy per 64-column
//     chunk: 2 npad rows x 128 B, ring of NB slots);
//   * warps 6-9: epilogue (TMEM lane quarter = warp % 4): corrected argmax with
//     the near-tie re-check, as score_st's Gram branch.
// Semantics: pkg/src/stmp/pursuit.py:134-162 (greedy level choice, first max of
// |score| in child order; leaf metadata for the last level).
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "score_epi.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;
using namespace epi;

int g_half_scores = 1;

namespace {

constexpr int kT = 128;
constexpr int kStagers = 128;
constexpr int kEpi = 128;
constexpr int kThreads = kStagers + 64 + kEpi;
constexpr uint32_t kSlot = kT * 128u;   // one landing slot: 128 rows x 64 halfs

struct ShLayout {
  uint32_t land, btab, hist, bars, slot, total;
};

__host__ __device__ inline uint32_t sh_align(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }
__host__ __device__ inline uint32_t sh_bslot(int npad) { return sh_align((uint32_t)npad * 128u * kPieces, 1024u); }

__host__ __device__ inline ShLayout sh_layout(int npad, int na, int nb) {
  ShLayout L{};
  uint32_t o = 0;
  L.land = o; o += (uint32_t)na * kSlot;
  L.btab = o; o += (uint32_t)nb * sh_bslot(npad);
  L.hist = o; o += 256 * 4;
  L.bars = sh_align(o, 8); o = L.bars + (uint32_t)(2 * nb + 2 * na + 4) * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

// Instruction descriptor: kind::f16, fp16 A and B, f32 accumulate, both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16, one CTA.
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int NA, int NB, int CPS>
__global__ void __launch_bounds__(kThreads, CPS) score_sh_kernel(ScoreArgs a, int nacc) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int npad = a.npad;
  const int kch = a.kchunks;   // 64-column chunks
  const bool last = a.leaf_sel != nullptr;
  const ShLayout Ly = sh_layout(npad, NA, NB);
  const uint32_t bslot = sh_bslot(npad);
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Ly.bars);   // [NB] table chunk landed (tx)
  uint64_t* done = full + NB;          // [NB] MMAs reading the table slot retired (commit)
  uint64_t* astaged = done + NB;       // [NA] row slot landed (128 stager threads)
  uint64_t* aempty = astaged + NA;     // [NA] MMAs reading the row slot retired (commit)
  uint64_t* accfull = aempty + NA;     // [2] accumulator complete (commit)
  uint64_t* accempty = accfull + 2;    // [2] accumulator read back by the 128 epilogue threads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.slot);

  if (warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&done[b], 1);
    }
    for (int b = 0; b < NA; ++b) {
      mbar_init(&astaged[b], kStagers);
      mbar_init(&aempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], kEpi);
    }
    fence_mbar_init();
  }
  for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int num_items = item_count(a);
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int i1 = min(num_items, i0 + per);
  const int total = i1 > i0 ? (i1 - i0) * kch : 0;   // chunks of this CTA
  const uint32_t tb = table_h_bytes(kch, npad);
  const uint32_t chunk_bytes = (uint32_t)npad * 128u * kPieces;
  const uint32_t accw = (uint32_t)(npad + 31) / 32 * 32;   // columns per piece group (npad % 32 == 0)
  const uint32_t accs = (uint32_t)kPieces * accw;                        // stride of the accumulator buffers

  if (warp == 5) {
    // ------------------------------------------------ table producer
    if (lane == 0) {
      const uint64_t tab_policy = l2_policy_evict_last();
      int bin = 0;
      for (int g = 0; g < total; ++g) {
        const int seq = g / kch, c = g - seq * kch;
        if (c == 0) bin = item_at(a, i0 + seq).x;
        const int s = g % NB;
        if (g >= NB) mbar_wait(&done[s], (uint32_t)(g / NB - 1) & 1u);
        mbar_arrive_expect_tx(&full[s], chunk_bytes);
        bulk_g2s_hint(base + Ly.btab + s * bslot, a.table_h + (size_t)bin * tb + (size_t)c * chunk_bytes, chunk_bytes,
                      &full[s], tab_policy);
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_f16(kT, kPieces * npad);
      const uint32_t a_s = smem_u32(base + Ly.land);
      const uint32_t b_s = smem_u32(base + Ly.btab);
      for (int g = 0; g < total; ++g) {
        const int seq = g / kch, c = g - seq * kch;
        const int sa = g % NA, s = g % NB;
        const int acc = nacc == 2 ? (seq & 1) : 0;
        const uint32_t dcol = tmem + (uint32_t)acc * accs;
        if (c == 0 && seq >= nacc) mbar_wait(&accempty[acc], (uint32_t)(seq / nacc - 1) & 1u);
        mbar_wait(&astaged[sa], (uint32_t)(g / NA) & 1u);
        mbar_wait(&full[s], (uint32_t)(g / NB) & 1u);
        tc_fence_after();
        const uint32_t ah = a_s + (uint32_t)sa * kSlot;
        const uint32_t bh = b_s + (uint32_t)s * bslot;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          if (c == kch - 1 && ks >= a.ks_last) break;   // zero padding on both operands
          mma_f16(dcol, sw128_kmajor_desc(ah + ks * 32u), sw128_kmajor_desc(bh + ks * 32u), idesc,
                  (c | ks) ? 1u : 0u);
        }
        mma_commit(&done[s]);
        mma_commit(&aempty[sa]);
        if (c == kch - 1) mma_commit(&accfull[acc]);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------ row gather (warps 0-3)
    const uint32_t land_s = smem_u32(base + Ly.land);
    const uint64_t row_policy = l2_policy_evict_first();
    int r_item = -1, r_row = -1;
    auto row_of = [&](int item) {
      if (item != r_item) {
        r_item = item;
        const int4 it = item_at(a, item);
        r_row = tid < it.z ? patch_of(a, row_at(a, it, tid)) : -1;
      }
      return r_row;
    };
    // chunk g of this warp's 32 rows -> landing slot g % NA: lanes 8q..8q+7 copy the
    // 128-byte chunk (64 halfs) of row 4i+q, four whole lines per instruction
    auto issue_a = [&](int g) {
      if (g < total) {
        const int seq = g / kch, c = g - seq * kch;
        const int rmine = row_of(i0 + seq);
        const uint32_t dst = land_s + (uint32_t)(g % NA) * kSlot;
        const int q = lane >> 3, j = lane & 7;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = 4 * i + q;   // row within the warp
          const int r = __shfl_sync(kFull, rmine, rl);
          const uint16_t* src = a.R16 + (r >= 0 ? (int64_t)r * a.ld + 64 * c + 8 * j : 0);
          cp_async16_hint(dst + sw128_offset((uint32_t)(warp * 32 + rl), (uint32_t)j), src, r >= 0 ? 16u : 0u,
                          row_policy);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int g = 0; g < NA; ++g) issue_a(g);
    for (int g = 0; g < total; ++g) {
      const int sa = g % NA;
      asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
      fence_proxy_async_smem();   // the tensor core reads the slot through the async proxy
      mbar_arrive(&astaged[sa]);
      // the slot is refilled with chunk g + NA once the MMAs of chunk g retire
      if (g + NA < total) {
        mbar_wait(&aempty[sa], (uint32_t)(g / NA) & 1u);
        __syncwarp();
      }
      issue_a(g + NA);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // ------------------------------------------------ epilogue (warps 6-9): TMEM lane quarter warp % 4
    const int et = (warp & 3) * 32 + lane;          // tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    for (int seq = 0; seq < i1 - i0; ++seq) {
      const int4 it = item_at(a, i0 + seq);
      const int cur_bin = it.x, cur_rows = it.z;
      const int p = et < it.z ? patch_of(a, row_at(a, it, et)) : -1;
      const int acc = nacc == 2 ? (seq & 1) : 0;
      mbar_wait(&accfull[acc], (uint32_t)(seq / nacc) & 1u);
      tc_fence_after();
      const int gnode = a.level_base + cur_bin;
      const int cb = __ldg(a.child_begin + gnode);
      const int cc = __ldg(a.child_count + gnode);
      int best = 0;
      float bestv = -1.f, rawbest = 0.f, second = -1.f;
      const bool valid = et < cur_rows && p >= 0;
      const float scale = valid ? __ldg(a.inv_scale + p) : 1.f;   // > 0 on every lane: the read-back is warp-collective
      const uint32_t taddr = tmem + lane_base + (uint32_t)acc * accs;
      corr_abs_argmax(taddr, accw, cc, a, valid ? p : -1, cb - a.corr_off, bestv, best, rawbest, second, scale);
      recheck_near_ties(taddr, accw, cc, cb, a, valid ? p : -1, second, bestv, best, rawbest, scale);
      tc_fence_before();
      mbar_arrive(&accempty[acc]);
      int leaf_info = 0, leaf_cnt = 0;
      if (last && valid) {   // the winner's leaf record, from the fp32 table block (L2-resident)
        const int* info = reinterpret_cast<const int*>(reinterpret_cast<const uint8_t*>(a.table) +
                                                       (size_t)cur_bin * table_bytes(a.ld / 32, npad, true) +
                                                       (size_t)(a.ld / 32) * npad * 256u);
        leaf_info = __ldg(info + best);
        leaf_cnt = __ldg(info + npad + best);
      }
      if (valid) {
        const int child = cb + best;
        a.path_ws[(int64_t)p * a.L + a.level] = child;
        if (a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = child;
        if (a.next_counts) atomicAdd(&s_hist[best], 1);
        if (last) a.leaf_sel[p] = leaf_info;
        if (last && a.bsel) a.bsel[p] = rawbest;
        if (a.ip) add_ip(a.ip, p, cc + leaf_cnt, cc);
      }
      if (a.next_counts) {
        named_sync(1, kEpi);
        for (int j = et; j < cc; j += kEpi) {
          const int h = s_hist[j];
          if (h) atomicAdd(&a.next_counts[cb + j - a.next_base], h);
          s_hist[j] = 0;
        }
        named_sync(1, kEpi);
      }
    }
  }
  __syncwarp();   // reconverge the single-lane roles before the CTA barrier
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

template <int NA, int NB, int CPS>
cudaError_t launch_sh(ScoreArgs s, int sms, cudaStream_t st) {
  const uint32_t smem = sh_layout(s.npad, NA, NB).total;
  const int accw = (s.npad + 31) / 32 * 32;
  constexpr int kCols = 512 / CPS;   // TMEM columns per CTA
  const int nacc = 2 * kPieces * accw <= kCols ? 2 : 1;
  int cols = 32;
  while (cols < nacc * kPieces * accw) cols <<= 1;
  s.tmem_cols = cols;
  cudaError_t e = cudaFuncSetAttribute(score_sh_kernel<NA, NB, CPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel(score_sh_kernel<NA, NB, CPS>, sms * CPS, kThreads, (size_t)smem, st, true, s, nacc);
}

// x16 = fp16(s x) with s = 2^(15 - e), max |x| = f 2^e, f in [0.5, 1): the largest
// element lands in [2^14, 2^15), so elements down to 2^-28 of it stay normal
// halfs.  One warp per patch row (ld floats, zero padding included).
__global__ void __launch_bounds__(256) half_rows_kernel(const float* __restrict__ X, int64_t N, int ld,
                                                        uint16_t* __restrict__ x16, float* __restrict__ inv_scale,
                                                        float* __restrict__ qerr) {
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= N) return;
  const float4* row = reinterpret_cast<const float4*>(X + p * ld);
  const int nq = ld / 4;
  float mx = 0.f;
  for (int i = lane; i < nq; i += 32) {
    const float4 v = __ldg(row + i);
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  int e = 0;
  if (mx > 0.f && mx < 3.0e38f) frexpf(mx, &e);
  const int sh = max(-100, min(100, 15 - e));
  const float s = ldexpf(1.f, sh), is = ldexpf(1.f, -sh);
  uint2* out = reinterpret_cast<uint2*>(x16 + p * ld);
  float err2 = 0.f;
  for (int i = lane; i < nq; i += 32) {
    const float4 v = __ldg(row + i);   // second read: the row is L1 / L2 hot
    const __half h0 = __float2half_rn(v.x * s), h1 = __float2half_rn(v.y * s), h2 = __float2half_rn(v.z * s),
                 h3 = __float2half_rn(v.w * s);
    const float d0 = v.x - __half2float(h0) * is, d1 = v.y - __half2float(h1) * is,
                d2 = v.z - __half2float(h2) * is, d3 = v.w - __half2float(h3) * is;
    err2 = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, err2))));
    uint2 w;
    w.x = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
    w.y = (uint32_t)__half_as_ushort(h2) | ((uint32_t)__half_as_ushort(h3) << 16);
    out[i] = w;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) err2 += __shfl_xor_sync(kFull, err2, o);
  if (lane == 0) {
    inv_scale[p] = is;
    qerr[p] = sqrtf(err2);
  }
}

// Per-node half-precision score tables of one level: each child centroid value
// c = p0 + 2^-11 p1 (+ 2^-22 p2, exact, when kPieces == 3) in fp16 pieces, round
// to nearest (p0 keeps 11 significant bits, p1 the next 11), laid out [chunk of
// 64 columns][piece][npad rows x 128 B] SW128 (the UMMA K-major B operand; the
// pieces are adjacent row blocks, one N = kPieces npad operand).  One CTA per node;
// the block is pre-zeroed.
__global__ void __launch_bounds__(256) table_h_kernel(const float* __restrict__ cent, int ld, const int* child_begin,
                                                      const int* child_count, int64_t level_base, int kch, int npad,
                                                      uint8_t* __restrict__ out) {
  const int64_t v = level_base + blockIdx.x;
  uint8_t* blk = out + (size_t)blockIdx.x * table_h_bytes(kch, npad);
  const int cb = child_begin[v], cc = child_count[v];
  const int width = 64 * kch;
  for (int e = threadIdx.x; e < cc * width; e += blockDim.x) {
    const int j = e / width, col = e - j * width;
    const float val = cent[(int64_t)(cb + j) * ld + col];
    const __half p0 = __float2half_rn(val);
    const float r1 = val - __half2float(p0);
    const __half p1 = __float2half_rn(r1 * 2048.f);
    const float r2 = r1 - __half2float(p1) * (1.f / 2048.f);
    const __half p2 = __float2half_rn(r2 * 4194304.f);
    const int kc = col >> 6, q = col & 63;
    const uint32_t off = sw128_offset((uint32_t)j, (uint32_t)(q >> 3)) + (uint32_t)(q & 7) * 2u;
    uint8_t* plane = blk + (size_t)kc * kPieces * npad * 128;
    *reinterpret_cast<__half*>(plane + off) = p0;
    *reinterpret_cast<__half*>(plane + (size_t)npad * 128 + off) = p1;
    if (kPieces == 3) *reinterpret_cast<__half*>(plane + (size_t)npad * 256 + off) = p2;
  }
}

}  // namespace

bool score_sh_fits(int ld, int npad) {
  // N = kPieces npad <= 256 per MMA, whole 32-column accumulator groups, 64-column chunks
  return ld % 64 == 0 && npad % 32 == 0 && npad >= 32 && npad <= 64;
}

cudaError_t launch_score_sh(const ScoreArgs& s, int sms, cudaStream_t st) {
  if (!score_sh_fits(s.ld, s.npad)) return cudaErrorNotSupported;
  if (s.npad > 32) return launch_sh<3, 3, 2>(s, sms, st);   // 48 KB of rows + 3 x 16 KB of table per CTA
  return launch_sh<4, 4, 2>(s, sms, st);                    // 64 KB + 4 x 8 KB
}

cudaError_t launch_half_rows(const float* X, int64_t N, int ld, uint16_t* x16, float* inv_scale, float* qerr,
                             cudaStream_t st) {
  return launch_kernel(half_rows_kernel, (unsigned)((N + 7) / 8), 256, 0, st, true, X, N, ld, x16, inv_scale, qerr);
}

uint8_t* build_half_table(const TreeHandle* t, int l, cudaStream_t st) {
  const int npad = t->staged_levels[l].npad;
  const int kch = t->ld / 64;
  const int64_t nodes = t->level_offsets[l + 1] - t->level_offsets[l];
  const size_t bytes = (size_t)table_h_bytes(kch, npad) * nodes;
  uint8_t* out = nullptr;
  if (cudaMalloc(&out, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaError_t e = cudaMemsetAsync(out, 0, bytes, st);
  if (e == cudaSuccess) {
    table_h_kernel<<<(unsigned)nodes, 256, 0, st>>>(t->cent, t->ld, t->child_begin, t->child_count,
                                                    t->level_offsets[l], kch, npad, out);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(out);
    cudaGetLastError();
    return nullptr;
  }
  return out;
}

}  // namespace stmp
