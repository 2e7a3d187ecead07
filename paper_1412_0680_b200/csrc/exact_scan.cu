// Exhaustive selection on the tensor cores: argmax_i |a_i . r| over the whole
// dictionary for 128-patch tiles, i.e. a GEMM R [N, n] x A^T [n, m] whose
// epilogue keeps only a running per-row (max |score|, lowest atom index).
//
// The dictionary is laid out once (lazily, per handle) as tf32 hi / lo atom
// blocks of BW = 128 or 256 atoms: [block][kchunk][hi|lo][BW rows x 128 B]
// SW128 -- the UMMA K-major B operand, one bulk copy per (block, chunk).  The
// kernel has the warp-specialised shape of score_st_kernel: a producer warp
// streams the block chunks through a ring of NB slots, an MMA warp issues the
// 3xTF32 tcgen05.mma (M = 128 patches, N = BW atoms, A from TMEM), and four
// stager warps gather the tile's rows chunk by chunk (re-staged for every atom
// block: the A tile is re-read from L2 / HBM, which costs less than a third of
// the MMA time even at n = 1600), split them into tf32 hi / lo in TMEM, and
// after each block fold the accumulator into the running argmax.  With BW =
// 128 two accumulators alternate, so the fold of block j overlaps the MMAs of
// block j + 1; BW = 256 (long rows, where a block's MMAs take tens of
// microseconds) uses one.
// F16 = true is the same scan with the 3xFP16 split of score_s16.cu (rows scaled
// by a power of two from the residual norm and split into two fp16 pieces in
// TMEM, atoms as two fp16 pieces of 2^8 a, 64-column chunks, three kind::f16
// MMAs per 16-column k-step): the accuracy class of 3xTF32 at twice the tensor
// rate and half the dictionary-table bytes; the running argmax is invariant
// under the positive row scale.
// Semantics: exact_select, pkg/src/stmp/pursuit.py:102-109 (np.argmax of |A r|:
// the first maximum, i.e. the lowest atom index; counter += m).
#include <cuda_fp16.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

namespace {

constexpr int kT = 128;
constexpr int kStagers = 128;
constexpr int kThreads = kStagers + 64;
constexpr uint32_t kSlot = kT * 128u;
constexpr int kNAB = 4;                    // TMEM A buffers (64 columns: hi | lo of one K chunk)
constexpr uint32_t kColAcc = 64u * kNAB;   // TMEM: A buffers [0, 256), accumulators from 256

struct XsLayout {
  uint32_t land, btab, bars, slot, total;
};

__host__ __device__ inline XsLayout xs_layout(int bw, int na, int nb, bool f16) {
  XsLayout L{};
  uint32_t o = 0;
  L.land = o; o += (uint32_t)na * kSlot * (f16 ? 2u : 1u);   // F16: 64-column chunks (two swizzled halves)
  L.btab = o; o += (uint32_t)nb * (uint32_t)bw * 256u;
  L.bars = o; o = L.bars + (uint32_t)(2 * nb + 2 * kNAB + 4) * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

template <int NA, int NB, bool F16>
__global__ void __launch_bounds__(kThreads, 1) exact_scan_kernel(ScoreArgs a, int nacc) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int bw = a.npad;           // atoms per block
  const int kch = a.kchunks;
  const int nblk = a.nblocks;
  const int m = a.m_atoms;
  const XsLayout Ly = xs_layout(bw, NA, NB, F16);
  constexpr uint32_t kLand = kSlot * (F16 ? 2u : 1u);
  const uint32_t bslot = (uint32_t)bw * 256u;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Ly.bars);
  uint64_t* done = full + NB;
  uint64_t* astaged = done + NB;
  uint64_t* aempty = astaged + kNAB;
  uint64_t* accfull = aempty + kNAB;
  uint64_t* accempty = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.slot);

  if (warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&done[b], 1);
    }
    for (int b = 0; b < kNAB; ++b) {
      mbar_init(&astaged[b], kStagers);
      mbar_init(&aempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], kStagers);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int num_items = item_count(a);
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int i1 = min(num_items, i0 + per);
  const int per_item = nblk * kch;
  const int total = i1 > i0 ? (i1 - i0) * per_item : 0;

  if (warp == 5) {
    // ------------------------------------------------ dictionary block producer
    if (lane == 0) {
      for (int g = 0; g < total; ++g) {
        const int bc = g % per_item;   // block * kch + chunk
        const int s = g % NB;
        if (g >= NB) mbar_wait(&done[s], (uint32_t)(g / NB - 1) & 1u);
        mbar_arrive_expect_tx(&full[s], bslot);
        bulk_g2s(base + Ly.btab + s * bslot,
                 (F16 ? a.table_h : reinterpret_cast<const uint8_t*>(a.table)) + (size_t)bc * bslot, bslot, &full[s]);
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = F16 ? idesc_f16(kT, bw) : idesc_tf32(kT, bw);
      const uint32_t b_s = smem_u32(base + Ly.btab);
      for (int g = 0; g < total; ++g) {
        const int bs = g / kch, c = g - bs * kch;   // bs: block sequence number of this CTA
        const int ab = g % kNAB, s = g % NB;
        const int acc = nacc == 2 ? (bs & 1) : 0;
        const uint32_t dcol = tmem + kColAcc + (uint32_t)acc * (uint32_t)bw;
        if (c == 0 && bs >= nacc) mbar_wait(&accempty[acc], (uint32_t)(bs / nacc - 1) & 1u);
        mbar_wait(&astaged[ab], (uint32_t)(g / kNAB) & 1u);
        mbar_wait(&full[s], (uint32_t)(g / NB) & 1u);
        tc_fence_after();
        const uint32_t bh = b_s + s * bslot;
        const uint32_t bl = bh + (uint32_t)bw * 128u;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t ah = tmem + (uint32_t)ab * 64u + ks * 8;
          const uint32_t al = ah + 32;
          const uint32_t o = ks * 32u;
          if (c == kch - 1 && ks >= a.ks_last) break;   // zero padding on both operands
          if (F16) {   // r_a.a_a + r_a.a_b + r_b.a_a: cells [0, 32) = r_a, [32, 64) = r_b; 16 columns per k-step
            mma_f16_ts(dcol, ah, sw128_kmajor_desc(bh + o), idesc, (c | ks) ? 1u : 0u);
            mma_f16_ts(dcol, ah, sw128_kmajor_desc(bl + o), idesc, 1u);
            mma_f16_ts(dcol, al, sw128_kmajor_desc(bh + o), idesc, 1u);
            continue;
          }
          mma_tf32_ts(dcol, ah, sw128_kmajor_desc(bh + o), idesc, (c | ks) ? 1u : 0u);
          mma_tf32_ts(dcol, ah, sw128_kmajor_desc(bl + o), idesc, 1u);
          mma_tf32_ts(dcol, al, sw128_kmajor_desc(bh + o), idesc, 1u);
        }
        mma_commit(&done[s]);
        mma_commit(&aempty[ab]);
        if (c == kch - 1) mma_commit(&accfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------ stagers + running argmax (warps 0-3)
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t land_s = smem_u32(base + Ly.land);
    int r_item = -1, r_row = -1;
    auto row_of = [&](int item) {
      if (item != r_item) {
        r_item = item;
        const int4 it = item_at(a, item);
        r_row = tid < it.z ? row_at(a, it, tid) : -1;
      }
      return r_row;
    };
    // chunk g (of the tile's rows) -> landing slot g % NA; lanes 8q..8q+7 copy
    // the 128-byte chunk of one row, four whole lines per instruction
    auto issue_a = [&](int g) {
      if (g < total) {
        const int c = g % kch;
        const int rmine = row_of(i0 + g / per_item);
        const int q = lane >> 3, j = lane & 7;
#pragma unroll
        for (int h = 0; h < (F16 ? 2 : 1); ++h) {
          const uint32_t dst = land_s + (uint32_t)(g % NA) * kLand + (uint32_t)h * kSlot;
          const int col0 = F16 ? 64 * c + 32 * h : 32 * c;
          const bool cols = col0 < a.ld;   // F16: the padded row may end inside the 64-column chunk
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rl = 4 * i + q;
            const int r = __shfl_sync(kFull, rmine, rl);
            const bool on = r >= 0 && cols;
            const float* src = a.R + (on ? (int64_t)r * a.ld + col0 + 4 * j : 0);
            cp_async16(dst + sw128_offset((uint32_t)(warp * 32 + rl), (uint32_t)j), src, on ? 16u : 0u);
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int g = 0; g < NA; ++g) issue_a(g);
    int cur_p = -1;
    bool valid = false;
    int best = 0;
    float bestv = -1.f;
    float rscale = 1.f;   // F16: the row's power-of-two scale
    for (int g = 0; g < total; ++g) {
      const int item = i0 + g / per_item, rem = g % per_item;
      const int blk = rem / kch, c = rem - blk * kch;
      const int bs = g / kch, ab = g % kNAB;
      if (rem == 0) {
        const int4 it = item_at(a, item);
        cur_p = tid < it.z ? row_at(a, it, tid) : -1;
        valid = cur_p >= 0;
        best = 0;
        bestv = -1.f;
      }
      asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
      __syncwarp();
      if (F16) {
        if (rem == 0) {   // s = 2^(14 - e) for ||r|| = f 2^e: every |r_i| s stays below 2^14
          int e = 0;
          const float nrm = cur_p >= 0 ? __ldg(a.rnorm + cur_p) : 0.f;
          if (nrm > 0.f && nrm < 3.0e38f) frexpf(nrm, &e);
          rscale = ldexpf(1.f, max(-100, min(100, 14 - e)));
        }
        if (g >= kNAB) {
          mbar_wait(&aempty[ab], (uint32_t)(g / kNAB - 1) & 1u);
          tc_fence_after();
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint8_t* slot = base + Ly.land + (uint32_t)(g % NA) * kLand + (uint32_t)h * kSlot;
          uint32_t ca[16], cb[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(slot + sw128_offset(tid, j));
            const __half2 a01 = __floats2half2_rn(v.x * rscale, v.y * rscale);
            const __half2 a23 = __floats2half2_rn(v.z * rscale, v.w * rscale);
            const float2 f01 = __half22float2(a01), f23 = __half22float2(a23);
            const __half2 b01 = __floats2half2_rn(fmaf(v.x, rscale, -f01.x), fmaf(v.y, rscale, -f01.y));
            const __half2 b23 = __floats2half2_rn(fmaf(v.z, rscale, -f23.x), fmaf(v.w, rscale, -f23.y));
            ca[2 * j] = *reinterpret_cast<const uint32_t*>(&a01);
            ca[2 * j + 1] = *reinterpret_cast<const uint32_t*>(&a23);
            cb[2 * j] = *reinterpret_cast<const uint32_t*>(&b01);
            cb[2 * j + 1] = *reinterpret_cast<const uint32_t*>(&b23);
          }
          tmem_st16(tmem + lane_base + (uint32_t)ab * 64u + 16u * h, ca);
          tmem_st16(tmem + lane_base + (uint32_t)ab * 64u + 32u + 16u * h, cb);
        }
        __syncwarp();
        issue_a(g + NA);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&astaged[ab]);
      } else {
      float hi[32], lo[32];
      const uint8_t* slot = base + Ly.land + (uint32_t)(g % NA) * kSlot;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(slot + sw128_offset(tid, j));
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hi[4 * j + q] = tf32_hi(x[q]);
          lo[4 * j + q] = x[q] - hi[4 * j + q];
        }
      }
      __syncwarp();
      issue_a(g + NA);
      if (g >= kNAB) {
        mbar_wait(&aempty[ab], (uint32_t)(g / kNAB - 1) & 1u);
        tc_fence_after();
      }
      tmem_st32(tmem + lane_base + (uint32_t)ab * 64u, hi);
      tmem_st32(tmem + lane_base + (uint32_t)ab * 64u + 32, lo);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&astaged[ab]);
      }
      if (c != kch - 1) continue;

      // ---- fold this block's scores into the running argmax
      const int acc = nacc == 2 ? (bs & 1) : 0;
      mbar_wait(&accfull[acc], (uint32_t)(bs / nacc) & 1u);
      tc_fence_after();
      const int a0 = blk * bw;
      const int cnt = min(bw, m - a0);
      {
        float bv;
        int bi;
        tmem_abs_argmax(tmem + lane_base + kColAcc + (uint32_t)acc * (uint32_t)bw, bw, cnt, bv, bi);
        if (bv > bestv) {   // strict: an earlier block keeps ties (lowest atom index)
          bestv = bv;
          best = a0 + bi;
        }
      }
      tc_fence_before();
      mbar_arrive(&accempty[acc]);
      if (blk == nblk - 1 && valid) {
        a.leaf_sel[cur_p] = best;
        if (a.ip) add_ip(a.ip, cur_p, m, 0);   // exact_select: counter += m (pursuit.py:106)
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

// Dictionary -> [block][kchunk][hi|lo][bw rows x 128 B] SW128 (rows past m zero).
__global__ void __launch_bounds__(256) xtable_kernel(const float* __restrict__ atoms, int64_t m, int ld, int bw,
                                                     float* __restrict__ out) {
  const int kch = ld / 32;
  const int blk = blockIdx.x / kch, kc = blockIdx.x - blk * kch;
  float* plane = out + ((size_t)blockIdx.x) * bw * 64;
  for (int e = threadIdx.x; e < bw * 32; e += blockDim.x) {
    const int j = e >> 5, q = e & 31;
    const int64_t atom = (int64_t)blk * bw + j;
    const float val = atom < m ? atoms[atom * ld + kc * 32 + q] : 0.f;
    const float hi = tf32_hi(val);
    const uint32_t off = sw128_offset((uint32_t)j, (uint32_t)(q >> 2)) / 4 + (q & 3);
    plane[off] = hi;
    plane[(size_t)bw * 32 + off] = val - hi;
  }
}

// Dictionary -> [block][chunk of 64 columns][a_a | a_b][bw rows x 128 B] SW128 with 2^8 a = a_a + a_b
// in fp16 pieces (rows past m and columns past ld zero).
__global__ void __launch_bounds__(256) xtable16_kernel(const float* __restrict__ atoms, int64_t m, int ld, int bw,
                                                       uint8_t* __restrict__ out) {
  const int kch = (ld + 63) / 64;
  const int blk = blockIdx.x / kch, kc = blockIdx.x - blk * kch;
  uint8_t* plane = out + ((size_t)blockIdx.x) * bw * 256;
  for (int e = threadIdx.x; e < bw * 64; e += blockDim.x) {
    const int j = e >> 6, q = e & 63;
    const int64_t atom = (int64_t)blk * bw + j;
    const int col = kc * 64 + q;
    const float val = atom < m && col < ld ? atoms[atom * ld + col] * 256.f : 0.f;
    const __half p0 = __float2half_rn(val);
    const __half p1 = __float2half_rn(val - __half2float(p0));
    const uint32_t off = sw128_offset((uint32_t)j, (uint32_t)(q >> 3)) + (uint32_t)(q & 7) * 2u;
    *reinterpret_cast<__half*>(plane + off) = p0;
    *reinterpret_cast<__half*>(plane + (size_t)bw * 128 + off) = p1;
  }
}

std::mutex g_xtable_mu;

template <int NA, int NB, bool F16>
cudaError_t launch_xs(ScoreArgs s, int sms, cudaStream_t st) {
  const uint32_t smem = xs_layout(s.npad, NA, NB, F16).total;
  if (F16) {   // 64-column chunks, 16-column k-steps
    s.kchunks = (s.ld + 63) / 64;
    s.ks_last = (s.ld - 64 * (s.kchunks - 1) + 15) / 16;
  }
  const int nacc = s.npad <= 128 ? 2 : 1;
  int cols = 32;
  while (cols < (int)kColAcc + nacc * s.npad) cols <<= 1;
  s.tmem_cols = cols;
  cudaError_t e = cudaFuncSetAttribute(exact_scan_kernel<NA, NB, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel(exact_scan_kernel<NA, NB, F16>, sms, kThreads, (size_t)smem, st, true, s, nacc);
}

}  // namespace

int xtable_block_width(int ld) { return ld / 32 <= 4 ? 128 : 256; }

const float* ensure_xtable(DictHandle* d, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_xtable_mu);
  if (d->xtable != nullptr || d->xtable_tried) return d->xtable;
  d->xtable_tried = true;
  const int bw = xtable_block_width(d->ld);
  const int64_t nblk = (d->m + bw - 1) / bw;
  float* tab = nullptr;
  if (cudaMalloc(&tab, (size_t)nblk * bw * d->ld * 8) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  xtable_kernel<<<(unsigned)(nblk * (d->ld / 32)), 256, 0, st>>>(d->atoms, d->m, d->ld, bw, tab);
  note_launch();
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
    cudaFree(tab);
    return nullptr;
  }
  d->xtable = tab;
  return tab;
}

const uint8_t* ensure_xtable16(DictHandle* d, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_xtable_mu);
  if (d->xtable16 != nullptr || d->xtable16_tried) return d->xtable16;
  d->xtable16_tried = true;
  const int bw = xtable_block_width(d->ld);
  const int64_t nblk = (d->m + bw - 1) / bw;
  const int kch = (d->ld + 63) / 64;
  uint8_t* tab = nullptr;
  if (cudaMalloc(&tab, (size_t)nblk * kch * bw * 256) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  xtable16_kernel<<<(unsigned)(nblk * kch), 256, 0, st>>>(d->atoms, d->m, d->ld, bw, tab);
  note_launch();
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
    cudaFree(tab);
    return nullptr;
  }
  d->xtable16 = tab;
  return tab;
}

cudaError_t launch_exact_scan(const ScoreArgs& s, int sms, cudaStream_t st) {
  // 128-atom blocks: 16 KB + 16 KB per chunk slot pair; 256-atom blocks: 64 KB slots
  if (s.table_h != nullptr && s.rnorm != nullptr) {   // 3xFP16 split (64-column chunks: 32 KB landing slots)
    if (s.npad == 128) return launch_xs<2, 3, true>(s, sms, st);
    if (s.npad == 256) return launch_xs<2, 2, true>(s, sms, st);
    return cudaErrorNotSupported;
  }
  if (s.npad == 128) return launch_xs<4, 3, false>(s, sms, st);
  if (s.npad == 256) return launch_xs<4, 2, false>(s, sms, st);
  return cudaErrorNotSupported;
}

}  // namespace stmp
