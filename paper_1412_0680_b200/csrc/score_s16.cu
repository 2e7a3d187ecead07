// Streamed score pass on the residual pipeline with a 3xFP16 split instead of
// 3xTF32 (opt-in: score_kernel = 4).
//
// score_st.cu scores fp32 residual rows as hi.hi + hi.lo + lo.hi of a tf32
// split: three tcgen05.mma.kind::tf32 per 8-column k-step.  The same 22 bits
// fit two fp16 pieces once a row is scaled by a power of two: with ||r|| (the
// residual norm every update writes; max |r_i| <= ||r||) = f 2^e and
// s = 2^(14 - e), r s = r_a + r_b with r_a = fp16(r s), r_b = fp16(r s - r_a),
// and the centroids c 2^8 = c_a + c_b likewise (|c| <= 1).  Then
// r_a.c_a + r_a.c_b + r_b.c_a is three tcgen05.mma.kind::f16 per 16-column
// k-step -- twice the tensor rate and half the instructions of the tf32 split,
// and tables of 4 instead of 8 bytes per value -- with the same accuracy class
// (dropped: r_b.c_b, 2^-22 relative, as 3xTF32 drops lo.lo).  The argmax of a
// row is invariant under its positive scale, so the epilogue is score_st's.
// A is read from tensor memory: the stager threads (thread = row) split their
// row chunk and store packed halfs (cell c of a lane = elements 2c | 2c+1 of
// the K step, low half first -- tools/tmem_f16_probe.cu).
// Roles per CTA (one per SM, 320 threads) as score_st: 4 stager warps (NA landing
// slots of 64 fp32 columns, NAB TMEM A buffers of 64 cells), MMA issuer, table
// producer (NB slots of [c_a | c_b][npad x 128 B] SW128), 4 epilogue warps.
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

namespace {

constexpr int kT = 128;
constexpr int kStagers = 128;
constexpr int kEpi = 128;
constexpr int kThreads = kStagers + 64 + kEpi;
constexpr uint32_t kHalfSlot = kT * 128u;      // 128 rows x 32 floats
constexpr uint32_t kSlot = 2u * kHalfSlot;     // one landing slot: 128 rows x 64 floats (two swizzled halves)
constexpr int kNA = 2, kNB = 2, kNAB = 4;
constexpr uint32_t kColAcc = 64u * kNAB;       // TMEM: A buffers at [0, 256), accumulators after them

struct S16Layout {
  uint32_t land, btab, hist, bars, slot, total;
};

__host__ __device__ inline uint32_t s16_align(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }
__host__ __device__ inline uint32_t s16_bslot(int npad) { return s16_align((uint32_t)npad * 256u, 1024u); }

__host__ __device__ inline S16Layout s16_layout(int npad) {
  S16Layout L{};
  uint32_t o = 0;
  L.land = o; o += (uint32_t)kNA * kSlot;
  L.btab = o; o += (uint32_t)kNB * s16_bslot(npad);
  L.hist = o; o += 256 * 4;
  L.bars = s16_align(o, 8); o = L.bars + (uint32_t)(2 * kNB + 2 * kNAB + 4) * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

__global__ void __launch_bounds__(kThreads, 1) score_s16_kernel(ScoreArgs a, int nacc) {
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
  const S16Layout Ly = s16_layout(npad);
  const uint32_t bslot = s16_bslot(npad);
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Ly.bars);   // [NB] table chunk landed (tx)
  uint64_t* done = full + kNB;         // [NB] MMAs reading the table slot retired (commit)
  uint64_t* astaged = done + kNB;      // [NAB] A buffer written by the 128 stagers
  uint64_t* aempty = astaged + kNAB;   // [NAB] MMAs reading the A buffer retired (commit)
  uint64_t* accfull = aempty + kNAB;   // [2] accumulator complete (commit)
  uint64_t* accempty = accfull + 2;    // [2] accumulator read back by the 128 epilogue threads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.slot);

  if (warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&done[b], 1);
    }
    for (int b = 0; b < kNAB; ++b) {
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
  const uint32_t tb = table_h_bytes(kch, npad);       // [kch][c_a | c_b][npad x 128 B]
  const uint32_t chunk_bytes = (uint32_t)npad * 256u;
  const uint32_t accw = (uint32_t)(npad + 31) / 32 * 32;

  if (warp == 5) {
    // ------------------------------------------------ table producer
    if (lane == 0) {
      const uint64_t tab_policy = l2_policy_evict_last();
      int bin = 0;
      for (int g = 0; g < total; ++g) {
        const int seq = g / kch, c = g - seq * kch;
        if (c == 0) bin = item_at(a, i0 + seq).x;
        const int s = g % kNB;
        if (g >= kNB) mbar_wait(&done[s], (uint32_t)(g / kNB - 1) & 1u);
        mbar_arrive_expect_tx(&full[s], chunk_bytes);
        bulk_g2s_hint(base + Ly.btab + s * bslot, a.table_h + (size_t)bin * tb + (size_t)c * chunk_bytes, chunk_bytes,
                      &full[s], tab_policy);
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_f16(kT, npad);
      const uint64_t bdesc0 = sw128_kmajor_desc(smem_u32(base + Ly.btab));
      const uint32_t plane = ((uint32_t)npad * 128u) >> 4;   // c_b plane, in descriptor address units
      int seq = 0, c = 0, ab = 0, s = 0;
      uint32_t pa = 0, pb = 0;
      for (int g = 0; g < total; ++g) {
        const int acc = nacc == 2 ? (seq & 1) : 0;
        const uint32_t dcol = tmem + kColAcc + (uint32_t)acc * accw;
        if (c == 0 && seq >= nacc) mbar_wait(&accempty[acc], (uint32_t)(seq / nacc - 1) & 1u);
        mbar_wait(&astaged[ab], pa);
        mbar_wait(&full[s], pb);
        tc_fence_after();
        const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)s * (bslot >> 4));
        const uint32_t aa = tmem + (uint32_t)ab * 64u;   // r_a cells [0, 32), r_b cells [32, 64)
        const int nks = c == kch - 1 ? a.ks_last : 4;    // the rest is zero padding on both operands
        for (int ks = 0; ks < nks; ++ks) {
          const uint32_t ka = aa + 8u * ks;
          const uint64_t kb = bd + 2u * ks;
          mma_f16_ts(dcol, ka, kb, idesc, (c | ks) ? 1u : 0u);          // r_a . c_a
          mma_f16_ts(dcol, ka, kb + plane, idesc, 1u);                  // r_a . c_b
          mma_f16_ts(dcol, ka + 32u, kb, idesc, 1u);                    // r_b . c_a
        }
        mma_commit(&done[s]);
        mma_commit(&aempty[ab]);
        if (c == kch - 1) mma_commit(&accfull[acc]);
        if (++c == kch) { c = 0; ++seq; }
        if (++ab == kNAB) { ab = 0; pa ^= 1u; }
        if (++s == kNB) { s = 0; pb ^= 1u; }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------ stagers (warps 0-3): thread = patch row = TMEM lane
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t land_s = smem_u32(base + Ly.land);
    const uint64_t row_policy = l2_policy_evict_first();
    // row ids per tile: the copies run ahead of the staging, so each keeps its own
    // cached tile (one fetch per tile each; the staging reuses the copier's row id)
    int i_item = -1, i_row = -1, i_prev_item = -1, i_prev_row = -1;
    auto row_of = [&](int item) {
      if (item != i_item) {
        i_prev_item = i_item;
        i_prev_row = i_row;
        i_item = item;
        const int4 it = item_at(a, item);
        i_row = tid < it.z ? patch_of(a, row_at(a, it, tid)) : -1;
      }
      return i_row;
    };
    int s_item = -1;
    float s_scale = 1.f;
    // s = 2^(14 - e) for ||r|| = f 2^e, f in [0.5, 1): every |r_i| s stays below 2^14
    auto scale_of = [&](int item) {
      if (item != s_item) {
        s_item = item;
        int row;
        if (item == i_item) row = i_row;
        else if (item == i_prev_item) row = i_prev_row;
        else {
          const int4 it = item_at(a, item);
          row = tid < it.z ? patch_of(a, row_at(a, it, tid)) : -1;
        }
        int e = 0;
        const float nrm = row >= 0 ? __ldg(a.rnorm + row) : 0.f;
        if (nrm > 0.f && nrm < 3.0e38f) frexpf(nrm, &e);
        s_scale = ldexpf(1.f, max(-100, min(100, 14 - e)));
      }
      return s_scale;
    };
    // chunk g (64 columns) of this warp's 32 rows -> landing slot g % NA, two swizzled
    // halves of 32 columns: lanes 8q..8q+7 copy a 128-byte line of row 4i+q
    auto issue_a = [&](int g) {
      if (g < total) {
        const int seq = g / kch, c = g - seq * kch;
        const int rmine = row_of(i0 + seq);
        const int q = lane >> 3, j = lane & 7;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t dst = land_s + (uint32_t)(g % kNA) * kSlot + (uint32_t)h * kHalfSlot;
          const bool cols = 64 * c + 32 * h < a.ld;   // the padded row may end inside the chunk
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rl = 4 * i + q;
            const int r = __shfl_sync(kFull, rmine, rl);
            const bool on = r >= 0 && cols;
            const float* src = a.R + (on ? (int64_t)r * a.ld + 64 * c + 32 * h + 4 * j : 0);
            cp_async16_hint(dst + sw128_offset((uint32_t)(warp * 32 + rl), (uint32_t)j), src, on ? 16u : 0u,
                            row_policy);
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int g = 0; g < kNA; ++g) issue_a(g);
    for (int g = 0; g < total; ++g) {
      const int ab = g % kNAB;
      asm volatile("cp.async.wait_group %0;" ::"n"(kNA - 1) : "memory");
      __syncwarp();   // the warp's rows were copied by all of its lanes
      const float s = scale_of(i0 + g / kch);
      if (g >= kNAB) {
        mbar_wait(&aempty[ab], (uint32_t)(g / kNAB - 1) & 1u);
        tc_fence_after();
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint8_t* slot = base + Ly.land + (uint32_t)(g % kNA) * kSlot + (uint32_t)h * kHalfSlot;
        uint32_t ca[16], cb[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(slot + sw128_offset(tid, j));
          // packed conversions: two elements per instruction, cell = (even K element low | odd high)
          const __half2 a01 = __floats2half2_rn(v.x * s, v.y * s), a23 = __floats2half2_rn(v.z * s, v.w * s);
          const float2 f01 = __half22float2(a01), f23 = __half22float2(a23);
          const __half2 b01 = __floats2half2_rn(fmaf(v.x, s, -f01.x), fmaf(v.y, s, -f01.y));
          const __half2 b23 = __floats2half2_rn(fmaf(v.z, s, -f23.x), fmaf(v.w, s, -f23.y));
          ca[2 * j] = *reinterpret_cast<const uint32_t*>(&a01);
          ca[2 * j + 1] = *reinterpret_cast<const uint32_t*>(&a23);
          cb[2 * j] = *reinterpret_cast<const uint32_t*>(&b01);
          cb[2 * j + 1] = *reinterpret_cast<const uint32_t*>(&b23);
        }
        tmem_st16(tmem + lane_base + (uint32_t)ab * 64u + 16u * h, ca);
        tmem_st16(tmem + lane_base + (uint32_t)ab * 64u + 32u + 16u * h, cb);
      }
      __syncwarp();      // every lane has read its row before the slot is refilled
      issue_a(g + kNA);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&astaged[ab]);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // ------------------------------------------------ epilogue (warps 6-9): TMEM lane quarter warp % 4
    const int et = (warp & 3) * 32 + lane;
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
      float bestv = -1.f;
      const bool valid = et < cur_rows && p >= 0;
      acc_abs_argmax(tmem + lane_base + kColAcc + (uint32_t)acc * accw, 0u, (int)accw, npad, bestv, best);
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

// Per-node tables of one level for the 3xFP16 pass: c 2^8 = c_a + c_b (fp16, round to
// nearest; c_b keeps the next 11 bits), laid out [chunk of 64 columns][c_a | c_b]
// [npad rows x 128 B] SW128 (the UMMA K-major B operand).  One CTA per node;
// the block is pre-zeroed.
__global__ void __launch_bounds__(256) table_s16_kernel(const float* __restrict__ cent, int ld, const int* child_begin,
                                                        const int* child_count, int64_t level_base, int kch,
                                                        int npad, uint8_t* __restrict__ out) {
  const int64_t v = level_base + blockIdx.x;
  uint8_t* blk = out + (size_t)blockIdx.x * table_h_bytes(kch, npad);
  const int cb = child_begin[v], cc = child_count[v];
  for (int e = threadIdx.x; e < cc * ld; e += blockDim.x) {
    const int j = e / ld, col = e - j * ld;
    const float val = cent[(int64_t)(cb + j) * ld + col] * 256.f;
    const __half p0 = __float2half_rn(val);
    const __half p1 = __float2half_rn(val - __half2float(p0));
    const int kc = col >> 6, q = col & 63;
    const uint32_t off = sw128_offset((uint32_t)j, (uint32_t)(q >> 3)) + (uint32_t)(q & 7) * 2u;
    uint8_t* plane = blk + (size_t)kc * 2 * npad * 128;
    *reinterpret_cast<__half*>(plane + off) = p0;
    *reinterpret_cast<__half*>(plane + (size_t)npad * 128 + off) = p1;
  }
}

}  // namespace

bool score_s16_fits(int ld, int npad) {
  if (ld % 32 != 0 || npad < 16 || npad > 256 || npad % 16 != 0) return false;
  return s16_layout(npad).total <= 227 * 1024;
}

cudaError_t launch_score_s16(const ScoreArgs& s_in, int sms, cudaStream_t st) {
  ScoreArgs s = s_in;
  if (!score_s16_fits(s.ld, s.npad) || s.table_h == nullptr || s.rnorm == nullptr) return cudaErrorNotSupported;
  const uint32_t smem = s16_layout(s.npad).total;
  const int accw = (s.npad + 31) / 32 * 32;
  const int nacc = (int)kColAcc + 2 * accw <= 512 ? 2 : 1;
  int cols = 32;
  while (cols < (int)kColAcc + nacc * accw) cols <<= 1;
  s.tmem_cols = cols;
  s.kchunks = (s.ld + 63) / 64;
  // 16-column k-steps holding data in the last 64-column chunk
  s.ks_last = (s.ld - 64 * (s.kchunks - 1) + 15) / 16;
  cudaError_t e = cudaFuncSetAttribute(score_s16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel(score_s16_kernel, sms, kThreads, (size_t)smem, st, true, s, nacc);
}

uint8_t* build_s16_table(const TreeHandle* t, int l, cudaStream_t st) {
  const int npad = t->staged_levels[l].npad;
  const int kch = (t->ld + 63) / 64;
  const int64_t nodes = t->level_offsets[l + 1] - t->level_offsets[l];
  const size_t bytes = (size_t)table_h_bytes(kch, npad) * nodes;
  uint8_t* out = nullptr;
  if (cudaMalloc(&out, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaError_t e = cudaMemsetAsync(out, 0, bytes, st);
  if (e == cudaSuccess) {
    table_s16_kernel<<<(unsigned)nodes, 256, 0, st>>>(t->cent, t->ld, t->child_begin, t->child_count,
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
