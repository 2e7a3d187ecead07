// Level passes of the Gram path on half-precision patch rows.
//
// On the Gram path (gram_path.cu) the rows the level passes multiply are the
// patches x themselves, never a residual, so they can be prepared once per
// encode (by the init kernel, encode_update.cu, in its pass over x): x16 =
// fp16(s_p x) with a power-of-two scale s_p per patch (half the bytes of every pass), and the exact near-tie re-check of the epilogue
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
#include <stdio.h>

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
  // this CTA's work items, read once: every role looks its tiles up here instead
  // of paying a global round trip at each tile boundary
  constexpr int kItemCache = 48;
  __shared__ int4 s_items[kItemCache];

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
#ifdef STMP_SH_TRACE   // timing experiments only: event times of CTA 0's first 64 chunks
  __shared__ long long tr[5][64];
  __shared__ long long trt[8][32];
  __shared__ int trn[32];
  const long long tr_t0 = clock64();
#define SH_TR(k, g) if (blockIdx.x == 0 && (g) < 64) tr[k][g] = clock64()
#define SH_TRT(k, seq) if ((seq) < 32) trt[k][seq] = clock64() - tr_t0
#else
#define SH_TR(k, g)
#define SH_TRT(k, seq)
#endif

  const int num_items = item_count(a);
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int i1 = min(num_items, i0 + per);
  const int total = i1 > i0 ? (i1 - i0) * kch : 0;   // chunks of this CTA
  for (int i = tid; i < min(i1 - i0, kItemCache); i += kThreads) s_items[i] = item_at(a, i0 + i);
  __syncthreads();
  auto item_of = [&](int seq) { return seq < kItemCache ? s_items[seq] : item_at(a, i0 + seq); };
  const uint32_t tb = table_h_bytes(kch, npad);
  const uint32_t chunk_bytes = (uint32_t)npad * 128u * kPieces;
  const uint32_t accw = (uint32_t)npad;   // columns per piece group: piece q's scores start at column q npad
  const uint32_t accs = (uint32_t)kPieces * accw;                        // stride of the accumulator buffers

  if (warp == 5) {
    // ------------------------------------------------ table producer
    if (lane == 0) {
      const uint64_t tab_policy = l2_policy_evict_last();
      int bin = 0;
      for (int g = 0; g < total; ++g) {
        const int seq = g / kch, c = g - seq * kch;
        if (c == 0) bin = item_of(seq).x;
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
      // one thread issues everything, so its instruction count per chunk is the
      // pipeline's clock: running counters instead of divisions, operand
      // descriptors advanced by adds (the address field counts 16-byte units)
      const uint32_t idesc = idesc_f16(kT, kPieces * npad);
      const uint64_t adesc0 = sw128_kmajor_desc(smem_u32(base + Ly.land));
      const uint64_t bdesc0 = sw128_kmajor_desc(smem_u32(base + Ly.btab));
      const int ks_last = a.ks_last;
      int seq = 0, c = 0, sa = 0, s = 0;
      uint32_t pa = 0, pb = 0;   // phase parities of the row / table rings
      for (int g = 0; g < total; ++g) {
        const int acc = nacc == 2 ? (seq & 1) : 0;
        const uint32_t dcol = tmem + (uint32_t)acc * accs;
        if (c == 0) { SH_TRT(0, seq); }
        if (c == 0 && seq >= nacc) mbar_wait(&accempty[acc], (uint32_t)(seq / nacc - 1) & 1u);
        if (c == 0) { SH_TRT(1, seq); }
        mbar_wait(&astaged[sa], pa);
        SH_TR(2, g);
        mbar_wait(&full[s], pb);
        SH_TR(3, g);
        tc_fence_after();
        const uint64_t ad = adesc0 + (uint64_t)((uint32_t)sa * (kSlot >> 4));
        const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)s * (bslot >> 4));
        const int nks = c == kch - 1 ? ks_last : 4;   // the rest is zero padding on both operands
        mma_f16(dcol, ad, bd, idesc, c ? 1u : 0u);
        if (nks > 1) mma_f16(dcol, ad + 2, bd + 2, idesc, 1u);
        if (nks > 2) mma_f16(dcol, ad + 4, bd + 4, idesc, 1u);
        if (nks > 3) mma_f16(dcol, ad + 6, bd + 6, idesc, 1u);
        mma_commit(&done[s]);
        mma_commit(&aempty[sa]);
        if (c == kch - 1) mma_commit(&accfull[acc]);
        SH_TR(4, g);
        if (++c == kch) { c = 0; ++seq; }
        if (++sa == NA) { sa = 0; pa ^= 1u; }
        if (++s == NB) { s = 0; pb ^= 1u; }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------ row gather (warps 0-3)
    const uint32_t land_s = smem_u32(base + Ly.land);
    const uint64_t row_policy = l2_policy_evict_first();
    // row id of this thread in tile `seq`; the next tile's is fetched one tile ahead
    auto row_fetch = [&](int seq) {
      if (i0 + seq >= i1) return -1;
      const int4 it = item_of(seq);
      return tid < it.z ? patch_of(a, row_at(a, it, tid)) : -1;
    };
    int r_next = row_fetch(0);
    // chunk g of this warp's 32 rows -> landing slot g % NA: lanes 8q..8q+7 copy the
    // 128-byte chunk (64 halfs) of row 4i+q, four whole lines per instruction; the
    // eight source pointers of a lane are set up once per tile
    const int q = lane >> 3, j = lane & 7;
    const uint16_t* rp[8];
    int rp_seq = -1;
    // chunks are issued in order: running (tile, chunk, slot) counters
    int ig = 0, iseq = 0, ic = 0, islot = 0;
    auto issue_next = [&]() {
      if (ig < total) {
        if (iseq != rp_seq) {
          rp_seq = iseq;
          const int rmine = r_next;
          r_next = row_fetch(iseq + 1);   // in flight during this tile's chunks
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = __shfl_sync(kFull, rmine, 4 * i + q);
            rp[i] = r >= 0 ? a.R16 + (int64_t)r * a.ld + 8 * j : nullptr;
          }
        }
        const uint32_t dst = land_s + (uint32_t)islot * kSlot;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          cp_async16_hint(dst + sw128_offset((uint32_t)(warp * 32 + 4 * i + q), (uint32_t)j),
                          rp[i] ? rp[i] + 64 * ic : a.R16, rp[i] ? 16u : 0u, row_policy);
        ++ig;
        if (++ic == kch) { ic = 0; ++iseq; }
        if (++islot == NA) islot = 0;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // Iteration g hands chunk g to the MMA warp first and only then refills the
    // slot of chunk g - 1 (whose MMAs were issued a whole iteration ago), so the
    // copy instructions of one chunk overlap the MMA issue of the next instead of
    // alternating with it (measured: the two took ~800 + ~700 cycles in turn).
    // Groups: chunks 0 .. NA-1 up front, then one per iteration from g = 1 on, so
    // NA - 2 groups follow chunk g's.
    for (int g = 0; g < NA; ++g) issue_next();
    int sa = 0, sp = NA - 1;   // slot of chunk g, slot of chunk g - 1
    uint32_t pp = 0;           // parity of chunk g - 1's use of its slot
    for (int g = 0; g < total; ++g) {
      asm volatile("cp.async.wait_group %0;" ::"n"(NA - 2) : "memory");
      if (tid == 0) { SH_TR(0, g); }
      fence_proxy_async_smem();   // the tensor core reads the slot through the async proxy
      mbar_arrive(&astaged[sa]);
      if (g >= 1) {
        if (ig < total) {
          mbar_wait(&aempty[sp], pp);
          if (tid == 0) { SH_TR(1, g); }
          __syncwarp();
        }
        issue_next();
      }
      sp = sa;
      if (g >= 1 && sp == 0) pp ^= 1u;   // chunk g - 1 wrapped to slot 0: next pass over the ring
      if (++sa == NA) sa = 0;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // ------------------------------------------------ epilogue (warps 6-9): TMEM lane quarter warp % 4
    const int et = (warp & 3) * 32 + lane;          // tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    for (int seq = 0; seq < i1 - i0; ++seq) {
      const int4 it = item_of(seq);
      const int cur_bin = it.x, cur_rows = it.z;
      const int p = et < it.z ? patch_of(a, row_at(a, it, et)) : -1;
      const int acc = nacc == 2 ? (seq & 1) : 0;
      const int gnode = a.level_base + cur_bin;
      const int cb = __ldg(a.child_begin + gnode);
      const int cc = __ldg(a.child_count + gnode);
      const bool valid = et < cur_rows && p >= 0;
      // Everything the row needs from global memory is requested before the wait
      // for the tile's MMAs (under the row stream a round trip costs thousands of
      // cycles, and the epilogue of a tile must fit into the next tile's MMAs):
      // 1 / s_p, the near-tie window, and the first 32 columns of the correction row.
      const bool has_corr = a.corr_pre != nullptr && a.sup_t > 0;
      const float4* crow = reinterpret_cast<const float4*>(a.corr_pre + (int64_t)(valid ? p : 0) * a.corr_pre_ld);
      float4 cr[4];   // corrections of the 16 columns at hand
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        cr[q4] = has_corr && valid && 4 * q4 < cc ? ld_now(crow + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float scale = valid ? ld_now(a.inv_scale + p) : 1.f;   // > 0 on every lane: the read-back is warp-collective
      const float delta =
          valid ? a.recheck_rel * (float)sqrt(ld_now(a.xn2 + p)) + a.recheck_q * ld_now(a.qerr + p) : 0.f;
      mbar_wait_backoff(&accfull[acc], (uint32_t)(seq / nacc) & 1u);   // a tile's MMAs take tens of microseconds
      if (et == 0) { SH_TRT(3, seq); }
      tc_fence_after();
      const uint32_t taddr = tmem + lane_base + (uint32_t)acc * accs;
      int best = 0;
      float bestv = -1.f, second = -1.f;
      if (et == 0) { SH_TRT(4, seq); }
      // corrected scores c . x - sum_k c_k P[S_k][child], first max of |score| in child
      // order (pursuit.py:151), 16 columns at a time
      for (int c0 = 0; c0 < cc; c0 += 16) {
        float4 cn[4];   // the next 16 columns' corrections, in flight during this step
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          cn[q4] = has_corr && valid && c0 + 16 + 4 * q4 < cc ? ld_now(crow + (c0 + 16) / 4 + q4)
                                                              : make_float4(0.f, 0.f, 0.f, 0.f);
        float v[16];
        acc_ld16h(taddr + (uint32_t)c0, accw, scale, v);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          v[4 * q4] -= cr[q4].x;
          v[4 * q4 + 1] -= cr[q4].y;
          v[4 * q4 + 2] -= cr[q4].z;
          v[4 * q4 + 3] -= cr[q4].w;
        }
        const int nc = min(16, cc - c0);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
          if (jj < nc) {
            const float m = fabsf(v[jj]);
            if (m > bestv) {
              second = bestv;
              bestv = m;
              best = c0 + jj;
            } else {
              second = fmaxf(second, m);
            }
          }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) cr[q4] = cn[q4];
      }
      if (et == 0) { SH_TRT(5, seq); }
      // Near ties (score_epi.cuh: recheck_near_ties, same rule): rows whose two best
      // scores are closer than delta note the children within 2 delta of the best
      // -- a second read of the accumulator --, the accumulator is released, and
      // only then are the candidates re-scored with exact dots.
      const bool flagged = valid && bestv - second < delta;
      const unsigned todo0 = __ballot_sync(kFull, flagged);
      unsigned cmask[2] = {0u, 0u};
      if (todo0) {
        const float lo = bestv - 2.f * delta;
        for (int c0 = 0; c0 < cc && c0 < 64; c0 += 16) {
          float v[16];
          acc_ld16h(taddr + (uint32_t)c0, accw, scale, v);
          if (flagged) {
            const int nc = min(16, cc - c0);
            unsigned mk = 0u;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const float corr = has_corr && jj < nc ? __ldg(a.corr_pre + (int64_t)p * a.corr_pre_ld + c0 + jj) : 0.f;
              if (jj < nc && fabsf(v[jj] - corr) >= lo) mk |= 1u << jj;
            }
            cmask[c0 >> 5] |= mk << (c0 & 16);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&accempty[acc]);
      {
        unsigned todo = todo0;
        while (todo) {
          const int src = __ffs(todo) - 1;
          todo &= todo - 1;
          const int q = __shfl_sync(kFull, p, src);
          const float* xrow = a.R + (int64_t)q * a.ld;
          // all lines of the row and of every candidate centroid are requested at
          // once (L2 prefetches), so the dots below pay one DRAM round trip together
          // instead of one per 128 columns each
          const unsigned cm0 = __shfl_sync(kFull, cmask[0], src), cm1 = __shfl_sync(kFull, cmask[1], src);
          const int nlines = a.ld / 32;
          for (int i = lane; i < nlines; i += 32) prefetch_l2(xrow + 32 * i);
          for (int h = 0; h < 2; ++h) {
            unsigned cand = h ? cm1 : cm0;
            while (cand) {
              const int jj = __ffs(cand) - 1;
              cand &= cand - 1;
              const float* crow_x = a.cent + (int64_t)(cb + 32 * h + jj) * a.ld;
              for (int i = lane; i < nlines; i += 32) prefetch_l2(crow_x + 32 * i);
            }
          }
          float nbv = -1.f;
          int nbest = 0;
          for (int h = 0; h < 2; ++h) {
            unsigned cand = h ? cm1 : cm0;
            while (cand) {
              const int jj = __ffs(cand) - 1;
              cand &= cand - 1;
              const int col = 32 * h + jj;
              const float raw = warp_dot(xrow, a.cent + (int64_t)(cb + col) * a.ld, a.ld);
              const float corr = has_corr ? __ldg(a.corr_pre + (int64_t)q * a.corr_pre_ld + col) : 0.f;
              const float sj = fabsf(raw - corr);
              if (sj > nbv) {   // columns visited in increasing order: strict > keeps the first max
                nbv = sj;
                nbest = col;
              }
            }
          }
          if (lane == src) {
            bestv = nbv;
            best = nbest;
          }
        }
      }
      if (et == 0) { SH_TRT(2, seq); }
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
#ifdef STMP_SH_TRACE
  if ((blockIdx.x == 0 || blockIdx.x == 101 || blockIdx.x == 290) && tid == 0 && a.sup_t == 5) {
    const long long tend = clock64() - tr_t0;
    for (int q = 0; q < i1 - i0 && q < 32; ++q)
      printf("TT L%d cta %d tile %d rows %d mma_start %lld acc_free %lld accfull %lld meta %lld argmax %lld epi_done %lld nrecheck(w0) %d end %lld\n", a.level, blockIdx.x, q,
             item_of(q).z, trt[0][q], trt[1][q], trt[3][q], trt[4][q], trt[5][q], trt[2][q], trn[q], tend);
  }
  if (blockIdx.x == 0 && tid == 0 && a.sup_t == 5)
    for (int g = 0; g < 64; ++g)
      printf("TR L%d g %d landed %lld aempty %lld astaged %lld full %lld issued %lld\n", a.level, g, tr[0][g] - tr[0][0],
             tr[1][g] - tr[0][0], tr[2][g] - tr[0][0], tr[3][g] - tr[0][0], tr[4][g] - tr[0][0]);
#endif
}

template <int NA, int NB, int CPS>
cudaError_t launch_sh(ScoreArgs s, int sms, cudaStream_t st) {
  const uint32_t smem = sh_layout(s.npad, NA, NB).total;
  const int accw = s.npad;
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
  // 64-column chunks; N = kPieces npad per MMA, the epilogue reads 16 columns at a time
  return ld % 64 == 0 && npad % 16 == 0 && npad >= 16 && npad <= 64;
}

cudaError_t launch_score_sh(const ScoreArgs& s, int sms, cudaStream_t st) {
  if (!score_sh_fits(s.ld, s.npad)) return cudaErrorNotSupported;
  // ring depths as a decimal code NA NB CPS (row slots, table slots, CTAs per SM);
  // developer hook for sweeps: -DSTMP_SH_WIDE=822
#ifndef STMP_SH_WIDE
#define STMP_SH_WIDE 422   // npad 64: 64 KB of rows + 2 x 16 KB of table per CTA
#endif
#ifndef STMP_SH_NARROW
#define STMP_SH_NARROW 532   // npad 32: 80 KB + 3 x 8 KB
#endif
  if (s.npad > 32) return launch_sh<STMP_SH_WIDE / 100, STMP_SH_WIDE / 10 % 10, STMP_SH_WIDE % 10>(s, sms, st);
  return launch_sh<STMP_SH_NARROW / 100, STMP_SH_NARROW / 10 % 10, STMP_SH_NARROW % 10>(s, sms, st);
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
