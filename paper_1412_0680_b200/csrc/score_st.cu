// Scoring pass for wide or long nodes: the node's child table streams through
// shared memory one 32-column K chunk at a time, with warp-specialised roles.
//
// score_ts_kernel keeps a whole per-node table resident in shared memory, which
// caps it at kchunks * npad * 256 B (+ a landing plane) per CTA.  Config 2
// (256 children of 144-dim rows -> 320 KB per node) and config 4 (1600-dim rows)
// do not fit, so this kernel streams.  One persistent CTA per SM, 192 threads:
//   * warps 0-3, stagers (thread = patch row = TMEM lane): each warp gathers
//     chunk c of its 32 rows (cp.async, four whole 128-byte lines per
//     instruction) into a ring of NA swizzled landing slots, NA chunks ahead --
//     a warp only reads the rows it copied, so the landing ring needs no CTA
//     barrier -- then each thread splits its row into tf32 hi / lo and stores
//     both into one of NAB TMEM A buffers (tcgen05.st);
//   * warps 6-9, epilogue (TMEM lane quarter = warp % 4): after a tile's last
//     chunk they read the accumulator back and reduce it to the argmax child
//     (Gram path: with the support correction and the near-tie re-check) while
//     the stagers already stage the next tile;
//   * warp 4, MMA issuer: per chunk, 3xTF32 tcgen05.mma (M = 128 patches,
//     N = npad <= 256 children, A from TMEM, B = the table chunk in shared
//     memory), commits that free the table slot and the A buffer, and at a
//     tile's end a commit that hands the accumulator to the epilogue;
//   * warp 5, table producer: one bulk copy per chunk (hi | lo planes, npad
//     rows x 128 B each, SW128) into a ring of NB slots, refilled as soon as
//     the MMAs of the slot's previous chunk retire (the last level's leaf
//     records are read by the epilogue straight from the table block in L2).
// The accumulator is double-buffered when 128 + 2 * npad TMEM columns fit, so
// a tile's epilogue overlaps the next tile's MMAs.
// Semantics: pkg/src/stmp/pursuit.py:134-162 (greedy level choice, first max of
// |score| in child order; leaf metadata for the last level).
#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "score_epi.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;
using namespace epi;

namespace {

constexpr int kT = 128;
constexpr int kStagers = 128;
constexpr int kEpi = 128;                 // epilogue warps 6-9 (TMEM lane quarter = warp % 4)
constexpr int kThreads = kStagers + 64 + kEpi;   // stagers, MMA warp, producer warp, epilogue
constexpr uint32_t kSlot = kT * 128u;     // one landing slot: 128 rows x 32 floats
// NAB TMEM A buffers (64 columns each: hi | lo of one K chunk) at [0, 64 NAB),
// accumulators from 64 NAB

struct StLayout {
  uint32_t land, btab, hist, bars, slot, total;
};

__host__ __device__ inline uint32_t st_align(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }

__host__ __device__ inline uint32_t st_bslot(int npad) { return st_align((uint32_t)npad * 256u, 1024u); }

__host__ __device__ inline StLayout st_layout(int npad, bool last, int na, int nb, int nab) {
  StLayout L{};
  uint32_t o = 0;
  L.land = o; o += (uint32_t)na * kSlot;
  L.btab = o; o += (uint32_t)nb * st_bslot(npad);
  o = st_align(o, 16);
  L.hist = o; o += 256 * 4;
  L.bars = st_align(o, 8); o = L.bars + (uint32_t)(2 * nb + 2 * nab + 4) * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

// Staged beam descent (pursuit.py:134-162), one entry (patch, node) per row,
// all 32 lanes of an epilogue warp call it (TMEM reads are warp-collective).
// Internal levels: the node's `keep` best children by |score| -- a stable sort
// on -|score|, i.e. the largest keys (|score| bits << 32 | ~position) -- become
// the next level's entries, in child order; the first survivor of the patch's
// first entry continues the reference's path (frontier[0]).  Last level: the
// survivors' leaf atoms are candidates; the top-1 child of every entry is a
// survivor, so the patch's pick -- max |score|, ties to the lowest atom index
// -- is one 64-bit atomicMax of (|score| bits << 32 | ~atom) per entry.
__device__ void beam_epilogue(uint32_t taddr, uint32_t off2, int cc, int cb, const ScoreArgs& a, bool valid, int p,
                              int e, bool last, const int* leaf_info, int* s_hist) {
  const int lane = (int)(threadIdx.x & 31);
  const int keep = a.beam_keep;
  const int npick = keep < cc ? keep : cc;
  const bool first = valid && (a.entry_first == nullptr || a.entry_first[e] != 0);
  auto key_at = [](float v, unsigned id) {
    return ((unsigned long long)__float_as_uint(fabsf(v)) << 32) | (unsigned long long)(0xFFFFFFFFu - id);
  };
  // top-npick children by position-tie-broken keys: each round takes the largest key below the previous one
  int pick[kMaxBeamKeep];
  unsigned long long prev = ~0ull;
  for (int q = 0; q < kMaxBeamKeep; ++q) {
    if (q >= npick) break;
    unsigned long long bk = 0ull;
    for (int c0 = 0; c0 < cc; c0 += 32) {
      float v[32];
      acc_ld32(taddr + (uint32_t)c0, off2, v);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c0 + j < cc) {
          const unsigned long long k = key_at(v[j], (unsigned)(c0 + j));
          if (k < prev && k > bk) bk = k;
        }
    }
    prev = bk;
    pick[q] = (int)(0xFFFFFFFFu - (unsigned)(bk & 0xFFFFFFFFull));
  }
  if (!last) {
    // survivors in child order
    for (int i = 1; i < npick; ++i) {
      const int v = pick[i];
      int j = i - 1;
      while (j >= 0 && pick[j] > v) {
        pick[j + 1] = pick[j];
        --j;
      }
      pick[j + 1] = v;
    }
    const int n = valid ? npick : 0;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    int base = 0;
    if (lane == 31 && total > 0) base = atomicAdd(a.out_count, total);
    base = __shfl_sync(kFull, base, 31) + incl - n;
    for (int i = 0; i < n; ++i) {
      a.out_patch[base + i] = p;
      a.out_node[base + i] = cb + pick[i];
      a.out_first[base + i] = (first && i == 0) ? 1 : 0;
      atomicAdd(&s_hist[pick[i]], 1);
    }
    if (valid) {
      if (first && a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = cb + pick[0];
      if (a.ip) add_ip(a.ip, p, cc, cc);
    }
  } else if (valid) {
    // the reference's path continues with the first survivor (in child order) of frontier[0]
    int minpos = pick[0];
    for (int i = 1; i < npick; ++i) minpos = pick[i] < minpos ? pick[i] : minpos;
    if (first && a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = cb + minpos;
    if (a.ip) add_ip(a.ip, p, cc + npick, cc);   // cc centroids + the survivors' single leaf atoms
  }
  if (last) {
    // candidates: the survivors' leaf atoms (pursuit.py:155-162), max |score|,
    // ties to the lowest atom index: one pass over the chunks (warp-collective)
    unsigned long long best = 0ull;
    for (int c0 = 0; c0 < cc; c0 += 32) {
      float v[32];
      acc_ld32(taddr + (uint32_t)c0, off2, v);
      if (!valid) continue;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        bool surv = false;
        for (int i = 0; i < kMaxBeamKeep; ++i) surv |= (i < npick && pick[i] == c0 + j);
        if (c0 + j < cc && surv) {
          const int atom = __ldg(leaf_info + c0 + j);
          const unsigned long long k = key_at(v[j], (unsigned)atom);
          best = k > best ? k : best;
        }
      }
    }
    if (valid) atomicMax(a.leaf_key + p, best);
  }
}

template <int NA, int NB, int NAB, int CPS>
__global__ void __launch_bounds__(kThreads, CPS) score_st_kernel(ScoreArgs a, int nacc, int chains) {
  constexpr int kNAB = NAB;
  constexpr uint32_t kColAcc = 64u * NAB;
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int npad = a.npad;
  const int kch = a.kchunks;
  const bool last = a.leaf_sel != nullptr;
  const StLayout Ly = st_layout(npad, last, NA, NB, NAB);
  const uint32_t bslot = st_bslot(npad);
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Ly.bars);   // [NB] table chunk landed (tx)
  uint64_t* done = full + NB;          // [NB] MMAs reading the slot retired (commit)
  uint64_t* astaged = done + NB;       // [kNAB] A buffer written by the 128 stagers
  uint64_t* aempty = astaged + kNAB;   // [kNAB] MMAs reading the A buffer retired (commit)
  uint64_t* accfull = aempty + kNAB;   // [2] accumulator complete (commit)
  uint64_t* accempty = accfull + 2;    // [2] accumulator read back by the 128 epilogue threads
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
  const uint32_t tb = table_bytes(kch, npad, last);
  const uint32_t chunk_bytes = (uint32_t)npad * 256u;
  const uint32_t accw = (uint32_t)(npad + 31) / 32 * 32;
  // wide-N mode (chains == 2, npad % 32 == 0): an accumulator buffer holds
  // [hi.hi | hi.lo + lo.hi]; one MMA with N = 2 npad multiplies x_hi by the
  // table's hi and lo planes at once (they are adjacent row blocks of the chunk),
  // a second adds x_lo . b_hi into the upper half -- two tensor instructions per
  // k-step instead of three; the epilogue sums the halves
  const uint32_t off2 = chains == 2 ? accw : 0u;
  const uint32_t accs = accw * (uint32_t)chains;   // stride of the accumulator buffers

#ifndef STMP_ST_L2HINTS
#define STMP_ST_L2HINTS 1
#endif
  if (warp == 5) {
    // ------------------------------------------------ table producer
    if (lane == 0) {
      const uint64_t tab_policy = STMP_ST_L2HINTS ? l2_policy_evict_last() : l2_policy_evict_first();
      int bin = 0;
      for (int g = 0; g < total; ++g) {
        const int seq = g / kch, c = g - seq * kch;
        if (c == 0) bin = item_at(a, i0 + seq).x;
        const int s = g % NB;
        if (g >= NB) mbar_wait(&done[s], (uint32_t)(g / NB - 1) & 1u);
        mbar_arrive_expect_tx(&full[s], chunk_bytes);
        bulk_g2s_hint(base + Ly.btab + s * bslot,
                      reinterpret_cast<const uint8_t*>(a.table) + (size_t)bin * tb + (size_t)c * chunk_bytes,
                      chunk_bytes, &full[s], tab_policy);
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(kT, npad);
      const uint32_t idesc2 = idesc_tf32(kT, 2 * npad);
      const uint32_t b_s = smem_u32(base + Ly.btab);
      for (int g = 0; g < total; ++g) {
        const int seq = g / kch, c = g - seq * kch;
        const int ab = g % kNAB, s = g % NB;
        const int acc = nacc == 2 ? (seq & 1) : 0;
        const uint32_t dcol = tmem + kColAcc + (uint32_t)acc * accs;
        const uint32_t dlo = dcol + off2;
        if (c == 0 && seq >= nacc) mbar_wait(&accempty[acc], (uint32_t)(seq / nacc - 1) & 1u);
        mbar_wait(&astaged[ab], (uint32_t)(g / kNAB) & 1u);
        mbar_wait(&full[s], (uint32_t)(g / NB) & 1u);
        tc_fence_after();
        const uint32_t bh = b_s + s * bslot;
        const uint32_t bl = bh + (uint32_t)npad * 128u;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t ah = tmem + (uint32_t)ab * 64u + ks * 8;
          const uint32_t al = ah + 32;
          const uint32_t o = ks * 32u;
          if (c == kch - 1 && ks >= a.ks_last) break;   // zero padding on both operands
#ifndef STMP_ST_MMAS   // timing experiments only: 0 = no MMAs, 1 = hi.hi only, 3 = 3xTF32 (default)
#define STMP_ST_MMAS 3
#endif
          if (off2) {
            mma_tf32_ts(dcol, ah, sw128_kmajor_desc(bh + o), idesc2, (c | ks) ? 1u : 0u);   // [hi.hi | hi.lo]
            if (STMP_ST_MMAS >= 3) mma_tf32_ts(dlo, al, sw128_kmajor_desc(bh + o), idesc, 1u);   // += lo.hi
          } else {
            if (STMP_ST_MMAS >= 1) mma_tf32_ts(dcol, ah, sw128_kmajor_desc(bh + o), idesc, (c | ks) ? 1u : 0u);
            if (STMP_ST_MMAS >= 3) {
              mma_tf32_ts(dcol, ah, sw128_kmajor_desc(bl + o), idesc, 1u);
              mma_tf32_ts(dcol, al, sw128_kmajor_desc(bh + o), idesc, 1u);
            }
          }
        }
        mma_commit(&done[s]);
        mma_commit(&aempty[ab]);
        if (c == kch - 1) mma_commit(&accfull[acc]);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------ stagers (warps 0-3)
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t land_s = smem_u32(base + Ly.land);
    const uint64_t row_policy = l2_policy_evict_first();
    // row ids of this warp's 32 rows for the item being gathered (lane l: row 32w + l)
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
    // 128-byte chunk of row 4i+q, so every cp.async instruction moves four whole
    // lines (one commit group per call; the warp syncs before reading)
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
          const float* src = a.R + (r >= 0 ? (int64_t)r * a.ld + 32 * c + 4 * j : 0);
          if (STMP_ST_L2HINTS)
            cp_async16_hint(dst + sw128_offset((uint32_t)(warp * 32 + rl), (uint32_t)j), src, r >= 0 ? 16u : 0u,
                            row_policy);
          else
            cp_async16(dst + sw128_offset((uint32_t)(warp * 32 + rl), (uint32_t)j), src, r >= 0 ? 16u : 0u);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int g = 0; g < NA; ++g) issue_a(g);
    for (int g = 0; g < total; ++g) {
      const int ab = g % kNAB;
      asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
      __syncwarp();   // the warp's rows were copied by all of its lanes
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
      __syncwarp();      // every lane has read its row before the slot is refilled
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
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // ------------------------------------------------ epilogue (warps 6-9): TMEM lane quarter warp % 4
    const int et = (warp & 3) * 32 + lane;          // tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    for (int seq = 0; seq < i1 - i0; ++seq) {
      const int4 it = item_at(a, i0 + seq);
      const int cur_bin = it.x, cur_rows = it.z;
      const int cur_e = et < it.z ? row_at(a, it, et) : -1;   // entry id (= patch id off the beam path)
      const int cur_p = patch_of(a, cur_e);
      const int tid = et;

      const int acc = nacc == 2 ? (seq & 1) : 0;
      mbar_wait(&accfull[acc], (uint32_t)(seq / nacc) & 1u);
      tc_fence_after();
      const int gnode = a.level_base + cur_bin;
      const int cb = __ldg(a.child_begin + gnode);
      const int cc = __ldg(a.child_count + gnode);
      int best = 0;
      float bestv = -1.f;
      const bool valid = tid < cur_rows && cur_p >= 0;
      const int p = cur_p;
      if (a.beam_keep > 0) {
        beam_epilogue(tmem + lane_base + kColAcc + (uint32_t)acc * accs, off2, cc, cb, a, valid, p, cur_e, last,
                      a.table == nullptr ? nullptr
                                         : reinterpret_cast<const int*>(reinterpret_cast<const uint8_t*>(a.table) +
                                                                        (size_t)cur_bin * tb +
                                                                        (size_t)kch * chunk_bytes),
                      s_hist);
        tc_fence_before();
        mbar_arrive(&accempty[acc]);
        if (a.out_count != nullptr) {   // next level's bin counts
          named_sync(1, kEpi);
          for (int j = tid; j < cc; j += kEpi) {
            const int h = s_hist[j];
            if (h) atomicAdd(&a.next_counts[cb + j - a.next_base], h);
            s_hist[j] = 0;
          }
          named_sync(1, kEpi);
        }
        continue;
      }
      if (a.corr != nullptr || a.raw_out != nullptr) {
        // Gram path: rows are x; score = c . x - sum_k c_k P[S_k][child] (gram_path.cu)
        float second = -1.f;
        corr_abs_argmax(tmem + lane_base + kColAcc + (uint32_t)acc * accs, off2, cc, a, valid ? p : -1,
                        cb - a.corr_off, bestv, best, second);
        if (a.cent != nullptr)
          recheck_near_ties(tmem + lane_base + kColAcc + (uint32_t)acc * accs, off2, cc, cb, a, valid ? p : -1,
                            second, bestv, best);
      } else {
        acc_abs_argmax(tmem + lane_base + kColAcc + (uint32_t)acc * accs, off2, (int)accw, npad, bestv, best);
      }
      tc_fence_before();
      mbar_arrive(&accempty[acc]);
      int leaf_info = 0, leaf_cnt = 0;
      if (last && valid) {   // the winner's leaf record, straight from the (L2-resident) table block
        const int* info = reinterpret_cast<const int*>(reinterpret_cast<const uint8_t*>(a.table) +
                                                       (size_t)cur_bin * tb + (size_t)kch * chunk_bytes);
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
        for (int j = tid; j < cc; j += kEpi) {
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

struct StCfg {
  int na, nb, nab, cps;   // landing slots, table slots, TMEM A buffers, CTAs per SM
};

// ring depths: wide nodes (c2: 64 KB table chunks) get three table slots and a
// two-deep landing ring (the table refill latency is the one to hide); narrow
// ones (c4: 8-16 KB) a deep ring on both sides
#ifndef STMP_ST_NAB_NARROW
#define STMP_ST_NAB_NARROW 4
#endif
// four A buffers leave room for a double-buffered accumulator up to npad 128;
// narrow nodes (c4: 32-64 children) get NAB A buffers, as many as TMEM holds
#ifndef STMP_ST_CPS_NARROW
#define STMP_ST_CPS_NARROW 2
#endif
// narrow nodes (<= 64 children): two CTAs per SM, each with half the rings and
// half of TMEM, so one CTA's epilogue / refills overlap the other's MMAs
inline StCfg st_cfg(int npad) {
  if (npad > 128) return StCfg{2, 3, 4, 1};
  if (npad > 64) return StCfg{4, 4, 4, 1};
  return STMP_ST_CPS_NARROW == 2 ? StCfg{3, 3, 2, 2} : StCfg{6, 6, STMP_ST_NAB_NARROW, 1};
}

template <int NA, int NB, int NAB, int CPS>
cudaError_t launch_st(ScoreArgs s, int sms, cudaStream_t st) {
  constexpr uint32_t kColAcc = 64u * NAB;
  const bool last = s.leaf_sel != nullptr;
  const uint32_t smem = st_layout(s.npad, last, NA, NB, NAB).total;
  const int accw = (s.npad + 31) / 32 * 32;
#ifndef STMP_ST_CHAINS
#define STMP_ST_CHAINS 2
#endif
  // wide-N MMAs (two accumulator halves) and two accumulator buffers when TMEM holds them
  constexpr int kCols = 512 / CPS;   // TMEM columns per CTA
  const int chains = (int)kColAcc + 2 * accw <= kCols && s.npad % 32 == 0 ? STMP_ST_CHAINS : 1;
  const int nacc = (int)kColAcc + 2 * chains * accw <= kCols ? 2 : 1;
  int cols = 32;
  while (cols < (int)kColAcc + nacc * chains * accw) cols <<= 1;
  s.tmem_cols = cols;
  cudaError_t e = cudaFuncSetAttribute(score_st_kernel<NA, NB, NAB, CPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel(score_st_kernel<NA, NB, NAB, CPS>, sms * CPS, kThreads, (size_t)smem, st, true, s, nacc,
                       chains);
}

}  // namespace

bool score_st_fits(int kchunks, int npad, bool last) {
  if (kchunks < 1 || npad < 16 || npad > 256) return false;
  const StCfg c = st_cfg(npad);
  return st_layout(npad, last, c.na, c.nb, c.nab).total <= 227 * 1024;
}

cudaError_t launch_score_st(const ScoreArgs& s, int sms, cudaStream_t st) {
  if (!score_st_fits(s.kchunks, s.npad, s.leaf_sel != nullptr)) return cudaErrorNotSupported;
  const StCfg c = st_cfg(s.npad);
  if (c.cps == 2) return launch_st<3, 3, 2, 2>(s, sms, st);
  if (c.nb == 3) return launch_st<2, 3, 4, 1>(s, sms, st);
  if (c.nb == 4) return launch_st<4, 4, 4, 1>(s, sms, st);
  return launch_st<6, 6, STMP_ST_NAB_NARROW, 1>(s, sms, st);
}

}  // namespace stmp
