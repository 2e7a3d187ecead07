// Scoring pass for wide or long nodes: the node's child table streams through
// shared memory one 32-column K chunk at a time.
//
// score_ts_kernel keeps a whole per-node table resident in shared memory, which
// caps it at kchunks * npad * 256 B (+ a landing plane) per CTA.  Config 2
// (256 children of 144-dim rows -> 320 KB per node) and config 4 (1600-dim rows)
// do not fit, so this kernel streams: for every 128-patch tile and K chunk c
//   * each thread gathers its own patch row's chunk c (8 x 16-B cp.async) into
//     a ring of NA swizzled landing slots, running NA chunks ahead -- a thread
//     only ever reads the row it copied, so no barrier guards the landing ring;
//   * the thread splits the chunk into tf32 hi / lo and stores both to one of
//     two TMEM A buffers (tcgen05.st), so the staging of chunk c+1 overlaps the
//     MMAs of chunk c;
//   * thread 0 keeps a ring of NB table-chunk slots (hi | lo planes, npad rows x
//     128 B each, SW128, one bulk copy per chunk) NB-1 chunks ahead and issues
//     the 3xTF32 MMAs of the chunk (M = 128 patches, N = npad <= 256 children,
//     A from TMEM), committing to the chunk's slot barrier, which frees both
//     the table slot and the TMEM A buffer;
//   * after the tile's last chunk the accumulator (npad TMEM columns) is read
//     back and reduced to the argmax child exactly like score_ts_kernel.
// Semantics: pkg/src/stmp/pursuit.py:134-162 (greedy level choice, first max of
// |score| in child order; leaf metadata for the last level).
#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

namespace {

constexpr int kT = 128;
constexpr int kThreads = 128;
constexpr uint32_t kSlot = kT * 128u;   // one landing slot: 128 rows x 32 floats
constexpr uint32_t kColAcc = 128;       // TMEM: A buffers at [0,64) and [64,128), accumulator from 128

struct StLayout {
  uint32_t land, btab, leaf, rows, hist, bars, slot, total;
};

__host__ __device__ inline uint32_t st_align(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }

__host__ __device__ inline StLayout st_layout(int npad, bool last, int na, int nb) {
  StLayout L{};
  uint32_t o = 0;
  L.land = o; o += (uint32_t)na * kSlot;
  L.btab = o; o += (uint32_t)nb * st_align((uint32_t)npad * 256u, 1024u);
  L.leaf = o; o += last ? (uint32_t)npad * 8u : 0u;
  o = st_align(o, 16);
  L.rows = o; o += kT * 4;
  L.hist = o; o += 256 * 4;
  L.bars = st_align(o, 8); o = L.bars + (uint32_t)(2 * nb + 1) * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

template <int NA, int NB>
__global__ void __launch_bounds__(kThreads, 1) score_st_kernel(ScoreArgs a) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int npad = a.npad;
  const int kch = a.kchunks;
  const bool last = a.leaf_sel != nullptr;
  const StLayout Ly = st_layout(npad, last, NA, NB);
  uint8_t* land = base + Ly.land;
  const uint32_t bslot = st_align((uint32_t)npad * 256u, 1024u);
  const int* s_leaf_info = reinterpret_cast<const int*>(base + Ly.leaf);
  const int* s_leaf_cnt = s_leaf_info + npad;
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Ly.bars);   // [NB] table chunk landed
  uint64_t* done = full + NB;                                      // [NB] MMAs of the chunk retired
  uint64_t* leafbar = done + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.slot);

  if (warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&done[b], 1);
    }
    mbar_init(leafbar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;

  const int num_items = *a.num_items;
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int i1 = min(num_items, i0 + per);
  if (i0 >= i1) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
    return;
  }
  const int total = (i1 - i0) * kch;   // chunks of this CTA
  const uint32_t idesc = idesc_tf32(kT, npad);
  const uint32_t tb = table_bytes(kch, npad, last);
  const uint32_t chunk_bytes = (uint32_t)npad * 256u;
  const uint32_t land_s = smem_u32(land);
  const uint32_t b_s = smem_u32(base + Ly.btab);

  // table chunk g -> ring slot g % NB (thread 0 only)
  int b_item = -1, b_bin = 0;
  auto issue_b = [&](int g) {
    const int item = i0 + g / kch, c = g - (g / kch) * kch;
    if (item != b_item) {
      b_item = item;
      b_bin = a.items[item].x;
    }
    const int s = g % NB;
    mbar_arrive_expect_tx(&full[s], chunk_bytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.table) + (size_t)b_bin * tb + (size_t)c * chunk_bytes;
    bulk_g2s(base + Ly.btab + s * bslot, src, chunk_bytes, &full[s]);
  };
  // this thread's row of item `item` (-1: padding row of a partial tile)
  int r_item = -1, r_row = -1;
  auto row_of = [&](int item) {
    if (item != r_item) {
      r_item = item;
      const int4 it = a.items[item];
      r_row = tid < it.z ? a.perm[it.y + tid] : -1;
    }
    return r_row;
  };
  // gather chunk g of this thread's row into landing slot g % NA (one commit group per call)
  auto issue_a = [&](int g) {
    if (g < total) {
      const int item = i0 + g / kch, c = g - (g / kch) * kch;
      const int r = row_of(item);
      const uint32_t dst = land_s + (uint32_t)(g % NA) * kSlot;
      const float* src = a.R + (r >= 0 ? (int64_t)r * a.ld + 32 * c : 0);
#pragma unroll
      for (int j = 0; j < 8; ++j) cp_async16(dst + sw128_offset(tid, j), src + 4 * j, r >= 0 ? 16u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  if (tid == 0) {
    for (int g = 0; g < NB && g < total; ++g) issue_b(g);
    if (last) {
      mbar_arrive_expect_tx(leafbar, 8u * npad);
      bulk_g2s(base + Ly.leaf, reinterpret_cast<const uint8_t*>(a.table) + (size_t)a.items[i0].x * tb +
                                   (size_t)kch * chunk_bytes, 8u * npad, leafbar);
    }
  }
  for (int g = 0; g < NA; ++g) issue_a(g);
  int b_next = min(NB, total);
  uint32_t leaf_phase = 0;

  int cur_item = -1, cur_p = -1, cur_bin = 0, cur_rows = 0;
  for (int g = 0; g < total; ++g) {
    const int item = i0 + g / kch, c = g - (g / kch) * kch;
    if (c == 0) {
      const int4 it = a.items[item];
      cur_item = item;
      cur_bin = it.x;
      cur_rows = it.z;
      cur_p = row_of(item);
    }
    // (1) own row's chunk landed
    asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
    // (2)-(3) read + split
    float hi[32], lo[32];
    const uint8_t* slot = land + (uint32_t)(g % NA) * kSlot;
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
    // landing slot consumed by this thread: refill it with chunk g + NA
    issue_a(g + NA);
    // (4) TMEM A buffer g & 1 is free once the MMAs of chunk g - 2 retired
    if (g >= 2) {
      const int gp = g - 2;
      mbar_wait(&done[gp % NB], (uint32_t)(gp / NB) & 1u);
      tc_fence_after();
    }
    const uint32_t abuf = (uint32_t)(g & 1) * 64u;
    tmem_st32(tmem + lane_base + abuf, hi);
    tmem_st32(tmem + lane_base + abuf + 32, lo);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      const int s = g % NB;
      mbar_wait(&full[s], (uint32_t)(g / NB) & 1u);
      tc_fence_after();
      const uint32_t bh = b_s + s * bslot;
      const uint32_t bl = bh + (uint32_t)npad * 128u;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t ah = tmem + abuf + ks * 8;
        const uint32_t al = ah + 32;
        const uint32_t o = ks * 32u;
        mma_tf32_ts(tmem + kColAcc, ah, sw128_kmajor_desc(bh + o), idesc, (c | ks) ? 1u : 0u);
        mma_tf32_ts(tmem + kColAcc, ah, sw128_kmajor_desc(bl + o), idesc, 1u);
        mma_tf32_ts(tmem + kColAcc, al, sw128_kmajor_desc(bh + o), idesc, 1u);
      }
      mma_commit(&done[s]);
      // refill the slot of chunk g - 1 (its MMAs were issued one chunk ago)
      if (g >= 1 && b_next < total && b_next == g - 1 + NB) {
        const int gp = g - 1;
        mbar_wait(&done[gp % NB], (uint32_t)(gp / NB) & 1u);
        issue_b(b_next++);
      }
    }
    if (c != kch - 1) continue;

    // ---- tile epilogue: argmax over the node's children
    mbar_wait(&done[g % NB], (uint32_t)(g / NB) & 1u);
    tc_fence_after();
    const int gnode = a.level_base + cur_bin;
    const int cb = __ldg(a.child_begin + gnode);
    const int cc = __ldg(a.child_count + gnode);
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
    const bool valid = tid < cur_rows;
    const int p = cur_p;
    const int child = cb + best;
    int leaf_info = 0, leaf_cnt = 0;
    if (last) {
      mbar_wait(leafbar, leaf_phase);
      leaf_phase ^= 1u;
      if (valid) {
        leaf_info = s_leaf_info[best];
        leaf_cnt = s_leaf_cnt[best];
      }
    }
    if (valid) {
      a.path_ws[(int64_t)p * a.L + a.level] = child;
      if (a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = child;
      if (a.next_counts) atomicAdd(&s_hist[best], 1);
      if (last) a.leaf_sel[p] = leaf_info;
      if (a.ip) add_ip(a.ip, p, cc + leaf_cnt, cc);
    }
    // generic reads of the leaf block before its async refill; hist complete
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (last && tid == 0 && item + 1 < i1) {
      mbar_arrive_expect_tx(leafbar, 8u * npad);
      bulk_g2s(base + Ly.leaf, reinterpret_cast<const uint8_t*>(a.table) + (size_t)a.items[item + 1].x * tb +
                                   (size_t)kch * chunk_bytes, 8u * npad, leafbar);
    }
    if (a.next_counts) {
      for (int j = tid; j < cc; j += kThreads) {
        const int h = s_hist[j];
        if (h) atomicAdd(&a.next_counts[cb + j - a.next_base], h);
        s_hist[j] = 0;
      }
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

template <int NA, int NB>
cudaError_t launch_st(ScoreArgs s, int sms, cudaStream_t st) {
  const bool last = s.leaf_sel != nullptr;
  const uint32_t smem = st_layout(s.npad, last, NA, NB).total;
  int cols = 32;
  while (cols < (int)kColAcc + (s.npad + 31) / 32 * 32) cols <<= 1;
  s.tmem_cols = cols;
  cudaError_t e = cudaFuncSetAttribute(score_st_kernel<NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int by_smem = (int)((228 * 1024) / (smem + 1024));
  const int by_tmem = 512 / cols;
  const int per_sm = std::max(1, std::min(4, std::min(by_smem, by_tmem)));
  return launch_kernel(score_st_kernel<NA, NB>, sms * per_sm, kThreads, (size_t)smem, st, true, s);
}

}  // namespace

bool score_st_fits(int kchunks, int npad, bool last) {
  if (kchunks < 1 || npad < 16 || npad > 256) return false;
  return st_layout(npad, last, 4, 2).total <= 227 * 1024;
}

cudaError_t launch_score_st(const ScoreArgs& s, int sms, cudaStream_t st) {
  if (!score_st_fits(s.kchunks, s.npad, s.leaf_sel != nullptr)) return cudaErrorNotSupported;
  // wide nodes: two 64 KB table slots; narrow ones: a deeper table ring
  if (s.npad > 128) return launch_st<4, 2>(s, sms, st);
  return launch_st<4, 3>(s, sms, st);
}

}  // namespace stmp
