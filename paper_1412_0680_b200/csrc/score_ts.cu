// Scoring pass with the residual operand in tensor memory ("TS" tcgen05.mma).
//
// Same work items and semantics as score_tc_kernel (encode_staged.cu), but the
// gathered residual rows are split into tf32 hi/lo in registers -- each thread
// owns one patch row, reads it from the SW128-swizzled landing buffer without
// bank conflicts -- and written to TMEM with tcgen05.st, one 32-column K chunk
// at a time.  The MMA then reads A from TMEM and only the node table from
// shared memory, which cuts the shared-memory traffic per tile ~2.5x and the
// footprint to one landing plane + one table, so four CTAs share an SM.  The
// next tile's gather is launched as soon as its rows are staged in TMEM, so it
// overlaps the MMAs and the argmax epilogue.
#include <string.h>

#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

namespace {

constexpr int kT = 128;
constexpr int kThreads = 128;   // thread = patch row; warp w owns TMEM lanes 32w..32w+31
constexpr uint32_t kColA = 0;   // A_hi chunk: 32 columns, A_lo chunk: next 32
constexpr uint32_t kColAcc = 64;

struct TsLayout {
  uint32_t raw, btab, rows, hist, leaf, bars, slot, total;
};

__host__ __device__ inline uint32_t align_up_u(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }

__host__ __device__ inline TsLayout ts_layout(int kch, int npad, bool last) {
  TsLayout L{};
  uint32_t o = 0;
  L.raw = o; o += (uint32_t)kch * kT * 128u;
  L.btab = o; o += align_up_u(table_bytes(kch, npad, last), 1024u);
  L.rows = o; o += 2 * kT * 4;
  L.hist = o; o += 256 * 4;
  L.leaf = o; o += 2 * 256 * 4;   // last level: the tile's leaf records, copied out of the table block
  L.bars = align_up_u(o, 8); o = L.bars + 3 * 8;
  L.slot = o; o += 16;
  L.total = o + 1024;
  return L;
}

template <int KCH>
__device__ __forceinline__ void gather_rows(const ScoreArgs& a, const int* rows_ids, int rows, uint32_t raw_s,
                                            int tid) {
  constexpr int F = 8 * KCH;   // 16-byte chunks per residual row
  if constexpr ((kThreads % F) == 0) {
    // each thread keeps one chunk column c and walks rows r0, r0 + RS, ...: the
    // source offset, the swizzled destination and the row stride are loop
    // invariants, so a chunk costs one row-id load, one wide multiply-add and
    // the copy (16 consecutive threads still cover a whole 256-byte row)
    constexpr int RS = kThreads / F;
    const int c = tid % F;
    const int r0 = tid / F;
    const char* base = reinterpret_cast<const char*>(a.R) + 16 * c;
    const int ldb = a.ld * 4;
#pragma unroll
    for (int k = 0; k < kT / RS; ++k) {
      const int row = r0 + k * RS;
      const int rid = rows_ids[row];   // -1 past the tile's rows and for skipped patches
      const uint32_t off = (uint32_t)(c >> 3) * (kT * 128u) + sw128_offset(row, c & 7);
      cp_async16_row(raw_s + off, base + (int64_t)rid * ldb, rid);
    }
  } else {
#pragma unroll 4
    for (int e = tid; e < kT * F; e += kThreads) {
      const int row = e / F;
      const int c = e - row * F;
      const uint32_t off = (uint32_t)(c >> 3) * (kT * 128u) + sw128_offset(row, c & 7);
      const int rid = row < rows ? rows_ids[row] : -1;
      const bool ok = rid >= 0;
      cp_async16(raw_s + off, a.R + (ok ? (int64_t)rid * a.ld + 4 * c : 0), ok ? 16u : 0u);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KCH>
__global__ void __launch_bounds__(kThreads, 4) score_ts_kernel(ScoreArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int npad = a.npad;
  const bool last = a.leaf_sel != nullptr;
  const TsLayout Ly = ts_layout(KCH, npad, last);
  uint8_t* raw = base + Ly.raw;
  uint8_t* btab = base + Ly.btab;
  const uint32_t tb = table_bytes(KCH, npad, last);
  const int* t_leaf = reinterpret_cast<const int*>(btab + (size_t)KCH * 2 * npad * 128);   // in the table block
  int* s_leaf_info = reinterpret_cast<int*>(base + Ly.leaf);   // copy: the block is refilled early
  int* s_rows = reinterpret_cast<int*>(base + Ly.rows);
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + Ly.bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.slot);

  if (warp == 0) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
  const int lane = tid & 31;
  // gather of one tile's rows (ids[0..rows)) into the landing plane
  auto issue_gather = [&](const int* ids, int rows) { gather_rows<KCH>(a, ids, rows, smem_u32(raw), tid); };
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  // TMEM, barriers and the histogram are set up while the previous kernel
  // drains (programmatic dependent launch); nothing above reads its output
  pdl_enter();

  const int num_items = item_count(a);
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int i1 = min(num_items, i0 + per);
  const uint32_t idesc = idesc_tf32(kT, npad);
  const uint32_t raw_s = smem_u32(raw), b_s = smem_u32(btab);
  uint32_t tab_phase = 0, mma_phase = 0;
  int loaded_bin = -1;
  bool table_pending = false;

  int4 it = i0 < i1 ? item_at(a, i0) : make_int4(0, 0, 0, 0);
  if (i0 < i1) {
    s_rows[tid] = tid < it.z ? row_at(a, it, tid) : -1;   // kThreads == kT: every slot written
    if (tid == 0) {
      mbar_arrive_expect_tx(&bars[0], tb);
      const uint8_t* src = reinterpret_cast<const uint8_t*>(a.table) + (size_t)it.x * tb;
      for (uint32_t off = 0; off < tb; off += 65536u)
        bulk_g2s(btab + off, src + off, min(65536u, tb - off), &bars[0]);
    }
    loaded_bin = it.x;
    table_pending = true;
    __syncthreads();
    issue_gather(s_rows, it.z);
  }

  for (int item = i0; item < i1; ++item) {
    const int buf = (item - i0) & 1;
    const int* rows_ids = s_rows + buf * kT;
    const int bin = it.x, rows = it.z;
    const int gnode = a.level_base + bin;
    const int cb = __ldg(a.child_begin + gnode);
    const int cc = __ldg(a.child_count + gnode);
    // the next tile's record and patch ids, consumed once this tile is in TMEM
    const bool has_next = item + 1 < i1;
    const int4 nit = has_next ? item_at(a, item + 1) : make_int4(0, 0, 0, 0);
    const int nperm = (has_next && tid < nit.z) ? row_at(a, nit, tid) : 0;

    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int row = tid;
#pragma unroll
    for (int kc = 0; kc < KCH; ++kc) {
      // this thread's row, K chunk kc: tf32 hi / lo split in registers, staged to TMEM
      float hi[32], lo[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 v = *reinterpret_cast<const float4*>(raw + kc * (kT * 128u) + sw128_offset(row, c));
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hi[4 * c + q] = tf32_hi(x[q]);
          lo[4 * c + q] = x[q] - hi[4 * c + q];
        }
      }
      if (kc > 0) {  // the previous chunk's MMAs must have consumed the A columns
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1u;
        tc_fence_after();  // order the tcgen05.st below after the MMAs' completion
      }
      tmem_st32(tmem + lane_base + kColA, hi);
      tmem_st32(tmem + lane_base + kColA + 32, lo);
      tmem_wait_st();
      tc_fence_before();
      __syncthreads();
      if (kc == KCH - 1 && has_next) {
        // every row is in TMEM: the landing plane and the rows buffer are free
        s_rows[(buf ^ 1) * kT + tid] = tid < nit.z ? nperm : -1;
      }
      if (tid == 0) {
        if (kc == 0 && table_pending) {
          mbar_wait(&bars[0], tab_phase);
          tab_phase ^= 1u;
          table_pending = false;
        }
        tc_fence_after();
        const uint32_t bh = b_s + kc * (2u * npad * 128u);
        const uint32_t bl = bh + npad * 128u;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t ah = tmem + kColA + ks * 8;
          const uint32_t al = ah + 32;
          const uint32_t o = ks * 32u;
          if (kc == KCH - 1 && ks >= a.ks_last) break;   // zero padding on both operands
          mma_tf32_ts(tmem + kColAcc, ah, sw128_kmajor_desc(bh + o), idesc, (kc | ks) ? 1u : 0u);
          mma_tf32_ts(tmem + kColAcc, ah, sw128_kmajor_desc(bl + o), idesc, 1u);
          mma_tf32_ts(tmem + kColAcc, al, sw128_kmajor_desc(bh + o), idesc, 1u);
        }
        mma_commit(&bars[1]);
      }
      table_pending = false;
    }
    // launch the next tile's gather; it overlaps the MMAs and this tile's epilogue
    if (has_next) {
      __syncthreads();  // s_rows of the next tile visible
      issue_gather(s_rows + (buf ^ 1) * kT, nit.z);
    }
    __syncwarp();
    mbar_wait(&bars[1], mma_phase);
    mma_phase ^= 1u;
    tc_fence_after();
    // the MMAs are done with the table block: copy the leaf records out and
    // start the next tile's table load now, so it overlaps this epilogue
    const bool reload = has_next && nit.x != loaded_bin;
    if (reload) {
      if (last)
        for (int j = tid; j < 2 * npad; j += kThreads) s_leaf_info[j] = t_leaf[j];
      fence_proxy_async_smem();   // generic reads of the block before its async refill
      __syncthreads();
      if (tid == 0) {
        mbar_arrive_expect_tx(&bars[0], tb);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.table) + (size_t)nit.x * tb;
        for (uint32_t off = 0; off < tb; off += 65536u)
          bulk_g2s(btab + off, src + off, min(65536u, tb - off), &bars[0]);
      }
      table_pending = true;
      loaded_bin = nit.x;
    }
    const int* leaf_rec = reload ? s_leaf_info : t_leaf;

    int best = 0;
    float bestv = -1.f;
    tmem_abs_argmax(tmem + lane_base + kColAcc, (npad + 31) & ~31, npad, bestv, best);
    const int p = row < rows ? rows_ids[row] : -1;
    const bool valid = p >= 0;
    const int child = cb + best;
    int leaf_info = 0, leaf_cnt = 0;
    if (last && valid) {
      leaf_info = leaf_rec[best];
      leaf_cnt = leaf_rec[npad + best];
    }
    __syncthreads();   // every row's leaf record read before the next tile copies records again
    if (valid) {
      a.path_ws[(int64_t)p * a.L + a.level] = child;
      if (a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = child;
      if (a.next_counts) atomicAdd(&s_hist[best], 1);
      if (last) a.leaf_sel[p] = leaf_info;
      if (a.ip) {
        add_ip(a.ip, p, cc + leaf_cnt, cc);
      }
    }
    if (a.next_counts) {
      __syncthreads();
      for (int j = tid; j < cc; j += kThreads) {
        const int h = s_hist[j];
        if (h) atomicAdd(&a.next_counts[cb + j - a.next_base], h);
        s_hist[j] = 0;
      }
    }
    tc_fence_before();
    it = nit;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

template <int KCH>
cudaError_t launch_ts_kch(ScoreArgs s, int sms, cudaStream_t st) {
  const bool last = s.leaf_sel != nullptr;
  const uint32_t smem = ts_layout(KCH, s.npad, last).total;
  int cols = 32;
  while (cols < (int)kColAcc + s.npad) cols <<= 1;
  s.tmem_cols = cols;
  auto kern = score_ts_kernel<KCH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int by_smem = (int)((228 * 1024) / (smem + 1024));
  const int by_tmem = 512 / cols;
  const int per_sm = std::max(1, std::min(4, std::min(by_smem, by_tmem)));
  return launch_kernel(kern, sms * per_sm, kThreads, smem, st, true, s);
}

}  // namespace

bool score_ts_fits(int kchunks, int npad, bool last) {
  if (kchunks < 1 || kchunks > 4 || npad > 256) return false;
  return ts_layout(kchunks, npad, last).total <= 227 * 1024;
}

cudaError_t launch_score_ts(const ScoreArgs& s, int sms, cudaStream_t st) {
  switch (s.kchunks) {
    case 1: return launch_ts_kch<1>(s, sms, st);
    case 2: return launch_ts_kch<2>(s, sms, st);
    case 3: return launch_ts_kch<3>(s, sms, st);
    case 4: return launch_ts_kch<4>(s, sms, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace stmp
