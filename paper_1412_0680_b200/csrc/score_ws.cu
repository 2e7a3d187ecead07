// Warp-specialized, multi-stage tcgen05 scoring pass of the staged encoder.
//
// One persistent CTA per SM walks a contiguous range of (node, <=128-patch)
// work items with three roles connected by mbarriers:
//   warps 0-3  producers: gather the tile's residual rows with cp.async into a
//              ring of NS landing stages (SW128 K-major slots; the landed rows
//              become the tf32 "hi" plane in place), bulk-copy the node's
//              pre-split centroid table (TMA engine) into the stage's B slot,
//              then split hi/lo and publish the tile;
//   warp 8     MMA issuer: 3xTF32 tcgen05.mma (hi*hi + hi*lo + lo*hi) into one of
//              two TMEM accumulators, commits to the epilogue;
//   warps 4-7  epilogue: tcgen05.ld, one thread per patch row, argmax with the
//              reference tie rule, path / leaf / counters.
// NS-1 tiles of gathers are in flight while the current tile is split,
// multiplied and reduced, so the pass streams the residual at near memory speed.
// Semantics identical to score_tc_kernel (encode_staged.cu).
#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

namespace {

constexpr int kT = 128;          // patches per tile (UMMA M)
constexpr int kWsThreads = 288;  // 4 producer + 4 epilogue + 1 MMA warp

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void cp_async_wait_n(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

struct StageMeta {
  int bin, start, rows, cb, cc, pad0, pad1, pad2;
};

struct WsLayoutSmem {
  uint32_t raw, alo, btab, st_rows, st_meta, ep_rows, ep_leaf, ep_meta, hist, bars, tmem_slot, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) & ~(a - 1); }

__host__ __device__ inline WsLayoutSmem ws_layout(int kch, int npad, bool last, int ns) {
  WsLayoutSmem L{};
  const uint32_t plane = (uint32_t)kch * kT * 128u;
  const uint32_t tb = align_up(table_bytes(kch, npad, last), 1024u);
  uint32_t o = 0;
  L.raw = o; o += ns * plane;
  L.alo = o; o += plane;
  L.btab = o; o += ns * tb;
  L.st_rows = o; o += ns * kT * 4;
  L.st_meta = o; o += ns * sizeof(StageMeta);
  L.ep_rows = o; o += 2 * kT * 4;
  L.ep_leaf = o; o += 2 * 2 * 256 * 4;
  L.ep_meta = o; o += 2 * sizeof(StageMeta);
  L.hist = o; o += 256 * 4;
  L.bars = align_up(o, 8); o = L.bars + (4 + 2 + 2 + ns) * 8;
  L.tmem_slot = o; o += 16;
  L.total = o + 1024;  // alignment slack
  return L;
}

template <int KCH, int NS>
__global__ void __launch_bounds__(kWsThreads, 1) score_ws_kernel(ScoreArgs a) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  constexpr int F = 8 * KCH;                     // 16-B chunks per residual row
  constexpr uint32_t kPlane = KCH * kT * 128u;   // one [128 x ld] SW128 plane
  const int npad = a.npad;
  const bool last = a.leaf_sel != nullptr;
  const WsLayoutSmem Ly = ws_layout(KCH, npad, last, NS);
  const uint32_t tb = table_bytes(KCH, npad, last);
  const uint32_t tb_al = align_up(tb, 1024u);
  uint8_t* raw = base + Ly.raw;
  uint8_t* alo = base + Ly.alo;
  uint8_t* btab = base + Ly.btab;
  int* st_rows = reinterpret_cast<int*>(base + Ly.st_rows);
  StageMeta* st_meta = reinterpret_cast<StageMeta*>(base + Ly.st_meta);
  int* ep_rows = reinterpret_cast<int*>(base + Ly.ep_rows);
  int* ep_leaf = reinterpret_cast<int*>(base + Ly.ep_leaf);
  StageMeta* ep_meta = reinterpret_cast<StageMeta*>(base + Ly.ep_meta);
  int* s_hist = reinterpret_cast<int*>(base + Ly.hist);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + Ly.bars);
  uint64_t* ab_full = bars + 0;     // producers -> MMA: tile split and published
  uint64_t* mma_done = bars + 1;    // MMA -> producers: lo plane / stage slot free
  uint64_t* acc_full = bars + 4;    // [2] MMA -> epilogue
  uint64_t* acc_empty = bars + 6;   // [2] epilogue -> producers
  uint64_t* tab_full = bars + 8;    // [NS] table bulk copy landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + Ly.tmem_slot);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (warp == 8) tmem_alloc(tmem_slot, a.tmem_cols);
  if (tid == 0) {
    mbar_init(ab_full, 128);
    mbar_init(mma_done, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, 128);
    }
    for (int s = 0; s < NS; ++s) mbar_init(tab_full + s, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 256; i += kWsThreads) s_hist[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int num_items = *a.num_items;
  const int per = (num_items + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per;
  const int n = max(0, min(num_items, i0 + per) - i0);

  if (warp < 4) {
    // ============================ producers ============================
    // Per tile: (1) prepare tile jj+NS-1 -- its item record, patch ids and node
    // metadata are loaded into registers (loads in flight, nothing waits);
    // (2) wait for tile jj's rows, split them, publish; (3) launch tile
    // jj+NS-1's gather + table copy from the prepared registers.  The id
    // round trip overlaps the split instead of sitting on the critical path.
    const int pt = tid;
    constexpr int kSlots = F;  // e-slots per thread: e = pt + 128*k
    int rid[kSlots];
    int4 pit = make_int4(0, 0, 0, 0);
    int pcb = 0, pcc = 0;
    auto prepare = [&](int q) {
      pit = a.items[i0 + q];
#pragma unroll
      for (int k = 0; k < kSlots; ++k) {
        const int row = (pt + 128 * k) / F;
        rid[k] = row < pit.z ? a.perm[pit.y + row] : 0;
      }
      if (pt == 0) {
        const int gnode = a.level_base + pit.x;
        pcb = __ldg(a.child_begin + gnode);
        pcc = __ldg(a.child_count + gnode);
      }
    };
    auto launch = [&](int q) {
      const int s = q % NS;
      const uint32_t dst = smem_u32(raw + s * kPlane);
#pragma unroll
      for (int k = 0; k < kSlots; ++k) {
        const int e = pt + 128 * k;
        const int row = e / F;
        const int c = e - row * F;
        const bool ok = row < pit.z;
        if (c == 0 && ok) st_rows[s * kT + row] = rid[k];
        const uint32_t off = (uint32_t)(c >> 3) * (kT * 128u) + sw128_offset(row, c & 7);
        cp_async16(dst + off, a.R + (int64_t)rid[k] * a.ld + 4 * c, ok ? 16u : 0u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (pt == 0) {
        StageMeta m;
        m.bin = pit.x; m.start = pit.y; m.rows = pit.z;
        m.cb = pcb; m.cc = pcc;
        m.pad0 = m.pad1 = m.pad2 = 0;
        st_meta[s] = m;
        mbar_arrive_expect_tx(tab_full + s, tb);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.table) + (size_t)pit.x * tb;
        for (uint32_t off = 0; off < tb; off += 65536u)
          bulk_g2s(btab + s * tb_al + off, src + off, min(65536u, tb - off), tab_full + s);
      }
    };
    for (int q = 0; q < NS - 1 && q < n; ++q) {
      prepare(q);
      launch(q);
    }
    for (int jj = 0; jj < n; ++jj) {
      const int s = jj % NS;
      const int q = jj + NS - 1;
      if (q < n) prepare(q);
      if (jj >= 1) mbar_wait(mma_done, (uint32_t)((jj - 1) & 1));
      // groups committed so far: tiles 0 .. min(n, jj+NS-1)-1
      cp_async_wait_n(min(NS - 2, n - 1 - jj));
      named_bar(1, 128);  // every producer's copies of tile jj have landed
      const int acc = jj & 1;
      if (jj >= 2) mbar_wait(acc_empty + acc, (uint32_t)(((jj >> 1) - 1) & 1));
      // split: hi in place (tf32 truncation), lo into the single lo plane
      uint8_t* hs = raw + s * kPlane;
#pragma unroll 4
      for (int e = pt; e < kT * F; e += 128) {
        const int row = e / F;
        const int c = e - row * F;
        const uint32_t off = (uint32_t)(c >> 3) * (kT * 128u) + sw128_offset(row, c & 7);
        float4* ph = reinterpret_cast<float4*>(hs + off);
        const float4 v = *ph;
        float4 h, l;
        h.x = tf32_hi(v.x); h.y = tf32_hi(v.y); h.z = tf32_hi(v.z); h.w = tf32_hi(v.w);
        l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
        *ph = h;
        *reinterpret_cast<float4*>(alo + off) = l;
      }
      // hand the tile's bookkeeping to the epilogue slot
      const StageMeta m = st_meta[s];
      if (pt < m.rows) ep_rows[acc * kT + pt] = st_rows[s * kT + pt];
      if (pt == 0) ep_meta[acc] = m;
      if (last) {
        mbar_wait(tab_full + s, (uint32_t)((jj / NS) & 1));
        const int* li = reinterpret_cast<const int*>(btab + s * tb_al + (size_t)KCH * 2 * npad * 128);
        for (int i = pt; i < 2 * npad; i += 128) ep_leaf[acc * 512 + i] = li[i];
      }
      fence_proxy_async_smem();
      mbar_arrive(ab_full);
      // slot (jj-1) % NS is free (MMA jj-1 done): launch the prepared tile into it
      if (q < n) {
        named_bar(1, 128);  // every producer has read st_meta / st_rows of tile jj
        launch(q);
      }
    }
  } else if (warp == 8) {
    // ============================ MMA issuer ============================
    if ((tid & 31) == 0) {
      const uint32_t idesc = idesc_tf32(kT, npad);
      const uint32_t alo_s = smem_u32(alo);
      for (int jj = 0; jj < n; ++jj) {
        const int s = jj % NS;
        const int acc = jj & 1;
        mbar_wait(ab_full, (uint32_t)(jj & 1));
        mbar_wait(tab_full + s, (uint32_t)((jj / NS) & 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * npad);
        const uint32_t ahi_s = smem_u32(raw + s * kPlane);
        const uint32_t b_s = smem_u32(btab + s * tb_al);
#pragma unroll
        for (int kc = 0; kc < KCH; ++kc) {
          const uint32_t ah = ahi_s + kc * (kT * 128u);
          const uint32_t al = alo_s + kc * (kT * 128u);
          const uint32_t bh = b_s + kc * (2u * npad * 128u);
          const uint32_t bl = bh + npad * 128u;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t o = ks * 32u;
            mma_tf32(d, sw128_kmajor_desc(ah + o), sw128_kmajor_desc(bh + o), idesc, (kc | ks) ? 1u : 0u);
            mma_tf32(d, sw128_kmajor_desc(ah + o), sw128_kmajor_desc(bl + o), idesc, 1u);
            mma_tf32(d, sw128_kmajor_desc(al + o), sw128_kmajor_desc(bh + o), idesc, 1u);
          }
        }
        mma_commit(mma_done);
        mma_commit(acc_full + acc);
      }
    }
    __syncwarp();
  } else {
    // ============================ epilogue ============================
    const int et = tid - 128;          // patch row of the tile
    const int quad = warp & 3;          // TMEM lane quadrant of this warp
    for (int jj = 0; jj < n; ++jj) {
      const int acc = jj & 1;
      mbar_wait(acc_full + acc, (uint32_t)((jj >> 1) & 1));
      tc_fence_after();
      const StageMeta m = ep_meta[acc];
      int best = 0;
      float bestv = -1.f;
      for (int col0 = 0; col0 < npad; col0 += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * npad + col0), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float mv = fabsf(v[j]);
          if (col0 + j < m.cc && mv > bestv) {
            bestv = mv;
            best = col0 + j;
          }
        }
      }
      tc_fence_before();
      const bool valid = et < m.rows;
      const int p = valid ? ep_rows[acc * kT + et] : 0;
      const int child = m.cb + best;
      int leaf_info = 0, leaf_cnt = 0;
      if (last && valid) {
        leaf_info = ep_leaf[acc * 512 + best];
        leaf_cnt = ep_leaf[acc * 512 + npad + best];
      }
      if (valid) {
        a.path_ws[(int64_t)p * a.L + a.level] = child;
        if (a.path_out) a.path_out[((int64_t)p * a.K + a.count[p]) * a.L + a.level] = child;
        if (a.next_counts) atomicAdd(&s_hist[best], 1);
        if (last) a.leaf_sel[p] = leaf_info;
        if (a.ip) {  // ScoreCounter: cc centroids at this level (+ the leaf atoms)
          add_ip(a.ip, p, m.cc + leaf_cnt, m.cc);
        }
      }
      // the tile's bookkeeping has been consumed: release the slot
      mbar_arrive(acc_empty + acc);
      if (a.next_counts) {
        named_bar(2, 128);
        for (int j = et; j < m.cc; j += 128) {
          const int h = s_hist[j];
          if (h) atomicAdd(&a.next_counts[m.cb + j - a.next_base], h);
          s_hist[j] = 0;
        }
        named_bar(2, 128);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, a.tmem_cols);
}

template <int KCH, int NS>
cudaError_t launch_ws(const ScoreArgs& s, int sms, cudaStream_t st) {
  const bool last = s.leaf_sel != nullptr;
  const uint32_t smem = ws_layout(KCH, s.npad, last, NS).total;
  cudaError_t e = cudaFuncSetAttribute(score_ws_kernel<KCH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel(score_ws_kernel<KCH, NS>, sms, kWsThreads, (size_t)smem, st, true, s);
}

template <int KCH>
cudaError_t launch_ws_kch(const ScoreArgs& s, int sms, cudaStream_t st) {
  const bool last = s.leaf_sel != nullptr;
  constexpr uint32_t kMax = 227 * 1024;
  if (ws_layout(KCH, s.npad, last, 4).total <= kMax) return launch_ws<KCH, 4>(s, sms, st);
  if (ws_layout(KCH, s.npad, last, 3).total <= kMax) return launch_ws<KCH, 3>(s, sms, st);
  if (ws_layout(KCH, s.npad, last, 2).total <= kMax) return launch_ws<KCH, 2>(s, sms, st);
  return cudaErrorNotSupported;
}

}  // namespace

bool score_ws_fits(int kchunks, int npad, bool last) {
  if (kchunks < 1 || kchunks > 4 || npad > 256) return false;
  return ws_layout(kchunks, npad, last, 2).total <= 227 * 1024;
}

cudaError_t launch_score_ws(const ScoreArgs& s, int sms, cudaStream_t st) {
  // TMEM: two accumulators of npad columns
  switch (s.kchunks) {
    case 1: return launch_ws_kch<1>(s, sms, st);
    case 2: return launch_ws_kch<2>(s, sms, st);
    case 3: return launch_ws_kch<3>(s, sms, st);
    case 4: return launch_ws_kch<4>(s, sms, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace stmp
