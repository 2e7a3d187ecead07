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
//                           patch row), count the winners for the next level;
//   update: MP step or OMP incremental-Cholesky refit, residual rebuilt and
//           written once (encode_update.cu).
// Reference semantics are the same as encode_fused.cu (see its header).
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "sm100.cuh"
#include "staged.cuh"

namespace stmp {

using namespace sm100;

int g_pdl = 1;          // programmatic dependent launch between staged kernels
int g_root_direct = 1;  // root pass over the batch in patch order (no scan / scatter at level 0)
int g_update_omp8 = 1;  // 1: lockstep OMP update (update_omp8_kernel, encode_update.cu)
int g_update_wide = 1;  // one-CTA-per-patch OMP update for rows wider than 160 floats
int g_score_ws = 2;  // 2: A operand in TMEM, whole node table in shared memory (default); 3: streamed table

namespace {

constexpr int kTile = 128;          // patches per work item (= UMMA M)
constexpr int kScoreThreads = 128;  // 4 warps: warp w owns TMEM lanes 32w..32w+31


// ------------------------------------------------------------------ scan (one CTA)
constexpr int kScanThreads = 1024;
constexpr int kScanSmemBins = 3072;   // 36 KB of dynamic shared memory (+ static CUB storage < 48 KB)
inline size_t scan_smem(int nbins) { return nbins <= kScanSmemBins ? (size_t)12 * nbins : 0; }

// `stripes` (root level only): kRootStripes partial counts of bin 0, folded
// into counts[0] and reset here.
__global__ void __launch_bounds__(kScanThreads) scan_kernel(int* counts, int nbins, int* offsets,
                                                             int4* items, int* num_items,
                                                             int* tile_off, int* cursor, int* stripes) {
  pdl_enter();
  using Scan = cub::BlockScan<int, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry[2];
  __shared__ int root_total;
  // bins' tile offsets / row offsets / counts, kept in shared memory for the item
  // search when they fit (dynamic size 12 * nbins, else 0)
  extern __shared__ int s_bins[];
  const bool in_smem = nbins <= kScanSmemBins;
  int* s_toff = s_bins;
  int* s_off = s_bins + nbins;
  int* s_cnt = s_bins + 2 * nbins;
  if (threadIdx.x == 0) carry[0] = carry[1] = root_total = 0;
  __syncthreads();
  if (stripes != nullptr) {
    if (threadIdx.x < kRootStripes) {
      int v = stripes[threadIdx.x];
      stripes[threadIdx.x] = 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      if ((threadIdx.x & 31) == 0) atomicAdd(&root_total, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) counts[0] += root_total;
    __syncthreads();
  }
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
      cursor[b] = 0;
      if (in_smem) {
        s_off[b] = carry[0] + pre_c;
        s_toff[b] = carry[1] + pre_t;
        s_cnt[b] = c;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] += tot_c;
      carry[1] += tot_t;
    }
    __syncthreads();
  }
  const int total_tiles = carry[1];
  const int* toff = in_smem ? s_toff : tile_off;
  const int* offs = in_smem ? s_off : offsets;
  const int* cnts = in_smem ? s_cnt : counts;
  // one item per tile: binary-search the bin owning tile i
  for (int i = threadIdx.x; i < total_tiles; i += kScanThreads) {
    int lo = 0, hi = nbins - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (toff[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int k = i - toff[lo];
    const int c = cnts[lo];
    items[i] = make_int4(lo, offs[lo] + k * kTile, min(kTile, c - k * kTile), 0);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += kScanThreads) counts[b] = 0;
  if (threadIdx.x == 0) *num_items = total_tiles;
}

// ------------------------------------------------------------------ scatter
// perm[offsets[bin] + slot] = p, slots claimed with one atomic per (warp, bin).
__global__ void scatter_kernel(int64_t N, const int* active, const int* path_ws, int L, int level,
                               int level_base, const int* offsets, int* cursor, int* perm) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool act = p < N && active[p];
  const int bin = act ? (level == 0 ? 0 : path_ws[p * L + level - 1] - level_base) : -1;
  const unsigned peers = __match_any_sync(kFull, bin);
  if (act) {
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cursor[bin], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    perm[offsets[bin] + base + __popc(peers & ((1u << lane) - 1u))] = (int)p;
  }
}

constexpr int kScatterThreads = 512;

// Scan fused into the scatter (levels >= 1 with few bins): every CTA scans the
// level's bin counts (written by the previous level's score pass) in shared
// memory, so no separate one-CTA scan launch sits between the two passes.  The
// CTAs also write the score pass's work items (one per 128-patch tile, bins in
// order) and zero the counters of the other iteration parity, which were last
// read one iteration ago and are produced again by the next iteration's score
// passes.  All loads of a patch are issued together (no active -> path chain).
constexpr int kScanRun = 8;   // bins per thread in the block scan: nbins <= 512 * 8
template <int kScatterPer>
__global__ void __launch_bounds__(kScatterThreads) scatter_scan_kernel(
    int64_t N, const int* active, const int* path_ws, int L, int level, int level_base, int nbins,
    const int* counts, int* cursor, int* zero_counts, int* zero_cursor, int* perm, int4* items,
    int* num_items) {
  pdl_enter();
  using Scan = cub::BlockScan<int, kScatterThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_total_tiles;
  extern __shared__ int sh[];  // [nbins] local counts | base | bin offsets | tile offsets
  int* s_loc = sh;
  int* s_base = sh + nbins;
  int* s_off = sh + 2 * nbins;
  int* s_toff = sh + 3 * nbins;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t p0 = (int64_t)blockIdx.x * kScatterThreads * kScatterPer + tid;
  int bins[kScatterPer], local[kScatterPer];
#pragma unroll
  for (int i = 0; i < kScatterPer; ++i) {
    const int64_t p = p0 + (int64_t)i * kScatterThreads;
    const bool in = p < N;
    const int act = in ? __ldg(active + p) : 0;
    const int pv = in ? __ldg(path_ws + p * L + level - 1) : level_base;
    bins[i] = act ? pv - level_base : -1;
  }
  const int b0 = tid * kScanRun;
  int cv[kScanRun];
  int csum = 0, tsum = 0;
#pragma unroll
  for (int j = 0; j < kScanRun; ++j) {
    cv[j] = b0 + j < nbins ? __ldg(counts + b0 + j) : 0;
    csum += cv[j];
    tsum += (cv[j] + kTile - 1) / kTile;
  }
  for (int b = blockIdx.x * kScatterThreads + tid; b < nbins; b += gridDim.x * kScatterThreads) {
    zero_counts[b] = 0;
    zero_cursor[b] = 0;
  }
  for (int b = tid; b < nbins; b += kScatterThreads) s_loc[b] = 0;
  int cpre, tpre, ttot;
  Scan(tmp).ExclusiveSum(csum, cpre);
  __syncthreads();
  Scan(tmp).ExclusiveSum(tsum, tpre, ttot);
#pragma unroll
  for (int j = 0; j < kScanRun; ++j) {
    if (b0 + j < nbins) {
      s_off[b0 + j] = cpre;
      s_toff[b0 + j] = tpre;
    }
    cpre += cv[j];
    tpre += (cv[j] + kTile - 1) / kTile;
  }
  if (tid == 0) s_total_tiles = ttot;
  __syncthreads();
  // one shared-memory atomic per (warp, bin)
#pragma unroll
  for (int i = 0; i < kScatterPer; ++i) {
    const unsigned peers = __match_any_sync(kFull, bins[i]);
    const int leader = __ffs(peers) - 1;
    int b = 0;
    if (lane == leader && bins[i] >= 0) b = atomicAdd(&s_loc[bins[i]], __popc(peers));
    b = __shfl_sync(kFull, b, leader);
    local[i] = b + __popc(peers & ((1u << lane) - 1u));
  }
  __syncthreads();
  for (int b = tid; b < nbins; b += kScatterThreads) {
    const int c = s_loc[b];
    s_base[b] = c ? s_off[b] + atomicAdd(&cursor[b], c) : 0;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScatterPer; ++i) {
    if (bins[i] >= 0) perm[s_base[bins[i]] + local[i]] = (int)(p0 + (int64_t)i * kScatterThreads);
  }
  // work items of the score pass: tile i -> (bin, first slot, rows)
  const int total = s_total_tiles;
  for (int i = blockIdx.x * kScatterThreads + tid; i < total; i += gridDim.x * kScatterThreads) {
    int lo = 0, hi = nbins - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_toff[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int k = i - s_toff[lo];
    const int c = (lo + 1 < nbins ? s_off[lo + 1] : s_off[lo] + __ldg(counts + lo)) - s_off[lo];
    items[i] = make_int4(lo, s_off[lo] + k * kTile, min(kTile, c - k * kTile), 0);
  }
  if (blockIdx.x == 0 && tid == 0) *num_items = total;
}

// Root level: a single bin holding every active patch.  One atomic per CTA.
__global__ void __launch_bounds__(256) scatter_root_kernel(int64_t N, const int* active, const int* offsets,
                                                           int* cursor, int* perm) {
  pdl_enter();
  __shared__ int warp_off[8];
  __shared__ int base;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool act = p < N && active[p];
  const unsigned m = __ballot_sync(kFull, act);
  if (lane == 0) warp_off[warp] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const int c = warp_off[w];
      warp_off[w] = s;
      s += c;
    }
    base = s ? atomicAdd(cursor, s) : 0;
  }
  __syncthreads();
  if (act) perm[offsets[0] + base + warp_off[warp] + __popc(m & ((1u << lane) - 1u))] = (int)p;
}

// Bucketing of the active patches by their level-(l-1) node for the score pass
// of level l >= 1: the scan fused into the scatter (counters double-buffered by
// iteration parity), or for more bins than one CTA scans, scan + scatter.
cudaError_t launch_level_scatter(int64_t N, const int* active, const int* path_ws, int L, int l, int level_base,
                                 int nb, int* counts_in, int* cursor_in, int* counts_next, int* cursor_next,
                                 int* offsets, int* tile_off, int* cursor, int* perm, int4* items, int* num_items,
                                 int sms, cudaStream_t st) {
  cudaError_t e;
  if (nb <= kScanRun * kScatterThreads) {
    const int per = N >= (int64_t)sms * kScatterThreads * 8 ? 8 : N >= (int64_t)sms * kScatterThreads * 2 ? 2 : 1;
    const int grid = (int)((N + kScatterThreads * per - 1) / (kScatterThreads * per));
    auto k = per == 8 ? scatter_scan_kernel<8> : per == 2 ? scatter_scan_kernel<2> : scatter_scan_kernel<1>;
    const size_t smem = (size_t)nb * 16;
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return e;
    return launch_kernel(k, grid, kScatterThreads, smem, st, true, N, active, path_ws, L, l, level_base, nb,
                         (const int*)counts_in, cursor_in, counts_next, cursor_next, perm, items, num_items);
  }
  e = launch_kernel(scan_kernel, 1, kScanThreads, scan_smem(nb), st, true, counts_in, nb, offsets, items, num_items,
                    tile_off, cursor, (int*)nullptr);
  if (e != cudaSuccess) return e;
  return launch_kernel(scatter_kernel, (int)((N + 255) / 256), 256, 0, st, true, N, active, path_ws, L, l, level_base,
                       (const int*)offsets, cursor, perm);
}

}  // namespace

size_t score_smem_bytes(int kchunks, int npad) {
  return 1024 + (size_t)kchunks * kTile * 128 * 2 + table_bytes(kchunks, npad, true) + 16 + 16 + 16 +
         (2 * kTile + 256) * 4;
}

bool staged_supported(const DictHandle* d, const TreeHandle* t, int K, int method) {
  if (method != kMethodMP && method != kMethodOMP) return false;
  UpdateCfg uc;
  if (!update_config(d->ld, K, uc)) return false;
  if (t == nullptr) return d->m < (1ll << 31) && K <= 64;   // exhaustive: exact_scan.cu
  if (t->staged_tables.empty()) return false;
  if (K > 64) return false;
  return true;
}

// Per-node score tables on the device: for every node of one level, its
// children's centroid rows split into tf32 hi / lo, laid out [kchunk][hi|lo]
// [npad rows x 128 B] SW128 (the UMMA K-major B operand), then for the last
// level npad leaf records {single leaf atom or -1 - leaf node} and npad leaf
// atom counts (pursuit.py:155-162).  One CTA per node; the block is pre-zeroed.
__global__ void __launch_bounds__(256) table_kernel(const float* __restrict__ cent, int ld, const int* child_begin,
                                                    const int* child_count, const int* leaf_atom, int64_t level_base,
                                                    int kch, int npad, int last, float* __restrict__ out) {
  const int64_t v = level_base + blockIdx.x;
  float* blk = out + (size_t)blockIdx.x * (table_bytes(kch, npad, last != 0) / 4);
  const int cb = child_begin[v], cc = child_count[v];
  const int width = 32 * kch;
  for (int e = threadIdx.x; e < cc * width; e += blockDim.x) {
    const int j = e / width, col = e - j * width;
    const float val = cent[(int64_t)(cb + j) * ld + col];
    const float hi = sm100::tf32_hi(val);
    const int kc = col >> 5, q = col & 31;
    const uint32_t off = sm100::sw128_offset((uint32_t)j, (uint32_t)(q >> 2)) / 4 + (q & 3);
    float* plane = blk + (size_t)kc * 2 * npad * 32;
    plane[off] = hi;
    plane[(size_t)npad * 32 + off] = val - hi;
  }
  if (last) {
    int32_t* info = reinterpret_cast<int32_t*>(blk + (size_t)kch * 2 * npad * 32);
    int32_t* cnt = info + npad;
    for (int j = threadIdx.x; j < cc; j += blockDim.x) {
      const int child = cb + j;
      const int lc = child_count[child];
      info[j] = lc == 1 ? leaf_atom[child_begin[child]] : -1 - child;
      cnt[j] = lc;
    }
  }
}

bool build_staged_tables(TreeHandle* t, const int32_t* child_begin, const int32_t* child_count,
                         const float* centroids, const int32_t* leaf_atom, cudaStream_t st,
                         std::string* err) {
  UpdateCfg uc;
  if (!update_config(t->ld, 1, uc)) return false;
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
    // whole-table kernels need the node table in shared memory; the streamed one does not
    if (score_smem_bytes(kch, levels[l].npad) > 227 * 1024 && !score_st_fits(kch, levels[l].npad, l == L - 1))
      return false;
  }
  std::vector<float*> tables(L, nullptr);
  (void)child_begin; (void)centroids; (void)leaf_atom;
  for (int l = 0; l < L; ++l) {
    const int npad = levels[l].npad;
    const bool last = l == L - 1;
    const int64_t nodes = t->level_offsets[l + 1] - t->level_offsets[l];
    const size_t bytes = (size_t)table_bytes(kch, npad, last) * nodes;
    cudaError_t e = cudaMalloc(&tables[l], bytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(tables[l], 0, bytes, st);
    if (e == cudaSuccess) {
      table_kernel<<<(unsigned)nodes, 256, 0, st>>>(t->cent, t->ld, t->child_begin, t->child_count, t->leaf_atom,
                                                    t->level_offsets[l], kch, npad, last ? 1 : 0, tables[l]);
      note_launch();
      e = cudaGetLastError();
    }
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

bool ensure_s16_tables(TreeHandle* t, cudaStream_t st) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (t->s16_tried) return !t->s16_tables.empty();
  t->s16_tried = true;
  std::vector<uint8_t*> tabs(t->levels, nullptr);
  bool good = true;
  for (int l = 0; l < t->levels && good; ++l)
    good = score_s16_fits(t->ld, t->staged_levels[l].npad) && (tabs[l] = build_s16_table(t, l, st)) != nullptr;
  if (!good) {
    for (uint8_t* p : tabs) cudaFree(p);
    cudaGetLastError();
    return false;
  }
  t->s16_tables = tabs;
  return true;
}

void free_staged_tables(TreeHandle* t) {
  for (uint8_t* p : t->s16_tables) cudaFree(p);
  t->s16_tables.clear();
  for (float* p : t->staged_tables) cudaFree(p);
  t->staged_tables.clear();
  t->staged_levels.clear();
}

namespace {

struct WsLayout {
  size_t total = 0;
  size_t R, Xpad, tol, active, perm, path_ws, leaf_sel, Lf, yv, S_ws, c_ws, counts, offsets, tile_off, cursor, items,
      num_items, cursor2;
  // Gram path only
  bool gram = false;
  size_t xn2 = 0, e_ws = 0, s0 = 0, corr = 0;
  // half-precision rows of the Gram path's level passes (score_sh.cu)
  bool half = false;
  size_t x16 = 0, inv_scale = 0, qerr = 0;
};

WsLayout layout(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method,
                std::vector<int64_t>* bin_off_out, int64_t* maxbins_out) {
  // exhaustive selection (t == nullptr): one pseudo level holding the single root bin
  const int L = t ? t->levels : 0;
  const int LB = t ? L : 1;
  int64_t maxbins = 1;
  std::vector<int64_t> bin_off(LB + 1, 0);
  for (int l = 0; l < LB; ++l) {
    const int64_t b = t ? t->level_offsets[l + 1] - t->level_offsets[l] : 1;
    maxbins = std::max(maxbins, b);
    bin_off[l + 1] = bin_off[l] + b;
  }
  WsLayout w;
  auto add = [&](size_t bytes) {
    const size_t at = w.total;
    w.total += (bytes + 255) & ~(size_t)255;
    return at;
  };
  w.R = add((size_t)N * d->ld * 4);
  w.Xpad = method == kMethodOMP ? add((size_t)N * d->ld * 4) : 0;
  w.tol = add((size_t)N * 4);
  w.active = add((size_t)N * 4);
  w.perm = add((size_t)N * 4);
  w.path_ws = add((size_t)N * L * 4);
  w.leaf_sel = add((size_t)N * 4);
  w.Lf = add((size_t)N * K * (K + 1) / 2 * 4);
  w.yv = add((size_t)N * K * 4);
  w.S_ws = add((size_t)N * K * 4);
  w.c_ws = add((size_t)N * K * 4);
  // bin counters, one set per iteration parity (scatter_scan_kernel), then the root stripes
  w.counts = add((size_t)(2 * bin_off[LB] + kRootStripes) * 4);
  w.cursor2 = add((size_t)2 * bin_off[LB] * 4);
  w.offsets = add((size_t)(maxbins + 1) * 4);
  w.tile_off = add((size_t)(maxbins + 1) * 4);
  w.cursor = add((size_t)(maxbins + 1) * 4);
  w.items = add((size_t)(N / kTile + maxbins + 2) * 16);
  w.num_items = add(16);
  if (t && gram_path_supported(d, t, K, method)) {
    w.gram = true;
    w.xn2 = add((size_t)N * 8);
    w.e_ws = add((size_t)N * 8);
    w.s0 = add((size_t)N * t->root_children * 4);
    w.corr = add((size_t)N * ((t->max_children + 3) & ~3) * 4);   // rows of whole float4
    // reserved whenever the shapes allow it (the option is read at encode time)
    w.half = true;
    for (int l = 1; l < L; ++l) w.half = w.half && score_sh_fits(d->ld, t->staged_levels[l].npad);
    if (w.half) {
      w.x16 = add((size_t)N * d->ld * 2);
      w.inv_scale = add((size_t)N * 4);
      w.qerr = add((size_t)N * 4);
    }
  }
  if (bin_off_out) *bin_off_out = bin_off;
  if (maxbins_out) *maxbins_out = maxbins;
  return w;
}

}  // namespace

size_t staged_workspace_bytes(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method) {
  return layout(d, t, N, K, method, nullptr, nullptr).total;
}

cudaError_t run_staged(const DictHandle* d, const TreeHandle* t, const float* X, int64_t N,
                       int64_t ldx, int K, int method, float tol_abs, int32_t* idx, float* coef,
                       int32_t* count, float* resnorm, int32_t* path, int32_t* ip, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  std::vector<int64_t> bin_off;
  int64_t maxbins = 1;
  const WsLayout w = layout(d, t, N, K, method, &bin_off, &maxbins);
  if (ws == nullptr || ws_bytes < w.total) return cudaErrorInvalidValue;
  const int L = t ? t->levels : 0;
  const int LB = t ? L : 1;   // bin levels (exhaustive: the root bin only)
  uint8_t* b = static_cast<uint8_t*>(ws);
  float* R = (float*)(b + w.R);
  float* Xpad = method == kMethodOMP ? (float*)(b + w.Xpad) : nullptr;
  float* tol = (float*)(b + w.tol);
  int* active = (int*)(b + w.active);
  int* perm = (int*)(b + w.perm);
  int* path_ws = (int*)(b + w.path_ws);
  int* leaf_sel = (int*)(b + w.leaf_sel);
  float* Lf = (float*)(b + w.Lf);
  float* yv = (float*)(b + w.yv);
  int* S_ws = (int*)(b + w.S_ws);
  float* c_ws = (float*)(b + w.c_ws);
  int* counts = (int*)(b + w.counts);
  int* offsets = (int*)(b + w.offsets);
  int* tile_off = (int*)(b + w.tile_off);
  int* cursor = (int*)(b + w.cursor);
  int4* items = (int4*)(b + w.items);
  int* num_items = (int*)(b + w.num_items);

  int* stripes = counts + 2 * bin_off[LB];
  int* cursor2 = (int*)(b + w.cursor2);
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)(2 * bin_off[LB] + kRootStripes) * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cursor2, 0, (size_t)2 * bin_off[LB] * 4, st);
  if (e != cudaSuccess) return e;
  // counters written by the score passes of iteration `it` (and read by its scatters)
  auto counts_of = [&](int it_) { return counts + (it_ & 1) * bin_off[LB]; };
  auto cursor_of = [&](int it_) { return cursor2 + (it_ & 1) * bin_off[LB]; };

  // Gram path: no residual in HBM (gram_path.cu); falls back to the residual
  // pipeline below when the pair tables cannot be built
  const bool gram = w.gram && ensure_pair_tables(const_cast<TreeHandle*>(t), d, st);

  UpdateCfg uc;
  update_config(d->ld, K, uc);
  UpdateArgs u{};
  u.X = X; u.ldx = ldx; u.n = d->n; u.R = R; u.ld = d->ld;
  u.X2 = Xpad; u.ld2 = d->ld;  // OMP rebuilds r from this padded copy of x
  u.atoms = d->atoms; u.child_begin = t ? t->child_begin : nullptr; u.child_count = t ? t->child_count : nullptr;
  u.leaf_atom = t ? t->leaf_atom : nullptr; u.L = L; u.path_ws = path_ws; u.K = K; u.method = method;
  u.tol_abs = tol_abs; u.idx = idx; u.coef = coef; u.count = count; u.resnorm = resnorm;
  u.ip = ip; u.path_out = path; u.Lf = Lf; u.yv = yv; u.tol = tol; u.active = active;
  u.root_count = stripes; u.N = N; u.S_ws = S_ws; u.c_ws = c_ws; u.leaf_sel = leaf_sel;
  // lockstep OMP update (update_omp8_kernel): K <= 8 with rows of <= 160 floats or K <= 16 with <= 64
  const bool lockstep = method == kMethodOMP && lockstep_lanes(d->ld, K) != 0 && g_update_omp8;
  u.m = d->m;
  // stage the support atoms in shared memory when the patch groups fit comfortably
  u.cache_atoms = update_smem_bytes(uc, K, d->ld, true) <= 96 * 1024 ? 1 : 0;

  const int gpb = 128 / uc.G;
  const int ublocks = (int)((N + gpb - 1) / gpb);
  // When the caller's rows are already padded (n == ld, contiguous) they serve
  // directly as the iteration-0 residual and as the x of the OMP rebuild;
  // otherwise init writes a padded copy into R (and Xpad for OMP).
  const bool direct = ldx == d->ld && d->n == d->ld;
  {
    UpdateArgs ui = u;
    if (direct) { ui.R = nullptr; ui.X2 = nullptr; }
    if (gram) {   // ||x||^2 for the Gram path's residual norms; no OMP rebuild copy
      ui.xn2 = (double*)(b + w.xn2);
      ui.e_ws = (double*)(b + w.e_ws);
      ui.X2 = nullptr;
      // level passes on fp16 rows (score_sh.cu): init writes the fp16 copy in the same pass over x
      if (w.half && g_half_scores != 0 && (int)t->half_tables.size() == L) {
        ui.x16 = (uint16_t*)(b + w.x16);
        ui.inv_scale = (float*)(b + w.inv_scale);
        ui.qerr = (float*)(b + w.qerr);
      }
    }
    if ((e = launch_init(uc, ui, ublocks, st)) != cudaSuccess) return e;
  }
  if (direct && method == kMethodOMP) u.X2 = X;
  const float* R0 = direct ? X : R;

  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int scatter_blocks = (int)((N + 255) / 256);
  const size_t usmem = update_smem_bytes(uc, K, d->ld, u.cache_atoms != 0);
  const bool wide = method == kMethodOMP && !lockstep && g_update_wide && wide_update_cpt(d->ld) != 0;
  // the root bin holds every active patch: its pass can walk the batch in patch
  // order (inactive rows skipped) instead of compacting them (score_ts / score_st /
  // exact_scan only)
  const bool root_direct = g_root_direct != 0;
  if (root_direct) u.root_count = nullptr;
  if (gram) {
    double* xn2 = (double*)(b + w.xn2);
    double* e_ws = (double*)(b + w.e_ws);
    float* s0 = (float*)(b + w.s0);
    GramArgs ga{};
    ga.N = N; ga.K = K; ga.L = L; ga.leaf_sel = leaf_sel;
    ga.gram = t->pair_tables[L - 1]; ga.gram_w = t->pair_width[L - 1]; ga.leaf_pos = t->leaf_pos;
    ga.root_tab = t->pair_tables[0]; ga.s0 = s0; ga.root_w = t->root_children;
    ga.root_cb = (int)t->level_offsets[1];
    ga.path_ws = path_ws; ga.path_out = path; ga.S_ws = S_ws; ga.c_ws = c_ws; ga.yv = yv;
    ga.Lf = Lf; ga.e_ws = e_ws; ga.xn2 = xn2; ga.tol = tol; ga.active = active; ga.idx = idx; ga.coef = coef;
    ga.count = count; ga.resnorm = resnorm; ga.ip = ip;
    ga.xr = R0; ga.atoms = d->atoms; ga.cent = t->cent; ga.ld = d->ld; ga.rho = 1e-2f; ga.recheck_rel = 1e-5f;
    // level passes on fp16 rows (score_sh.cu) when the tree carries the fp16 piece tables (init wrote x16)
    const bool half = w.half && g_half_scores != 0 && (int)t->half_tables.size() == L;
    uint16_t* x16 = half ? (uint16_t*)(b + w.x16) : nullptr;
    float* inv_scale = half ? (float*)(b + w.inv_scale) : nullptr;
    float* qerr = half ? (float*)(b + w.qerr) : nullptr;
    for (int it = 0; it < K; ++it) {
      for (int l = it == 0 ? 0 : 1; l < L; ++l) {
        const StagedLevel& lv = t->staged_levels[l];
        const int nb = (int)(t->level_offsets[l + 1] - t->level_offsets[l]);
        if (l > 0 &&
            (e = launch_level_scatter(N, active, path_ws, L, l, (int)t->level_offsets[l], nb,
                                      counts_of(it) + bin_off[l], cursor_of(it) + bin_off[l],
                                      counts_of(it + 1) + bin_off[l], cursor_of(it + 1) + bin_off[l], offsets,
                                      tile_off, cursor, perm, items, num_items, sms, st)) != cudaSuccess)
          return e;
#ifndef STMP_GRAM_CORR_PRE
#define STMP_GRAM_CORR_PRE 1
#endif
        float* corr_pre = STMP_GRAM_CORR_PRE && l > 0 && it > 0 ? (float*)(b + w.corr) : nullptr;
        if (corr_pre != nullptr &&
            (e = launch_gram_corr(N, active, path_ws, L, l, t->child_begin, t->child_count,
                                  (int)t->level_offsets[l + 1], t->pair_tables[l], t->pair_width[l], S_ws, c_ws, K,
                                  it, corr_pre, (t->max_children + 3) & ~3, st)) != cudaSuccess)
          return e;
        ScoreArgs s{};
        s.R = R0; s.ld = d->ld; s.nrows = N; s.perm = l == 0 ? nullptr : perm; s.items = items;
        s.num_items = num_items; s.active = active;
        s.table = t->staged_tables[l]; s.npad = lv.npad; s.kchunks = d->ld / 32; s.tmem_cols = lv.tmem_cols;
        s.level = l; s.level_base = (int)t->level_offsets[l]; s.child_begin = t->child_begin;
        s.child_count = t->child_count; s.path_ws = path_ws; s.path_out = path; s.count = count;
        s.K = K; s.L = L; s.ip = ip; s.leaf_atom = t->leaf_atom;
        s.ks_last = (d->n - 32 * (s.kchunks - 1) + 7) / 8;
        if (l + 1 < L) {
          s.next_counts = counts_of(it) + bin_off[l + 1];
          s.next_base = (int)t->level_offsets[l + 1];
        } else {
          s.leaf_sel = leaf_sel;
        }
        // the rows are x: scores corrected by the support's pair-table products
        s.corr = t->pair_tables[l]; s.corr_w = t->pair_width[l]; s.corr_off = (int)t->level_offsets[l + 1];
        s.sup = S_ws; s.supc = c_ws; s.sup_t = it; s.sup_ld = K;
        s.cent = t->cent; s.xn2 = xn2; s.recheck_rel = 1e-5f;
        s.corr_pre = corr_pre; s.corr_pre_ld = (t->max_children + 3) & ~3;
        if (l == 0) { s.raw_out = s0; s.raw_w = t->root_children; }   // iteration 0: cache c_v . x of the root
        if (half && l > 0) {   // (the root pass stays on fp32 rows: its raw scores are cached for every later root choice)
          s.R16 = x16; s.table_h = t->half_tables[l]; s.inv_scale = inv_scale; s.qerr = qerr;
          // window += 16 sigma of the rows' quantisation noise on a unit centroid's score (||e|| / sqrt(n))
          s.recheck_q = 16.f / sqrtf((float)d->n);
          s.kchunks = d->ld / 64;
          s.ks_last = (d->n - 64 * (s.kchunks - 1) + 15) / 16;
          if ((e = launch_score_sh(s, sms, st)) != cudaSuccess) return e;
          continue;
        }
        if ((e = launch_score_st(s, sms, st)) != cudaSuccess) return e;
      }
      ga.iter = it;
      ga.root_counts = counts_of(it + 1) + bin_off[1];
      if ((e = launch_update_gram(ga, st)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const float* xtable = t ? nullptr : ensure_xtable(const_cast<DictHandle*>(d), st);
  if (!t && xtable == nullptr) return cudaErrorMemoryAllocation;
  // exhaustive scan with the 3xFP16 split (exact_scan.cu) unless score_kernel = 3 asks for 3xTF32
  const uint8_t* xtable16 = (!t && g_score_ws != 3) ? ensure_xtable16(const_cast<DictHandle*>(d), st) : nullptr;

  for (int it = 0; it < K; ++it) {
    if (!t) {
      // exhaustive selection: (compact the active patches, then) one tensor-core scan
      if (!root_direct) {
        e = launch_kernel(scan_kernel, 1, kScanThreads, scan_smem(1), st, true, counts_of(it), 1, offsets, items,
                          num_items, tile_off, cursor, stripes);
        if (e == cudaSuccess)
          e = launch_kernel(scatter_root_kernel, scatter_blocks, 256, 0, st, true, N, (const int*)active,
                            (const int*)offsets, cursor, perm);
        if (e != cudaSuccess) return e;
      }
      ScoreArgs s{};
      s.R = it == 0 ? R0 : R; s.ld = d->ld; s.nrows = N; s.perm = root_direct ? nullptr : perm; s.items = items;
      s.num_items = num_items; s.active = active;
      s.table = xtable; s.npad = xtable_block_width(d->ld); s.kchunks = d->ld / 32;
      if (xtable16 != nullptr) { s.table_h = xtable16; s.rnorm = resnorm; }
      s.nblocks = (int)((d->m + s.npad - 1) / s.npad); s.m_atoms = (int)d->m;
      s.leaf_sel = leaf_sel; s.ip = ip; s.K = K; s.L = 0;
      s.ks_last = (d->n - 32 * (s.kchunks - 1) + 7) / 8;
      if ((e = launch_exact_scan(s, sms, st)) != cudaSuccess) return e;
    }
    for (int l = 0; l < L; ++l) {
      const StagedLevel& lv = t->staged_levels[l];
      const int nb = (int)(t->level_offsets[l + 1] - t->level_offsets[l]);
      const bool direct_pass = l == 0 && root_direct;
      if (!direct_pass && l > 0) {
        if ((e = launch_level_scatter(N, active, path_ws, L, l, (int)t->level_offsets[l], nb, counts_of(it) + bin_off[l],
                                      cursor_of(it) + bin_off[l], counts_of(it + 1) + bin_off[l],
                                      cursor_of(it + 1) + bin_off[l], offsets, tile_off, cursor, perm, items,
                                      num_items, sms, st)) != cudaSuccess)
          return e;
      } else if (!direct_pass) {   // root bin compaction (root_direct off)
        e = launch_kernel(scan_kernel, 1, kScanThreads, scan_smem(nb), st, true, counts_of(it) + bin_off[l], nb,
                          offsets, items, num_items, tile_off, cursor, stripes);
        if (e == cudaSuccess)
          e = launch_kernel(scatter_root_kernel, scatter_blocks, 256, 0, st, true, N, (const int*)active,
                            (const int*)offsets, cursor, perm);
        if (e != cudaSuccess) return e;
      }
      ScoreArgs s{};
      s.R = it == 0 ? R0 : R; s.ld = d->ld; s.nrows = N; s.perm = direct_pass ? nullptr : perm; s.items = items;
      s.num_items = num_items; s.active = active;
      s.table = t->staged_tables[l]; s.npad = lv.npad; s.kchunks = d->ld / 32; s.tmem_cols = lv.tmem_cols;
      s.level = l; s.level_base = (int)t->level_offsets[l]; s.child_begin = t->child_begin;
      s.child_count = t->child_count; s.path_ws = path_ws; s.path_out = path; s.count = count;
      s.K = K; s.L = L; s.ip = ip; s.leaf_atom = t->leaf_atom;
      s.ks_last = (d->n - 32 * (s.kchunks - 1) + 7) / 8;
      if (l + 1 < L) {
        s.next_counts = counts_of(it) + bin_off[l + 1];
        s.next_base = (int)t->level_offsets[l + 1];
      } else {
        s.leaf_sel = leaf_sel;
      }
      s.tmem_cols = lv.tmem_cols;
      const bool whole = score_smem_bytes(s.kchunks, lv.npad) <= 227 * 1024;
      // streamed passes over wide nodes (> 128 children: config 2) are tensor-bound: 3xFP16 split by
      // default (score_kernel = 3 keeps them on 3xTF32, 4 takes the 3xFP16 pass at every level)
      const bool streamed = !whole || !score_ts_fits(s.kchunks, lv.npad, l + 1 == L);
      const bool want16 = g_score_ws == 4 || (g_score_ws == 2 && streamed && lv.npad > 128);
      if (want16 && score_s16_fits(d->ld, lv.npad) && ensure_s16_tables(const_cast<TreeHandle*>(t), st)) {
        s.table_h = t->s16_tables[l];   // 3xFP16 split, rows scaled by the residual norm the update wrote
        s.rnorm = resnorm;
        e = launch_score_s16(s, sms, st);
      } else if (g_score_ws == 3 || !whole || !score_ts_fits(s.kchunks, lv.npad, l + 1 == L))
        e = launch_score_st(s, sms, st);
      else
        e = launch_score_ts(s, sms, st);
      if (e != cudaSuccess) return e;
    }
    u.R_in = it == 0 ? R0 : R;
    u.iter = it;
    if (lockstep) e = launch_update_omp8(u, st);
    else if (wide) e = launch_update_wide(u, st);
    else e = launch_update(uc, u, ublocks, usmem, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}


// ======================================================================================
// Staged beam descent (non-greedy alpha, pursuit.py:134-162).
//
// The greedy pipeline keeps one node per patch per level; with retained_count
// > 1 a patch owns a frontier of nodes.  Each level pass therefore scores
// *entries* (patch, node): the entries are bucketed by node exactly like the
// greedy pass buckets patches, every entry's row is its patch's residual, and
// the epilogue keeps the `keep` best children (score_st.cu: beam_epilogue) as
// the next level's entries -- or, at the last level, folds the survivors' leaf
// atoms into one 64-bit max per patch.  Node tables are shared by all entries
// of a node, so the tensor-core passes stay as they are; the work grows with
// the frontier (c4 at alpha 0.1: 1 + 7 + 49 entries per patch per iteration).
// ======================================================================================
namespace {

__global__ void __launch_bounds__(256) scatter_entries_kernel(const int* count, const int* node, int level_base,
                                                              const int* offsets, int* cursor, int* perm) {
  pdl_enter();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool act = e < *count;
  const int bin = act ? node[e] - level_base : -1;
  const unsigned peers = __match_any_sync(kFull, bin);
  if (act) {
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cursor[bin], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    perm[offsets[bin] + base + __popc(peers & ((1u << lane) - 1u))] = e;
  }
}

// the patch's pick of the last beam level -> leaf_sel; the key is reset for the next iteration
__global__ void __launch_bounds__(256) beam_resolve_kernel(int64_t N, const int* active,
                                                           unsigned long long* key, int* leaf_sel) {
  pdl_enter();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  if (active[p]) leaf_sel[p] = (int)(0xFFFFFFFFu - (unsigned)(key[p] & 0xFFFFFFFFull));
  key[p] = 0ull;
}

struct BeamLayout {
  size_t total = 0;
  size_t R, Xpad, tol, active, path_ws, leaf_sel, Lf, yv, S_ws, c_ws, key, perm, items, num_items, offsets, tile_off,
      cursor, counts, ecount, epatch[2], enode[2], efirst[2];
  int64_t maxE = 0, maxbins = 1;
  std::vector<int64_t> frontier;   // entries per patch bound, per level
  std::vector<int64_t> bin_off;    // counts of level l at bin_off[l]
};

BeamLayout beam_layout(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method, const int* keep) {
  BeamLayout w;
  const int L = t->levels;
  w.frontier.assign(L, 1);
  w.bin_off.assign(L + 1, 0);
  for (int l = 1; l < L; ++l) {
    const int64_t nodes = t->level_offsets[l + 1] - t->level_offsets[l];
    w.frontier[l] = std::min<int64_t>(w.frontier[l - 1] * std::min(keep[l - 1], t->max_children), nodes);
  }
  for (int l = 0; l < L; ++l) {
    const int64_t nb = t->level_offsets[l + 1] - t->level_offsets[l];
    w.maxbins = std::max(w.maxbins, nb);
    w.bin_off[l + 1] = w.bin_off[l] + nb;
    w.maxE = std::max(w.maxE, N * w.frontier[l]);
  }
  auto add = [&](size_t bytes) {
    const size_t at = w.total;
    w.total += (bytes + 255) & ~(size_t)255;
    return at;
  };
  w.R = add((size_t)N * d->ld * 4);
  w.Xpad = method == kMethodOMP ? add((size_t)N * d->ld * 4) : 0;
  w.tol = add((size_t)N * 4);
  w.active = add((size_t)N * 4);
  w.path_ws = add((size_t)N * L * 4);
  w.leaf_sel = add((size_t)N * 4);
  w.Lf = add((size_t)N * K * (K + 1) / 2 * 4);
  w.yv = add((size_t)N * K * 4);
  w.S_ws = add((size_t)N * K * 4);
  w.c_ws = add((size_t)N * K * 4);
  w.key = add((size_t)N * 8);
  w.perm = add((size_t)w.maxE * 4);
  w.items = add((size_t)(w.maxE / kTile + w.maxbins + 2) * 16);
  w.num_items = add(16);
  w.offsets = add((size_t)(w.maxbins + 1) * 4);
  w.tile_off = add((size_t)(w.maxbins + 1) * 4);
  w.cursor = add((size_t)(w.maxbins + 1) * 4);
  w.counts = add((size_t)(w.bin_off[L] + 1) * 4);
  w.ecount = add(16);
  for (int i = 0; i < 2; ++i) {
    w.epatch[i] = add((size_t)w.maxE * 4);
    w.enode[i] = add((size_t)w.maxE * 4);
    w.efirst[i] = add((size_t)w.maxE);
  }
  return w;
}

}  // namespace

bool staged_beam_supported(const DictHandle* d, const TreeHandle* t, int K, int method, const int* keep) {
  if (t == nullptr || t->staged_tables.empty() || (method != kMethodMP && method != kMethodOMP) || K > 64) return false;
  if (t->max_leaf_children != 1 || t->levels > kMaxBeamLevels) return false;   // single-atom leaves
  UpdateCfg uc;
  if (!update_config(d->ld, K, uc)) return false;
  for (int l = 0; l < t->levels; ++l)
    if (keep[l] > kMaxBeamKeep || !score_st_fits(d->ld / 32, t->staged_levels[l].npad, l + 1 == t->levels))
      return false;
  return true;
}

size_t staged_beam_workspace(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method,
                             const int* keep) {
  return beam_layout(d, t, N, K, method, keep).total;
}

static bool beam_debug() {
  static const bool on = getenv("STMP_BEAM_DEBUG") != nullptr;
  return on;
}

cudaError_t run_staged_beam(const DictHandle* d, const TreeHandle* t, const float* X, int64_t N, int64_t ldx, int K,
                            int method, float tol_abs, const int* keep, int max_frontier, int32_t* idx, float* coef,
                            int32_t* count, float* resnorm, int32_t* path, int32_t* ip, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  (void)max_frontier;
  const BeamLayout w = beam_layout(d, t, N, K, method, keep);
  if (ws == nullptr || ws_bytes < w.total) return cudaErrorInvalidValue;
  const int L = t->levels;
  uint8_t* b = static_cast<uint8_t*>(ws);
  float* R = (float*)(b + w.R);
  float* Xpad = method == kMethodOMP ? (float*)(b + w.Xpad) : nullptr;
  int* active = (int*)(b + w.active);
  int* leaf_sel = (int*)(b + w.leaf_sel);
  int* perm = (int*)(b + w.perm);
  int4* items = (int4*)(b + w.items);
  int* num_items = (int*)(b + w.num_items);
  int* offsets = (int*)(b + w.offsets);
  int* tile_off = (int*)(b + w.tile_off);
  int* cursor = (int*)(b + w.cursor);
  int* counts = (int*)(b + w.counts);
  int* ecount = (int*)(b + w.ecount);
  unsigned long long* key = (unsigned long long*)(b + w.key);
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)(w.bin_off[L] + 1) * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(key, 0, (size_t)N * 8, st);
  if (e != cudaSuccess) return e;

  UpdateCfg uc;
  update_config(d->ld, K, uc);
  UpdateArgs u{};
  u.X = X; u.ldx = ldx; u.n = d->n; u.R = R; u.ld = d->ld;
  u.X2 = Xpad; u.ld2 = d->ld;
  u.atoms = d->atoms; u.child_begin = t->child_begin; u.child_count = t->child_count;
  u.leaf_atom = t->leaf_atom; u.L = L; u.path_ws = (int*)(b + w.path_ws); u.K = K; u.method = method;
  u.tol_abs = tol_abs; u.idx = idx; u.coef = coef; u.count = count; u.resnorm = resnorm;
  u.ip = ip; u.path_out = path; u.Lf = (float*)(b + w.Lf); u.yv = (float*)(b + w.yv); u.tol = (float*)(b + w.tol);
  u.active = active; u.root_count = nullptr; u.N = N; u.S_ws = (int*)(b + w.S_ws); u.c_ws = (float*)(b + w.c_ws);
  u.leaf_sel = leaf_sel; u.m = d->m;
  u.cache_atoms = update_smem_bytes(uc, K, d->ld, true) <= 96 * 1024 ? 1 : 0;
  const bool lockstep = method == kMethodOMP && lockstep_lanes(d->ld, K) != 0 && g_update_omp8;
  const bool wide = method == kMethodOMP && !lockstep && g_update_wide && wide_update_cpt(d->ld) != 0;
  const int gpb = 128 / uc.G;
  const int ublocks = (int)((N + gpb - 1) / gpb);
  const bool direct = ldx == d->ld && d->n == d->ld;
  {
    UpdateArgs ui = u;
    if (direct) { ui.R = nullptr; ui.X2 = nullptr; }
    if ((e = launch_init(uc, ui, ublocks, st)) != cudaSuccess) return e;
  }
  if (direct && method == kMethodOMP) u.X2 = X;
  const float* R0 = direct ? X : R;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t usmem = update_smem_bytes(uc, K, d->ld, u.cache_atoms != 0);

  for (int it = 0; it < K; ++it) {
    int cur = 0;
    for (int l = 0; l < L; ++l) {
      const StagedLevel& lv = t->staged_levels[l];
      const int nb = (int)(t->level_offsets[l + 1] - t->level_offsets[l]);
      const bool lastl = l + 1 == L;
      if (l > 0) {
        // bucket the level's entries by node
        e = launch_kernel(scan_kernel, 1, kScanThreads, scan_smem(nb), st, true, counts + w.bin_off[l], nb, offsets,
                          items, num_items, tile_off, cursor, (int*)nullptr);
        if (e == cudaSuccess)
          e = launch_kernel(scatter_entries_kernel, (int)((N * w.frontier[l] + 255) / 256), 256, 0, st, true,
                            (const int*)(ecount + cur), (const int*)(b + w.enode[cur]), (int)t->level_offsets[l],
                            (const int*)offsets, cursor, perm);
        if (e != cudaSuccess) return e;
        if (beam_debug() && (e = cudaStreamSynchronize(st)) != cudaSuccess) {
          fprintf(stderr, "beam: scatter level %d it %d: %s\n", l, it, cudaGetErrorString(e));
          return e;
        }
      }
      if (!lastl && (e = cudaMemsetAsync(ecount + (1 - cur), 0, 4, st)) != cudaSuccess) return e;
      ScoreArgs s{};
      s.R = it == 0 ? R0 : R; s.ld = d->ld; s.nrows = N; s.perm = l == 0 ? nullptr : perm; s.items = items;
      s.num_items = num_items; s.active = active;
      s.table = t->staged_tables[l]; s.npad = lv.npad; s.kchunks = d->ld / 32; s.tmem_cols = lv.tmem_cols;
      s.level = l; s.level_base = (int)t->level_offsets[l]; s.child_begin = t->child_begin;
      s.child_count = t->child_count; s.path_ws = (int*)(b + w.path_ws); s.path_out = path; s.count = count;
      s.K = K; s.L = L; s.ip = ip; s.leaf_atom = t->leaf_atom;
      s.ks_last = (d->n - 32 * (s.kchunks - 1) + 7) / 8;
      s.beam_keep = keep[l];
      if (l > 0) {
        s.entry_patch = (const int*)(b + w.epatch[cur]);
        s.entry_first = (const uint8_t*)(b + w.efirst[cur]);
      }
      if (!lastl) {
        s.out_patch = (int*)(b + w.epatch[1 - cur]);
        s.out_node = (int*)(b + w.enode[1 - cur]);
        s.out_first = (uint8_t*)(b + w.efirst[1 - cur]);
        s.out_count = ecount + (1 - cur);
        s.next_counts = counts + w.bin_off[l + 1];
        s.next_base = (int)t->level_offsets[l + 1];
      } else {
        s.leaf_sel = leaf_sel;   // marks the last level (leaf records in the table block)
        s.leaf_key = key;
      }
      if ((e = launch_score_st(s, sms, st)) != cudaSuccess) return e;
      if (beam_debug() && (e = cudaStreamSynchronize(st)) != cudaSuccess) {
        fprintf(stderr, "beam: score level %d it %d: %s\n", l, it, cudaGetErrorString(e));
        return e;
      }
      cur = 1 - cur;   // the next level's entries are in the buffer this pass filled
    }
    if ((e = launch_kernel(beam_resolve_kernel, (int)((N + 255) / 256), 256, 0, st, true, N, (const int*)active,
                           key, leaf_sel)) != cudaSuccess)
      return e;
    u.R_in = it == 0 ? R0 : R;
    u.iter = it;
    if (lockstep) e = launch_update_omp8(u, st);
    else if (wide) e = launch_update_wide(u, st);
    else e = launch_update(uc, u, ublocks, usmem, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace stmp
