// Micro-benchmark (not part of the library): the score passes' two input
// streams together -- the 128-row x gather (cp.async, 128 B of every row per K
// chunk, as score_st's stagers) and the node-table chunk stream (one bulk copy
// per K chunk into a ring of NB slots, as score_st's producer warp) -- with no
// MMAs, to find what the memory system alone allows when a pass reads as many
// table bytes (from L2 or DRAM) as patch bytes (from DRAM).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1412_0680_b200/csrc -o tools/_stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "sm100.cuh"

using namespace stmp::sm100;

// warps 0-3: gather; warp 4: table producer.  RPT = tiles (of 128 rows) that
// share one table chunk before it is released (1 = the score kernels; the paired
// variants faulted on the box and were dropped with the idea).
template <int NA, int NB, int RPT>
__global__ void __launch_bounds__(160) tab_kernel(const float* __restrict__ X, int ld, const int* __restrict__ perm,
                                                  int ntiles, int kch, const uint8_t* __restrict__ table,
                                                  uint32_t tbytes, int tiles_per_node, int hint, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NB], done[NB];
  constexpr int SLOT = 32 * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = sm + warp * NA * SLOT;
  uint8_t* tab = sm + 4 * NA * SLOT;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&done[b], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int groups = (ntiles + RPT - 1) / RPT;          // tile groups sharing table chunks
  const int per = (groups + gridDim.x - 1) / gridDim.x;
  const int g0 = blockIdx.x * per, g1 = min(groups, g0 + per);
  const int tsteps = (g1 - g0) * kch;                   // table chunks of this CTA
  const int total = tsteps * RPT;                       // gather chunks
  float acc = 0.f;
  if (warp == 4) {
    if (lane == 0 && tbytes) {
      const uint64_t pol = hint ? l2_policy_evict_last() : l2_policy_evict_first();
      for (int t = 0; t < tsteps; ++t) {
        const int grp = g0 + t / kch, c = t % kch;
        const int node = (grp * RPT) / tiles_per_node;
        const int s = t % NB;
        if (t >= NB) mbar_wait(&done[s], (uint32_t)(t / NB - 1) & 1u);
        mbar_arrive_expect_tx(&full[s], tbytes);
        bulk_g2s_hint(tab + (size_t)s * tbytes, table + ((size_t)node * kch + c) * tbytes, tbytes, &full[s], pol);
      }
    }
    return;
  }
  const uint64_t rpol = l2_policy_evict_first();
  // gather chunk q: table step t = q / RPT, tile (g0 + t / kch) * RPT + q % RPT, K chunk t % kch
  auto issue = [&](int q) {
    if (q < total) {
      const int t = q / RPT, sub = q % RPT;
      const int tile = min(ntiles - 1, (g0 + t / kch) * RPT + sub), c = t % kch;
      uint8_t* dst = ring + (q % NA) * SLOT;
      for (int e = lane; e < 32 * 8; e += 32) {
        const int r = e / 8, j = e % 8;
        const int row = perm[tile * 128 + warp * 32 + r];
        cp_async16_hint(smem_u32(dst + (r * 8 + (j ^ (r & 7))) * 16), X + (int64_t)row * ld + c * 32 + 4 * j, 16u,
                        rpol);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int q = 0; q < NA; ++q) issue(q);
  for (int q = 0; q < total; ++q) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
    __syncwarp();
    const float4* s = reinterpret_cast<const float4*>(ring + (q % NA) * SLOT) + lane * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 v = s[j ^ (lane & 7)];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    issue(q + NA);
    if (tbytes && q % RPT == RPT - 1) {
      const int t = q / RPT, sl = t % NB;
      mbar_wait(&full[sl], (uint32_t)(t / NB) & 1u);
      acc += reinterpret_cast<const float*>(tab + (size_t)sl * tbytes)[threadIdx.x];
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[sl]);
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

template <int NA, int NB, int RPT>
float run(const float* X, int ld, const int* perm, int ntiles, int kch, const uint8_t* table, uint32_t tbytes,
          int tiles_per_node, int hint, float* out, int cps, int sms) {
  const size_t smem = (size_t)4 * NA * 4096 + (size_t)NB * tbytes;
  cudaFuncSetAttribute(tab_kernel<NA, NB, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tab_kernel<NA, NB, RPT><<<sms * cps, 160, smem>>>(X, ld, perm, ntiles, kch, table, tbytes, tiles_per_node, hint, out);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int i = 0; i < reps; ++i)
    tab_kernel<NA, NB, RPT><<<sms * cps, 160, smem>>>(X, ld, perm, ntiles, kch, table, tbytes, tiles_per_node, hint,
                                                     out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / reps;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
  const int N = 524288, ld = 1600, kch = ld / 32;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* X;
  int* perms[3];
  float* out;
  uint8_t* table;
  const size_t tab_total = (size_t)4096 * kch * 8192;   // level 2: 4096 nodes x 50 chunks x 8 KB = 1.68 GB
  CK(cudaMalloc(&X, (size_t)N * ld * 4));
  CK(cudaMemset(X, 0, (size_t)N * ld * 4));
  CK(cudaMalloc(&table, tab_total));
  CK(cudaMemset(table, 0, tab_total));
  CK(cudaMalloc(&out, 4));
  printf("allocated\n");
  std::vector<int> h(N);
  for (int i = 0; i < N; ++i) h[i] = i;
  for (int k = 0; k < 3; ++k) cudaMalloc(&perms[k], N * 4);
  cudaMemcpy(perms[0], h.data(), N * 4, cudaMemcpyHostToDevice);
  srand(1);
  // "bucket64": stable bucketing by a random bin of 64 (level 1: rows of a tile ascend with stride ~64)
  {
    std::vector<int> bin(N), o(N);
    for (int i = 0; i < N; ++i) bin[i] = rand() % 64;
    for (int i = 0; i < N; ++i) o[i] = i;
    std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return bin[a] < bin[b]; });
    cudaMemcpy(perms[1], o.data(), N * 4, cudaMemcpyHostToDevice);
  }
  for (int i = N - 1; i > 0; --i) {
    const int j = rand() % (i + 1);
    std::swap(h[i], h[j]);
  }
  cudaMemcpy(perms[2], h.data(), N * 4, cudaMemcpyHostToDevice);
  CK(cudaDeviceSynchronize());
  printf("perms ready\n");
  const char* pname[3] = {"inorder", "bucket64", "random"};
  const int ntiles = N / 128;
  const double bytes = (double)N * ld * 4;
  struct V {
    const char* name;
    float (*fn)(const float*, int, const int*, int, int, const uint8_t*, uint32_t, int, int, float*, int, int);
    uint32_t tbytes;
    int tiles_per_node, hint, cps;
  } vs[] = {
      {"no table            NA3 x2", run<3, 3, 1>, 0, 64, 1, 2},
      {"no table            NA6 x1", run<6, 3, 1>, 0, 64, 1, 1},
      {"L1 16KB/chunk L2res NA3 NB3 x2", run<3, 3, 1>, 16384, 64, 1, 2},
      {"L1 16KB/chunk L2res NA6 NB6 x1", run<6, 6, 1>, 16384, 64, 1, 1},
      {"L1  8KB/chunk L2res NA3 NB3 x2", run<3, 3, 1>, 8192, 64, 1, 2},
      {"L2  8KB/chunk DRAM  NA3 NB3 x2", run<3, 3, 1>, 8192, 1, 0, 2},
      {"L2  8KB/chunk DRAM  NA6 NB6 x1", run<6, 6, 1>, 8192, 1, 0, 1},
      {"L2  4KB/chunk DRAM  NA3 NB3 x2", run<3, 3, 1>, 4096, 1, 0, 2},
  };
  for (auto& v : vs) {
    for (int k = 0; k < 3; ++k) {
      const float ms = v.fn(X, ld, perms[k], ntiles, kch, table, v.tbytes, v.tiles_per_node, v.hint, out, v.cps, sms);
      printf("%-34s %-8s %8.3f ms  x %7.1f GB/s\n", v.name, pname[k], ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
