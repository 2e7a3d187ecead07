// Micro-benchmark of the score passes' row-gather pattern (not part of the
// library): one persistent CTA per SM streams "tiles" of 128 rows, one
// 32-float (128 B) K chunk of every row at a time, through a ring of NA landing
// slots -- exactly the access pattern of score_st's stagers -- and only sums
// the data (no MMA), so the time is the gather's.  Variants: warps per CTA,
// ring depth, bytes per row per chunk, rows in order (root pass) or permuted
// (bucketed levels), CTAs per SM.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// Stager work per chunk after the gather (thread = row, W = 4):
//   MODE 1: tf32 hi/lo split + two tcgen05.st (32 columns each) + wait::st  (score_st today)
//   MODE 2: lo = x - trunc_tf32(x) written back to a shared-memory lo slot (A operand from SMEM)
template <int NA, int MODE>
__global__ void __launch_bounds__(128) stage_kernel(const float* __restrict__ X, int ld, const int* __restrict__ perm,
                                                     int ntiles, int kch, float* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint32_t tslot;
  constexpr int SLOT = 32 * 128;             // a warp's 32 rows x 128 B
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = sm + warp * NA * SLOT;
  uint8_t* lo_slots = sm + 4 * NA * SLOT + warp * 2 * SLOT;
  if ((MODE == 1 || MODE == 3) && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  const int total = (t1 - t0) * kch;
  float acc = 0.f;
  auto issue = [&](int g) {
    if (g < total) {
      const int tile = t0 + g / kch, c = g % kch;
      uint8_t* dst = ring + (g % NA) * SLOT;
      for (int e = lane; e < 32 * 8; e += 32) {
        const int r = e / 8, j = e % 8;
        const int row = perm[tile * 128 + warp * 32 + r];
        cp_async16(smem_u32(dst + (r * 8 + (j ^ (r & 7))) * 16), X + (int64_t)row * ld + c * 32 + 4 * j);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int g = 0; g < NA; ++g) issue(g);
  for (int g = 0; g < total; ++g) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
    __syncwarp();
    const float4* s = reinterpret_cast<const float4*>(ring + (g % NA) * SLOT) + lane * 8;
    float hi[32], lo[32];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 v = s[j ^ (lane & 7)];
      const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hi[4 * j + q] = __uint_as_float(__float_as_uint(x[q]) & 0xFFFFE000u);
        lo[4 * j + q] = x[q] - hi[4 * j + q];
      }
    }
    if (MODE == 1 || MODE == 3) {
      __syncwarp();
      issue(g + NA);
      const uint32_t lb = (uint32_t)(warp * 32) << 16;
      if (MODE == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");   // previous chunk's stores
      tmem_st32(tmem + lb + (g & 1) * 64, hi);
      tmem_st32(tmem + lb + (g & 1) * 64 + 32, lo);
      if (MODE == 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      float4* d = reinterpret_cast<float4*>(lo_slots + (g & 1) * SLOT) + lane * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) d[j ^ (lane & 7)] = make_float4(lo[4 * j], lo[4 * j + 1], lo[4 * j + 2], lo[4 * j + 3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      issue(g + NA);
      acc += hi[0];
    }
  }
  if (acc == 123.456f) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((MODE == 1 || MODE == 3) && warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

template <int NA, int MODE>
float run_stage(const float* X, int ld, const int* perm, int ntiles, int kch, float* out, int cps, int sms) {
  const size_t smem = (size_t)4 * NA * 4096 + 4 * 2 * 4096;
  cudaFuncSetAttribute(stage_kernel<NA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  stage_kernel<NA, MODE><<<sms * cps, 128, smem>>>(X, ld, perm, ntiles, kch, out);
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) stage_kernel<NA, MODE><<<sms * cps, 128, smem>>>(X, ld, perm, ntiles, kch, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / 3;
}

// W warps, each owning 128 / W rows of a tile; CB = 16-byte pieces per row per chunk
template <int W, int NA, int CB>
__global__ void __launch_bounds__(W * 32) gather_kernel(const float* __restrict__ X, int ld, const int* __restrict__ perm,
                                                         int ntiles, int kch, float* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int RPW = 128 / W;               // rows per warp
  constexpr int SLOT = RPW * CB * 16;        // bytes per warp per slot
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = sm + warp * NA * SLOT;
  const int chunks = kch / (CB / 8);         // chunks of CB*4 floats
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  const int total = (t1 - t0) * chunks;
  float acc = 0.f;
  auto issue = [&](int g) {
    if (g < total) {
      const int tile = t0 + g / chunks, c = g % chunks;
      uint8_t* dst = ring + (g % NA) * SLOT;
      // piece e = (row r, 16-byte piece j) of this warp's rows
      for (int e = lane; e < RPW * CB; e += 32) {
        const int r = e / CB, j = e % CB;
        const int row = perm[tile * 128 + warp * RPW + r];
        cp_async16(smem_u32(dst + e * 16), X + (int64_t)row * ld + c * CB * 4 + 4 * j);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int g = 0; g < NA; ++g) issue(g);
  for (int g = 0; g < total; ++g) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NA - 1) : "memory");
    __syncwarp();
    const float4* s = reinterpret_cast<const float4*>(ring + (g % NA) * SLOT);
    for (int e = lane; e < RPW * CB; e += 32) {
      const float4 v = s[e];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    issue(g + NA);
  }
  if (acc == 123.456f) out[0] = acc;
}

template <int W, int NA, int CB>
float run(const float* X, int ld, const int* perm, int ntiles, int kch, float* out, int ctas_per_sm, int sms) {
  const size_t smem = (size_t)W * NA * (128 / W) * CB * 16;
  cudaFuncSetAttribute(gather_kernel<W, NA, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather_kernel<W, NA, CB><<<sms * ctas_per_sm, W * 32, smem>>>(X, ld, perm, ntiles, kch, out);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int i = 0; i < reps; ++i) gather_kernel<W, NA, CB><<<sms * ctas_per_sm, W * 32, smem>>>(X, ld, perm, ntiles, kch, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / reps;
}

int main() {
  const int N = 524288, ld = 1600, kch = ld / 32;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* X;
  int *pin, *prnd;
  float* out;
  cudaMalloc(&X, (size_t)N * ld * 4);
  cudaMemset(X, 0, (size_t)N * ld * 4);
  cudaMalloc(&pin, N * 4);
  cudaMalloc(&prnd, N * 4);
  cudaMalloc(&out, 4);
  std::vector<int> h(N);
  for (int i = 0; i < N; ++i) h[i] = i;
  cudaMemcpy(pin, h.data(), N * 4, cudaMemcpyHostToDevice);
  srand(1);
  for (int i = N - 1; i > 0; --i) {
    const int j = rand() % (i + 1);
    std::swap(h[i], h[j]);
  }
  cudaMemcpy(prnd, h.data(), N * 4, cudaMemcpyHostToDevice);
  const int ntiles = N / 128;
  const double bytes = (double)N * ld * 4;
  struct V {
    const char* name;
    float (*fn)(const float*, int, const int*, int, int, float*, int, int);
    int cps;
  } vs[] = {
      {"W4 NA6 CB8 (score_st today)", run<4, 6, 8>, 1},   {"W4 NA12 CB8", run<4, 12, 8>, 1},
      {"W4 NA6 CB16", run<4, 6, 16>, 1},                   {"W8 NA6 CB8", run<8, 6, 8>, 1},
      {"W8 NA12 CB8", run<8, 12, 8>, 1},                   {"W4 NA6 CB8 x2 CTA/SM", run<4, 6, 8>, 2},
      {"W4 NA8 CB8 x2 CTA/SM", run<4, 8, 8>, 2},           {"W16 NA6 CB8", run<16, 6, 8>, 1},
      {"stage TMEM (split+2 STTM+wait) NA6", run_stage<6, 1>, 1},
      {"stage SMEM lo NA6", run_stage<6, 2>, 1},
      {"stage TMEM deferred wait NA6", run_stage<6, 3>, 1},
      {"stage TMEM NA6 x2 CTA/SM", run_stage<6, 1>, 2},
      {"stage SMEM lo NA6 x2 CTA/SM", run_stage<6, 2>, 2},
  };
  for (auto& v : vs) {
    for (int rnd = 0; rnd < 2; ++rnd) {
      const float ms = v.fn(X, ld, rnd ? prnd : pin, ntiles, kch, out, v.cps, sms);
      printf("%-32s %-8s %8.3f ms  %7.1f GB/s\n", v.name, rnd ? "random" : "inorder", ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
