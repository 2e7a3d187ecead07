// Probe (not part of the library): how tcgen05.mma.kind::f16 reads a 16-bit A
// operand from tensor memory.  A[r][k] = k + 1 (fp16) is stored under a layout
// hypothesis, B = identity (16 x 16, shared memory, K-major SW128), so D[r][n]
// shows which A element the hardware took for K index n.
//   hypothesis 0: 32-bit cell c of lane r holds (A[r][2c] low half, A[r][2c+1] high half)
//   hypothesis 1: the reverse pairing
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_1412_0680_b200/csrc -o tools/_tmem_f16_probe tools/tmem_f16_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "sm100.cuh"

using namespace stmp::sm100;

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__global__ void __launch_bounds__(128) probe(int hyp, float* out) {
  __shared__ __align__(1024) uint8_t btab[2048];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc(&slot, 64);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 2048; i += 128) btab[i] = 0;
  __syncthreads();
  if (tid < 16) {   // B[n][k] = (n == k), row n of 128 B, 16-byte chunks swizzled
    const int n = tid, k = tid;
    const uint32_t off = sw128_offset((uint32_t)n, (uint32_t)(k >> 3)) + (uint32_t)(k & 7) * 2u;
    *reinterpret_cast<__half*>(btab + off) = __float2half(1.f);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // A: lane = row = tid, 8 cells = 16 halfs; value = 100 * (tid % 8) + k + 1 so rows differ
  uint32_t cells[8];
  for (int c = 0; c < 8; ++c) {
    const float lo = 100.f * (tid % 8) + 2 * c + 1, hi = 100.f * (tid % 8) + 2 * c + 2;
    const uint32_t l = __half_as_ushort(__float2half(hyp == 0 ? lo : hi));
    const uint32_t h = __half_as_ushort(__float2half(hyp == 0 ? hi : lo));
    cells[c] = l | (h << 16);
  }
  tmem_st8(tmem + ((uint32_t)(warp * 32) << 16), cells);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mma_f16_ts(tmem + 32, tmem, sw128_kmajor_desc(smem_u32(btab)), idesc_f16(128, 16), 0u);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + 32, v);
  for (int j = 0; j < 16; ++j) out[tid * 16 + j] = v[j];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

int main() {
  float* out;
  cudaMalloc(&out, 128 * 16 * 4);
  for (int hyp = 0; hyp < 2; ++hyp) {
    cudaMemset(out, 0, 128 * 16 * 4);
    probe<<<1, 128>>>(hyp, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("hypothesis %d: %s\n", hyp, cudaGetErrorString(e));
      return 1;
    }
    float h[128 * 16];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    for (int r : {0, 1, 37, 127}) {
      printf("hyp %d row %3d:", hyp, r);
      for (int j = 0; j < 16; ++j) printf(" %g", h[r * 16 + j]);
      printf("\n");
    }
  }
  return 0;
}
