// Atom Gram matrix G = A A^T of a (padded) dictionary, built once per
// dictionary handle for the staged OMP update: the Gram column of a newly
// selected atom against the support (the omp_refit normal equations,
// pkg/src/stmp/pursuit.py:247-249) becomes t scalar gathers instead of t
// n-length dot products.  Plain fp32 FFMA accumulation, the precision of the
// on-the-fly dots it replaces.
#include <mutex>

#include "common.cuh"
#include "staged.cuh"

namespace stmp {

namespace {

constexpr int kGT = 64;   // output tile
constexpr int kGK = 32;   // k step

__global__ void __launch_bounds__(256) gram_kernel(const float* __restrict__ A, int64_t m, int ld,
                                                    float* __restrict__ G) {
  __shared__ float As[kGK][kGT + 4];
  __shared__ float Bs[kGK][kGT + 4];
  const int64_t bi = (int64_t)blockIdx.y * kGT, bj = (int64_t)blockIdx.x * kGT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < ld; k0 += kGK) {
    for (int e = threadIdx.x; e < kGT * kGK; e += 256) {
      const int r = e / kGK, k = e % kGK;
      As[k][r] = bi + r < m ? A[(bi + r) * ld + k0 + k] : 0.f;
      Bs[k][r] = bj + r < m ? A[(bj + r) * ld + k0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kGK; ++k) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[k][ty * 4 + i];
        bv[i] = Bs[k][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = bi + ty * 4 + i, c = bj + tx * 4 + j;
      if (r < m && c < m) G[r * m + c] = acc[i][j];
    }
}

std::mutex g_gram_mutex;

}  // namespace

const float* ensure_gram(DictHandle* d, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_gram_mutex);
  if (d->gram_tried) return d->gram;
  d->gram_tried = true;
  if (d->m > kGramMaxAtoms) return nullptr;
  float* g = nullptr;
  if (cudaMalloc(&g, (size_t)d->m * d->m * sizeof(float)) != cudaSuccess) {
    cudaGetLastError();  // clear: fall back to on-the-fly dots
    return nullptr;
  }
  const dim3 grid((unsigned)((d->m + kGT - 1) / kGT), (unsigned)((d->m + kGT - 1) / kGT));
  gram_kernel<<<grid, 256, 0, st>>>(d->atoms, d->m, d->ld, g); note_launch();
  // one-time build: finish it before any stream can read the table
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
    cudaFree(g);
    return nullptr;
  }
  d->gram = g;
  return g;
}

}  // namespace stmp
