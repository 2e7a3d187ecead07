// Kernel launch interfaces shared between the ABI layer and the kernel files.
#pragma once

#include "common.cuh"

namespace stmp {

constexpr int kMethodMP = 0;
constexpr int kMethodOMP = 1;
constexpr int kMethodSelect = 2;

struct FusedArgs {
  const float* X;
  int64_t N;
  int64_t ldx;
  int n;
  const float* atoms;
  int64_t m;
  int ld;
  int vpl;
  TreeView tree;
  int has_tree;
  int K;
  int method;
  float tol_abs;          // < 0: relative tolerance 1e-6 * ||x||
  int32_t* idx;
  float* coef;
  int32_t* count;
  float* resnorm;
  int32_t* path;
  int32_t* ip;
  int root_smem_rows;     // > 0: the root's child centroids are staged in shared memory
  int root_begin;
  int cache_atoms;        // support atoms cached per warp in shared memory
  int warp_smem_floats;   // per-warp shared scratch (OMP factor + optional atom cache)
  // non-greedy alpha (beam descent, pkg/src/stmp/pursuit.py:134-162): children kept
  // per node at each level, and per-warp global scratch for the frontiers
  int beam;               // 0: greedy (one child per level)
  int keep[8];            // retained_count(alpha, k_l) per level
  int max_frontier;       // largest frontier (nodes) over the levels
  int* scratch;           // [warps][2 * max_frontier ints | 256 floats]
};
constexpr int kMaxBeamLevels = 8;
// per-warp scratch of the beam descent (ints): two frontiers and a score row
__host__ __device__ inline int64_t beam_scratch_ints(int max_frontier) { return 2 * (int64_t)max_frontier + 256; }

int fused_vpl_for(int n);

// batch driver (driver.cu): DC split before the encoder, lift + reconstruct after it
cudaError_t launch_dc_split(const float* Y, int64_t N, int64_t ldy, int n, const double* dc_meas, double denom,
                            float* Yc, int64_t ldc, double* dc, cudaStream_t st);
cudaError_t launch_reconstruct(const DictHandle* d, const int32_t* idx, const float* coef, const int32_t* count,
                               int64_t N, int K, const double* scale, const double* dc, double* out, int64_t ldo,
                               cudaStream_t st);

// data formats either side of the path (tensor_ops.cu)
cudaError_t launch_extract(const float* t, int rank, const int64_t* shape, const int64_t* patch,
                           const int64_t* nstarts, const int64_t* starts_dev, float* out, cudaStream_t st);
cudaError_t launch_aggregate(const float* patches, int rank, const int64_t* shape, const int64_t* patch,
                             const int64_t* nstarts, const int64_t* starts_dev, float* out, cudaStream_t st);
cudaError_t launch_row_select(const float* X, int64_t N, int n_in, const int64_t* rows_dev, int n_out, double* Y,
                              cudaStream_t st);
cudaError_t launch_coded_exposure(const float* X, int64_t N, int n_in, const float* mask_dev, int pixels,
                                  int windows, int frames, double* Y, cudaStream_t st);
cudaError_t launch_block_average(const float* X, int64_t N, int rank, const int64_t* in_shape,
                                 const int64_t* factors, double* Y, cudaStream_t st);
cudaError_t launch_encode_fused(const FusedArgs& a, cudaStream_t stream);
// warps of the fused kernel's persistent grid for N patches (beam scratch sizing)
int64_t fused_warps(int64_t N);

}  // namespace stmp
