// Batch driver around the encoder: the per-patch work that
// pipelines._code_patches (pkg/src/stmp/pipelines.py:180-217) does before and
// after matching_pursuit, on the device.
//
//   dc_split:     dc = (y . dc_meas) / denom,  y_c = y - dc * dc_meas
//                 (pipelines.py:201-203), f64 arithmetic on the f32 patch,
//                 y_c rounded to f32 for the encoder;
//   reconstruct:  out = sum_k (c_k / scale[i_k]) a_{i_k} + dc
//                 (lift_code, operators.py:199-215, then reconstruct,
//                 pursuit.py:224-232, then "+ dc", pipelines.py:204): f64,
//                 entries in selection order, multiply and add rounded
//                 separately exactly like NumPy's `out += c * atoms[i]`.
#include "common.cuh"
#include "kernels.cuh"

namespace stmp {

namespace {

// one warp per patch
__global__ void __launch_bounds__(256) dc_split_kernel(const float* __restrict__ Y, int64_t N, int64_t ldy, int n,
                                                       const double* __restrict__ dc_meas, double denom,
                                                       float* __restrict__ Yc, int64_t ldc, double* __restrict__ dc) {
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= N) return;
  const float* y = Y + p * ldy;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s = fma((double)y[i], dc_meas[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  const double d = s / denom;
  float* yc = Yc + p * ldc;
  for (int i = lane; i < n; i += 32) yc[i] = (float)__dsub_rn((double)y[i], __dmul_rn(d, dc_meas[i]));
  if (lane == 0) dc[p] = d;
}

// one CTA row of 128 threads per patch, threads over the full-space dimension
__global__ void __launch_bounds__(128) reconstruct_kernel(const float* __restrict__ atoms, int ld, int n,
                                                          const int32_t* __restrict__ idx,
                                                          const float* __restrict__ coef,
                                                          const int32_t* __restrict__ count, int K,
                                                          const double* __restrict__ scale,
                                                          const double* __restrict__ dc, double* __restrict__ out,
                                                          int64_t ldo) {
  const int64_t p = blockIdx.x;
  const int cnt = count[p];
  double* o = out + p * ldo;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < cnt; ++k) {
      const int a = idx[p * K + k];
      double c = (double)coef[p * K + k];
      if (scale) c = __ddiv_rn(c, scale[a]);
      acc = __dadd_rn(acc, __dmul_rn(c, (double)atoms[(int64_t)a * ld + i]));
    }
    if (dc) acc = __dadd_rn(acc, dc[p]);
    o[i] = acc;
  }
}

}  // namespace

cudaError_t launch_dc_split(const float* Y, int64_t N, int64_t ldy, int n, const double* dc_meas, double denom,
                            float* Yc, int64_t ldc, double* dc, cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  dc_split_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(Y, N, ldy, n, dc_meas, denom, Yc, ldc, dc);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_reconstruct(const DictHandle* d, const int32_t* idx, const float* coef, const int32_t* count,
                               int64_t N, int K, const double* scale, const double* dc, double* out, int64_t ldo,
                               cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  reconstruct_kernel<<<(unsigned)N, 128, 0, st>>>(d->atoms, d->ld, d->n, idx, coef, count, K, scale, dc, out, ldo);
  note_launch();
  return cudaGetLastError();
}

}  // namespace stmp
