// Data formats either side of the hot path: sliding-window
// patch extraction / deterministic overlap-average aggregation
// (pkg/src/stmp/tensor.py:104-136) and the batched observation operators
// (pkg/src/stmp/operators.py:115-141).
//
// Geometry is passed as small per-axis arrays (rank <= kMaxRank): tensor
// extents, patch extents and, per axis, the sorted window start positions
// (PatchLayout.axis_starts, concatenated).  Patches are numbered in row-major
// origin order (first axis slowest) and their n values in row-major order of
// the patch window, exactly as np.ix_ + reshape orders them.
#include "common.cuh"
#include "kernels.cuh"

namespace stmp {

namespace {

struct Geometry {
  int rank;
  int64_t shape[kMaxRank];     // tensor extents
  int64_t patch[kMaxRank];     // window extents
  int64_t nstarts[kMaxRank];   // window starts per axis
  int64_t soff[kMaxRank];      // offset of each axis's starts in `starts`
};

// one thread per (patch, element): a pure copy, bit-exact with np.ix_ indexing
__global__ void __launch_bounds__(256) extract_kernel(const float* __restrict__ t, Geometry g,
                                                      const int64_t* __restrict__ starts, int64_t N, int64_t n,
                                                      float* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * n) return;
  int64_t p = e / n, i = e - p * n;
  int64_t src = 0, stride = 1;
  for (int a = g.rank - 1; a >= 0; --a) {
    const int64_t si = p % g.nstarts[a];
    p /= g.nstarts[a];
    const int64_t oi = i % g.patch[a];
    i /= g.patch[a];
    src += (starts[g.soff[a] + si] + oi) * stride;
    stride *= g.shape[a];
  }
  out[e] = t[src];
}

// first start index j with starts[j] >= v (the axis's starts ascend)
__device__ __forceinline__ int64_t lower_bound(const int64_t* s, int64_t len, int64_t v) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (s[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One thread per output cell: the windows covering a cell are a box of start
// indices (a contiguous range per axis); they are visited in row-major origin
// order -- the order in which aggregate_patches adds patches -- and summed in
// f64, so each cell's sum, count and mean are bitwise those of the reference.
__global__ void __launch_bounds__(256) aggregate_kernel(const float* __restrict__ patches, Geometry g,
                                                        const int64_t* __restrict__ starts, int64_t cells,
                                                        int64_t n, float* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  int64_t x[kMaxRank], lo[kMaxRank], hi[kMaxRank];
  int64_t rem = c;
  for (int a = g.rank - 1; a >= 0; --a) {
    x[a] = rem % g.shape[a];
    rem /= g.shape[a];
    const int64_t* s = starts + g.soff[a];
    lo[a] = lower_bound(s, g.nstarts[a], x[a] - g.patch[a] + 1);   // starts[j] + patch - 1 >= x
    hi[a] = lower_bound(s, g.nstarts[a], x[a] + 1);                // starts[j] <= x
  }
  int64_t idx[kMaxRank];
  for (int a = 0; a < g.rank; ++a) idx[a] = lo[a];
  double acc = 0.0;
  int64_t cnt = 0;
  bool more = true;
  for (int a = 0; a < g.rank; ++a) more = more && lo[a] < hi[a];
  while (more) {
    int64_t p = 0, off = 0;
    for (int a = 0; a < g.rank; ++a) {
      p = p * g.nstarts[a] + idx[a];
      off = off * g.patch[a] + (x[a] - starts[g.soff[a] + idx[a]]);
    }
    acc = __dadd_rn(acc, (double)patches[p * n + off]);
    ++cnt;
    // next index in row-major order (last axis fastest)
    int a = g.rank - 1;
    for (; a >= 0; --a) {
      if (++idx[a] < hi[a]) break;
      idx[a] = lo[a];
    }
    more = a >= 0;
  }
  out[c] = (float)__ddiv_rn(acc, (double)cnt);
}

// Observation operators on a batch of rows (apply_batch): f32 rows in, f64 rows out.
__global__ void __launch_bounds__(256) row_select_kernel(const float* __restrict__ X, int64_t N, int n_in,
                                                         const int64_t* __restrict__ rows, int n_out,
                                                         double* __restrict__ Y) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * n_out) return;
  const int64_t p = e / n_out;
  const int j = (int)(e - p * n_out);
  Y[e] = (double)X[p * n_in + rows[j]];
}

// coded exposure: the patch is (spatial..., windows, frames) row-major; each
// measurement sums its frames weighted by the pixel's binary mask, in f64
__global__ void __launch_bounds__(256) coded_exposure_kernel(const float* __restrict__ X, int64_t N, int n_in,
                                                             const float* __restrict__ mask, int pixels,
                                                             int windows, int frames, double* __restrict__ Y) {
  const int n_out = pixels * windows;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * n_out) return;
  const int64_t p = e / n_out;
  const int q = (int)(e - p * n_out);
  const int px = q / windows;
  const float* x = X + p * n_in + (int64_t)q * frames;
  const float* m = mask + (int64_t)px * frames;
  double s = 0.0;
  for (int t = 0; t < frames; ++t) s = __dadd_rn(s, __dmul_rn((double)x[t], (double)m[t]));
  Y[e] = s;
}

// block average: mean over each factor block of the patch grid (in_shape row-major)
__global__ void __launch_bounds__(256) block_average_kernel(const float* __restrict__ X, int64_t N, int n_in,
                                                            Geometry g, double* __restrict__ Y, int n_out) {
  // g.shape = in_shape, g.patch = factors
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * n_out) return;
  const int64_t p = e / n_out;
  int64_t q = e - p * n_out;
  int64_t ob[kMaxRank];
  for (int a = g.rank - 1; a >= 0; --a) {
    const int64_t oe = g.shape[a] / g.patch[a];
    ob[a] = q % oe;
    q /= oe;
  }
  int64_t idx[kMaxRank];
  for (int a = 0; a < g.rank; ++a) idx[a] = 0;
  double s = 0.0;
  int64_t cnt = 0;
  bool more = true;
  while (more) {
    int64_t src = 0;
    for (int a = 0; a < g.rank; ++a) src = src * g.shape[a] + ob[a] * g.patch[a] + idx[a];
    s = __dadd_rn(s, (double)X[p * n_in + src]);
    ++cnt;
    int a = g.rank - 1;
    for (; a >= 0; --a) {
      if (++idx[a] < g.patch[a]) break;
      idx[a] = 0;
    }
    more = a >= 0;
  }
  Y[e] = __ddiv_rn(s, (double)cnt);
}

Geometry make_geometry(int rank, const int64_t* shape, const int64_t* patch, const int64_t* nstarts) {
  Geometry g{};
  g.rank = rank;
  int64_t off = 0;
  for (int a = 0; a < rank; ++a) {
    g.shape[a] = shape[a];
    g.patch[a] = patch[a];
    g.nstarts[a] = nstarts ? nstarts[a] : 0;
    g.soff[a] = off;
    off += g.nstarts[a];
  }
  return g;
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t launch_extract(const float* t, int rank, const int64_t* shape, const int64_t* patch,
                           const int64_t* nstarts, const int64_t* starts_dev, float* out, cudaStream_t st) {
  const Geometry g = make_geometry(rank, shape, patch, nstarts);
  int64_t N = 1, n = 1;
  for (int a = 0; a < rank; ++a) {
    N *= nstarts[a];
    n *= patch[a];
  }
  if (N * n == 0) return cudaSuccess;
  extract_kernel<<<blocks_for(N * n), 256, 0, st>>>(t, g, starts_dev, N, n, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_aggregate(const float* patches, int rank, const int64_t* shape, const int64_t* patch,
                             const int64_t* nstarts, const int64_t* starts_dev, float* out, cudaStream_t st) {
  const Geometry g = make_geometry(rank, shape, patch, nstarts);
  int64_t cells = 1, n = 1;
  for (int a = 0; a < rank; ++a) {
    cells *= shape[a];
    n *= patch[a];
  }
  if (cells == 0) return cudaSuccess;
  aggregate_kernel<<<blocks_for(cells), 256, 0, st>>>(patches, g, starts_dev, cells, n, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_row_select(const float* X, int64_t N, int n_in, const int64_t* rows_dev, int n_out, double* Y,
                              cudaStream_t st) {
  if (N * n_out == 0) return cudaSuccess;
  row_select_kernel<<<blocks_for(N * n_out), 256, 0, st>>>(X, N, n_in, rows_dev, n_out, Y);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_coded_exposure(const float* X, int64_t N, int n_in, const float* mask_dev, int pixels,
                                  int windows, int frames, double* Y, cudaStream_t st) {
  const int64_t total = N * pixels * windows;
  if (total == 0) return cudaSuccess;
  coded_exposure_kernel<<<blocks_for(total), 256, 0, st>>>(X, N, n_in, mask_dev, pixels, windows, frames, Y);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_average(const float* X, int64_t N, int rank, const int64_t* in_shape,
                                 const int64_t* factors, double* Y, cudaStream_t st) {
  const Geometry g = make_geometry(rank, in_shape, factors, nullptr);
  int n_in = 1, n_out = 1;
  for (int a = 0; a < rank; ++a) {
    n_in *= (int)in_shape[a];
    n_out *= (int)(in_shape[a] / factors[a]);
  }
  if (N * n_out == 0) return cudaSuccess;
  block_average_kernel<<<blocks_for(N * n_out), 256, 0, st>>>(X, N, n_in, g, Y, n_out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace stmp
