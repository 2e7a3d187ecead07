// Shared device helpers and handle layouts for the STMP B200 library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

namespace stmp {

// process-wide count of kernel launches (stmp_kernel_launches)
inline std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}
inline void note_launch() { launch_counter().fetch_add(1, std::memory_order_relaxed); }

// Optional per-launch timing (stmp_kernel_timing / stmp_kernel_times): CUDA
// events recorded on the launch stream right before and after every kernel
// launched through launch_kernel, aggregated per kernel name on request.
// Encodes run eagerly (no graph replay) while it is on.
struct KernelTimer {
  struct Rec {
    const void* fn;
    cudaEvent_t e0, e1;
  };
  bool on = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
inline KernelTimer& kernel_timer() {
  static KernelTimer t;
  return t;
}

// Programmatic dependent launch between the kernels of one encode: a kernel
// launched with `pdl` is set up while its predecessor's last CTAs drain (the
// trigger is the implicit one at CTA exit -- an early explicit trigger let
// successor CTAs crowd out the persistent score kernels and measured slower);
// pdl_enter(), the first statement of every staged kernel, waits for the
// predecessor's completion and memory flush.  Every kernel waits before it can
// complete, so a kernel still sees everything written by all earlier kernels.
extern int g_pdl;

__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && g_pdl) ? 1 : 0;
  note_launch();
  KernelTimer& kt = kernel_timer();
  if (!kt.on) return cudaLaunchKernelEx(&cfg, k, args...);
  KernelTimer::Rec r{reinterpret_cast<const void*>(k), kt.take(), kt.take()};
  cudaEventRecord(r.e0, st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  cudaEventRecord(r.e1, st);
  kt.recs.push_back(r);
  return e;
}

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxRank = 8;   // tensor / patch ranks of the data-format kernels (tensor_ops.cu)

// ScoreCounter update of one patch: both int32 counters {all, centroid} in one
// 64-bit add (the low word never carries: counts stay far below 2^32).
__device__ __forceinline__ void add_ip(int32_t* ip, int64_t p, int all, int cent) {
  atomicAdd(reinterpret_cast<unsigned long long*>(ip + 2 * p),
            ((unsigned long long)(unsigned)cent << 32) | (unsigned)all);
}
constexpr float kRidge = 1e-8f;     // pkg/src/stmp/pursuit.py:249
constexpr float kRelTol = 1e-6f;    // pkg/src/stmp/pursuit.py:209

struct DictHandle {
  float* atoms = nullptr;  // [m, ld] f32, zero-padded columns n..ld
  int64_t m = 0;
  int n = 0;
  int ld = 0;              // padded row stride = 32 * vpl
  int vpl = 0;             // values per lane for the warp-per-patch kernels
  uint64_t fingerprint = 0;
  uint64_t generation = 0; // process-unique id (the graph cache keys on it, never on the address)
  float* xtable = nullptr; // tf32 hi/lo atom blocks for the exhaustive scan (built lazily)
  bool xtable_tried = false;
  uint8_t* xtable16 = nullptr;  // fp16 piece atom blocks for the 3xFP16 exhaustive scan (built lazily)
  bool xtable16_tried = false;
};



struct StagedLevel {
  int npad = 0;       // children per node padded to the UMMA N granularity (16)
  int tmem_cols = 0;  // TMEM columns allocated for the [128 x npad] f32 accumulator
};

struct TreeHandle {
  std::vector<float*> staged_tables;        // per level: [nodes][kchunks][hi|lo][npad x 32] SW128
  std::vector<StagedLevel> staged_levels;
  int levels = 0;
  std::vector<int> branching;
  std::vector<int64_t> level_offsets;  // L+2
  int64_t num_internal = 0;
  int64_t num_leaves = 0;
  int* child_begin = nullptr;   // [num_internal]
  int* child_count = nullptr;   // [num_internal]
  float* cent = nullptr;        // [num_internal, ld]
  int* leaf_atom = nullptr;     // [num_leaves]
  int n = 0, ld = 0;
  int root_children = 0;
  int max_children = 0;         // over all internal nodes
  int max_leaf_children = 0;    // over depth-L nodes
  uint64_t fingerprint = 0;
  uint64_t generation = 0;      // process-unique id (graph cache key)
  const DictHandle* dict = nullptr;
  // Gram path (gram_path.cu): per level l, the [m][nodes at depth l + 1] table of
  // child-centroid . atom products; leaf_pos[a] = column of atom a at the last level
  int leaf_is_atom = -1;        // -1 unknown, 0/1: every depth-L node is one atom equal to its centroid
  std::vector<float*> pair_tables;
  std::vector<int64_t> pair_width;
  int* leaf_pos = nullptr;
  bool pair_tried = false;
  std::vector<uint8_t*> s16_tables;    // per level: [c_a | c_b] fp16 tables of the 3xFP16 pass (score_s16.cu), built on first use
  bool s16_tried = false;
  std::vector<uint8_t*> half_tables;   // per level >= 1: fp16 piece tables (score_sh.cu), built with the pair tables
};

// Device-side view passed to kernels by value.
struct TreeView {
  const int* child_begin;
  const int* child_count;
  const float* cent;
  const int* leaf_atom;
  int levels;
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Ordering key for "max |score|, ties to the lowest id": |s| as IEEE bits is
// order-preserving for non-negative floats; the low word inverts the id so a
// larger key means a smaller id (pursuit.py:108,151,159-161).
__device__ __forceinline__ unsigned long long score_key(float s, unsigned id) {
  return ((unsigned long long)__float_as_uint(fabsf(s)) << 32) |
         (unsigned long long)(0xFFFFFFFFu - id);
}

// Reduce-scatter of 32 per-lane partial sums: afterwards p[0] on lane l holds
// the warp-wide sum of p[l].  31 shuffles instead of 32 x 5.
__device__ __forceinline__ float reduce_scatter32(float (&p)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const float send = upper ? p[j] : p[j + o];
      const float keep = upper ? p[j + o] : p[j];
      p[j] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
  return p[0];
}

}  // namespace stmp
