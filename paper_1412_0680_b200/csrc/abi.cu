// extern "C" boundary of the STMP B200 library (declared in include/stmp_b200.h).
// Validation mirrors the reference's error behaviour:
// ValueError cases -> STMP_EINVAL, fingerprint mismatch -> STMP_ESTALE,
// CUDA failures -> STMP_ECUDA.  No CPU fallback exists.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/stmp_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "staged.cuh"

struct stmp_dict : stmp::DictHandle {};
struct stmp_tree : stmp::TreeHandle {};

namespace {

thread_local std::string g_err;
int g_path_mode = 0;          // 0 auto, 1 fused warp-per-patch, 2 staged tensor-core
int64_t g_staged_min = 4096;  // auto: staged path from this batch size on (c0: 0.19 vs 0.41 ms at 10,000)
int64_t g_exact_min = 512;    // auto: tensor-core exhaustive scan from this batch size on
int g_graphs = 1;             // replay repeated staged encodes as CUDA graphs

// CUDA-graph cache of staged encodes.  A call whose every argument (handles,
// buffers, sizes, stream) and kernel option matches a previous one is replayed
// from an instantiated graph: the second occurrence is captured, later ones
// only launch.  Removes the ~60 host launches per encode from the critical path
// of small batches and of the chunked host-buffer path.
struct GraphKey {
  const void* p[14];
  int64_t v[16];
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  bool seen = false;
  uint64_t stamp = 0;
};
std::mutex g_graph_mu;
GraphEntry g_graph_cache[32];   // host path: 3 streams x ramped chunk sizes
uint64_t g_graph_clock = 0;
std::atomic<uint64_t> g_generation{0};   // handle ids: a freed handle's id is never reused

// Drop every cached graph that was built for handle generation `gen` (called
// when a dictionary or tree is freed: its graphs reference its device memory).
void purge_graphs(uint64_t gen) {
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (GraphEntry& ge : g_graph_cache) {
    if (!ge.seen) continue;
    if ((uint64_t)ge.key.v[8] == gen || (uint64_t)ge.key.v[10] == gen) {
      if (ge.exec) cudaGraphExecDestroy(ge.exec);
      ge = GraphEntry();
    }
  }
}

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(STMP_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define STMP_CUDA(call, what)                   \
  do {                                          \
    cudaError_t _e = (call);                    \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

int check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "no CUDA device (the B200 path has no CPU fallback)");
  int major = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  if (major != 10)
    return fail(STMP_ECUDA, "device compute capability %d.x: this library is built for sm_100a only", major);
  return STMP_OK;
}

// Device staging of the host-buffer entry point, one per stream, grown on demand.
struct HostStage {
  cudaStream_t st = nullptr;
  int64_t cap_rows = 0;
  int cap_n = 0, cap_K = 0;
  size_t cap_ws = 0;
  float* dX = nullptr;
  int32_t* dI = nullptr;
  float* dC = nullptr;
  int32_t* dN = nullptr;
  float* dR = nullptr;
  int32_t* dP = nullptr;
  void* dW = nullptr;
};
constexpr int kHostStreams = 3;
std::mutex g_host_mutex;
HostStage g_host[kHostStreams];

int ensure_stage(HostStage& h, int64_t rows, int n, int K, size_t ws) {
  if (h.st == nullptr) STMP_CUDA(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking), "stream create");
  if (rows > h.cap_rows || n > h.cap_n || K > h.cap_K) {
    cudaStreamSynchronize(h.st);
    cudaFree(h.dX); cudaFree(h.dI); cudaFree(h.dC); cudaFree(h.dN); cudaFree(h.dR); cudaFree(h.dP);
    h.cap_rows = std::max(rows, h.cap_rows);
    h.cap_n = std::max(n, h.cap_n);
    h.cap_K = std::max(K, h.cap_K);
    STMP_CUDA(cudaMalloc(&h.dX, h.cap_rows * h.cap_n * sizeof(float)), "staging alloc");
    STMP_CUDA(cudaMalloc(&h.dI, h.cap_rows * h.cap_K * sizeof(int32_t)), "staging alloc");
    STMP_CUDA(cudaMalloc(&h.dC, h.cap_rows * h.cap_K * sizeof(float)), "staging alloc");
    STMP_CUDA(cudaMalloc(&h.dN, h.cap_rows * sizeof(int32_t)), "staging alloc");
    STMP_CUDA(cudaMalloc(&h.dR, h.cap_rows * sizeof(float)), "staging alloc");
    STMP_CUDA(cudaMalloc(&h.dP, h.cap_rows * 2 * sizeof(int32_t)), "staging alloc");
  }
  if (ws > h.cap_ws) {
    cudaStreamSynchronize(h.st);
    cudaFree(h.dW);
    STMP_CUDA(cudaMalloc(&h.dW, ws), "workspace alloc");
    h.cap_ws = ws;
  }
  return STMP_OK;
}

// pursuit.py:29-33
int retained_count(double alpha, int k) {
  int c = (int)ceil(alpha * k - 1e-9);
  return c < 1 ? 1 : c;
}

}  // namespace

extern "C" {

const char* stmp_version(void) { return "stmp_b200 0.1.0 (sm_100a)"; }

const char* stmp_last_error(void) { return g_err.c_str(); }

uint64_t stmp_fnv1a64(const void* data, size_t len, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}

int stmp_kernel_launches(int64_t* out) {
  if (out == nullptr) return fail(STMP_EINVAL, "null output");
  *out = stmp::launch_counter().load(std::memory_order_relaxed);
  return STMP_OK;
}

int stmp_kernel_timing(int32_t enable) {
  g_err.clear();
  stmp::KernelTimer& kt = stmp::kernel_timer();
  for (auto& r : kt.recs) {
    kt.pool.push_back(r.e0);
    kt.pool.push_back(r.e1);
  }
  kt.recs.clear();
  kt.on = enable != 0;
  return STMP_OK;
}

int stmp_kernel_times(int32_t max_entries, char* names, int32_t name_len, int64_t* launches, double* total_ms,
                      int32_t* n_entries) {
  g_err.clear();
  if (n_entries == nullptr || (max_entries > 0 && (names == nullptr || launches == nullptr || total_ms == nullptr)) ||
      name_len < 2)
    return fail(STMP_EINVAL, "NULL output or name_len < 2");
  stmp::KernelTimer& kt = stmp::kernel_timer();
  std::vector<const void*> fns;
  std::vector<int64_t> cnt;
  std::vector<double> ms;
  for (auto& r : kt.recs) {
    cudaError_t e = cudaEventSynchronize(r.e1);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.e0, r.e1);
    if (e != cudaSuccess) return cuda_fail(e, "kernel timing");
    size_t i = 0;
    while (i < fns.size() && fns[i] != r.fn) ++i;
    if (i == fns.size()) {
      fns.push_back(r.fn);
      cnt.push_back(0);
      ms.push_back(0.0);
    }
    cnt[i] += 1;
    ms[i] += t;
  }
  *n_entries = (int32_t)fns.size();
  for (size_t i = 0; i < fns.size() && (int32_t)i < max_entries; ++i) {
    const char* nm = nullptr;
    if (cudaFuncGetName(&nm, fns[i]) != cudaSuccess || nm == nullptr) nm = "?";
    snprintf(names + i * name_len, (size_t)name_len, "%s", nm);
    launches[i] = cnt[i];
    total_ms[i] = ms[i];
  }
  return STMP_OK;
}

int stmp_stream_sync(void* stream) {
  STMP_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
  return STMP_OK;
}

int stmp_dict_create(const float* atoms, int64_t m, int32_t n, int32_t atoms_on_device,
                     uint64_t fingerprint, void* stream, stmp_dict** out) {
  g_err.clear();
  if (out == nullptr) return fail(STMP_EINVAL, "out handle pointer is NULL");
  *out = nullptr;
  if (atoms == nullptr || m <= 0 || n <= 0)
    return fail(STMP_EINVAL, "atoms must form a non-empty 2-D array, got shape (%lld, %d)",
                (long long)m, n);
  if (m > 0x7fffffffLL) return fail(STMP_EINVAL, "atom count %lld exceeds 2^31-1", (long long)m);
  const int vpl = stmp::fused_vpl_for(n);
  if (vpl < 0) return fail(STMP_EINVAL, "atom dimension %d exceeds the supported maximum 2048", n);
  if (int rc = check_device()) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  stmp_dict* d = new stmp_dict();
  d->m = m;
  d->n = n;
  d->vpl = vpl;
  d->ld = 32 * vpl;
  d->fingerprint = fingerprint;
  d->generation = ++g_generation;
  const size_t bytes = (size_t)m * d->ld * sizeof(float);
  cudaError_t e = cudaMalloc(&d->atoms, bytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(d->atoms, 0, bytes, s);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(d->atoms, d->ld * sizeof(float), atoms, (size_t)n * sizeof(float),
                          (size_t)n * sizeof(float), (size_t)m,
                          atoms_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(d->atoms);
    delete d;
    return cuda_fail(e, "dictionary upload");
  }
  *out = d;
  return STMP_OK;
}

void stmp_dict_free(stmp_dict* d) {
  if (d == nullptr) return;
  purge_graphs(d->generation);
  cudaFree(d->atoms);
  cudaFree(d->xtable);
  cudaFree(d->xtable16);
  delete d;
}

int stmp_dict_info(const stmp_dict* d, int64_t* m, int32_t* n, int32_t* ld, uint64_t* fp) {
  if (d == nullptr) return fail(STMP_EINVAL, "dictionary handle is NULL");
  if (m) *m = d->m;
  if (n) *n = d->n;
  if (ld) *ld = d->ld;
  if (fp) *fp = d->fingerprint;
  return STMP_OK;
}

int stmp_tree_create(const stmp_dict* d, int32_t levels, const int32_t* branching,
                     const int64_t* level_offsets, const int32_t* child_begin,
                     const int32_t* child_count, const float* centroids, int64_t num_leaves,
                     const int32_t* leaf_atom, uint64_t fingerprint, void* stream,
                     stmp_tree** out) {
  g_err.clear();
  if (out == nullptr) return fail(STMP_EINVAL, "out handle pointer is NULL");
  *out = nullptr;
  if (d == nullptr) return fail(STMP_EINVAL, "dictionary handle is NULL");
  if (fingerprint != d->fingerprint)
    return fail(STMP_ESTALE, "tree fingerprint %#018llx does not match dictionary fingerprint %#018llx",
                (unsigned long long)fingerprint, (unsigned long long)d->fingerprint);
  if (levels < 1) return fail(STMP_EINVAL, "branching must name at least one level");
  if (!branching || !level_offsets || !child_begin || !child_count || !centroids || !leaf_atom)
    return fail(STMP_EINVAL, "tree arrays must not be NULL");
  for (int l = 0; l < levels; ++l)
    if (branching[l] < 2)
      return fail(STMP_EINVAL, "branching entry %d at level %d must be at least 2", branching[l], l);
  if (level_offsets[0] != 0 || level_offsets[1] != 1) return fail(STMP_EINVAL, "tree must have one root");
  const int64_t ni = level_offsets[levels + 1];
  // structural checks: BFS contiguity, non-empty nodes, leaf coverage
  for (int dd = 0; dd <= levels; ++dd) {
    int64_t expect = dd < levels ? level_offsets[dd + 1] : 0;
    for (int64_t v = level_offsets[dd]; v < level_offsets[dd + 1]; ++v) {
      if (child_count[v] < 1) return fail(STMP_EINVAL, "internal node %lld has no children", (long long)v);
      if (child_begin[v] != expect)
        return fail(STMP_EINVAL, "children of node %lld are not contiguous in BFS order", (long long)v);
      expect += child_count[v];
    }
    const int64_t end = dd < levels ? level_offsets[dd + 2] : num_leaves;
    if (expect != end) return fail(STMP_EINVAL, "child counts at depth %d do not cover the next level", dd);
  }
  for (int64_t j = 0; j < num_leaves; ++j)
    if (leaf_atom[j] < 0 || leaf_atom[j] >= d->m)
      return fail(STMP_EINVAL, "leaf atom index %d outside [0, %lld)", leaf_atom[j], (long long)d->m);
  if (int rc = check_device()) return rc;

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  stmp_tree* t = new stmp_tree();
  t->levels = levels;
  t->branching.assign(branching, branching + levels);
  t->level_offsets.assign(level_offsets, level_offsets + levels + 2);
  t->num_internal = ni;
  t->num_leaves = num_leaves;
  t->n = d->n;
  t->ld = d->ld;
  t->fingerprint = fingerprint;
  t->generation = ++g_generation;
  t->dict = d;
  t->root_children = child_count[0];
  for (int64_t v = 0; v < ni; ++v) t->max_children = std::max(t->max_children, child_count[v]);
  for (int64_t v = level_offsets[levels]; v < ni; ++v)
    t->max_leaf_children = std::max(t->max_leaf_children, child_count[v]);
  cudaError_t e = cudaMalloc(&t->child_begin, ni * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->child_count, ni * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->leaf_atom, num_leaves * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->cent, (size_t)ni * t->ld * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->child_begin, child_begin, ni * sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->child_count, child_count, ni * sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->leaf_atom, leaf_atom, num_leaves * sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(t->cent, 0, (size_t)ni * t->ld * sizeof(float), s);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(t->cent, t->ld * sizeof(float), centroids, (size_t)t->n * sizeof(float),
                          (size_t)t->n * sizeof(float), (size_t)ni, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    stmp_tree_free(t);
    return cuda_fail(e, "tree upload");
  }
  std::string berr;
  if (!stmp::build_staged_tables(t, child_begin, child_count, centroids, leaf_atom, s, &berr) && !berr.empty()) {
    stmp_tree_free(t);
    return fail(STMP_ECUDA, "staged table upload: %s", berr.c_str());
  }
  // Gram path (gram_path.cu): each atom must be exactly one depth-L leaf
  if (t->max_leaf_children == 1 && num_leaves == d->m) {
    std::vector<char> seen((size_t)d->m, 0);
    bool unique = true;
    for (int64_t j = 0; j < num_leaves && unique; ++j) unique = !seen[leaf_atom[j]]++;
    if (unique && !stmp::build_leaf_pos(t, d->m, s)) cudaGetLastError();
  }
  *out = t;
  return STMP_OK;
}

void stmp_tree_free(stmp_tree* t) {
  if (t == nullptr) return;
  purge_graphs(t->generation);
  cudaFree(t->child_begin);
  cudaFree(t->child_count);
  cudaFree(t->leaf_atom);
  cudaFree(t->cent);
  stmp::free_staged_tables(t);
  stmp::free_pair_tables(t);
  delete t;
}

// Beam descent (retained_count(alpha, k_l) > 1 at some level, pursuit.py:141-153):
// children kept per level and a bound on the frontier size.  Returns false for
// greedy alpha (one child per level).
static bool beam_plan(const stmp_tree* t, double alpha, int* keep, int* max_frontier) {
  if (t == nullptr || !(alpha > 0.0 && alpha <= 1.0)) return false;
  bool beam = false;
  int64_t f = 1, mx = 1;
  for (int l = 0; l < t->levels; ++l) {
    const int k = retained_count(alpha, t->branching[l]);
    if (keep && l < stmp::kMaxBeamLevels) keep[l] = k;
    beam |= k > 1;
    const int64_t nodes = (l + 2 < (int)t->level_offsets.size() ? t->level_offsets[l + 2] - t->level_offsets[l + 1]
                                                                 : t->num_leaves);
    f = std::min<int64_t>(f * std::min(k, t->max_children), nodes);
    mx = std::max(mx, f);
  }
  if (max_frontier) *max_frontier = (int)std::min<int64_t>(mx, 1 << 30);
  return beam;
}

int g_staged_beam = 1;   // beam descent on the staged pipeline where supported (else the fused kernel)

static bool use_staged(const stmp_dict* d, const stmp_tree* t, int64_t N, int32_t K, int32_t method,
                       double alpha = 0.0) {
  if (g_path_mode == 1 || d == nullptr) return false;
  int keep[stmp::kMaxBeamLevels] = {0};
  if (beam_plan(t, alpha, keep, nullptr)) {   // beam descent: staged entries, or the fused kernel
    if (!g_staged_beam || t->levels > stmp::kMaxBeamLevels || !stmp::staged_beam_supported(d, t, K, method, keep))
      return false;
    return g_path_mode == 2 || N >= g_staged_min;
  }
  if (!stmp::staged_supported(d, t, K, method)) return false;
  // exhaustive selection: the tensor-core scan wins as soon as one tile fills an SM
  return g_path_mode == 2 || N >= (t == nullptr ? g_exact_min : g_staged_min);
}

int stmp_set_option(const char* key, int64_t value) {
  g_err.clear();
  if (key == nullptr) return fail(STMP_EINVAL, "option key is NULL");
  if (strcmp(key, "path") == 0) {
    if (value < 0 || value > 2) return fail(STMP_EINVAL, "path must be 0 (auto), 1 (fused) or 2 (staged)");
    g_path_mode = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "root_direct") == 0) {
    if (value < 0 || value > 1) return fail(STMP_EINVAL, "root_direct must be 0 or 1");
    stmp::g_root_direct = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "graphs") == 0) {
    if (value < 0 || value > 1) return fail(STMP_EINVAL, "graphs must be 0 or 1");
    g_graphs = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "pdl") == 0) {
    if (value < 0 || value > 1) return fail(STMP_EINVAL, "pdl must be 0 or 1");
    stmp::g_pdl = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "update_kernel") == 0) {
    if (value < 0 || value > 1)
      return fail(STMP_EINVAL, "update_kernel must be 0 (generic) or 1 (lockstep / wide-row OMP)");
    stmp::g_update_omp8 = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "score_kernel") == 0) {
    if (value < 2 || value > 4)
      return fail(STMP_EINVAL, "score_kernel must be 2 (node table in shared memory), 3 (streamed table) or "
                               "4 (streamed table, 3xFP16 split)");
    stmp::g_score_ws = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "gram_path") == 0) {
    if (value < 0 || value > 2) return fail(STMP_EINVAL, "gram_path must be 0 (off), 1 (auto) or 2 (when supported)");
    stmp::g_gram_path = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "half_scores") == 0) {
    if (value < 0 || value > 1)
      return fail(STMP_EINVAL, "half_scores must be 0 (fp32 rows) or 1 (fp16 rows on the Gram path's level passes)");
    stmp::g_half_scores = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "staged_beam") == 0) {
    if (value < 0 || value > 1) return fail(STMP_EINVAL, "staged_beam must be 0 or 1");
    g_staged_beam = (int)value;
    return STMP_OK;
  }
  if (strcmp(key, "staged_min_batch") == 0) {
    if (value < 1) return fail(STMP_EINVAL, "staged_min_batch must be positive");
    g_staged_min = value;
    return STMP_OK;
  }
  return fail(STMP_EINVAL, "unknown option '%s'", key);
}

size_t stmp_encode_workspace(const stmp_dict* d, const stmp_tree* t, int64_t N, int32_t K,
                             int32_t method, double alpha) {
  if (N <= 0 || d == nullptr) return 0;
  int mf = 0;
  int keep[stmp::kMaxBeamLevels] = {0};
  if (beam_plan(t, alpha, keep, &mf)) {
    if (use_staged(d, t, N, K, method, alpha)) return stmp::staged_beam_workspace(d, t, N, K, method, keep);
    return (size_t)stmp::fused_warps(N) * (size_t)stmp::beam_scratch_ints(mf) * sizeof(int);
  }
  if (!use_staged(d, t, N, K, method, alpha)) return 0;
  return stmp::staged_workspace_bytes(d, t, N, K, method);
}

static int validate_encode(const stmp_dict* d, const stmp_tree* t, int64_t N, int64_t ldx,
                           int32_t K, int32_t method, double alpha, double tol_abs) {
  if (d == nullptr) return fail(STMP_EINVAL, "dictionary handle is NULL");
  if (N < 0) return fail(STMP_EINVAL, "patch count must be non-negative, got %lld", (long long)N);
  if (ldx < d->n) return fail(STMP_EINVAL, "row stride %lld below atom dimension %d", (long long)ldx, d->n);
  if (K < 1) return fail(STMP_EINVAL, "sparsity K must be at least 1, got %d", K);
  if (K > STMP_MAX_K) return fail(STMP_EINVAL, "sparsity K=%d exceeds the GPU maximum %d", K, STMP_MAX_K);
  if (method != STMP_METHOD_MP && method != STMP_METHOD_OMP && method != STMP_METHOD_SELECT)
    return fail(STMP_EINVAL, "unknown method %d", method);
  if (method == STMP_METHOD_OMP && K > d->n)
    return fail(STMP_EINVAL, "support size %d exceeds atom dimension %d", K, d->n);
  if (std::isnan(tol_abs)) return fail(STMP_EINVAL, "residual tolerance is NaN");
  if (t != nullptr) {
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(STMP_EINVAL, "alpha must lie in (0, 1], got %g", alpha);
    if (t->fingerprint != d->fingerprint)
      return fail(STMP_ESTALE, "tree fingerprint %#018llx does not match dictionary fingerprint %#018llx",
                  (unsigned long long)t->fingerprint, (unsigned long long)d->fingerprint);
    if (t->dict != d && t->n != d->n) return fail(STMP_EINVAL, "tree dimension differs from dictionary");
    if (beam_plan(t, alpha, nullptr, nullptr) && t->levels > stmp::kMaxBeamLevels)
      return fail(STMP_EINVAL, "beam descent supports at most %d tree levels, got %d", stmp::kMaxBeamLevels,
                  t->levels);
  }
  return STMP_OK;
}

int stmp_encode(const stmp_dict* d, const stmp_tree* t, const float* X, int64_t N, int64_t ldx,
                int32_t K, int32_t method, double alpha, double tol_abs, int32_t* idx, float* coef,
                int32_t* count, float* resnorm, int32_t* path, int32_t* ip, void* workspace,
                size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (int rc = validate_encode(d, t, N, ldx, K, method, alpha, tol_abs)) return rc;
  if (N == 0) return STMP_OK;
  if (X == nullptr || idx == nullptr || coef == nullptr || count == nullptr || resnorm == nullptr)
    return fail(STMP_EINVAL, "X, idx, coef, count and resnorm must be device pointers");
  if (reinterpret_cast<uintptr_t>(ip) % 8 != 0)
    return fail(STMP_EINVAL, "ip must be 8-byte aligned (its two counters are updated as one 64-bit word)");
  if (use_staged(d, t, N, K, method, alpha)) {
    int keep[stmp::kMaxBeamLevels] = {0};
    int mf = 0;
    const bool beam = beam_plan(t, alpha, keep, &mf);
    const size_t need = beam ? stmp::staged_beam_workspace(d, t, N, K, method, keep)
                             : stmp::staged_workspace_bytes(d, t, N, K, method);
    if (workspace == nullptr || workspace_bytes < need)
      return fail(STMP_EINVAL, "workspace of %zu bytes is below the required %zu (stmp_encode_workspace)",
                  workspace_bytes, need);
    const float tol = tol_abs < 0 ? -1.f : (float)tol_abs;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto run = [&] {
      if (beam)
        return stmp::run_staged_beam(d, t, X, N, ldx, K, method, tol, keep, mf, idx, coef, count, resnorm, path, ip,
                                     workspace, workspace_bytes, st);
      return stmp::run_staged(d, t, X, N, ldx, K, method, tol, idx, coef, count, resnorm, path, ip, workspace,
                              workspace_bytes, st);
    };
    // the legacy default stream cannot be captured; timed encodes run eagerly
    if (!g_graphs || stmp::kernel_timer().on || st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) {
      cudaError_t e = run();
      if (e != cudaSuccess) return cuda_fail(e, "staged encode");
      return STMP_OK;
    }
    GraphKey k;
    memset(&k, 0, sizeof(k));
    // handles enter the key by generation, not address: a new handle allocated
    // where a freed one lived must not replay the freed one's graph
    const void* ps[14] = {nullptr, nullptr, X, idx, coef, count, resnorm, path, ip, workspace, stream, nullptr,
                          nullptr, nullptr};
    for (int i = 0; i < 14; ++i) k.p[i] = ps[i];
    const int64_t vs[16] = {N, ldx, K, method, (int64_t)workspace_bytes, stmp::g_root_direct, stmp::g_score_ws,
                            stmp::g_update_omp8, (int64_t)d->generation, stmp::g_pdl,
                            t ? (int64_t)t->generation : 0, 0, stmp::g_gram_path, 0, g_staged_beam, stmp::g_half_scores};
    memcpy(k.v, vs, sizeof(vs));
    memcpy(&k.v[11], &tol, sizeof(float));
    memcpy(&k.v[13], &alpha, sizeof(double));   // beam: the kept children per level
    std::lock_guard<std::mutex> lock(g_graph_mu);
    GraphEntry* hit = nullptr;
    GraphEntry* lru = &g_graph_cache[0];
    for (GraphEntry& ge : g_graph_cache) {
      if (ge.seen && memcmp(&ge.key, &k, sizeof(k)) == 0) hit = &ge;
      if (ge.stamp < lru->stamp) lru = &ge;
    }
    if (hit && hit->exec) {
      hit->stamp = ++g_graph_clock;
      stmp::launch_counter().fetch_add(hit->launches, std::memory_order_relaxed);
      cudaError_t e = cudaGraphLaunch(hit->exec, st);
      if (e != cudaSuccess) return cuda_fail(e, "graph launch");
      return STMP_OK;
    }
    if (hit) {   // second occurrence: capture, instantiate, launch
      const int64_t before = stmp::launch_counter().load();
      cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      cudaGraph_t g = nullptr;
      if (e == cudaSuccess) {
        cudaError_t er = run();
        e = cudaStreamEndCapture(st, &g);
        if (e == cudaSuccess) e = er;
      }
      cudaGraphExec_t exec = nullptr;
      if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, g, 0);
      if (g) cudaGraphDestroy(g);
      if (e == cudaSuccess) {
        hit->exec = exec;
        hit->launches = stmp::launch_counter().load() - before;
        hit->stamp = ++g_graph_clock;
        e = cudaGraphLaunch(exec, st);
        if (e != cudaSuccess) return cuda_fail(e, "graph launch");
        return STMP_OK;
      }
      // capture unsupported here: forget the entry and run eagerly
      cudaGetLastError();
      stmp::launch_counter().store(before);
      hit->seen = false;
      e = run();
      if (e != cudaSuccess) return cuda_fail(e, "staged encode");
      return STMP_OK;
    }
    if (lru->exec) cudaGraphExecDestroy(lru->exec);
    lru->exec = nullptr;
    lru->key = k;
    lru->seen = true;
    lru->stamp = ++g_graph_clock;
    cudaError_t e = run();
    if (e != cudaSuccess) return cuda_fail(e, "staged encode");
    return STMP_OK;
  }
  stmp::FusedArgs a{};
  a.X = X;
  a.N = N;
  a.ldx = ldx;
  a.n = d->n;
  a.atoms = d->atoms;
  a.m = d->m;
  a.ld = d->ld;
  a.vpl = d->vpl;
  a.has_tree = t != nullptr;
  if (t) a.tree = stmp::TreeView{t->child_begin, t->child_count, t->cent, t->leaf_atom, t->levels};
  else a.tree = stmp::TreeView{nullptr, nullptr, nullptr, nullptr, 0};
  a.K = K;
  a.method = method;
  a.tol_abs = tol_abs < 0 ? -1.f : (float)tol_abs;
  a.beam = beam_plan(t, alpha, a.keep, &a.max_frontier) ? 1 : 0;
  if (a.beam) {
    const size_t need = (size_t)stmp::fused_warps(N) * (size_t)stmp::beam_scratch_ints(a.max_frontier) * sizeof(int);
    if (workspace == nullptr || workspace_bytes < need)
      return fail(STMP_EINVAL, "beam descent needs a workspace of %zu bytes (stmp_encode_workspace), got %zu", need,
                  workspace_bytes);
    a.scratch = static_cast<int*>(workspace);
  }
  a.idx = idx;
  a.coef = coef;
  a.count = count;
  a.resnorm = resnorm;
  a.path = t ? path : nullptr;
  a.ip = ip;
  const int wpb = 8;
  const size_t atom_cache = (size_t)K * d->ld;
  const size_t base_ws = (size_t)K * (K + 1) / 2 + 4 * (size_t)K;
  a.cache_atoms = (method == STMP_METHOD_OMP && atom_cache * 4 <= 8192) ? 1 : 0;
  a.warp_smem_floats = (int)(((base_ws + (a.cache_atoms ? atom_cache : 0)) + 3) / 4 * 4);
  a.root_smem_rows = 0;
  a.root_begin = 1;
  if (t) {
    const size_t root_bytes = (size_t)t->root_children * t->ld * 4;
    if (root_bytes <= 48 * 1024) a.root_smem_rows = t->root_children;
  }
  const size_t smem = 4 * ((size_t)a.root_smem_rows * a.ld + (size_t)wpb * a.warp_smem_floats);
  if (smem > 200 * 1024) return fail(STMP_EINVAL, "K=%d needs too much shared memory", K);
  cudaError_t e = stmp::launch_encode_fused(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "encode launch");
  return STMP_OK;
}

int stmp_encode_host(const stmp_dict* d, const stmp_tree* t, const float* X, int64_t N,
                     int64_t ldx, int32_t K, int32_t method, double alpha, double tol_abs,
                     int32_t* idx, float* coef, int32_t* count, float* resnorm, int32_t* ip,
                     int64_t chunk) {
  g_err.clear();
  if (int rc = validate_encode(d, t, N, ldx, K, method, alpha, tol_abs)) return rc;
  if (N == 0) return STMP_OK;
  if (X == nullptr || idx == nullptr || coef == nullptr || count == nullptr || resnorm == nullptr)
    return fail(STMP_EINVAL, "X, idx, coef, count and resnorm must be host pointers");
  if (chunk <= 0) chunk = 1 << 17;
  if (chunk > N) chunk = N;
  // Persistent staging: device buffers and streams are kept between calls
  // (allocating ~1 GB of workspace per call would dominate the host path).
  std::lock_guard<std::mutex> lock(g_host_mutex);
  const size_t wsz = stmp_encode_workspace(d, t, chunk, K, method, alpha);
  for (int i = 0; i < kHostStreams; ++i)
    if (int rc = ensure_stage(g_host[i], chunk, d->n, K, wsz)) return rc;
  // Chunk schedule: ramp up (chunk/4, chunk/2) so the first encode starts
  // after a short copy, full chunks in the middle, ramp down at the end so the
  // last encode + D2H (the part no copy overlaps) is short.
  std::vector<int64_t> sizes;
  if (N >= 4 * chunk && chunk >= 4096) {
    const int64_t ramp[2] = {chunk / 4, chunk / 2};
    int64_t mid = N - 2 * (ramp[0] + ramp[1]);
    sizes.push_back(ramp[0]);
    sizes.push_back(ramp[1]);
    for (; mid > 0; mid -= chunk) sizes.push_back(std::min(chunk, mid));
    sizes.push_back(ramp[1]);
    sizes.push_back(ramp[0]);
  } else {
    for (int64_t s0 = 0; s0 < N; s0 += chunk) sizes.push_back(std::min(chunk, N - s0));
  }
  int rc = STMP_OK;
  int64_t s0 = 0;
  for (size_t ci = 0; ci < sizes.size() && rc == STMP_OK; s0 += sizes[ci], ++ci) {
    HostStage& h = g_host[ci % kHostStreams];
    const int64_t rows = sizes[ci];
    cudaError_t e = ldx == d->n
        ? cudaMemcpyAsync(h.dX, X + s0 * ldx, rows * d->n * sizeof(float), cudaMemcpyHostToDevice, h.st)
        : cudaMemcpy2DAsync(h.dX, d->n * sizeof(float), X + s0 * ldx, ldx * sizeof(float),
                            d->n * sizeof(float), rows, cudaMemcpyHostToDevice, h.st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D"); break; }
    rc = stmp_encode(d, t, h.dX, rows, d->n, K, method, alpha, tol_abs, h.dI, h.dC, h.dN, h.dR,
                     nullptr, h.dP, h.dW, h.cap_ws, h.st);
    if (rc != STMP_OK) break;
    e = cudaMemcpyAsync(idx + s0 * K, h.dI, rows * K * sizeof(int32_t), cudaMemcpyDeviceToHost, h.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(coef + s0 * K, h.dC, rows * K * sizeof(float), cudaMemcpyDeviceToHost, h.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(count + s0, h.dN, rows * sizeof(int32_t), cudaMemcpyDeviceToHost, h.st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(resnorm + s0, h.dR, rows * sizeof(float), cudaMemcpyDeviceToHost, h.st);
    if (e == cudaSuccess && ip) e = cudaMemcpyAsync(ip + 2 * s0, h.dP, rows * 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, h.st);
    if (e != cudaSuccess) rc = cuda_fail(e, "D2H");
  }
  for (int i = 0; i < kHostStreams; ++i) {
    cudaError_t e = cudaStreamSynchronize(g_host[i].st);
    if (e != cudaSuccess && rc == STMP_OK) rc = cuda_fail(e, "encode_host sync");
  }
  return rc;
}

int stmp_dc_split(const float* Y, int64_t N, int64_t ldy, int32_t n, const double* dc_meas, double denom,
                  float* Yc, int64_t ldc, double* dc, void* stream) {
  g_err.clear();
  if (N < 0) return fail(STMP_EINVAL, "patch count must be non-negative, got %lld", (long long)N);
  if (n < 1) return fail(STMP_EINVAL, "measurement dimension must be positive, got %d", n);
  if (ldy < n || ldc < n) return fail(STMP_EINVAL, "row stride below the measurement dimension %d", n);
  if (!(denom > 0.0)) return fail(STMP_EINVAL, "dc_meas . dc_meas must be positive, got %g", denom);
  if (N > 0 && (Y == nullptr || dc_meas == nullptr || Yc == nullptr || dc == nullptr))
    return fail(STMP_EINVAL, "NULL buffer");
  if (int rc = check_device()) return rc;
  cudaError_t e = stmp::launch_dc_split(Y, N, ldy, n, dc_meas, denom, Yc, ldc, dc, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "dc_split");
  return STMP_OK;
}

int stmp_reconstruct(const stmp_dict* base, const int32_t* idx, const float* coef, const int32_t* count, int64_t N,
                     int32_t K, const double* scale, const double* dc, double* out, int64_t ldo, void* stream) {
  g_err.clear();
  if (base == nullptr) return fail(STMP_EINVAL, "dictionary handle is NULL");
  if (N < 0) return fail(STMP_EINVAL, "patch count must be non-negative, got %lld", (long long)N);
  if (K < 1) return fail(STMP_EINVAL, "sparsity K must be at least 1, got %d", K);
  if (ldo < base->n) return fail(STMP_EINVAL, "output row stride below the atom dimension %d", base->n);
  if (N > 0 && (idx == nullptr || coef == nullptr || count == nullptr || out == nullptr))
    return fail(STMP_EINVAL, "NULL buffer");
  if (int rc = check_device()) return rc;
  cudaError_t e = stmp::launch_reconstruct(base, idx, coef, count, N, K, scale, dc, out, ldo,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "reconstruct");
  return STMP_OK;
}

static int check_geometry(int32_t rank, const int64_t* shape, const int64_t* patch, const int64_t* nstarts) {
  if (rank < 1 || rank > stmp::kMaxRank) return fail(STMP_EINVAL, "rank must lie in [1, %d], got %d", stmp::kMaxRank, rank);
  if (shape == nullptr || patch == nullptr || nstarts == nullptr) return fail(STMP_EINVAL, "NULL geometry array");
  for (int a = 0; a < rank; ++a) {
    if (shape[a] < 1 || patch[a] < 1 || nstarts[a] < 1)
      return fail(STMP_EINVAL, "non-positive extent on axis %d", a);
    if (patch[a] > shape[a])
      return fail(STMP_EINVAL, "patch extent %lld exceeds tensor extent %lld on axis %d", (long long)patch[a],
                  (long long)shape[a], a);
  }
  return STMP_OK;
}

int stmp_extract_patches(const float* t, int32_t rank, const int64_t* shape, const int64_t* patch,
                         const int64_t* nstarts, const int64_t* starts, float* out, void* stream) {
  g_err.clear();
  if (int rc = check_geometry(rank, shape, patch, nstarts)) return rc;
  if (t == nullptr || starts == nullptr || out == nullptr) return fail(STMP_EINVAL, "NULL buffer");
  if (int rc = check_device()) return rc;
  cudaError_t e = stmp::launch_extract(t, rank, shape, patch, nstarts, starts, out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "extract_patches");
  return STMP_OK;
}

int stmp_aggregate_patches(const float* patches, int32_t rank, const int64_t* shape, const int64_t* patch,
                           const int64_t* nstarts, const int64_t* starts, float* out, void* stream) {
  g_err.clear();
  if (int rc = check_geometry(rank, shape, patch, nstarts)) return rc;
  if (patches == nullptr || starts == nullptr || out == nullptr) return fail(STMP_EINVAL, "NULL buffer");
  if (int rc = check_device()) return rc;
  cudaError_t e = stmp::launch_aggregate(patches, rank, shape, patch, nstarts, starts, out,
                                         static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "aggregate_patches");
  return STMP_OK;
}

int stmp_apply_operator(int32_t kind, const float* X, int64_t N, int32_t n_in, const int64_t* rows, int32_t n_rows,
                        const float* mask, int32_t pixels, int32_t windows, int32_t frames, int32_t rank,
                        const int64_t* in_shape, const int64_t* factors, double* Y, void* stream) {
  g_err.clear();
  if (N < 0) return fail(STMP_EINVAL, "patch count must be non-negative, got %lld", (long long)N);
  if (n_in < 1) return fail(STMP_EINVAL, "operator input dimension must be positive, got %d", n_in);
  if (N > 0 && (X == nullptr || Y == nullptr)) return fail(STMP_EINVAL, "NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  switch (kind) {
    case STMP_OP_ROW_SELECT:
      if (rows == nullptr || n_rows < 1) return fail(STMP_EINVAL, "row selection keeps no coordinates");
      if (int rc = check_device()) return rc;
      e = stmp::launch_row_select(X, N, n_in, rows, n_rows, Y, st);
      break;
    case STMP_OP_CODED_EXPOSURE:
      if (mask == nullptr || pixels < 1 || windows < 1 || frames < 1 ||
          (int64_t)pixels * windows * frames != n_in)
        return fail(STMP_EINVAL, "coded exposure geometry %d x %d x %d does not match dimension %d", pixels, windows,
                    frames, n_in);
      if (int rc = check_device()) return rc;
      e = stmp::launch_coded_exposure(X, N, n_in, mask, pixels, windows, frames, Y, st);
      break;
    case STMP_OP_BLOCK_AVERAGE: {
      if (rank < 1 || rank > stmp::kMaxRank || in_shape == nullptr || factors == nullptr)
        return fail(STMP_EINVAL, "block average needs 1..%d axes", stmp::kMaxRank);
      int64_t prod = 1;
      for (int a = 0; a < rank; ++a) {
        if (factors[a] < 1 || in_shape[a] % factors[a] != 0)
          return fail(STMP_EINVAL, "factor %lld must divide extent %lld", (long long)factors[a], (long long)in_shape[a]);
        prod *= in_shape[a];
      }
      if (prod != n_in) return fail(STMP_EINVAL, "block shape does not match dimension %d", n_in);
      if (int rc = check_device()) return rc;
      e = stmp::launch_block_average(X, N, rank, in_shape, factors, Y, st);
      break;
    }
    default:
      return fail(STMP_EINVAL, "unknown operator kind %d", kind);
  }
  if (e != cudaSuccess) return cuda_fail(e, "apply_operator");
  return STMP_OK;
}

}  // extern "C"
