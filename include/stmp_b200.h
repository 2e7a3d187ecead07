/*
 * stmp_b200.h -- C ABI of the B200-native Shallow Tree Matching Pursuit
 * encoding path (arXiv 1412.0680).
 *
 * The reference (package `stmp`, pure Python + NumPy) has no FFI: its plugin
 * seam is the duck-typed selector protocol consumed by `matching_pursuit`
 * (pkg/src/stmp/pursuit.py:194-221): an object with `.dictionary` and
 * `.select(r, counter) -> (index, signed_score)`.  Each entry point below
 * names the reference interface it replaces; INTEGRATION.md shows the
 * ctypes binding a maintainer adds on the reference side.
 *
 * Conventions:
 *   - plain pointers and sizes only; `stream` is a cudaStream_t (NULL = legacy default);
 *   - every encode/select buffer is a DEVICE pointer owned by the caller; the
 *     library owns only the immutable dictionary / tree handles;
 *   - all device work is asynchronous on `stream`;
 *   - status codes map to the reference's exceptions:
 *       STMP_OK 0, STMP_EINVAL 1 -> ValueError, STMP_ESTALE 2 -> StaleTreeError,
 *       STMP_ECUDA 3 -> RuntimeError; message via stmp_last_error() (thread-local);
 *   - there is no CPU fallback: without a usable sm_100 device every device
 *     entry point returns STMP_ECUDA.
 */
#ifndef STMP_B200_H
#define STMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STMP_OK 0
#define STMP_EINVAL 1
#define STMP_ESTALE 2
#define STMP_ECUDA 3

#define STMP_METHOD_MP 0      /* matching_pursuit step update, pursuit.py:219-220            */
#define STMP_METHOD_OMP 1     /* omp_refit per iteration (pursuit.py:235-250)     */
#define STMP_METHOD_SELECT 2  /* one selection per row, no update: stmp_select/exact_select   */

#define STMP_MAX_K 128

typedef struct stmp_dict stmp_dict;
typedef struct stmp_tree stmp_tree;

/* Library identification and error text (thread-local, valid until the next call). */
const char* stmp_version(void);
const char* stmp_last_error(void);

/* FNV-1a 64 over a byte buffer, continuing from `state` (pass
 * STMP_FNV_OFFSET to start).  Replaces the pure-Python `fnv1a64` +
 * `Dictionary.fingerprint` (pkg/src/stmp/dictionary.py:32-37,105-109).     */
#define STMP_FNV_OFFSET 0xCBF29CE484222325ULL
uint64_t stmp_fnv1a64(const void* data, size_t len, uint64_t state);

/* Upload a dictionary: m unit-norm atoms of dimension n, atom-major f32
 * (the layout of `Dictionary.atoms`, pkg/src/stmp/dictionary.py:68-100).
 * `atoms` is a host pointer when atoms_on_device == 0, else a device pointer.
 * `fingerprint` is the FNV-1a of the f32 payload (stmp_fnv1a64) and binds
 * trees to this dictionary.  Replaces `Dictionary.scoring_atoms`.           */
int stmp_dict_create(const float* atoms, int64_t m, int32_t n, int32_t atoms_on_device,
                     uint64_t fingerprint, void* stream, stmp_dict** out);
void stmp_dict_free(stmp_dict* d);
int stmp_dict_info(const stmp_dict* d, int64_t* m, int32_t* n, int32_t* ld, uint64_t* fingerprint);

/* Upload a flattened cluster tree (host arrays, BFS order):
 *   levels L = len(branching); internal nodes have global ids in BFS order,
 *   level_offsets[L+2] delimits depths 0..L; child_begin/child_count per
 *   internal node index the next depth's ids (depth < L) or leaf_atom
 *   (depth L); centroids is num_internal x n f32.
 * Replaces `ClusterTree`/`TreeNode.child_matrix`/`child_atom_indices`
 * (pkg/src/stmp/clustering.py:217-264).  Returns STMP_ESTALE when
 * `fingerprint` differs from the dictionary's (pursuit.py:181-185).        */
int stmp_tree_create(const stmp_dict* d, int32_t levels, const int32_t* branching,
                     const int64_t* level_offsets, const int32_t* child_begin,
                     const int32_t* child_count, const float* centroids, int64_t num_leaves,
                     const int32_t* leaf_atom, uint64_t fingerprint, void* stream,
                     stmp_tree** out);
void stmp_tree_free(stmp_tree* t);

/* Batch encode N patches X[N x ldx] (f32, device).
 *   tree == NULL selects exhaustively (ExactSelector, pursuit.py:165-172),
 *   otherwise tree descent (TreeSelector, pursuit.py:175-191) with
 *   retained_count(alpha, k_l) children kept per node at level l: greedy
 *   (one child per level, alpha <= 1/max(branching)) runs on the
 *   staged tensor-core pipeline for large batches; non-greedy alpha (beam
 *   descent, pursuit.py:134-162) on the warp-per-patch kernel (<= 8 levels).
 *   method: STMP_METHOD_MP / STMP_METHOD_OMP / STMP_METHOD_SELECT.
 *   tol_abs < 0 means the reference default 1e-6 * ||x|| (pursuit.py:207-209).
 * Outputs (device; idx, coef, count and resnorm are required, path and ip
 * may be NULL):
 *   idx[N*K] int32 selected atoms in selection order (-1 padded),
 *   coef[N*K] f32 (MP: step scores; OMP: final refit; SELECT: signed score),
 *   count[N] int32 atoms selected, resnorm[N] f32 final ||r|| (the staged
 *   pipeline also keeps its per-patch iteration state in count),
 *   path[N*K*L] int32 BFS node id kept at each level (optional),
 *   ip[N*2] int32 {inner products, centroid inner products} per patch
 *   (ScoreCounter, pkg/src/stmp/dictionary.py:40-65) (optional; 8-byte aligned).
 * Replaces `matching_pursuit` (pursuit.py:194-221) driven by the batch loop
 * of `_code_patches` (pkg/src/stmp/pipelines.py:180-217).
 * Workspace: stmp_encode_workspace() bytes of device memory, caller-owned
 * (the same alpha as the encode: beam descent needs frontier scratch).      */
size_t stmp_encode_workspace(const stmp_dict* d, const stmp_tree* t, int64_t N, int32_t K,
                             int32_t method, double alpha);
int stmp_encode(const stmp_dict* d, const stmp_tree* t, const float* X, int64_t N, int64_t ldx,
                int32_t K, int32_t method, double alpha, double tol_abs, int32_t* idx,
                float* coef, int32_t* count, float* resnorm, int32_t* path, int32_t* ip,
                void* workspace, size_t workspace_bytes, void* stream);

/* Host-buffer variant for end-to-end use: X and every output are HOST
 * pointers (pinned memory recommended); the library stages chunks through
 * device buffers, overlapping H2D copies, encode and D2H copies on its own
 * streams, and returns after the results are on the host.                   */
int stmp_encode_host(const stmp_dict* d, const stmp_tree* t, const float* X, int64_t N,
                     int64_t ldx, int32_t K, int32_t method, double alpha, double tol_abs,
                     int32_t* idx, float* coef, int32_t* count, float* resnorm, int32_t* ip,
                     int64_t chunk);

/* Batch driver around the encoder: the per-patch arithmetic
 * of pipelines._code_patches (pkg/src/stmp/pipelines.py:180-217) on the device.
 *
 * stmp_dc_split replaces pipelines.py:201-203: for each measured patch
 * y = Y[p] (f32, device, row stride ldy), dc[p] = (y . dc_meas) / denom (f64,
 * denom = dc_meas . dc_meas) and Yc[p] = f32(y - dc[p] * dc_meas), the input
 * the encoder codes.  dc_meas is a device f64 [n] vector.                     */
int stmp_dc_split(const float* Y, int64_t N, int64_t ldy, int32_t n, const double* dc_meas, double denom,
                  float* Yc, int64_t ldc, double* dc, void* stream);

/* stmp_reconstruct replaces lift_code (pkg/src/stmp/operators.py:199-215),
 * reconstruct (pkg/src/stmp/pursuit.py:224-232) and "+ dc"
 * (pipelines.py:204): out[p] = sum_{k < count[p]} (coef[p,k] / scale[idx[p,k]])
 * * base_atom[idx[p,k]] + dc[p], in f64, entries in selection order, with the
 * multiply and the add rounded separately as in NumPy.  `base` holds the
 * full-space atoms (ProjectedDictionary.base); scale (device f64 [m]) and dc
 * (device f64 [N]) may be NULL for 1 and 0.  Unusable atoms must be rejected
 * by the caller before (lift_code raises RuntimeError, operators.py:209-213). */
int stmp_reconstruct(const stmp_dict* base, const int32_t* idx, const float* coef, const int32_t* count, int64_t N,
                     int32_t K, const double* scale, const double* dc, double* out, int64_t ldo, void* stream);

/* Data formats either side of the path.  Device buffers;
 * the geometry arrays (rank entries) are HOST arrays, the window starts a
 * DEVICE int64 array: axis 0's nstarts[0] starts, then axis 1's, ...
 * (PatchLayout.axis_starts, pkg/src/stmp/tensor.py:49-99).
 *
 * stmp_extract_patches replaces extract_patches (tensor.py:104-111): row p of
 * out[N x n] is window p of the row-major f32 tensor t, windows in row-major
 * origin order, values in row-major window order; bit-exact.
 * stmp_aggregate_patches replaces aggregate_patches (tensor.py:114-136): each
 * cell of out (f32, tensor shape) is the f64 mean of every covering patch
 * value, summed in origin order -- bitwise the reference's result.           */
int stmp_extract_patches(const float* t, int32_t rank, const int64_t* shape, const int64_t* patch,
                         const int64_t* nstarts, const int64_t* starts, float* out, void* stream);
int stmp_aggregate_patches(const float* patches, int32_t rank, const int64_t* shape, const int64_t* patch,
                           const int64_t* nstarts, const int64_t* starts, float* out, void* stream);

/* stmp_apply_operator replaces apply_batch (pkg/src/stmp/operators.py:115-141)
 * for N f32 rows X[N x n_in] -> f64 rows Y[N x n_out]:
 *   STMP_OP_ROW_SELECT      rows (device int64 [n_rows]) kept, in order;
 *   STMP_OP_CODED_EXPOSURE  mask (device f32 [pixels x frames], binary): the
 *                           patch is (pixels, windows, frames) row-major and
 *                           each output sums its frames times the pixel's mask;
 *   STMP_OP_BLOCK_AVERAGE   in_shape / factors (host int64 [rank]): the mean
 *                           of each factor block.
 * (IDENTITY is a copy and needs no kernel.)  f64 arithmetic; sums in index
 * order, so results equal NumPy's pairwise sums to rounding (1e-15 relative). */
#define STMP_OP_ROW_SELECT 1
#define STMP_OP_CODED_EXPOSURE 2
#define STMP_OP_BLOCK_AVERAGE 3
int stmp_apply_operator(int32_t kind, const float* X, int64_t N, int32_t n_in, const int64_t* rows, int32_t n_rows,
                        const float* mask, int32_t pixels, int32_t windows, int32_t frames, int32_t rank,
                        const int64_t* in_shape, const int64_t* factors, double* Y, void* stream);

/* Process-wide tuning knobs (no reference counterpart):
 *   "path": 0 auto (default), 1 fused warp-per-patch kernel, 2 staged tensor-core pipeline;
 *   "staged_min_batch": batch size from which `auto` picks the staged pipeline;
 *   "score_kernel": staged score pass 2 node table in shared memory where it fits (default; where it
 *                   does not, the streamed pass -- on nodes of > 128 children with the 3xFP16 split),
 *                   3 streamed table, 3xTF32, at every level, 4 streamed table, 3xFP16 split, at every
 *                   level of the residual pipeline;
 *   "update_kernel": staged OMP update 0 generic, 1 lockstep / wide-row (default);
 *   "gram_path": tree OMP without a residual in HBM, on per-tree pair tables of
 *                child-centroid . atom products (the Gram matrix at the last level;
 *                needs single-atom depth-L nodes and m x nodes x 4 B of free device
 *                memory): 0 off, 1 auto = rows >= 256 and >= 8x the widest node
 *                (default), 2 whenever supported;
 *   "half_scores": 1 (default) the Gram path's level passes multiply fp16 copies of the
 *                patch rows (x16 = fp16(s x), one power-of-two scale per patch) by two fp16
 *                pieces of every centroid; the exact near-tie re-check widens its window by
 *                the rows' quantisation noise, so decisions stay the fp32 ones; 0 = fp32 rows
 *                (3xTF32).  Applies where every level >= 1 has nodes of <= 64 children and
 *                the padded row length is a multiple of 64;
 *   "pdl": 1 (default) launch the staged kernels with programmatic dependent launch, 0 plain;
 *   "graphs": 1 (default) replay repeated staged encodes (same buffers, sizes, stream) as CUDA graphs. */
int stmp_set_option(const char* key, int64_t value);

/* Instrumentation: cumulative number of CUDA kernels this library has launched. */
int stmp_kernel_launches(int64_t* out);

/* Instrumentation: per-kernel device time.  stmp_kernel_timing(1) clears the
 * record and brackets every later kernel launch with CUDA events on its stream
 * (encodes run eagerly, without graph replay, while on); stmp_kernel_timing(0)
 * stops recording.  stmp_kernel_times synchronises the recorded events and
 * returns, per kernel (up to max_entries, names truncated to name_len bytes,
 * NUL-terminated, in names[i * name_len]), the launch count and the summed
 * duration in ms; *n_entries is the number of distinct kernels.             */
int stmp_kernel_timing(int32_t enable);
int stmp_kernel_times(int32_t max_entries, char* names, int32_t name_len, int64_t* launches, double* total_ms,
                      int32_t* n_entries);

/* Device synchronisation helper for hosts without a CUDA runtime binding. */
int stmp_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STMP_B200_H */
