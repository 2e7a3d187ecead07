// Argument blocks and entry points of the staged (level-synchronous) encoder.
#pragma once

#include "common.cuh"

namespace stmp {

// striped counters of the root bin (count_root / scan_kernel)
constexpr int kRootStripes = 128;

struct ScoreArgs {
  const float* R;        // residual rows [N, ld]
  int ld;
  int64_t nrows;         // N (extent of R for the row tensor map)
  const int* perm;       // patch ids grouped by bin
  const int4* items;     // {bin, start in perm, rows, 0}
  const int* num_items;
  const float* table;    // per-bin SW128 hi/lo child-centroid blocks
  int npad, kchunks, tmem_cols;
  int level, level_base;
  const int* child_begin;
  const int* child_count;
  int* path_ws;          // [N, L] node chosen at each level this iteration
  int* path_out;         // optional [N, K, L]
  const int* count;      // current support size per patch (path slot)
  int K, L;
  int* next_counts;      // bin counters of the next level (nullptr at the last level)
  int next_base;

  int32_t* ip;           // optional per-patch {inner products, centroid inner products}
  int* leaf_sel;         // last level: the single leaf atom, or -1-node for multi-atom leaves
  const int* leaf_atom;
  int nblocks;           // exhaustive scan: atom blocks of npad atoms
  int m_atoms;           // exhaustive scan: dictionary size
  const int* active;     // root pass in patch order (perm == nullptr): skip inactive rows
  int ks_last;           // 8-column k-steps holding data in the last 32-column chunk (1..4): the
                         // rest are zero padding on both operands and their MMAs are skipped

  // ---- Gram path (gram_path.cu): the rows are the patches x, not residuals, and
  // a child's score is corrected to c . r = c . x - sum_k c_k (c . a_{S_k})
  const float* corr;     // pair table of this level: [m][corr_w], row = atom, column = child node
  int64_t corr_w;        // columns per row (nodes at depth level + 1)
  int corr_off;          // global id of the first depth-(level + 1) node (column 0)
  const int* sup;        // support atoms [N][sup_ld] (S_ws), the first `sup_t` entries valid
  const float* supc;     // current coefficients [N][sup_ld] (c_ws)
  int sup_t;             // support size of every active patch (the iteration index)
  int64_t sup_ld;        // K
  float* raw_out;        // root pass of iteration 0: raw scores c . x of all children -> [N][raw_w]
  int raw_w;
  // exact re-check of near ties: the tensor cores' truncating fp32 accumulation
  // leaves ~1e-6 ||x|| of error on c . x, so decisions whose top-2 corrected
  // scores are closer than recheck_rel * ||x|| are re-scored with FFMA dots
  const float* cent;     // centroid rows [nodes][ld] (global ids)
  const double* xn2;     // ||x||^2 per patch
  float recheck_rel;
  // corrections precomputed by gram_corr_kernel: [N][corr_pre_ld], column j =
  // child j of the patch's node (nullptr: gathered from the pair table here)
  const float* corr_pre;
  int corr_pre_ld;
  // half-precision rows (score_sh.cu, Gram path levels >= 1): x16 = fp16(s_p x)
  // with a power-of-two scale per patch, the node tables as three fp16 pieces
  const uint16_t* R16;      // [N][ld] halfs
  const uint8_t* table_h;   // per node: [ld / 64][2 pieces][npad rows x 128 B] SW128
  const float* inv_scale;   // 1 / s_p
  const float* qerr;        // ||x - x16 / s_p|| per patch
  float recheck_q;          // near-tie window += recheck_q * qerr
  // 3xFP16 pass of the residual pipeline (score_s16.cu): table_h = [c_a | c_b] pieces of 2^8 c
  const float* rnorm;       // ||r|| per patch (the resnorm output every update writes): the row scale

  // ---- staged beam descent (run_staged_beam): the pass scores (patch, node)
  // entries instead of patches; perm holds entry ids
  int beam_keep;            // > 0: retained_count(alpha, k_level) children kept per entry
  const int* entry_patch;   // entry -> patch (nullptr: rows are patches)
  const uint8_t* entry_first;   // the entry is frontier[0] of its patch (the reference's path)
  int* out_patch;           // internal levels: survivors appended as the next level's entries
  int* out_node;
  uint8_t* out_first;
  int* out_count;
  unsigned long long* leaf_key;   // last level: per patch max of (|score| << 32 | ~atom)
};
constexpr int kMaxBeamKeep = 16;   // staged beam: children kept per node (larger: warp-per-patch kernel)

// Work items of a score pass: (bin, first slot in perm, rows) from the scan, or
// -- the root pass over the whole batch in patch order, perm == nullptr -- the
// i-th 128-patch tile of the batch, whose inactive rows carry row id -1.
__device__ __forceinline__ int item_count(const ScoreArgs& a) {
  return a.perm ? *a.num_items : (int)((a.nrows + 127) / 128);
}
__device__ __forceinline__ int4 item_at(const ScoreArgs& a, int i) {
  if (a.perm) return a.items[i];
  return make_int4(0, i * 128, (int)min((int64_t)128, a.nrows - (int64_t)i * 128), 0);
}
// patch of row r (< it.z) of item `it`, -1 for a skipped row
__device__ __forceinline__ int row_at(const ScoreArgs& a, int4 it, int r) {
  if (a.perm) return a.perm[it.y + r];
  const int p = it.y + r;
  return a.active[p] ? p : -1;
}
// patch of a row id (an entry id on the staged beam path), -1 stays -1
__device__ __forceinline__ int patch_of(const ScoreArgs& a, int id) {
  return (a.entry_patch != nullptr && id >= 0) ? a.entry_patch[id] : id;
}

struct UpdateArgs {
  const float* X;        // caller's patches (row stride ldx, n valid columns)
  int64_t ldx;
  int n;
  float* R;              // residual [N, ld] (written)
  const float* R_in;     // residual read by this pass (x itself on the first iteration)
  int ld;
  const float* X2;       // padded copy of X used by the OMP rebuild (OMP only)
  int ld2;
  const float* atoms;    // padded dictionary [m, ld]
  const int* child_begin;
  const int* child_count;
  const int* leaf_atom;
  int L;
  const int* path_ws;
  int K, method;
  float tol_abs;
  int32_t* idx;
  float* coef;
  int32_t* count;
  float* resnorm;
  int32_t* ip;
  int32_t* path_out;
  float* Lf;             // packed inverse Cholesky factor M = L^{-1} per patch
  float* yv;             // y = M A_S x per patch
  float* tol;
  int* active;

  int* root_count;       // kRootStripes counters of the next root bin
  const int* leaf_sel;   // written by the last score pass
  int64_t m;
  int cache_atoms;       // stage the support atoms in shared memory
  int64_t N;
  // lockstep OMP kernel (update_omp8): state laid out [entry][patch]
  int* S_ws;             // support atoms [K][N]
  float* c_ws;           // coefficients [K][N]
  int iter;              // iteration index = support size of every active patch
  double* xn2;           // Gram path: ||x||^2 per patch (init), and the running ||r||^2
  double* e_ws;
  // Gram path with fp16 level passes (score_sh.cu): init also writes the fp16 row
  // copy x16 = fp16(s_p x), 1 / s_p and ||x - x16 / s_p|| (nullptr: not needed)
  uint16_t* x16;
  float* inv_scale;
  float* qerr;
};

// Gram path (gram_path.cu, OMP on trees whose depth-L nodes are single atoms):
// no residual is kept; every score is c . x minus the support's contribution
// read from per-level pair tables, and the OMP update works on Gram entries.
struct GramArgs {
  int64_t N;
  int K, L, iter;
  const int* leaf_sel;     // atom chosen by the last score pass
  const float* gram;       // pair table of the last level = the Gram matrix in leaf order [m][m]
  int64_t gram_w;
  const int* leaf_pos;     // [m] column of each atom in the last-level table
  const float* root_tab;   // pair table of level 0 [m][root_w]
  float* s0;               // cached root scores c . x [N][root_w] (near-tie re-checks write exact values back)
  int root_w, root_cb;     // root children: count, first global id
  int* root_counts;        // level-1 bin counters of the next iteration
  int* path_ws;
  int32_t* path_out;
  int* S_ws;
  float* c_ws;
  float* yv;
  float* Lf;
  double* e_ws;            // ||r||^2 = ||x||^2 - sum_j y_j^2 (f64)
  const double* xn2;       // ||x||^2
  const float* tol;
  int* active;
  int32_t* idx;
  float* coef;
  int32_t* count;
  float* resnorm;
  int32_t* ip;
  // exact dots (b = a . x, root near ties) and the explicit residual norm for
  // patches whose ||r||^2 estimate falls below rho ||x||^2 (cancellation)
  const float* xr;         // patch rows x, zero-padded [N][ld]
  const float* atoms;
  const float* cent;       // centroid rows [nodes][ld] (root children: root_cb ..)
  int ld;
  float rho;
  float recheck_rel;       // near-tie window: recheck_rel * ||x||
};
bool gram_path_supported(const DictHandle* d, const TreeHandle* t, int K, int method);
// builds the pair tables on first use; false if they cannot be allocated
bool ensure_pair_tables(TreeHandle* t, const DictHandle* d, cudaStream_t st);
cudaError_t launch_update_gram(const GramArgs& a, cudaStream_t st);
// sum_k c_k P_l[S_k][children of the patch's level-l node] for every active patch,
// written to out[N][ld] before the level-l score pass (one warp per patch: the
// support's pair-table rows are read coalesced, the epilogue then reads one row)
cudaError_t launch_gram_corr(int64_t N, const int* active, const int* path_ws, int L, int level,
                             const int* child_begin, const int* child_count, int col_off, const float* tab,
                             int64_t tab_w, const int* S_ws, const float* c_ws, int K, int T, float* out, int ld,
                             cudaStream_t st);
// leaf_pos of a tree whose depth-L nodes are single atoms covering the dictionary
bool build_leaf_pos(TreeHandle* t, int64_t m, cudaStream_t st);
void free_pair_tables(TreeHandle* t);
extern int g_gram_path;   // 0 off, 1 auto (wide rows), 2 whenever supported

struct UpdateCfg {
  int G = 0;   // lanes per patch
  int E = 0;   // row elements per lane (G * E == ld)
  int KC = 0;  // support atoms cached in registers (0: reload)
};

bool update_config(int ld, int K, UpdateCfg& c);
cudaError_t launch_init(const UpdateCfg& c, const UpdateArgs& a, int blocks, cudaStream_t st);
cudaError_t launch_update(const UpdateCfg& c, const UpdateArgs& a, int blocks, size_t smem,
                          cudaStream_t st);
size_t update_smem_bytes(const UpdateCfg& c, int K, int ld, bool cache_atoms);
// Lockstep OMP update (K <= 8 with rows of <= 160 floats, K <= 16 with <= 64):
// 8 lanes per patch, each owning one or two rows of the inverse Cholesky factor,
// support size a.iter fixed at compile time, state in the [entry][patch] layout.  Returns cudaErrorNotSupported when not applicable.
cudaError_t launch_update_omp8(const UpdateArgs& a, cudaStream_t st);
// OMP update with one CTA per patch for rows wider than 160 floats (0: not applicable)
int wide_update_cpt(int ld);
cudaError_t launch_update_wide(const UpdateArgs& a, cudaStream_t st);
extern int g_update_wide;
// lanes per patch of the lockstep OMP update for this shape (8 or 16), 0 if unsupported
int lockstep_lanes(int ld, int K);

size_t score_smem_bytes(int kchunks, int npad);

// Per-bin table block: [kchunks][hi|lo][npad rows x 128 B] SW128, then (last
// level only) npad ints leaf_info (single leaf atom, or -1-child) and npad
// ints leaf count.
__host__ __device__ inline uint32_t table_bytes(int kch, int npad, bool last) {
  return (uint32_t)kch * 2u * npad * 128u + (last ? 8u * npad : 0u);
}

extern int g_score_ws;
extern int g_update_omp8;
extern int g_root_direct;
bool score_ts_fits(int kchunks, int npad, bool last);
// exhaustive selection (exact_scan.cu): dictionary blocks of xtable_block_width(ld)
// atoms; a.table = ensure_xtable(d), a.npad = block width, a.leaf_sel = best atom
int xtable_block_width(int ld);
const float* ensure_xtable(DictHandle* d, cudaStream_t st);
const uint8_t* ensure_xtable16(DictHandle* d, cudaStream_t st);   // fp16 pieces, nullptr if it cannot be built
cudaError_t launch_exact_scan(const ScoreArgs& s, int sms, cudaStream_t st);
// streamed-table score pass (score_st.cu): any K, npad <= 256
bool score_st_fits(int kchunks, int npad, bool last);
cudaError_t launch_score_st(const ScoreArgs& s, int sms, cudaStream_t st);
// half-precision streamed pass of the Gram path (score_sh.cu): s.kchunks = ld / 64,
// s.ks_last = 16-column k-steps holding data in the last chunk
bool score_sh_fits(int ld, int npad);
cudaError_t launch_score_sh(const ScoreArgs& s, int sms, cudaStream_t st);
// bytes of one node's half-precision table block
__host__ __device__ inline uint32_t table_h_bytes(int kch64, int npad) { return (uint32_t)kch64 * 2u * npad * 128u; }
// per-node fp16 piece tables of level l (nullptr on allocation failure)
uint8_t* build_half_table(const TreeHandle* t, int l, cudaStream_t st);
// 3xFP16 streamed pass of the residual pipeline (score_s16.cu, score_kernel = 4)
bool score_s16_fits(int ld, int npad);
cudaError_t launch_score_s16(const ScoreArgs& s, int sms, cudaStream_t st);
uint8_t* build_s16_table(const TreeHandle* t, int l, cudaStream_t st);
bool ensure_s16_tables(TreeHandle* t, cudaStream_t st);
extern int g_half_scores;   // 1: Gram-path level passes read fp16 rows (default), 0: fp32 rows / 3xTF32
cudaError_t launch_score_ts(const ScoreArgs& s, int sms, cudaStream_t st);
bool staged_supported(const DictHandle* d, const TreeHandle* t, int K, int method);
size_t staged_workspace_bytes(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method);
// staged beam descent (non-greedy alpha, single-atom depth-L nodes, keep <= kMaxBeamKeep):
// keep[l] children per node at level l, max_frontier = largest entries-per-patch count
bool staged_beam_supported(const DictHandle* d, const TreeHandle* t, int K, int method, const int* keep);
size_t staged_beam_workspace(const DictHandle* d, const TreeHandle* t, int64_t N, int K, int method,
                             const int* keep);
cudaError_t run_staged_beam(const DictHandle* d, const TreeHandle* t, const float* X, int64_t N, int64_t ldx, int K,
                            int method, float tol_abs, const int* keep, int max_frontier, int32_t* idx, float* coef,
                            int32_t* count, float* resnorm, int32_t* path, int32_t* ip, void* ws, size_t ws_bytes,
                            cudaStream_t st);
cudaError_t run_staged(const DictHandle* d, const TreeHandle* t, const float* X, int64_t N,
                       int64_t ldx, int K, int method, float tol_abs, int32_t* idx, float* coef,
                       int32_t* count, float* resnorm, int32_t* path, int32_t* ip, void* ws,
                       size_t ws_bytes, cudaStream_t st);
// host-side construction of the per-level SW128 hi/lo tables
bool build_staged_tables(TreeHandle* t, const int32_t* child_begin, const int32_t* child_count,
                         const float* centroids, const int32_t* leaf_atom, cudaStream_t st,
                         std::string* err);
void free_staged_tables(TreeHandle* t);

}  // namespace stmp
