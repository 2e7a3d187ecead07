"""Algorithmic work per patch and the roofline it implies.

Per patch, with n dims, K iterations, L levels, greedy branching k_1..k_L:

* ``IP_sel`` -- inner products one selection spends (the reference's own
  ScoreCounter count): ``sum_i k_i + leaf_atoms`` for the tree, ``m`` for the
  exhaustive scan (pursuit.py:139-140,157-158,107).
* FLOPs ``F = K * 2n * IP_sel + 2n * K(K+1)`` (OMP: Gram column + rhs +
  residual rebuild, ``sum_k 4nk``); MP replaces the second term by ``2nK``.
* HBM bytes of the SURVEY's staged design
  ``B = 4n + K((L+2) 4n + 8L) + 8K + 4`` (x in; per iteration L level
  stages each read r, the fused update reads x and writes r, 8 B node ids per
  level; outputs), plus for dictionaries larger than L2 the support-atom
  gathers ``4n K(K+1)/2`` and the non-resident centroid tables amortised per
  patch.  Exhaustive: ``4n + K(12n + 4nm/N) + 4n K(K+1)/2 + 8K + 4``.

``achieved = B * N / t`` (GB/s) or ``F * N / t`` (FLOP/s) with ``t`` the
measured kernel time, i.e. ``frac = T_roof(model) / T_measured``.
"""

from __future__ import annotations

import math

L2_BYTES = 126 * 1024 * 1024
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: FFMA peak at max clock


def ip_per_selection(branching, m: int, exhaustive: bool) -> int:
    if exhaustive:
        return int(m)
    leaves = max(1, round(m / math.prod(branching)))
    return int(sum(branching)) + leaves


def flops_per_patch(n: int, K: int, branching, m: int, method: str = "omp", exhaustive=False) -> float:
    ips = ip_per_selection(branching, m, exhaustive)
    upd = 2 * n * K * (K + 1) if method == "omp" else 2 * n * K
    return float(K * 2 * n * ips + upd)


def bytes_per_patch(n: int, K: int, branching, m: int, N: int, method: str = "omp",
                    exhaustive=False, table_bytes: int = 0) -> float:
    dict_bytes = 4 * n * m
    if exhaustive:
        return float(4 * n + K * (12 * n + 4 * n * m / N) + 4 * n * K * (K + 1) / 2 + 8 * K + 4)
    L = len(branching)
    b = 4 * n + K * ((L + 2) * 4 * n + 8 * L) + 8 * K + 4
    if dict_bytes > L2_BYTES:
        b += 4 * n * K * (K + 1) / 2
        b += K * table_bytes / N
    return float(b)


def model(cfg, N: int | None = None, method: str = "omp", exhaustive: bool = False,
          hbm_gbs: float = 6548.2, tensor_tflops: float = 300.0) -> dict:
    """Roofline numbers for a workload config (see workloads.CONFIGS).
    ``tensor_tflops`` is the fp32-accurate tensor rate: the MEASURED dense TF32
    GEMM rate / 3 (3xTF32, three tf32 products per k-step)."""
    N = cfg.N if N is None else N
    L = len(cfg.branching)
    # centroid tables of depths 1..L (excluding single-atom depth L, which is the dictionary)
    nodes = [math.prod(cfg.branching[:d + 1]) for d in range(L)]
    table_bytes = sum(4 * cfg.n * v for v in nodes if 4 * cfg.n * v > L2_BYTES)
    F = flops_per_patch(cfg.n, cfg.K, cfg.branching, cfg.m, method, exhaustive)
    B = bytes_per_patch(cfg.n, cfg.K, cfg.branching, cfg.m, N, method, exhaustive, table_bytes)
    P = tensor_tflops * 1e12
    t_hbm = B / (hbm_gbs * 1e9)
    t_fl = F / P
    return dict(flops_per_patch=F, bytes_per_patch=B, bound="hbm" if t_hbm >= t_fl else "tensor",
                t_roof_per_patch=max(t_hbm, t_fl), patches_per_s_roof=1.0 / max(t_hbm, t_fl))


# ---------------------------------------------------------------- per kernel family
# Kernel families of one staged encode, by (mangled) kernel name.
FAMILIES = (("corr", ("gram_corr_kernel",)),
            ("score", ("score_ts_kernel", "score_st_kernel", "score_sh_kernel", "score_s16_kernel")),
            ("exact_scan", ("exact_scan_kernel",)),
            ("update", ("update_omp8_kernel", "update_wide_kernel", "update_gram_kernel", "update_kernel")),
            ("scatter", ("scatter_scan_kernel", "scatter_kernel", "scatter_root_kernel", "scan_kernel",
                         "scatter_entries_kernel", "beam_resolve_kernel")),
            ("init", ("init_kernel",)),
            ("fused", ("encode_fused_kernel",)))


def family_of(name: str) -> str:
    for fam, keys in FAMILIES:
        if any(k in name for k in keys):
            return fam
    return "other"


# fp32-accurate tensor rate of the score passes (3xTF32: three tf32 products per
# k-step) against HBM, to decide which roof binds a tensor-core pass; bench.py
# passes the TF32 rate it measures live (profiles/r02_peaks_tf32.json: 776)
HBM_GBS_DEFAULT = 6548.2
TF32X3_TFLOPS_DEFAULT = 776.3 / 3


def binding(work: dict, hbm_gbs: float = HBM_GBS_DEFAULT, tensor_tflops: float = TF32X3_TFLOPS_DEFAULT) -> dict:
    """Mark a tensor-core family "tensor"- or "hbm"-bound by its roofline time."""
    t_hbm = work["bytes"] / (hbm_gbs * 1e9)
    t_tc = work["flops"] / (tensor_tflops * 1e12)
    return dict(work, bound="tensor" if t_tc > t_hbm else "hbm")


def beam_ip(branching, alpha: float, m: int) -> int:
    """Inner products of one beam selection (pursuit.py:134-162): the frontier of
    level l holds F_l nodes, each scoring its k_l children; the survivors' leaf
    atoms are scored at the end (balanced tree: m / prod(k) atoms per leaf node)."""
    f, ips = 1, 0
    for k in branching:
        ips += f * k
        f *= min(k, max(1, math.ceil(alpha * k - 1e-9)))
    return ips + f * max(1, round(m / math.prod(branching)))


def fused_work(cfg, N: int, alpha: float, method: str = "omp") -> dict:
    """The warp-per-patch kernel (encode_fused.cu): FFMA dot products of every
    scored centroid / atom with the residual held in registers -- SIMT-FLOP
    bound; HBM bytes are x in and the outputs."""
    n, K = cfg.n, cfg.K
    ips = beam_ip(cfg.branching, alpha, cfg.m)
    upd = 2 * n * K * (K + 1) if method == "omp" else 2 * n * K
    return {"bytes": float(N * (4 * n + 8 * K + 16)), "flops": float(N * (K * 2 * n * ips + upd)), "bound": "fp32"}


def gram_family_work(cfg, family: str, N: int, half: bool = False) -> dict:
    """Algorithmic work of one kernel family of the Gram path (gram_path.cu: tree
    OMP without a residual, single-atom depth-L nodes) over a whole encode of N
    patches, every patch running all K iterations, T = support size at iteration T.

    * score: x rows per pass -- the root once (iteration 0, 4n B, plus its raw
      scores 4 k_1 B cached), levels 1..L-1 every iteration (4n B, or 2n B with
      ``half``: fp16 rows, score_sh.cu) plus the precomputed correction row
      (4 k_{l+1} B), node tables only where a level's centroids exceed L2 (each
      visited node once per iteration; 4 B per value either way: tf32 hi | lo or
      two fp16 pieces); FLOPs 2n per scored child.
    * corr (gram_corr_kernel, one launch per level >= 1 and iteration >= 1): the
      support's T x k_{l+1} pair-table floats in, one k_{l+1}-float row out.
    * init (``half``): the init pass also writes the fp16 row copy, 2n B per patch.
    * update: x and the chosen atom (2 x 4n B) for the exact right-hand side, T Gram
      entries, the cached root scores (4 k_1 B) and the solver state (M row, c, y).
    * scatter / init as in family_work.
    """
    n, K = cfg.n, cfg.K
    br = cfg.branching
    L = len(br)
    T_sum = K * (K - 1) // 2
    kids = [math.prod(br[:d + 1]) for d in range(L)]
    tables = sum(4 * n * k for k in kids[1:] if 4 * n * k > L2_BYTES)
    if family == "score":
        row = 2 * n if half else 4 * n
        b = 4 * n + 4 * br[0] + K * (L - 1) * (row + 8) + (K - 1) * 4 * sum(br[1:])
        return binding({"bytes": float(N * b + K * tables),
                        "flops": float(N * 2 * n * (br[0] + K * sum(br[1:])))})
    if family == "corr":
        b = (T_sum + K - 1) * 4 * sum(br[1:])
        return {"bytes": float(N * b), "flops": float(N * 2 * T_sum * sum(br[1:])), "bound": "hbm"}
    if family == "update":
        b = sum(8 * n + 4 * T + 4 * br[0] + 4 * 3 * (T + 1) for T in range(K))
        return {"bytes": float(N * b), "flops": float(N * K * 2 * n), "bound": "hbm"}
    if family == "init" and half:
        return {"bytes": float(N * (4 * n * 2 + 2 * n)), "flops": 0.0, "bound": "hbm"}
    return family_work(cfg, family, N, "omp", False)


def gram_model(cfg, N: int, hbm_gbs: float = 6548.2, half: bool = False) -> dict:
    """The Gram path's whole-step algorithmic bytes per patch (sum of its families)."""
    fams = ("score", "corr", "update", "scatter", "init")
    B = sum(gram_family_work(cfg, f, N, half)["bytes"] for f in fams) / N
    F = sum(gram_family_work(cfg, f, N, half)["flops"] for f in fams) / N
    return dict(flops_per_patch=F, bytes_per_patch=B, bound="hbm", t_roof_per_patch=B / (hbm_gbs * 1e9),
                patches_per_s_roof=hbm_gbs * 1e9 / B)


def beam_frontiers(branching, alpha: float) -> list:
    """Entries (frontier nodes) per patch at each level of a beam descent."""
    f, out = 1, []
    for k in branching:
        out.append(f)
        f *= min(k, max(1, math.ceil(alpha * k - 1e-9)))
    return out


def family_work(cfg, family: str, N: int, method: str = "omp", exhaustive: bool = False,
                alpha: float | None = None) -> dict:
    """Algorithmic work of one kernel family over a whole encode of N patches,
    assuming every patch runs all K iterations (the noisy BASELINE inputs never
    reach the 1e-6 tolerance early).  Returns {"bytes": B, "flops": F, "bound"}.

    * score (tree): every level pass reads each residual row (4n B) and the
      patch's node id (8 B); centroid tables count only when the level's table
      exceeds L2 (config 4's last level: each visited node table once per
      iteration).  FLOPs 2n per scored child.
    * exact_scan: FLOPs 2nm per patch per iteration (tensor-bound).
    * update (OMP, iteration T): x read, new atom read, r written (3 x 4n B),
      plus the T support rows when the dictionary exceeds L2; MP: r read, atom
      read, r written.
    * scatter: active flag, node id and permutation slot (12 B per patch and level).
    """
    n, K, m = cfg.n, cfg.K, cfg.m
    L = len(cfg.branching)
    big = 4 * n * m > L2_BYTES
    if family == "exact_scan":
        return {"bytes": float(N * K * 4 * n + K * 4 * n * m), "flops": float(N * K * 2 * n * m), "bound": "tensor"}
    if family == "score":
        kids = [math.prod(cfg.branching[:d + 1]) for d in range(L)]
        tables = sum(4 * n * k for k in kids if 4 * n * k > L2_BYTES)
        if alpha is not None:   # staged beam: one residual row per (patch, frontier node) entry
            fr = beam_frontiers(cfg.branching, alpha)
            return binding({"bytes": float(N * K * sum(fr) * (4 * n + 12) + K * tables),
                            "flops": float(N * K * 2 * n * sum(f * k for f, k in zip(fr, cfg.branching)))})
        return binding({"bytes": float(N * K * L * (4 * n + 8) + K * tables),
                        "flops": float(N * K * 2 * n * sum(cfg.branching))})
    if family == "update":
        if method == "omp":
            per = sum(4 * n * (3 + (T if big else 0)) for T in range(K))
            fl = sum(4 * n * (T + 1) for T in range(K))
        else:
            per, fl = K * 3 * 4 * n, K * 2 * n
        return {"bytes": float(N * per), "flops": float(N * fl), "bound": "hbm"}
    if family == "scatter":
        return {"bytes": float(N * K * max(L - 1, 0) * 12), "flops": 0.0, "bound": "hbm"}
    if family == "init":
        return {"bytes": float(N * 4 * n * 2), "flops": 0.0, "bound": "hbm"}
    return {"bytes": 0.0, "flops": 0.0, "bound": "hbm"}
