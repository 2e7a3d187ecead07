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
TF32_DENSE_TFLOPS_EST = 1686.0 / 2                  # half the measured bf16 rate (estimate)


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
          hbm_gbs: float = 6548.2, tensor_tflops: float | None = None) -> dict:
    """Roofline numbers for a workload config (see workloads.CONFIGS)."""
    N = cfg.N if N is None else N
    L = len(cfg.branching)
    # centroid tables of depths 1..L (excluding single-atom depth L, which is the dictionary)
    nodes = [math.prod(cfg.branching[:d + 1]) for d in range(L)]
    table_bytes = sum(4 * cfg.n * v for v in nodes if 4 * cfg.n * v > L2_BYTES)
    F = flops_per_patch(cfg.n, cfg.K, cfg.branching, cfg.m, method, exhaustive)
    B = bytes_per_patch(cfg.n, cfg.K, cfg.branching, cfg.m, N, method, exhaustive, table_bytes)
    P = (tensor_tflops or TF32_DENSE_TFLOPS_EST / 3) * 1e12
    t_hbm = B / (hbm_gbs * 1e9)
    t_fl = F / P
    return dict(flops_per_patch=F, bytes_per_patch=B, bound="hbm" if t_hbm >= t_fl else "tensor",
                t_roof_per_patch=max(t_hbm, t_fl), patches_per_s_roof=1.0 / max(t_hbm, t_fl))
