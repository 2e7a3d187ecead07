"""CPU ORACLE -- test infrastructure only, never the product.

Runs the f64 oracle of ``oracle.stmp_oracle`` over many patches at once, so
parity checks on large prefixes (16,384+ patches of configs 1-3,
hundreds of config-4 exhaustive patches) finish in seconds on the GPU box's
host cores:

* tree selectors: the per-patch oracle loop (``encode_one``) on a fork pool,
  contiguous shards, one BLAS thread per process;
* the exhaustive selector: ``encode_exact_batched``, which restates
  ``exact_select`` (pkg/src/stmp/pursuit.py:102-109) for a block of residuals
  at once -- ``scores = R A^T`` as one GEMM instead of one GEMV per patch,
  argmax of |scores| per row with the lowest index on ties -- and otherwise
  follows ``encode_one`` step for step.  The GEMM sums in a different order
  than the GEMV, so scores differ in the last bits; only decisions whose
  top-2 gap is that small can differ, and those are near ties the parity
  contract already excuses.  ``tests/test_oracle.py`` checks it against the
  per-patch oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os

import numpy as np

from . import stmp_oracle as O

_STATE: dict = {}


def _limit_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl is optional
        pass


def _tree_worker(bounds):
    lo, hi = bounds
    _limit_blas()
    st = _STATE
    sel = O.tree_selector(st["otree"], st["a64"], st["alpha"])
    return [O.encode_one(sel, st["a64"], x, st["K"], st["method"], st["tol"]) for x in st["X"][lo:hi]]


def _exact_worker(bounds):
    lo, hi = bounds
    _limit_blas()
    st = _STATE
    return encode_exact_batched(st["a64"], st["X"][lo:hi], st["K"], st["method"], st["tol"])


def procs_default() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def encode_parallel(otree, a64, X, K, method="omp", tol=None, alpha=None, procs=None, keep_residual=False):
    """Oracle results (the ``encode_one`` dicts) for every row of X.
    ``otree`` None selects the exhaustive oracle."""
    X = np.asarray(X)
    procs = min(procs or procs_default(), max(1, len(X)))
    _STATE.update(otree=otree, a64=a64, X=X, K=K, method=method, tol=tol, alpha=alpha)
    worker = _tree_worker if otree is not None else _exact_worker
    step = max(1, -(-len(X) // (procs * 4)))
    bounds = [(s, min(s + step, len(X))) for s in range(0, len(X), step)]
    if procs == 1 or len(bounds) == 1:
        parts = [worker(b) for b in bounds]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            parts = pool.map(worker, bounds)
    out = [r for part in parts for r in part]
    if not keep_residual:
        for r in out:
            r.pop("residual", None)
    return out


def encode_exact_batched(a64, X, K, method="omp", tol=None, block=64):
    """``encode_one`` with ``exact_selector`` for a block of patches at once
    (see the module docstring).  Same control flow per patch: tolerance check
    before selecting, stop on a zero score, OMP stops on a re-selected atom."""
    X = np.asarray(X, dtype=np.float64)
    out = []
    for s0 in range(0, len(X), block):
        Xb = X[s0:s0 + block]
        nb = len(Xb)
        xn = np.linalg.norm(Xb, axis=1)
        tols = O.REL_TOL * xn if tol is None else np.full(nb, float(tol))
        R = Xb.copy()
        res = [dict(indices=[], coefs=np.zeros(0), steps=[], ip=0, cip=0, paths=[], gaps=[], rnorms=[])
               for _ in range(nb)]
        live = np.ones(nb, dtype=bool)
        m = a64.shape[0]
        for _ in range(K):
            rn = np.linalg.norm(R, axis=1)
            live &= ~(rn <= tols)
            ids = np.flatnonzero(live)
            if ids.size == 0:
                break
            S = R[ids] @ a64.T                      # [live, m]
            mags = np.abs(S)
            best = np.argmax(mags, axis=1)          # first maximum = lowest atom index
            top2 = np.partition(mags, m - 2, axis=1)[:, -2:] if m >= 2 else None
            for j, p in enumerate(ids):
                r = res[p]
                r["rnorms"].append(rn[p] / xn[p] if xn[p] > 0 else 0.0)
                i = int(best[j])
                sc = float(S[j, i])
                hi = float(top2[j, 1]) if top2 is not None else 0.0
                gap = math.inf if top2 is None or hi == 0.0 else (hi - float(top2[j, 0])) / hi
                r["ip"] += m
                if sc == 0.0:
                    live[p] = False
                    continue
                if method == "omp" and i in r["indices"]:
                    r["gaps"].append(gap)
                    live[p] = False
                    continue
                r["indices"].append(i)
                r["paths"].append([])
                r["gaps"].append(gap)
                if method == "mp":
                    r["steps"].append(sc)
                    R[p] = R[p] - sc * a64[i]
                else:
                    r["coefs"] = O.omp_refit(a64, r["indices"], Xb[p])
                    R[p] = Xb[p] - a64[r["indices"]].T @ r["coefs"]
        for p in range(nb):
            r = res[p]
            if method == "mp":
                r["coefs"] = np.asarray(r["steps"])
            r.pop("steps")
            r["resnorm"] = float(np.linalg.norm(R[p]))
            r["residual"] = R[p]
        out.extend(res)
    return out
