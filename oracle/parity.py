"""CPU ORACLE side -- test infrastructure only.  Parity comparator between GPU
outputs and the CPU oracle (SURVEY §8c contract); used by tests/ and by
bench.py's parity block.

* Atom indices and tree paths must be equal, except from the first iteration
  at which the oracle's decision had a relative top-2 gap < 1e-5 (a near-tie),
  or was taken on a residual already at fp32 rounding level (||r|| < 1e-5 ||x||,
  e.g. an exactly sparse patch coded with tolerance 0): that patch is counted
  as excused from then on.
* Coefficients and residual norms within 1e-4 relative (plus an absolute floor
  of 1e-6 * ||x|| for values that are themselves ~0).
* Inner-product counts equal.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NEAR_TIE = 1e-5
# A selection made on a residual whose norm is below 1e-5 ||x|| is fp32 rounding
# noise on the GPU (the f64 oracle sees ~1e-16 noise instead): excused like a tie.
NOISE_RESIDUAL = 1e-5
RTOL = 1e-4
ATOL_REL_X = 1e-6


@dataclass
class ParityReport:
    patches: int = 0
    excused: int = 0
    excused_by_reason: dict = field(default_factory=lambda: {"near_tie": 0, "noise_residual": 0,
                                                             "noise_stop_ip": 0})
    failures: list = field(default_factory=list)
    failures_by_kind: dict = field(default_factory=lambda: {"idx": 0, "coef": 0, "resnorm": 0, "ip": 0, "path": 0})
    max_coef_rel: float = 0.0
    max_res_rel: float = 0.0

    @property
    def ok(self) -> bool:
        return not self.failures

    def summary(self) -> str:
        head = (f"{self.patches} patches, {self.excused} excused {self.excused_by_reason}, "
                f"{len(self.failures)} failures {self.failures_by_kind}, max coef rel err {self.max_coef_rel:.2e}, "
                f"max resnorm rel err {self.max_res_rel:.2e}")
        return head + ("" if self.ok else "\n  " + "\n  ".join(self.failures[:10]))

    def as_dict(self) -> dict:
        return {"patches": self.patches, "excused_near_ties": self.excused_by_reason["near_tie"],
                "excused_by_reason": dict(self.excused_by_reason), "failures": len(self.failures),
                "failures_by_kind": dict(self.failures_by_kind),
                "max_coef_rel": self.max_coef_rel, "max_resnorm_rel": self.max_res_rel}


def compare(gpu: dict, ref: dict, X: np.ndarray, check_ip: bool = True, check_path: bool = True,
            near_tie: float = NEAR_TIE) -> ParityReport:
    """``gpu`` and ``ref`` hold idx [N,K], coef [N,K], count [N], resnorm [N],
    ip [N,2] (optional), path [N,K,L] (optional); ``ref`` also holds ``gaps``
    [N,K] (oracle relative top-2 gap per iteration, inf when unknown)."""
    rep = ParityReport(patches=len(X))
    xnorm = np.linalg.norm(np.asarray(X, dtype=np.float64), axis=1)
    gi, ri = np.asarray(gpu["idx"]), np.asarray(ref["idx"])
    gc, rc = np.asarray(gpu["count"]), np.asarray(ref["count"])
    gaps = ref.get("gaps")
    rnorm_rel = ref.get("rnorm_rel")
    for p in range(len(X)):
        K = gi.shape[1]
        # first iteration where the decisions differ
        diff_at = None
        for it in range(K):
            a = gi[p, it] if it < gc[p] else -1
            b = ri[p, it] if it < rc[p] else -1
            if a != b:
                diff_at = it
                break
        if diff_at is not None:
            g = gaps[p, diff_at] if gaps is not None and diff_at < gaps.shape[1] else np.inf
            rr = rnorm_rel[p, diff_at] if rnorm_rel is not None and diff_at < rnorm_rel.shape[1] else np.inf
            if g < near_tie or rr < NOISE_RESIDUAL:
                rep.excused += 1
                rep.excused_by_reason["near_tie" if g < near_tie else "noise_residual"] += 1
                continue
            rep.failures_by_kind["idx"] += 1
            rep.failures.append(f"patch {p}: iteration {diff_at} gpu {gi[p, :gc[p]].tolist()} "
                                f"ref {ri[p, :rc[p]].tolist()} (gap {g:.2e})")
            continue
        c = int(rc[p])
        atol = ATOL_REL_X * xnorm[p]
        gcoef = np.asarray(gpu["coef"][p, :c], dtype=np.float64)
        rcoef = np.asarray(ref["coef"][p, :c], dtype=np.float64)
        err = np.abs(gcoef - rcoef)
        if c:
            rel = float(np.max(err / np.maximum(np.abs(rcoef), atol / RTOL + 1e-300)))
            rep.max_coef_rel = max(rep.max_coef_rel, rel)
            if np.any(err > RTOL * np.abs(rcoef) + atol):
                rep.failures_by_kind["coef"] += 1
                rep.failures.append(f"patch {p}: coef gpu {gcoef} ref {rcoef}")
                continue
        gr, rr = float(gpu["resnorm"][p]), float(ref["resnorm"][p])
        rep.max_res_rel = max(rep.max_res_rel, abs(gr - rr) / max(rr, atol / RTOL, 1e-300))
        if abs(gr - rr) > RTOL * rr + atol:
            rep.failures_by_kind["resnorm"] += 1
            rep.failures.append(f"patch {p}: resnorm gpu {gr} ref {rr}")
            continue
        noisy = rnorm_rel is not None and bool(np.any(rnorm_rel[p] < NOISE_RESIDUAL))
        if noisy and gpu["ip"] is not None and not np.array_equal(
                np.asarray(gpu["ip"][p], dtype=np.int64), np.asarray(ref["ip"][p], dtype=np.int64)):
            # the stop after a noise-level residual (exact-zero tests) differs between f32 and f64
            rep.excused += 1
            rep.excused_by_reason["noise_stop_ip"] += 1
            continue
        if check_ip and "ip" in gpu and "ip" in ref and gpu["ip"] is not None:
            if not np.array_equal(np.asarray(gpu["ip"][p], dtype=np.int64), np.asarray(ref["ip"][p], dtype=np.int64)):
                rep.failures_by_kind["ip"] += 1
                rep.failures.append(f"patch {p}: ip gpu {gpu['ip'][p]} ref {ref['ip'][p]}")
                continue
        if check_path and gpu.get("path") is not None and ref.get("path") is not None:
            gp = np.asarray(gpu["path"][p, :c])
            rp = np.asarray(ref["path"][p, :c])
            bad = np.flatnonzero((gp != rp).any(axis=-1)) if gp.ndim > 1 else np.flatnonzero(gp != rp)
            if bad.size and gaps is not None and gaps[p, bad[0]] < near_tie:
                # the path (frontier[0]) can differ alone at a near tie of a beam boundary
                rep.excused += 1
                rep.excused_by_reason["near_tie"] += 1
                continue
            if not np.array_equal(gp, rp):
                rep.failures_by_kind["path"] += 1
                rep.failures.append(f"patch {p}: path gpu {gp.tolist()} ref {rp.tolist()}")
    return rep
