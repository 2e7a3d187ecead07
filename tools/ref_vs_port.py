"""Time the UNMODIFIED reference against the oracle port on the same patches
(build container only: /root/reference does not exist on the GPU box).

`bench.py --impl reference` has to time the oracle port (oracle/stmp_oracle.py)
because a Python reference cannot travel to the GPU box.  This script shows
what that stands in for: on identical f32 inputs it runs

* the reference itself -- `stmp.TreeSelector` / `stmp.ExactSelector`
  (pkg/src/stmp/pursuit.py:165-191) driven through `stmp.matching_pursuit`
  (MP, :194-221) or the SURVEY §8c OMP composition of `selector.select` +
  `stmp.omp_refit` (:235-250), tree loaded with the reference's `load_tree`
  from the .tree bytes our `tree.write_tree_file` emits;
* the oracle port's `encode_one` on the same patches,

one process each, single-threaded BLAS, and checks that both produce the same
supports, coefficients and residual norms.  Output: one JSON line per config
(profiles/r02_reference_vs_port.jsonl).

Usage: OPENBLAS_NUM_THREADS=1 python tools/ref_vs_port.py [cid ...]
"""

import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import stmp  # noqa: E402

from oracle import stmp_oracle as O  # noqa: E402
from paper_1412_0680_b200 import tree as T  # noqa: E402
from paper_1412_0680_b200 import workloads as W  # noqa: E402

SAMPLE = {0: 400, 1: 300, 2: 100, 3: 200, 4: 40}


def ref_omp(selector, d, x, K):
    """SURVEY §8c OMP loop from the reference's own pieces (as tests/golden/make_golden.py)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    counter = stmp.ScoreCounter()
    tol = 1e-6 * float(np.linalg.norm(x))
    r = x.copy()
    S, c = [], np.zeros(0)
    for _ in range(K):
        if float(np.linalg.norm(r)) <= tol:
            break
        i, s = selector.select(r, counter)
        if s == 0.0 or i in S:
            break
        S.append(i)
        c = stmp.omp_refit(d, S, x)
        r = x - d.scoring_atoms[S].T @ c
    return S, list(c), float(np.linalg.norm(r))


def ref_mp(selector, d, x, K):
    code = stmp.matching_pursuit(selector, x, stmp.SearchParams(K=K))
    resid = np.asarray(x, dtype=np.float64) - stmp.reconstruct(d, code)
    return [i for i, _ in code.entries], [c for _, c in code.entries], float(np.linalg.norm(resid))


def run(cid, method="omp", selector="tree"):
    cfg = W.CONFIGS[cid]
    wl = W.make_dictionary(cfg)
    n = SAMPLE[cid] if selector == "tree" else 4
    X = W.make_patches(wl, n)
    flat = T.load_structure(os.path.join(ROOT, "tests", "golden", "trees", f"c{cid}.npz"), wl.atoms)
    d = stmp.Dictionary(wl.atoms)
    a64 = wl.atoms.astype(np.float64)
    if selector == "tree":
        path = f"/tmp/ref_vs_port_c{cid}.tree"
        with open(path, "wb") as fh:
            fh.write(T.write_tree_file(flat))
        tree = stmp.load_tree(path)
        rsel = stmp.TreeSelector(tree, d, cfg.alpha)
        osel = O.tree_selector(O.OracleTree.from_flat(flat), a64, cfg.alpha)
    else:
        rsel = stmp.ExactSelector(d)
        osel = O.exact_selector(a64)
    d.scoring_atoms  # the lazily built f64 copy is set-up, not per-patch work
    fn = ref_omp if method == "omp" else ref_mp
    fn(rsel, d, X[0], cfg.K)  # warm caches
    t0 = time.perf_counter()
    ref = [fn(rsel, d, X[p], cfg.K) for p in range(n)]
    t_ref = time.perf_counter() - t0
    O.encode_one(osel, a64, X[0], cfg.K, method)
    t0 = time.perf_counter()
    port = [O.encode_one(osel, a64, X[p], cfg.K, method) for p in range(n)]
    t_port = time.perf_counter() - t0
    same_idx = sum(list(r[0]) == [int(i) for i in q["indices"]] for r, q in zip(ref, port))
    coef_err = max((float(np.max(np.abs(np.asarray(r[1]) - np.asarray(q["coefs"]))
                                 / np.maximum(np.abs(np.asarray(r[1])), 1e-30)))
                    if len(r[1]) else 0.0) for r, q in zip(ref, port) if list(r[0]) == [int(i) for i in q["indices"]])
    return {
        "workload": f"{cfg.name}/{selector}-{method.upper()}", "patches": n,
        "reference_patches_per_s_1core": n / t_ref, "port_patches_per_s_1core": n / t_port,
        "port_over_reference": t_ref / t_port,
        "identical_supports": same_idx, "max_coef_rel_diff": coef_err,
        "reference": "pkg/src/stmp (unmodified, imported from /root/reference) TreeSelector/ExactSelector + "
                     "matching_pursuit / select+omp_refit", "port": "oracle/stmp_oracle.encode_one",
        "cpu": open("/proc/cpuinfo").read().split("model name")[1].split(":")[1].split("\n")[0].strip(),
    }


if __name__ == "__main__":
    cids = [int(c) for c in sys.argv[1:]] or [0, 1, 2, 3, 4]
    for cid in cids:
        print(json.dumps(run(cid)), flush=True)
        if cid == 1:
            print(json.dumps(run(cid, "mp")), flush=True)
        if cid == 4:
            print(json.dumps(run(cid, "omp", "exact")), flush=True)
