"""Generate the golden fixtures from the REFERENCE itself (build container only).

Every expected value in tests/golden/*.npz is produced here by importing the
unmodified reference package from /root/reference/pkg/src.  The
GPU box has no /root/reference, so the tests there compare against these
committed vectors.

Fixtures
--------
fnv.npz            fnv1a64 golden vectors (incl. pkg/tests/test_dictionary.py:21-25)
ipcount.npz        retained_count / predicted_ip_count cases (pkg/tests/test_pursuit.py:35-51)
select_small.npz   stmp_select (greedy and beam alpha) + exact_select on a (10,5) tree
select_ragged.npz  greedy stmp_select on a ragged (7,5) tree over m=97 atoms
pursuit_small.npz  matching_pursuit (tree + exact) and the restated OMP loop, K=6
c0_prefix.npz      config 0, first 1024 patches: tree-OMP / tree-MP / exhaustive-OMP
edge.npz           zero patch, atom patch (early stop), tolerance 0, r == 0 selects

Usage:  python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import stmp  # noqa: E402
from paper_1412_0680_b200 import tree as T  # noqa: E402
from paper_1412_0680_b200 import workloads as W  # noqa: E402


def flat_arrays(tree):
    f = T.from_reference_tree(tree)
    return dict(t_branching=np.asarray(f.branching), t_n=f.n,
                t_fingerprint=np.array([f.fingerprint], dtype=np.uint64),
                t_level_offsets=f.level_offsets, t_child_begin=f.child_begin,
                t_child_count=f.child_count, t_centroids=f.centroids, t_leaf_atom=f.leaf_atom)


def ref_omp(selector, d, x, K, tol=None):
    """The SURVEY §8c OMP restatement composed from the reference's own
    selector.select and omp_refit (pursuit.py:203-221, 235-250)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    counter = stmp.ScoreCounter()
    if tol is None:
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
    return S, c, float(np.linalg.norm(r)), counter


def ref_mp(selector, d, x, K, tol=None):
    counter = stmp.ScoreCounter()
    code = stmp.matching_pursuit(selector, x, stmp.SearchParams(K=K, residual_tolerance=tol), counter)
    resid = np.asarray(x, dtype=np.float64) - stmp.reconstruct(d, code)
    return [i for i, _ in code.entries], [c for _, c in code.entries], float(np.linalg.norm(resid)), counter


def pack_runs(runs, K):
    N = len(runs)
    idx = np.full((N, K), -1, np.int64)
    coef = np.zeros((N, K))
    cnt = np.zeros(N, np.int64)
    res = np.zeros(N)
    ip = np.zeros((N, 2), np.int64)
    for p, (S, c, rn, ctr) in enumerate(runs):
        cnt[p] = len(S)
        idx[p, :len(S)] = S
        coef[p, :len(S)] = c
        res[p] = rn
        ip[p] = (ctr.inner_products, ctr.centroid_inner_products)
    return idx, coef, cnt, res, ip


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name)


def main():
    # --- FNV golden vectors
    msgs = [b"", b"a", b"foobar", bytes(range(256)), b"stmp-b200" * 37]
    save("fnv.npz", lengths=np.array([len(m) for m in msgs]),
         payload=np.frombuffer(b"".join(msgs), dtype=np.uint8),
         hashes=np.array([stmp.fnv1a64(m) for m in msgs], dtype=np.uint64))

    # --- counting cases
    rng = np.random.default_rng(0)
    cases = [((100, 10, 10), 0.1), ((100, 10), 0.1), ((100, 10, 10, 10), 0.1), ((7,), 0.05),
             ((16, 16, 16), 1 / 16), ((32, 32, 16), 1 / 32), ((256, 256), 1 / 256),
             ((64, 40, 40), 1 / 64), ((64, 64, 32), 1 / 64)]
    for _ in range(30):
        depth = int(rng.integers(1, 5))
        cases.append((tuple(int(k) for k in rng.integers(2, 30, size=depth)), float(rng.uniform(0.02, 1.0))))
    br = np.zeros((len(cases), 4), np.int64)
    for i, (b, _) in enumerate(cases):
        br[i, :len(b)] = b
    rc_cases = [(1.0, 10), (0.1, 100), (0.1, 10), (0.05, 10), (0.25, 10)]
    save("ipcount.npz", branching=br, alpha=np.array([a for _, a in cases]),
         predicted=np.array([stmp.predicted_ip_count(b, a) for b, a in cases]),
         rc_alpha=np.array([a for a, _ in rc_cases]), rc_k=np.array([k for _, k in rc_cases]),
         rc_out=np.array([stmp.retained_count(a, k) for a, k in rc_cases]))

    # --- small tree selection (greedy + beam alphas) and exhaustive
    d = stmp.normalize_columns(np.random.default_rng(3).standard_normal((500, 10)))
    tree = stmp.build_tree(d, (10, 5), seed=4)
    Q = np.random.default_rng(5).standard_normal((200, 10)).astype(np.float32)
    out = {}
    for tag, alpha in (("greedy", 0.1), ("beam", 0.3), ("full", 1.0)):
        res = [stmp.stmp_select(tree, d, q, alpha, c := stmp.ScoreCounter()) + (c.inner_products, c.centroid_inner_products) for q in Q]
        out[f"{tag}_idx"] = np.array([r[0] for r in res])
        out[f"{tag}_score"] = np.array([r[1] for r in res])
        out[f"{tag}_ip"] = np.array([[r[2], r[3]] for r in res])
    ex = [stmp.exact_select(d, q, stmp.ScoreCounter()) for q in Q]
    save("select_small.npz", atoms=d.atoms, Q=Q, exact_idx=np.array([e[0] for e in ex]),
         exact_score=np.array([e[1] for e in ex]), **out, **flat_arrays(tree))

    # --- ragged tree (m not a product of the branching)
    d = stmp.normalize_columns(np.random.default_rng(6).standard_normal((97, 12)))
    tree = stmp.build_tree(d, (7, 5), seed=7)
    Q = np.random.default_rng(8).standard_normal((300, 12)).astype(np.float32)
    res = [stmp.stmp_select(tree, d, q, 1 / 7, c := stmp.ScoreCounter()) + (c.inner_products, c.centroid_inner_products) for q in Q]
    save("select_ragged.npz", atoms=d.atoms, Q=Q, idx=np.array([r[0] for r in res]),
         score=np.array([r[1] for r in res]), ip=np.array([[r[2], r[3]] for r in res]),
         **flat_arrays(tree))

    # --- pursuit runs on a small (16,8) tree, n=24
    d = stmp.normalize_columns(np.random.default_rng(9).standard_normal((1024, 24)))
    tree = stmp.build_tree(d, (16, 8), seed=10)
    X = np.random.default_rng(11).standard_normal((150, 24)).astype(np.float32)
    K = 6
    tsel = stmp.TreeSelector(tree, d, 1 / 16)
    esel = stmp.ExactSelector(d)
    arrays = {}
    for tag, sel in (("tree", tsel), ("exact", esel)):
        for meth, fn in (("omp", ref_omp), ("mp", ref_mp)):
            i, c, n_, r, ip = pack_runs([fn(sel, d, x, K) for x in X], K)
            arrays.update({f"{tag}_{meth}_idx": i, f"{tag}_{meth}_coef": c, f"{tag}_{meth}_count": n_,
                           f"{tag}_{meth}_resnorm": r, f"{tag}_{meth}_ip": ip})
    save("pursuit_small.npz", atoms=d.atoms, X=X, K=K, **arrays, **flat_arrays(tree))

    # --- config 0 prefix (tree from the shipped structure == reference build_tree)
    cfg = W.CONFIGS[0]
    wl = W.make_dictionary(cfg)
    d = stmp.Dictionary(wl.atoms)
    tree = stmp.build_tree(d, cfg.branching, W.tree_seed(0))
    X = W.make_patches(wl, 1024)
    tsel = stmp.TreeSelector(tree, d, cfg.alpha)
    arrays = {}
    for tag, sel, fn, rows in (("tree_omp", tsel, ref_omp, 1024), ("tree_mp", tsel, ref_mp, 1024),
                               ("exact_omp", stmp.ExactSelector(d), ref_omp, 128)):
        i, c, n_, r, ip = pack_runs([fn(sel, d, x, cfg.K) for x in X[:rows]], cfg.K)
        arrays.update({f"{tag}_idx": i, f"{tag}_coef": c, f"{tag}_count": n_, f"{tag}_resnorm": r, f"{tag}_ip": ip})
    save("c0_prefix.npz", X=X, **arrays)

    # --- edge cases on the pursuit_small dictionary
    d = stmp.normalize_columns(np.random.default_rng(9).standard_normal((1024, 24)))
    tree = stmp.build_tree(d, (16, 8), seed=10)
    tsel = stmp.TreeSelector(tree, d, 1 / 16)
    E = np.stack([np.zeros(24), d.atoms[5], 2.5 * d.atoms[700] - 0.5 * d.atoms[3],
                  np.full(24, 1e-3), -d.atoms[1023]]).astype(np.float32)
    arrays = {}
    for tol_tag, tol in (("deftol", None), ("tol0", 0.0), ("tol05", 0.5)):
        for meth, fn in (("omp", ref_omp), ("mp", ref_mp)):
            i, c, n_, r, ip = pack_runs([fn(tsel, d, x, 4, tol) for x in E], 4)
            arrays.update({f"{meth}_{tol_tag}_idx": i, f"{meth}_{tol_tag}_coef": c,
                           f"{meth}_{tol_tag}_count": n_, f"{meth}_{tol_tag}_resnorm": r, f"{meth}_{tol_tag}_ip": ip})
    sel0 = stmp.stmp_select(tree, d, np.zeros(24), 1 / 16, stmp.ScoreCounter())
    ex0 = stmp.exact_select(d, np.zeros(24), stmp.ScoreCounter())
    save("edge.npz", E=E, zero_tree_select=np.array([sel0[0], sel0[1]]),
         zero_exact_select=np.array([ex0[0], ex0[1]]), **arrays)


if __name__ == "__main__":
    main()
