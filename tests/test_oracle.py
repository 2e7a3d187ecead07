"""Pin the CPU oracle: golden vectors everywhere, the live reference where mounted."""

import numpy as np
import pytest

from conftest import flat_from_fixture, golden
from oracle import stmp_oracle as O


def test_fnv_golden_vectors():
    z = golden("fnv.npz")
    payload = z["payload"].tobytes()
    pos = 0
    for length, h in zip(z["lengths"], z["hashes"]):
        assert O.fnv1a64(payload[pos:pos + length]) == int(h)
        pos += length
    # pkg/tests/test_dictionary.py:21-25
    assert O.fnv1a64(b"") == 0xCBF29CE484222325
    assert O.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert O.fnv1a64(b"foobar") == 0x85944171F73967E8


def test_counting_golden():
    z = golden("ipcount.npz")
    for b, a, p in zip(z["branching"], z["alpha"], z["predicted"]):
        br = tuple(int(k) for k in b if k)
        assert O.predicted_ip_count(br, float(a)) == int(p)
    for a, k, r in zip(z["rc_alpha"], z["rc_k"], z["rc_out"]):
        assert O.retained_count(float(a), int(k)) == int(r)
    with pytest.raises(ValueError):
        O.retained_count(0.0, 10)


def _tree(z):
    return O.OracleTree.from_flat(flat_from_fixture(z))


@pytest.mark.parametrize("tag,alpha", [("greedy", 0.1), ("beam", 0.3), ("full", 1.0)])
def test_tree_select_matches_golden(tag, alpha):
    z = golden("select_small.npz")
    t = _tree(z)
    a64 = z["atoms"].astype(np.float64)
    for q, i, s, ip in zip(z["Q"], z[f"{tag}_idx"], z[f"{tag}_score"], z[f"{tag}_ip"]):
        gi, gs, cip, aip, path, gap = O.tree_select(t, a64, q.astype(np.float64), alpha)
        assert gi == int(i)
        assert gs == pytest.approx(float(s), rel=1e-12, abs=1e-12)
        assert (cip + aip, cip) == (int(ip[0]), int(ip[1]))


def test_exact_select_matches_golden():
    z = golden("select_small.npz")
    a64 = z["atoms"].astype(np.float64)
    for q, i, s in zip(z["Q"], z["exact_idx"], z["exact_score"]):
        gi, gs, ips, _ = O.exact_select(a64, q.astype(np.float64))
        assert gi == int(i) and gs == pytest.approx(float(s), rel=1e-12, abs=1e-12)
        assert ips == a64.shape[0]


def test_ragged_tree_greedy_matches_golden():
    z = golden("select_ragged.npz")
    t = _tree(z)
    counts = set(t.child_count[1:].tolist())
    assert len(counts) > 1, "fixture must be ragged"
    a64 = z["atoms"].astype(np.float64)
    for q, i, s, ip in zip(z["Q"], z["idx"], z["score"], z["ip"]):
        gi, gs, cip, aip, path, _ = O.tree_select(t, a64, q.astype(np.float64), 1 / 7)
        assert gi == int(i) and gs == pytest.approx(float(s), rel=1e-12, abs=1e-12)
        assert (cip + aip, cip) == (int(ip[0]), int(ip[1]))
        # path is consistent with the tree: each node is a child of the previous one
        prev = 0
        for node in path:
            b, c = t.child_begin[prev], t.child_count[prev]
            assert b <= node < b + c
            prev = node
        b, c = t.child_begin[prev], t.child_count[prev]
        assert gi in t.leaf_atom[b:b + c]


def _check_runs(res, z, prefix, K):
    packed = O.pack(res, K)
    np.testing.assert_array_equal(packed["count"], z[f"{prefix}_count"])
    np.testing.assert_array_equal(packed["idx"], z[f"{prefix}_idx"])
    np.testing.assert_allclose(packed["coef"], z[f"{prefix}_coef"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(packed["resnorm"], z[f"{prefix}_resnorm"], rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal(packed["ip"], z[f"{prefix}_ip"])


@pytest.mark.parametrize("sel", ["tree", "exact"])
@pytest.mark.parametrize("method", ["omp", "mp"])
def test_pursuit_matches_golden(sel, method):
    z = golden("pursuit_small.npz")
    K = int(z["K"])
    a64 = z["atoms"].astype(np.float64)
    select = O.tree_selector(_tree(z), a64, 1 / 16) if sel == "tree" else O.exact_selector(a64)
    res = O.encode_batch(select, a64, z["X"], K, method)
    _check_runs(res, z, f"{sel}_{method}", K)


@pytest.mark.parametrize("tag,method,rows", [("tree_omp", "omp", 256), ("tree_mp", "mp", 256),
                                             ("exact_omp", "omp", 32)])
def test_config0_prefix_matches_golden(tag, method, rows):
    from paper_1412_0680_b200 import tree as T
    from paper_1412_0680_b200 import workloads as W
    import os
    from conftest import GOLDEN
    cfg = W.CONFIGS[0]
    wl = W.make_dictionary(cfg)
    flat = T.load_structure(os.path.join(GOLDEN, "trees", "c0.npz"), wl.atoms)
    z = golden("c0_prefix.npz")
    a64 = wl.atoms.astype(np.float64)
    X = z["X"][:rows]
    np.testing.assert_array_equal(X, W.make_patches(wl, rows))
    select = (O.tree_selector(O.OracleTree.from_flat(flat), a64, cfg.alpha) if tag.startswith("tree")
              else O.exact_selector(a64))
    res = O.encode_batch(select, a64, X, cfg.K, method)
    sub = {k: z[k][:rows] for k in z.files if k.startswith(tag)}
    _check_runs(res, sub, tag, cfg.K)


@pytest.mark.parametrize("tol_tag,tol", [("deftol", None), ("tol0", 0.0), ("tol05", 0.5)])
@pytest.mark.parametrize("method", ["omp", "mp"])
def test_edge_cases_match_golden(tol_tag, tol, method):
    z = golden("edge.npz")
    p = golden("pursuit_small.npz")
    a64 = p["atoms"].astype(np.float64)
    select = O.tree_selector(_tree(p), a64, 1 / 16)
    res = O.encode_batch(select, a64, z["E"], 4, method, tol)
    _check_runs(res, z, f"{method}_{tol_tag}", 4)
    i, s, *_ = select(np.zeros(24))
    assert (i, s) == (int(z["zero_tree_select"][0]), float(z["zero_tree_select"][1]))


def test_oracle_tree_select_matches_live_reference(stmp_ref):
    """The oracle walk vs the reference's own stmp_select on fresh random trees,
    index and score bitwise (f64, same arithmetic)."""
    from paper_1412_0680_b200 import tree as T
    rng = np.random.default_rng(42)
    for m, n, br in ((300, 9, (6, 5)), (1000, 16, (10, 10, 3)), (257, 20, (9, 4))):
        d = stmp_ref.normalize_columns(rng.standard_normal((m, n)))
        tree = stmp_ref.build_tree(d, br, seed=int(rng.integers(1 << 30)))
        t = O.OracleTree.from_flat(T.from_reference_tree(tree))
        a64 = d.scoring_atoms
        alpha = 1 / max(br)
        for _ in range(60):
            q = rng.standard_normal(n)
            ri, rs = stmp_ref.stmp_select(tree, d, q, alpha, stmp_ref.ScoreCounter())
            gi, gs, *_ = O.tree_select(t, a64, q, alpha)
            assert (gi, gs) == (ri, rs)


def test_oracle_omp_refit_matches_reference(stmp_ref):
    rng = np.random.default_rng(26)
    d = stmp_ref.normalize_columns(rng.standard_normal((60, 20)))
    for _ in range(10):
        support = sorted(rng.choice(60, size=5, replace=False).tolist())
        x = rng.standard_normal(20)
        np.testing.assert_allclose(O.omp_refit(d.scoring_atoms, support, x),
                                   stmp_ref.omp_refit(d, support, x), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("method", ["omp", "mp"])
def test_batched_exact_oracle_equals_per_patch(method):
    """oracle/parallel.py's GEMM-batched exhaustive oracle (used for the large
    exhaustive parity prefixes) against the per-patch restatement."""
    from oracle import parallel as OP
    z = golden("pursuit_small.npz")
    a64 = z["atoms"].astype(np.float64)
    K = int(z["K"])
    X = np.concatenate([z["X"], np.zeros((1, z["X"].shape[1]), np.float32)])
    ref = O.pack(O.encode_batch(O.exact_selector(a64), a64, X, K, method), K)
    got = O.pack(OP.encode_exact_batched(a64, X, K, method, block=7), K)
    np.testing.assert_array_equal(got["idx"], ref["idx"])
    np.testing.assert_array_equal(got["count"], ref["count"])
    np.testing.assert_array_equal(got["ip"], ref["ip"])
    np.testing.assert_allclose(got["coef"], ref["coef"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(got["resnorm"], ref["resnorm"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got["gaps"], ref["gaps"], rtol=1e-9)
    # and it reproduces the reference's own recorded exhaustive runs
    np.testing.assert_array_equal(got["idx"][:-1], z[f"exact_{method}_idx"])


def test_parallel_tree_oracle_equals_serial():
    from oracle import parallel as OP
    z = golden("pursuit_small.npz")
    a64 = z["atoms"].astype(np.float64)
    t = _tree(z)
    K = int(z["K"])
    ref = O.pack(O.encode_batch(O.tree_selector(t, a64, 1 / 16), a64, z["X"], K, "omp"), K)
    got = O.pack(OP.encode_parallel(t, a64, z["X"], K, "omp", alpha=1 / 16, procs=2), K)
    for k in ("idx", "coef", "count", "resnorm", "ip", "path", "gaps"):
        np.testing.assert_array_equal(got[k], ref[k])
