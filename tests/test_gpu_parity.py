"""GPU parity: the sm_100a path through the C ABI vs the golden vectors and the
CPU oracle (SURVEY §8c contract, comparator in tests/parity.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, flat_from_fixture, golden
from oracle import stmp_oracle as O
from parity import compare

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1412_0680_b200 import build
    build.build()


def P():
    import paper_1412_0680_b200 as pkg
    return pkg


# (score_kernel, update_kernel, gram_path) per staged variant; library defaults
# are (2, 1, 1).  Every id runs a distinct kernel set: the whole-table score pass
# (score_ts) or the streamed one (score_st) at every level; the lockstep /
# wide-row OMP update or the generic one; the Gram path (no residual, pair
# tables; auto = config 4) forced on, or off; the streamed pass with the 3xFP16
# split (score_s16) at every level of the residual pipeline.
STAGED_KERNELS = {"staged-ts": (2, 1, 1), "staged-st": (3, 1, 1), "staged-generic": (2, 0, 0),
                  "staged-resid": (2, 1, 0), "staged-gram": (2, 1, 2), "staged-s16": (4, 1, 0)}
PATHS = ["fused", *STAGED_KERNELS]


def restore_defaults(_lib):
    _lib.set_option("path", _lib.PATH_AUTO)
    _lib.set_option("score_kernel", 2)
    _lib.set_option("update_kernel", 1)
    _lib.set_option("gram_path", 1)
    _lib.set_option("half_scores", 1)


@pytest.fixture(params=PATHS)
def path(request):
    """Force one encoder implementation (the C ABI 'path' / 'score_kernel' /
    'update_kernel' options)."""
    from paper_1412_0680_b200 import _lib
    mode = request.param
    _lib.set_option("path", _lib.PATH_FUSED if mode == "fused" else _lib.PATH_STAGED)
    sk, uk, gp = STAGED_KERNELS.get(mode, (2, 1, 1))
    _lib.set_option("score_kernel", sk)
    _lib.set_option("update_kernel", uk)
    _lib.set_option("gram_path", gp)
    yield mode
    restore_defaults(_lib)


@pytest.mark.parametrize("kernels", sorted(set(STAGED_KERNELS.values()) - {(2, 1, 0)}))
def test_staged_is_deterministic_and_batch_invariant(kernels):
    """262,144 config-1 patches: two runs and a run in 8192-patch batches must agree
    bitwise (each patch's arithmetic is independent of bucketing order)."""
    from paper_1412_0680_b200 import _lib
    from paper_1412_0680_b200 import workloads as W
    cfg, wl, flat = config(1)
    X = torch.as_tensor(W.make_patches(wl, 262144)).cuda()
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    _lib.set_option("path", _lib.PATH_STAGED)
    _lib.set_option("score_kernel", kernels[0])
    _lib.set_option("update_kernel", kernels[1])
    _lib.set_option("gram_path", kernels[2])
    try:
        a = P().encode(sel, X, cfg.K, method="omp")
        b = P().encode(sel, X, cfg.K, method="omp")
        c = [P().encode(sel, X[s:s + 8192], cfg.K, method="omp") for s in range(0, len(X), 8192)]
        torch.cuda.synchronize()
        ci = torch.cat([r.idx for r in c])
        cc = torch.cat([r.coef for r in c])
        assert int((a.idx != b.idx).any(1).sum()) == 0
        assert int((a.idx != ci).any(1).sum()) == 0
        assert bool(torch.equal(a.coef, cc))
    finally:
        restore_defaults(_lib)


def as_np(res):
    out = {k: getattr(res, k) for k in ("idx", "coef", "count", "resnorm", "ip", "path")}
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items() if v is not None}


def oracle_pack(select, a64, X, K, method, tol=None):
    return O.pack(O.encode_batch(select, a64, X, K, method, tol), K)


def run(selector, X, K, method, tol=None, paths=True):
    Xd = torch.as_tensor(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    res = P().encode(selector, Xd, K, method=method, tol=tol, paths=paths)
    torch.cuda.synchronize()
    return as_np(res)


# ----------------------------------------------------------------- small fixtures

def test_tree_select_small_matches_reference():
    z = golden("select_small.npz")
    flat = flat_from_fixture(z)
    sel = P().TreeSelector(flat, z["atoms"], 0.1)
    out = run(sel, z["Q"], 1, "select")
    t = O.OracleTree.from_flat(flat)
    a64 = z["atoms"].astype(np.float64)
    gaps = np.array([O.tree_select(t, a64, q.astype(np.float64), 0.1)[5] for q in z["Q"]])
    ok = (out["idx"][:, 0] == z["greedy_idx"]) | (gaps < 1e-5)
    assert ok.all()
    same = out["idx"][:, 0] == z["greedy_idx"]
    np.testing.assert_allclose(out["coef"][same, 0], z["greedy_score"][same], rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(out["ip"], z["greedy_ip"])


def test_exact_select_small_matches_reference():
    z = golden("select_small.npz")
    sel = P().ExactSelector(z["atoms"])
    out = run(sel, z["Q"], 1, "select")
    assert (out["idx"][:, 0] == z["exact_idx"]).mean() == 1.0
    np.testing.assert_allclose(out["coef"][:, 0], z["exact_score"], rtol=1e-5, atol=1e-6)
    assert (out["ip"][:, 0] == 500).all() and (out["ip"][:, 1] == 0).all()


def test_ragged_tree_select_matches_reference():
    z = golden("select_ragged.npz")
    flat = flat_from_fixture(z)
    sel = P().TreeSelector(flat, z["atoms"], 1 / 7)
    out = run(sel, z["Q"], 1, "select")
    np.testing.assert_array_equal(out["idx"][:, 0], z["idx"])
    np.testing.assert_allclose(out["coef"][:, 0], z["score"], rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(out["ip"], z["ip"])


@pytest.mark.parametrize("sel_kind", ["tree", "exact"])
@pytest.mark.parametrize("method", ["omp", "mp"])
def test_pursuit_small_matches_reference(sel_kind, method, path):
    z = golden("pursuit_small.npz")
    K = int(z["K"])
    flat = flat_from_fixture(z)
    a64 = z["atoms"].astype(np.float64)
    if sel_kind == "tree":
        sel = P().TreeSelector(flat, z["atoms"], 1 / 16)
        osel = O.tree_selector(O.OracleTree.from_flat(flat), a64, 1 / 16)
    else:
        sel = P().ExactSelector(z["atoms"])
        osel = O.exact_selector(a64)
    out = run(sel, z["X"], K, method)
    ref = oracle_pack(osel, a64, z["X"], K, method)
    # the oracle itself equals the reference run recorded in the fixture
    np.testing.assert_array_equal(ref["idx"], z[f"{sel_kind}_{method}_idx"])
    rep = compare(out, ref, z["X"], check_path=sel_kind == "tree")
    assert rep.ok, rep.summary()
    assert rep.excused <= 2


@pytest.mark.parametrize("tol_tag,tol", [("deftol", None), ("tol0", 0.0), ("tol05", 0.5)])
@pytest.mark.parametrize("method", ["omp", "mp"])
def test_edge_cases(tol_tag, tol, method, path):
    z = golden("edge.npz")
    p = golden("pursuit_small.npz")
    sel = P().TreeSelector(flat_from_fixture(p), p["atoms"], 1 / 16)
    out = run(sel, z["E"], 4, method, tol)
    ref = {k.split("_", 2)[2]: z[k] for k in z.files if k.startswith(f"{method}_{tol_tag}_")}
    a64 = p["atoms"].astype(np.float64)
    orc = oracle_pack(O.tree_selector(O.OracleTree.from_flat(flat_from_fixture(p)), a64, 1 / 16),
                      a64, z["E"], 4, method, tol)
    ref["gaps"], ref["rnorm_rel"] = orc["gaps"], orc["rnorm_rel"]
    rep = compare(out, ref, z["E"], check_path=False)
    assert rep.ok, rep.summary()
    # zero patch: empty code, zero residual (pursuit.py:214 with tolerance 0)
    assert out["count"][0] == 0 and out["resnorm"][0] == 0.0


def test_zero_residual_select_matches_reference():
    z = golden("edge.npz")
    p = golden("pursuit_small.npz")
    sel = P().TreeSelector(flat_from_fixture(p), p["atoms"], 1 / 16)
    out = run(sel, np.zeros((1, 24), np.float32), 1, "select")
    assert out["idx"][0, 0] == int(z["zero_tree_select"][0])
    assert out["coef"][0, 0] == 0.0
    ex = P().ExactSelector(p["atoms"])
    out = run(ex, np.zeros((1, 24), np.float32), 1, "select")
    assert out["idx"][0, 0] == int(z["zero_exact_select"][0]) == 0


def test_selector_protocol_drop_in():
    """The GPU selector plugs into the reference's MP control flow unchanged
    (pursuit.py:194-221, restated by the oracle loop) and gives the same codes."""
    z = golden("pursuit_small.npz")
    flat = flat_from_fixture(z)
    sel = P().TreeSelector(flat, z["atoms"], 1 / 16)
    a64 = z["atoms"].astype(np.float64)
    counter = P().ScoreCounter()

    def gpu_select(r):
        before = (counter.inner_products, counter.centroid_inner_products)
        i, s = sel.select(r, counter)
        ci = counter.centroid_inner_products - before[1]
        return i, s, ci, counter.inner_products - before[0] - ci, [], np.inf

    for p_, x in enumerate(z["X"][:20]):
        got = O.encode_one(gpu_select, a64, x, int(z["K"]), "mp")
        assert got["indices"] == [int(i) for i in z["tree_mp_idx"][p_, :z["tree_mp_count"][p_]]]
        np.testing.assert_allclose(got["coefs"], z["tree_mp_coef"][p_, :z["tree_mp_count"][p_]],
                                   rtol=1e-4, atol=1e-5)
        assert got["ip"] == int(z["tree_mp_ip"][p_, 0])
    # single-patch API mirrors
    code = P().matching_pursuit(sel, z["X"][0], P().SearchParams(K=int(z["K"])))
    assert [i for i, _ in code.entries] == [int(i) for i in z["tree_mp_idx"][0, :z["tree_mp_count"][0]]]
    code = P().orthogonal_matching_pursuit(sel, z["X"][0], P().SearchParams(K=int(z["K"])))
    assert [i for i, _ in code.entries] == [int(i) for i in z["tree_omp_idx"][0, :z["tree_omp_count"][0]]]


def test_error_behaviour_matches_reference():
    z = golden("pursuit_small.npz")
    flat = flat_from_fixture(z)
    with pytest.raises(ValueError):
        P().TreeSelector(flat, z["atoms"], 1.5)   # alpha outside (0, 1] (pursuit.py:179-180)
    with pytest.raises(ValueError):
        P().TreeSelector(flat, z["atoms"], 0.0)
    other = np.ascontiguousarray(z["atoms"][::-1])
    with pytest.raises(P().StaleTreeError):
        P().TreeSelector(flat, other, 1 / 16)
    sel = P().TreeSelector(flat, z["atoms"], 1 / 16)
    X = torch.zeros((4, 24), device="cuda")
    with pytest.raises(ValueError):
        P().encode(sel, X, 0)
    with pytest.raises(ValueError):
        P().encode(sel, torch.zeros((4, 23), device="cuda"), 3)
    with pytest.raises(ValueError):
        P().encode(sel, X, 3, tol=-1.0)


def test_encode_host_equals_device_path(path):
    z = golden("pursuit_small.npz")
    sel = P().TreeSelector(flat_from_fixture(z), z["atoms"], 1 / 16)
    X = np.ascontiguousarray(np.tile(z["X"], (7, 1)))
    dev = run(sel, X, int(z["K"]), "omp", paths=False)
    host = P().encode_host(sel, X, int(z["K"]), "omp", chunk=200)
    for k in ("idx", "coef", "count", "resnorm", "ip"):
        np.testing.assert_array_equal(getattr(host, k), dev[k])


# ----------------------------------------------------------------- benchmark configs

def _config(cid):
    from paper_1412_0680_b200 import tree as T
    cfg, wl = dictionary(cid)
    flat = T.load_structure(os.path.join(GOLDEN, "trees", f"c{cid}.npz"), wl.atoms)
    return cfg, wl, flat


_CACHE = {}


def dictionary(cid):
    """The config's seeded dictionary only (the exhaustive selector needs no tree)."""
    from paper_1412_0680_b200 import workloads as W
    key = ("dict", cid)
    if key not in _CACHE:
        cfg = W.CONFIGS[cid]
        _CACHE[key] = (cfg, W.make_dictionary(cfg))
    return _CACHE[key]


def config(cid):
    if cid not in _CACHE:
        _CACHE[cid] = _config(cid)
    return _CACHE[cid]


_ORACLE = {}


def oracle_config(cid, rows, method, exhaustive=False):
    """Oracle results for the first `rows` patches of a config (computed once per
    module on a fork pool of the host cores, shared by every path variant)."""
    from oracle import parallel as OP
    from paper_1412_0680_b200 import workloads as W
    key = (cid, rows, method, exhaustive)
    if key not in _ORACLE:
        if exhaustive:
            cfg, wl = dictionary(cid)
            otree = None
        else:
            cfg, wl, flat = config(cid)
            otree = O.OracleTree.from_flat(flat)
        X = W.make_patches(wl, rows)
        a64 = wl.atoms.astype(np.float64)
        res = OP.encode_parallel(otree, a64, X, cfg.K, method, alpha=cfg.alpha)
        _ORACLE[key] = (X, O.pack(res, cfg.K))
    return _ORACLE[key]


def _tree_cases():
    cases = [(0, 10_000, "omp"), (0, 10_000, "mp"), (1, 16_384, "omp"), (1, 4096, "mp"),
             (2, 16_384, "omp"), (3, 16_384, "omp"), (4, 512, "omp"), (4, 256, "mp")]
    # ids that would rerun the default kernels of a config are left out:
    # config 4 already streams every node table ("staged-st"; config 2 streams the 3xFP16
    # pass by default, so "staged-st" is its 3xTF32 variant); only config 4
    # takes the Gram path by default ("staged-resid" elsewhere = "staged-ts"); config
    # 3's ragged last level has a centroid that is not its atom and config 4 is on
    # the Gram path already ("staged-gram"); the Gram path is OMP only.
    skip = {("staged-st", 4), ("staged-resid", 0), ("staged-resid", 1), ("staged-resid", 2),
            ("staged-resid", 3), ("staged-gram", 3), ("staged-gram", 4)}
    return [(c, r, m, p) for c, r, m in cases for p in PATHS
            if (p, c) not in skip and not (m == "mp" and p in ("staged-gram", "staged-resid"))]


def launched(fn):
    """Run fn() and return (its result, the set of library kernel names it launched)."""
    from paper_1412_0680_b200 import _lib
    _lib.kernel_timing(True)
    try:
        res = fn()
        torch.cuda.synchronize()
        names = set(_lib.kernel_times())
    finally:
        _lib.kernel_timing(False)
    return res, names


def expects_gram(cid, method, path):
    return method == "omp" and ((path in ("staged-ts", "staged-st") and cid == 4) or
                                (path == "staged-gram" and cid in (0, 1, 2)))


@pytest.mark.parametrize("cid,rows,method,path", _tree_cases(), indirect=["path"])
def test_config_tree_parity(cid, rows, method, path):
    cfg, wl, flat = config(cid)
    X, ref = oracle_config(cid, rows, method)
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    out, names = launched(lambda: run(sel, X, cfg.K, method))
    gram = any("update_gram_kernel" in k for k in names)
    assert gram == expects_gram(cid, method, path), sorted(names)
    # the 3xFP16 pass: forced, or by default on config 2's streamed 256-child nodes
    s16 = path == "staged-s16" or (cid == 2 and path in ("staged-ts", "staged-generic"))
    assert any("score_s16_kernel" in k for k in names) == s16, sorted(names)
    rep = compare(out, ref, X)
    print(f"c{cid} {method} {path}: {rep.summary()}")
    assert rep.ok, rep.summary()
    assert rep.excused <= max(2, rows // 500)


def test_config0_golden_prefix():
    """GPU vs the reference's own recorded runs on config 0 (no oracle in between)."""
    cfg, wl, flat = config(0)
    z = golden("c0_prefix.npz")
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    esel = P().ExactSelector(wl.atoms)
    a64 = wl.atoms.astype(np.float64)
    t = O.OracleTree.from_flat(flat)
    for tag, s, os_, method, rows in (("tree_omp", sel, O.tree_selector(t, a64, cfg.alpha), "omp", 1024),
                                      ("tree_mp", sel, O.tree_selector(t, a64, cfg.alpha), "mp", 1024),
                                      ("exact_omp", esel, O.exact_selector(a64), "omp", 128)):
        X = z["X"][:rows]
        out = run(s, X, cfg.K, method, paths=False)
        ref = {k[len(tag) + 1:]: z[k][:rows] for k in z.files if k.startswith(tag + "_")}
        ref["gaps"] = oracle_pack(os_, a64, X, cfg.K, method)["gaps"]
        rep = compare(out, ref, X, check_path=False)
        assert rep.ok, f"{tag}: {rep.summary()}"


# "staged-ts": the scan with the 3xFP16 split (default); "staged-st" (score_kernel = 3): 3xTF32
@pytest.mark.parametrize("path", ["fused", "staged-ts", "staged-st"], indirect=True)
@pytest.mark.parametrize("cid,rows", [(1, 256), (1, 4096), (4, 8), (4, 300)])
def test_config_exhaustive_parity(cid, rows, path):
    cfg, wl = dictionary(cid)
    X, ref = oracle_config(cid, rows, "omp", exhaustive=True)
    sel = P().ExactSelector(wl.atoms)
    out, names = launched(lambda: run(sel, X, cfg.K, "omp"))
    f16 = [k for k in names if "exact_scan_kernel" in k and ("Lb1E" in k or "true" in k)]   # <NA, NB, F16 = true>
    if path != "fused":
        assert any("exact_scan_kernel" in k for k in names), sorted(names)
        assert bool(f16) == (path == "staged-ts"), sorted(names)
    rep = compare(out, ref, X, check_path=False)
    print(f"c{cid} exhaustive {path}: {rep.summary()}")
    assert rep.ok, rep.summary()
    assert rep.excused <= max(2, rows // 500)


@pytest.mark.parametrize("path", ["staged-ts"], indirect=True)
def test_config1_full_size_properties(path):
    """All 1,048,576 config-1 patches: size-independent invariants of OMP."""
    from paper_1412_0680_b200 import workloads as W
    cfg, wl, flat = config(1)
    X = W.make_patches(wl)
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    Xd = torch.as_tensor(X).cuda()
    res = P().encode(sel, Xd, cfg.K, method="omp", paths=True)
    torch.cuda.synchronize()
    A = torch.as_tensor(wl.atoms).cuda().double()
    idx, coef, cnt = res.idx.long(), res.coef.double(), res.count.long()
    valid = idx >= 0
    assert bool((valid.sum(1) == cnt).all())
    assert bool((cnt >= 1).all()) and bool((cnt <= cfg.K).all())
    # residual norm equals ||x - A_S c|| recomputed in f64 (all patches)
    recon = torch.einsum("pk,pkn->pn", coef * valid, A[idx.clamp(min=0)])
    r = Xd.double() - recon
    rn = r.norm(dim=1)
    rel = (rn - res.resnorm.double()).abs() / rn.clamp(min=1e-12)
    assert float(rel.max()) < 1e-4
    # OMP optimality: the residual is orthogonal to every selected atom
    ortho = torch.einsum("pkn,pn->pk", A[idx.clamp(min=0)], r).abs() * valid
    assert float((ortho.max(1).values / Xd.double().norm(dim=1)).max()) < 1e-4
    # support atoms are distinct per patch
    srt = torch.sort(torch.where(valid, idx, -torch.arange(1, cfg.K + 1, device="cuda")), dim=1).values
    assert bool((srt[:, 1:] != srt[:, :-1]).all())
    # paths follow the tree and end at the selected atom's leaf parent
    cb = torch.as_tensor(flat.child_begin).cuda().long()
    cc = torch.as_tensor(flat.child_count).cuda().long()
    la = torch.as_tensor(flat.leaf_atom).cuda().long()
    path = res.path.long()
    prev = torch.zeros_like(idx)
    for lvl in range(flat.levels):
        node = path[:, :, lvl]
        ok = (node >= cb[prev]) & (node < cb[prev] + cc[prev])
        assert bool((ok | ~valid).all())
        prev = node.clamp(min=0)
    assert bool(((la[cb[prev]] == idx) | ~valid).all())  # single-atom leaves in config 1
    # cost accounting: 32 + 32 + 16 centroids + 1 leaf atom per selection
    sel_per = torch.div(res.ip[:, 0].long(), 81, rounding_mode="floor")
    assert bool((res.ip[:, 0].long() % 81 == 0).all())
    assert bool(((sel_per == cnt) | (sel_per == cnt + 1)).all())
    assert bool((res.ip[:, 1].long() == sel_per * 80).all())
    # the first rows equal an independent small-batch run (batch-size invariance)
    head = run(sel, X[:3000], cfg.K, "omp", paths=False)
    np.testing.assert_array_equal(head["idx"], res.idx[:3000].cpu().numpy())
    np.testing.assert_array_equal(head["coef"], res.coef[:3000].cpu().numpy())


# ----------------------------------------------------------------- synthetic shapes for the update variants

def _synthetic(seed, m, n, counts_by_depth, branching):
    """Random unit atoms and a random tree over them (any centroids define a
    valid greedy descent; the oracle scores the same centroids)."""
    from paper_1412_0680_b200 import tree as T
    rng = np.random.default_rng(seed)
    atoms = rng.standard_normal((m, n))
    atoms = (atoms / np.linalg.norm(atoms, axis=1, keepdims=True)).astype(np.float32)
    n_internal = sum(len(c) for c in counts_by_depth)
    leaf_atom = rng.permutation(m)
    # centroids: the normalised mean of each node's descendant atoms (like a k-means tree)
    cent = np.zeros((n_internal, n), dtype=np.float32)
    flat = T._from_counts(branching, n, P().fingerprint_atoms(atoms), counts_by_depth, cent, leaf_atom)
    off = flat.level_offsets
    L = len(branching)
    sums = np.zeros((n_internal, n))
    for v in range(off[L], off[L + 1]):
        sums[v] = atoms[leaf_atom[flat.child_begin[v]:flat.child_begin[v] + flat.child_count[v]]].sum(0)
    for d in range(L - 1, -1, -1):
        for v in range(off[d], off[d + 1]):
            sums[v] = sums[flat.child_begin[v]:flat.child_begin[v] + flat.child_count[v]].sum(0)
    cent = (sums / np.linalg.norm(sums, axis=1, keepdims=True)).astype(np.float32)
    flat = T._from_counts(branching, n, P().fingerprint_atoms(atoms), counts_by_depth, cent, leaf_atom)
    return atoms, flat


@pytest.mark.parametrize("shape", ["k16-lockstep-two-rows", "wide-multi-atom-leaves"])
def test_update_variants_match_oracle(shape):
    """K = 16 on 64-dim rows (lockstep update, two Cholesky rows per lane) and
    200-dim rows with two-atom leaves (one-CTA-per-patch wide update, leaf
    scoring inside the update), staged pipeline, against the f64 oracle."""
    from paper_1412_0680_b200 import _lib
    if shape.startswith("k16"):
        m, n, K, cbd, br = 512, 64, 16, [[8], [8] * 8, [8] * 64, [1] * 512], (8, 8, 8)
    else:
        m, n, K, cbd, br = 128, 200, 6, [[8], [8] * 8, [2] * 64], (8, 8)
    atoms, flat = _synthetic(7, m, n, cbd, br)
    rng = np.random.default_rng(8)
    N = 4096
    X = np.zeros((N, n), dtype=np.float64)
    for p in range(N):
        sup = rng.choice(m, 4, replace=False)
        X[p] = rng.standard_normal(4) @ atoms[sup].astype(np.float64) + 0.05 * rng.standard_normal(n)
    X = X.astype(np.float32)
    sel = P().TreeSelector(flat, atoms, 1 / 8)
    _lib.set_option("path", _lib.PATH_STAGED)
    try:
        out = run(sel, X, K, "omp")
    finally:
        restore_defaults(_lib)
    a64 = atoms.astype(np.float64)
    rows = slice(0, 512)   # the oracle on a prefix keeps the test short; the GPU encoded all N
    ref = oracle_pack(O.tree_selector(O.OracleTree.from_flat(flat), a64, 1 / 8), a64, X[rows], K, "omp")
    rep = compare({k: v[rows] for k, v in out.items()}, ref, X[rows], check_path=True)
    assert rep.ok, rep.summary()


@pytest.mark.parametrize("tol_tag,tol", [("deftol", None), ("tol0", 0.0)])
def test_gram_path_exact_sparse_and_tolerance(tol_tag, tol):
    """Gram path (no residual) on exactly sparse patches: the ||r||^2 estimate
    ||x||^2 - sum y^2 cancels, so the update must fall back to the explicit
    residual norm for the stopping rule (pursuit.py:214) and the reported norm.
    256-dim rows (auto-enabled), single-atom leaves equal to their centroids."""
    from paper_1412_0680_b200 import _lib
    from paper_1412_0680_b200 import tree as T
    rng = np.random.default_rng(21)
    m, n, br = 1024, 256, (8, 8, 16)
    atoms = rng.standard_normal((m, n))
    atoms = (atoms / np.linalg.norm(atoms, axis=1, keepdims=True)).astype(np.float32)
    cbd = [[8], [8] * 8, [16] * 64, [1] * 1024]
    leaf = rng.permutation(m)
    ni = sum(len(c) for c in cbd)
    flat = T._from_counts(br, n, P().fingerprint_atoms(atoms), cbd, np.zeros((ni, n), np.float32), leaf)
    off = flat.level_offsets
    sums = np.zeros((ni, n))
    for v in range(off[3], off[4]):
        sums[v] = atoms[leaf[flat.child_begin[v]]]
    for d in (2, 1, 0):
        for v in range(off[d], off[d + 1]):
            sums[v] = sums[flat.child_begin[v]:flat.child_begin[v] + flat.child_count[v]].sum(0)
    cent = (sums / np.linalg.norm(sums, axis=1, keepdims=True)).astype(np.float32)
    cent[off[3]:off[4]] = atoms[leaf]          # depth-L centroids are the atoms themselves
    flat = T._from_counts(br, n, P().fingerprint_atoms(atoms), cbd, cent, leaf)
    N, K = 4096, 8
    X = np.zeros((N, n))
    for p in range(N):
        sup = rng.choice(m, 3, replace=False)
        X[p] = rng.standard_normal(3) @ atoms[sup].astype(np.float64)
        if p % 2:
            X[p] += 0.05 * rng.standard_normal(n)   # half the patches noisy
    X = X.astype(np.float32)
    sel = P().TreeSelector(flat, atoms, 1 / 16)
    _lib.set_option("path", _lib.PATH_STAGED)
    try:
        out, names = launched(lambda: run(sel, X, K, "omp", tol))
    finally:
        restore_defaults(_lib)
    assert any("update_gram_kernel" in k for k in names), sorted(names)
    a64 = atoms.astype(np.float64)
    rows = slice(0, 1024)
    ref = oracle_pack(O.tree_selector(O.OracleTree.from_flat(flat), a64, 1 / 16), a64, X[rows], K, "omp", tol)
    rep = compare({k: v[rows] for k, v in out.items()}, ref, X[rows], check_path=True)
    print(f"gram exact-sparse {tol_tag}: {rep.summary()}")
    assert rep.ok, rep.summary()


@pytest.mark.parametrize("cid,rows", [(4, 512), (1, 4096), (0, 4096)])
@pytest.mark.parametrize("half", [0, 1])
def test_gram_level_passes_fp16_rows_and_fp32_rows(cid, rows, half):
    """Gram path with the level passes on fp16 patch rows (score_sh.cu, the default)
    and on fp32 rows (score_st.cu, half_scores = 0): both must meet the oracle, and
    the option must select the kernel."""
    from paper_1412_0680_b200 import _lib
    cfg, wl, flat = config(cid)
    X, ref = oracle_config(cid, rows, "omp")
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    _lib.set_option("path", _lib.PATH_STAGED)
    _lib.set_option("gram_path", 2)
    _lib.set_option("half_scores", half)
    try:
        out, names = launched(lambda: run(sel, X, cfg.K, "omp"))
    finally:
        restore_defaults(_lib)
    assert any("update_gram_kernel" in k for k in names), sorted(names)
    assert any("score_sh_kernel" in k for k in names) == bool(half), sorted(names)
    rep = compare(out, ref, X)
    print(f"c{cid} gram half_scores={half}: {rep.summary()}")
    assert rep.ok, rep.summary()
    assert rep.excused <= max(2, rows // 500)


def test_fp16_and_fp32_rows_give_identical_outputs():
    """The fp16 row copies only pre-rank the children (near ties are re-taken with
    exact f32 dots on either path), so 16,384 config-4 patches must come out the
    same with half_scores = 1 and 0: supports equal, coefficients and norms bitwise."""
    from paper_1412_0680_b200 import _lib
    from paper_1412_0680_b200 import workloads as W
    cfg, wl, flat = config(4)
    X = torch.as_tensor(W.make_patches(wl, 16384)).cuda()
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    _lib.set_option("path", _lib.PATH_STAGED)
    outs = []
    try:
        for half in (1, 0):
            _lib.set_option("half_scores", half)
            r = P().encode(sel, X, cfg.K, method="omp", paths=True)
            torch.cuda.synchronize()
            outs.append(r)
    finally:
        restore_defaults(_lib)
    a, b = outs
    differing = int((a.idx != b.idx).any(1).sum())
    print(f"fp16 vs fp32 rows: {differing} of {len(X)} patches differ")
    assert differing == 0
    assert bool(torch.equal(a.coef, b.coef)) and bool(torch.equal(a.resnorm, b.resnorm))
    assert bool(torch.equal(a.path, b.path)) and bool(torch.equal(a.ip, b.ip))


def test_fp16_rows_many_tiles_per_cta_and_ragged_batch():
    """score_sh with more work items per CTA than its shared-memory item cache holds
    (4,000,003 config-1 patches on the forced Gram path: ~110 tiles per CTA at level
    1) and a batch that is not a multiple of the tile: outputs equal the f32-row path."""
    from paper_1412_0680_b200 import _lib
    from paper_1412_0680_b200 import workloads as W
    cfg, wl, flat = config(1)
    base = W.make_patches(wl, 1 << 18)
    N = 4_000_003
    X = torch.as_tensor(base).cuda().repeat(16, 1)[:N].contiguous()
    X += 1e-3 * torch.randn(X.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    _lib.set_option("path", _lib.PATH_STAGED)
    _lib.set_option("gram_path", 2)
    outs = []
    try:
        for half in (1, 0):
            _lib.set_option("half_scores", half)
            (r, names) = launched(lambda: P().encode(sel, X, cfg.K, method="omp"))
            assert any("score_sh_kernel" in k for k in names) == bool(half), sorted(names)
            outs.append(r)
    finally:
        restore_defaults(_lib)
    a, b = outs
    differing = int((a.idx != b.idx).any(1).sum())
    print(f"c1 gram, {N} patches, fp16 vs fp32 rows: {differing} patches differ")
    assert differing == 0
    assert bool(torch.equal(a.coef, b.coef)) and bool(torch.equal(a.count, b.count))


def test_fp16_rows_follow_the_patch_scale():
    """The fp16 row copies carry one power-of-two scale per patch: patches scaled
    by 2^-60 .. 2^60 (exact in fp32, so the f64 oracle's results scale exactly too)
    must give the same selections and exactly scaled coefficients and norms."""
    from paper_1412_0680_b200 import _lib
    cfg, wl, flat = config(4)
    X, ref = oracle_config(4, 512, "omp")
    scale = np.ldexp(1.0, np.resize(np.array([-60, -7, 0, 9, 60]), len(X))).astype(np.float64)
    Xs = (X.astype(np.float64) * scale[:, None]).astype(np.float32)
    assert np.array_equal(Xs.astype(np.float64), X.astype(np.float64) * scale[:, None])
    sref = dict(ref)
    sref["coef"] = ref["coef"] * scale[:, None]
    sref["resnorm"] = ref["resnorm"] * scale
    sel = P().TreeSelector(flat, wl.atoms, cfg.alpha)
    _lib.set_option("path", _lib.PATH_STAGED)
    try:
        out, names = launched(lambda: run(sel, Xs, cfg.K, "omp"))
    finally:
        restore_defaults(_lib)
    assert any("score_sh_kernel" in k for k in names), sorted(names)
    rep = compare(out, sref, Xs)
    print(f"c4 fp16 rows, scaled patches: {rep.summary()}")
    assert rep.ok, rep.summary()
    assert rep.excused <= 2


# ----------------------------------------------------------------- beam (non-greedy alpha) descent

@pytest.mark.parametrize("tag,alpha", [("beam", 0.3), ("full", 1.0)])
def test_tree_select_beam_matches_reference(tag, alpha):
    """stmp_select with retained_count > 1 (pursuit.py:134-162) against the
    reference's own recorded selections (select_small.npz)."""
    z = golden("select_small.npz")
    flat = flat_from_fixture(z)
    sel = P().TreeSelector(flat, z["atoms"], alpha)
    out, names = launched(lambda: run(sel, z["Q"], 1, "select"))
    assert any("encode_fused_kernel" in k for k in names)
    t = O.OracleTree.from_flat(flat)
    a64 = z["atoms"].astype(np.float64)
    gaps = np.array([O.tree_select(t, a64, q.astype(np.float64), alpha)[5] for q in z["Q"]])
    ok = (out["idx"][:, 0] == z[f"{tag}_idx"]) | (gaps < 1e-5)
    assert ok.all()
    same = out["idx"][:, 0] == z[f"{tag}_idx"]
    np.testing.assert_allclose(out["coef"][same, 0], z[f"{tag}_score"][same], rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(out["ip"], z[f"{tag}_ip"])


@pytest.mark.parametrize("method", ["omp", "mp"])
def test_beam_pursuit_matches_oracle(method):
    z = golden("pursuit_small.npz")
    flat = flat_from_fixture(z)
    K = int(z["K"])
    a64 = z["atoms"].astype(np.float64)
    sel = P().TreeSelector(flat, z["atoms"], 0.3)
    out = run(sel, z["X"], K, method)
    ref = oracle_pack(O.tree_selector(O.OracleTree.from_flat(flat), a64, 0.3), a64, z["X"], K, method)
    rep = compare(out, ref, z["X"], check_path=True)
    assert rep.ok, rep.summary()
    assert rep.excused <= 2


@pytest.mark.parametrize("path", ["fused", "staged-ts"], indirect=True)
@pytest.mark.parametrize("cid,rows,alpha", [(1, 4096, 0.1), (4, 512, 0.1), (0, 4096, 0.2)])
def test_config_beam_parity(cid, rows, alpha, path):
    """The paper's alpha = 0.1 setting on config trees: frontiers
    of ceil(0.1 k) children per node (c1: 4, 16, 32 nodes; c4: 7, 49, 196), on the
    warp-per-patch kernel and on the staged pipeline (node-bucketed entries)."""
    from paper_1412_0680_b200 import workloads as W
    from oracle import parallel as OP
    cfg, wl, flat = config(cid)
    X = W.make_patches(wl, rows)
    sel = P().TreeSelector(flat, wl.atoms, alpha)
    out, names = launched(lambda: run(sel, X, cfg.K, "omp"))
    staged = any("beam_resolve_kernel" in k for k in names)
    assert staged == (path != "fused"), sorted(names)
    a64 = wl.atoms.astype(np.float64)
    ref = O.pack(OP.encode_parallel(O.OracleTree.from_flat(flat), a64, X, cfg.K, "omp", alpha=alpha), cfg.K)
    rep = compare(out, ref, X, check_path=True)
    print(f"c{cid} beam alpha={alpha}: {rep.summary()}")
    assert rep.ok, rep.summary()
    assert rep.excused <= max(2, rows // 200)


# ----------------------------------------------------------------- API robustness (round-1 advisor findings)

def test_encode_on_a_side_stream_matches_default_stream():
    """encode(stream=s) allocates its outputs and workspace on s and orders s after
    the producer of X: results equal the default-stream run."""
    z = golden("pursuit_small.npz")
    sel = P().TreeSelector(flat_from_fixture(z), z["atoms"], 1 / 16)
    X = torch.as_tensor(np.ascontiguousarray(np.tile(z["X"], (300, 1)))).cuda()   # staged pipeline
    ref = P().encode(sel, X, int(z["K"]), "omp")
    s = torch.cuda.Stream()
    Y = X * 1.0                                   # produced on the current stream
    out = P().encode(sel, Y, int(z["K"]), "omp", stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    assert torch.equal(out.idx, ref.idx) and torch.equal(out.coef, ref.coef)


def test_encode_host_rejects_bad_output_buffers():
    z = golden("pursuit_small.npz")
    sel = P().TreeSelector(flat_from_fixture(z), z["atoms"], 1 / 16)
    X = np.ascontiguousarray(z["X"])
    N, K = X.shape[0], int(z["K"])
    good = dict(idx=np.empty((N, K), np.int32), coef=np.empty((N, K), np.float32), count=np.empty(N, np.int32),
                resnorm=np.empty(N, np.float32), ip=np.empty((N, 2), np.int32))
    P().encode_host(sel, X, K, "omp", out=good)
    for key, bad in (("idx", np.empty((N - 1, K), np.int32)), ("coef", np.empty((N, K), np.float64)),
                     ("ip", np.empty((2, N), np.int32).T), ("count", np.empty(N, np.int64))):
        out = dict(good)
        out[key] = bad
        with pytest.raises(ValueError):
            P().encode_host(sel, X, K, "omp", out=out)


def test_encode_requires_count_and_resnorm():
    import ctypes as C
    from paper_1412_0680_b200 import _lib
    z = golden("pursuit_small.npz")
    sel = P().TreeSelector(flat_from_fixture(z), z["atoms"], 1 / 16)
    X = torch.as_tensor(np.ascontiguousarray(z["X"])).cuda()
    N, K = X.shape[0], int(z["K"])
    idx = torch.empty((N, K), dtype=torch.int32, device="cuda")
    coef = torch.empty((N, K), dtype=torch.float32, device="cuda")
    lib = _lib.load()
    rc = lib.stmp_encode(sel.gdict.handle, sel.tree.handle, X.data_ptr(), N, X.shape[1], K, _lib.METHOD_OMP,
                         1 / 16, -1.0, idx.data_ptr(), coef.data_ptr(), None, None, None, None, None, 0,
                         C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == _lib.STMP_EINVAL


def test_graph_cache_never_replays_a_freed_tree():
    """A tree handle allocated where a freed one lived must not replay the freed
    one's CUDA graph (the cache keys on handle generations, and freeing a handle
    drops its graphs)."""
    import gc
    from paper_1412_0680_b200 import tree as T
    from paper_1412_0680_b200 import workloads as W
    cfg, wl, flat = config(0)
    rng = np.random.default_rng(5)
    other = T._from_counts(flat.branching, flat.n, flat.fingerprint,
                           [flat.child_count[flat.level_offsets[d]:flat.level_offsets[d + 1]]
                            for d in range(flat.levels + 1)],
                           flat.centroids, rng.permutation(flat.leaf_atom))   # same dictionary, other leaves
    X = torch.as_tensor(W.make_patches(wl, 8192)).cuda()
    s = torch.cuda.Stream()

    def three_on_side_stream(tree):
        sel = P().TreeSelector(tree, wl.atoms, cfg.alpha)
        with torch.cuda.stream(s):
            for _ in range(3):     # eager, capture, replay
                r = P().encode(sel, X, cfg.K, "omp")
        torch.cuda.synchronize()
        out = r.idx.clone()
        del sel, r
        gc.collect()
        return out

    a = three_on_side_stream(flat)
    b = three_on_side_stream(other)
    fresh = P().encode(P().TreeSelector(other, wl.atoms, cfg.alpha), X, cfg.K, "omp").idx
    torch.cuda.synchronize()
    assert not torch.equal(a, b)
    assert torch.equal(b, fresh)


@pytest.mark.parametrize("method", ["omp", "mp"])
def test_staged_beam_equals_fused_beam(method):
    """Staged beam descent and the warp-per-patch beam give the same codes
    (decisions; coefficients to fp32 rounding) on 8192 config-1 patches."""
    from paper_1412_0680_b200 import _lib
    from paper_1412_0680_b200 import workloads as W
    cfg, wl, flat = config(1)
    X = W.make_patches(wl, 8192)
    sel = P().TreeSelector(flat, wl.atoms, 0.1)
    try:
        _lib.set_option("path", _lib.PATH_FUSED)
        a = run(sel, X, cfg.K, method)
        _lib.set_option("path", _lib.PATH_STAGED)
        b = run(sel, X, cfg.K, method)
    finally:
        restore_defaults(_lib)
    same = (a["idx"] == b["idx"]).all(axis=1)
    assert same.mean() > 0.999, same.mean()
    np.testing.assert_array_equal(a["ip"][same], b["ip"][same])
    np.testing.assert_allclose(a["coef"][same], b["coef"][same], rtol=1e-4, atol=1e-5)
