"""Host-side tree flattening / shipping format and the seeded workloads."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, flat_from_fixture, golden
from paper_1412_0680_b200 import tree as T
from paper_1412_0680_b200 import workloads as W


def test_tree_file_round_trip_from_fixture():
    flat = flat_from_fixture(golden("select_ragged.npz"))
    data = T.write_tree_file(flat)
    back = T.read_tree_file(data)
    assert back.centroid_digest() == flat.centroid_digest()
    np.testing.assert_array_equal(back.child_count, flat.child_count)
    np.testing.assert_array_equal(back.leaf_atom, flat.leaf_atom)
    assert T.write_tree_file(back) == data


def test_tree_file_rejects_corruption():
    flat = flat_from_fixture(golden("select_small.npz"))
    data = bytearray(T.write_tree_file(flat))
    with pytest.raises(T.TreeFormatError):
        T.read_tree_file(bytes(data[:-3]))
    bad = bytearray(data)
    bad[0:8] = b"NOTATREE"
    with pytest.raises(T.TreeFormatError):
        T.read_tree_file(bytes(bad))
    bad = bytearray(data)
    bad[8] = 9   # version
    with pytest.raises(T.TreeFormatError):
        T.read_tree_file(bytes(bad))


def test_flatten_matches_reference_tree_file(stmp_ref, tmp_path):
    rng = np.random.default_rng(3)
    d = stmp_ref.normalize_columns(rng.standard_normal((211, 9)))
    tree = stmp_ref.build_tree(d, (7, 4), seed=5)
    flat = T.from_reference_tree(tree)
    stmp_ref.save_tree(tree, tmp_path / "t.tree")
    parsed = T.read_tree_file(tmp_path / "t.tree")
    assert parsed.centroid_digest() == flat.centroid_digest()
    assert (tmp_path / "t.tree").read_bytes() == T.write_tree_file(flat)
    # and the reference can read what we write
    (tmp_path / "u.tree").write_bytes(T.write_tree_file(flat))
    back = stmp_ref.load_tree(tmp_path / "u.tree")
    assert stmp_ref.validate_tree(back, d).ok


@pytest.mark.parametrize("cid", [0, 1, 2, 3, 4])
def test_shipped_structures_rebuild_bitwise(cid):
    cfg = W.CONFIGS[cid]
    wl = W.make_dictionary(cfg)
    flat = T.load_structure(os.path.join(GOLDEN, "trees", f"c{cid}.npz"), wl.atoms)
    assert flat.branching == cfg.branching
    assert flat.m == cfg.m
    assert sorted(flat.leaf_atom.tolist()) == list(range(cfg.m))


def test_structure_rejects_wrong_dictionary():
    cfg = W.CONFIGS[0]
    wl = W.make_dictionary(cfg)
    atoms = wl.atoms.copy()
    atoms[[0, 1]] = atoms[[1, 0]]
    with pytest.raises(T.TreeFormatError):
        T.load_structure(os.path.join(GOLDEN, "trees", "c0.npz"), atoms)


def test_dictionary_restatement_matches_reference(stmp_ref):
    for cid in (0, 1):
        cfg = W.CONFIGS[cid]
        rng = np.random.default_rng(W.seed_sequence(cid, 0))
        ref = stmp_ref.normalize_columns(rng.standard_normal((cfg.m, cfg.n)))
        np.testing.assert_array_equal(ref.atoms.view(np.uint32), W.make_dictionary(cfg).atoms.view(np.uint32))


def test_patch_prefix_is_stable_and_shards_are_disjoint():
    cfg = W.CONFIGS[1]
    wl = W.make_dictionary(cfg)
    a = W.make_patches(wl, 1000)
    b = W.make_patches(wl, 70000)
    np.testing.assert_array_equal(a, b[:1000])
    c = W.make_patches(wl, 1000, start=cfg.chunk)
    np.testing.assert_array_equal(c, b[cfg.chunk:cfg.chunk + 1000])
    with pytest.raises(ValueError):
        W.make_patches(wl, 10, start=3)
    assert a.dtype == np.float32 and a.shape == (1000, 64)


def test_membership_format_detects_a_wrong_rebuild(tmp_path):
    """The membership-only file rebuilds centroids as _unit_mean of the members
    (clustering.py:145-153); any disagreement fails the SHA-256 check loudly."""
    cfg = W.CONFIGS[0]
    wl = W.make_dictionary(cfg)
    src = os.path.join(GOLDEN, "trees", "c0.npz")
    z = dict(np.load(src))
    assert str(z["format"]) == T.MEMBERSHIP_FORMAT
    bad = dict(z)
    bad["norms"] = z["norms"].copy()
    bad["norms"][3] *= 1 + 1e-6
    np.savez(tmp_path / "bad.npz", **bad)
    with pytest.raises(T.TreeFormatError):
        T.load_structure(tmp_path / "bad.npz", wl.atoms)
    swapped = dict(z)
    la = z["leaf_atom"].copy()
    la[[0, 100]] = la[[100, 0]]
    swapped["leaf_atom"] = la
    np.savez(tmp_path / "swapped.npz", **swapped)
    with pytest.raises(T.TreeFormatError):
        T.load_structure(tmp_path / "swapped.npz", wl.atoms)
