"""Build the benchmark-config trees with the REFERENCE's own CPU tree learner.

Runs only in the build container, where the reference is importable from
/root/reference/pkg/src.  For each config it

1. regenerates the coding dictionary with ``paper_1412_0680_b200.workloads``
   and checks it bitwise against the reference's ``normalize_columns`` /
   ``project_dictionary`` on the same raw draw;
2. calls the reference ``build_tree(d, branching, seed)``
   (pkg/src/stmp/clustering.py:285-316) and ``validate_tree``;
3. flattens the tree and writes the membership-only structure file from which
   the GPU box rebuilds every centroid bitwise (``tree.save_membership`` /
   ``tree.load_structure``, checked by the stored SHA-256), plus the
   reference ``.tree`` bytes round-trip check.

Usage: python tools/make_trees.py 0 1 2 3 [4] [--out DIR]
"""

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import stmp  # noqa: E402
from paper_1412_0680_b200 import tree as T  # noqa: E402
from paper_1412_0680_b200 import workloads as W  # noqa: E402


def reference_dictionary(cfg):
    rng = np.random.default_rng(W.seed_sequence(cfg.cid, 0))
    if cfg.n_base == 0:
        return stmp.normalize_columns(rng.standard_normal((cfg.m, cfg.n)))
    base = stmp.normalize_columns(rng.standard_normal((cfg.m, cfg.n_base)))
    op = stmp.coded_exposure_operator(W.exposure_mask(cfg))
    return stmp.project_dictionary(base, op).dictionary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", type=int)
    ap.add_argument("--out", default="tests/golden/trees")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    for cid in args.configs:
        cfg = W.CONFIGS[cid]
        t0 = time.time()
        ref_d = reference_dictionary(cfg)
        wl = W.make_dictionary(cfg)
        assert np.array_equal(ref_d.atoms.view(np.uint32), wl.atoms.view(np.uint32)), "dictionary restatement differs"
        print(f"[c{cid}] dictionary ok ({time.time() - t0:.1f}s)", flush=True)
        tree = stmp.build_tree(ref_d, cfg.branching, W.tree_seed(cid))
        print(f"[c{cid}] build_tree {time.time() - t0:.1f}s", flush=True)
        rep = stmp.validate_tree(tree, ref_d)
        assert rep.ok, rep.violation
        flat = T.from_reference_tree(tree)
        path = os.path.join(args.out, f"c{cid}.npz")
        T.save_membership(flat, wl.atoms, path)
        back = T.load_structure(path, wl.atoms)
        assert back.centroid_digest() == flat.centroid_digest()
        if cid <= 1:
            import tempfile
            with tempfile.NamedTemporaryFile(suffix=".tree") as fh:
                stmp.save_tree(tree, fh.name)
                parsed = T.read_tree_file(fh.name)
                assert parsed.centroid_digest() == flat.centroid_digest()
                assert np.array_equal(parsed.leaf_atom, flat.leaf_atom)
                assert open(fh.name, "rb").read() == T.write_tree_file(flat)
        print(f"[c{cid}] wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB, "
              f"{flat.num_internal} internal nodes, fingerprint {flat.fingerprint:#018x}) "
              f"total {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
