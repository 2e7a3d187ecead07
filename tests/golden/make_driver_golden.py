"""Golden fixture of the batch driver (``pipelines._code_patches``) from the
REFERENCE itself (build container only; /root/reference is absent on the GPU box).

driver.npz, two cases coded with the reference's own ``_code_patches``
(pkg/src/stmp/pipelines.py:180-217) and tree selector:
  * id_*  identity operator (denoise shape): m=64 atoms of 16 dims, tree (8, 8);
  * ce_*  coded-exposure operator (pkg/src/stmp/operators.py:67-93) with a
          3x3x4 mask: base atoms of 36 dims, 9-dim measurements, projected
          dictionary of m=96 atoms, tree (8, 12).
Measured patches are f32-representable so the GPU sees the same inputs.

Usage:  python tests/golden/make_driver_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import stmp  # noqa: E402
from stmp import pipelines as refpipe  # noqa: E402
from stmp import operators as refops  # noqa: E402
from paper_1412_0680_b200 import tree as T  # noqa: E402


def case(prefix, rng, base_atoms, op, branching, N, K, seed):
    d = stmp.normalize_columns(base_atoms)
    pd = refops.project_dictionary(d, op)
    tree = stmp.build_tree(pd.dictionary, branching, seed)
    alpha = 1.0 / max(branching)
    sel = stmp.TreeSelector(tree, pd.dictionary, alpha)
    n_meas = op.n_out
    # measured patches: a few atoms' images plus a flat offset and noise, rounded to f32
    Y = np.zeros((N, n_meas))
    for p in range(N):
        sup = rng.choice(pd.dictionary.m, 3, replace=False)
        Y[p] = rng.standard_normal(3) @ pd.dictionary.atoms[sup].astype(np.float64)
        Y[p] += 0.3 * rng.standard_normal() + 0.05 * rng.standard_normal(n_meas)
    Y = Y.astype(np.float32).astype(np.float64)
    dc_meas = refops.apply(op, np.ones(d.n))
    params = stmp.SearchParams(K=K, alpha=alpha, branching=branching)
    out, counter = refpipe._code_patches(Y, dc_meas, sel, pd, params, 1)
    f = T.from_reference_tree(tree)
    return {
        f"{prefix}_base": d.atoms, f"{prefix}_atoms": pd.dictionary.atoms, f"{prefix}_scale": pd.scale,
        f"{prefix}_usable": pd.usable.astype(np.uint8), f"{prefix}_Y": Y.astype(np.float32),
        f"{prefix}_dc_meas": np.asarray(dc_meas, dtype=np.float64), f"{prefix}_out": out,
        f"{prefix}_ip": np.array([counter.inner_products, counter.centroid_inner_products], dtype=np.int64),
        f"{prefix}_K": np.array([K]), f"{prefix}_branching": np.asarray(branching),
        f"{prefix}_t_level_offsets": f.level_offsets, f"{prefix}_t_child_begin": f.child_begin,
        f"{prefix}_t_child_count": f.child_count, f"{prefix}_t_centroids": f.centroids,
        f"{prefix}_t_leaf_atom": f.leaf_atom, f"{prefix}_t_fingerprint": np.array([f.fingerprint], dtype=np.uint64),
    }


def main():
    rng = np.random.default_rng(1412)
    arrays = {}
    arrays.update(case("id", rng, rng.standard_normal((64, 16)), refops.identity_operator(16), (8, 8), 40, 4, 7))
    mask = (rng.random((3, 3, 4)) < 0.5).astype(np.float32)
    mask[..., 0] = 1.0   # every pixel open in at least one frame (operators.py:79-80)
    arrays.update(case("ce", rng, rng.standard_normal((96, 36)), refops.coded_exposure_operator(mask), (8, 12),
                       40, 3, 11))
    np.savez_compressed(os.path.join(HERE, "driver.npz"), **arrays)
    print("wrote driver.npz")


if __name__ == "__main__":
    main()
