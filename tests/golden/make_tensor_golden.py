"""Golden fixture of the data-format functions from the REFERENCE itself
(build container only): tensor.extract_patches / aggregate_patches
(pkg/src/stmp/tensor.py:104-136) and operators.apply_batch
(pkg/src/stmp/operators.py:115-141) on seeded inputs.

tensor.npz: for case i, t{i} (tensor), g{i} (shape | patch | stride rows),
P{i} (extract output), A{i} (aggregate of perturbed patches Q{i});
operators: X (f32 rows) and Y_<kind> with their parameters.

Usage:  python tests/golden/make_tensor_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from stmp import operators as ops  # noqa: E402
from stmp import tensor as ten  # noqa: E402

CASES = [((9, 7), (3, 2), (2, 2)),          # pkg/tests/test_tensor.py:73-79
         ((6, 6, 4), (3, 3, 2), (3, 3, 2)),  # test_tensor.py:82-87
         ((10, 9), (4, 3), (2, 2)),          # test_tensor.py:98-104
         ((5, 6, 7), (3, 2, 4), (1, 2, 3)),  # overlapping 3-D, ragged final starts
         ((33, 17), (8, 8), (3, 5))]


def main():
    rng = np.random.default_rng(4321)
    arrays = {}
    for i, (shape, patch, stride) in enumerate(CASES):
        t = rng.random(shape).astype(np.float32)
        layout, P = ten.extract_patches(t, patch, stride)
        Q = (P + rng.standard_normal(P.shape).astype(np.float32) * 0.1).astype(np.float32)
        arrays[f"t{i}"] = t
        arrays[f"g{i}"] = np.array([shape, patch, stride], dtype=np.int64)
        arrays[f"P{i}"] = P
        arrays[f"Q{i}"] = Q
        arrays[f"A{i}"] = ten.aggregate_patches(layout, Q)
    # operators on 37 f32 rows
    X = rng.standard_normal((37, 72)).astype(np.float32)
    arrays["X"] = X
    rows = np.array([0, 3, 4, 10, 31, 32, 50, 71], dtype=np.int64)
    arrays["rows"] = rows
    arrays["Y_row_select"] = ops.apply_batch(ops.row_select_operator(72, rows), X)
    mask = (rng.random((3, 3, 4)) < 0.5).astype(np.float32)
    mask[..., 0] = 1.0
    arrays["mask"] = mask
    arrays["Y_coded_exposure"] = ops.apply_batch(ops.coded_exposure_operator(mask, windows=2), X)
    arrays["in_shape"] = np.array([4, 6, 3], dtype=np.int64)
    arrays["factors"] = np.array([2, 3, 1], dtype=np.int64)
    arrays["Y_block_average"] = ops.apply_batch(ops.block_average_operator((4, 6, 3), (2, 3, 1)), X)
    arrays["Y_identity"] = ops.apply_batch(ops.identity_operator(72), X)
    np.savez_compressed(os.path.join(HERE, "tensor.npz"), **arrays)
    print("wrote tensor.npz")


if __name__ == "__main__":
    main()
