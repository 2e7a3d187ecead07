"""Data formats either side of the path: patch extraction,
overlap-average aggregation and the observation operators.

The oracle restatement is pinned to the reference's own outputs
(tests/golden/tensor.npz from tests/golden/make_tensor_golden.py); the GPU
kernels are compared with the golden vectors: extraction and aggregation
bit-exact, operators within 1e-12 relative (the reference's NumPy sums use
pairwise order).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import stmp_oracle as O

NCASES = 5


def _case(z, i):
    shape, patch, stride = (tuple(int(v) for v in row) for row in z[f"g{i}"])
    return shape, patch, stride


@pytest.mark.parametrize("i", range(NCASES))
def test_oracle_extract_aggregate_match_reference(i):
    z = golden("tensor.npz")
    shape, patch, stride = _case(z, i)
    np.testing.assert_array_equal(O.extract_patches(z[f"t{i}"], patch, stride), z[f"P{i}"])
    np.testing.assert_array_equal(O.aggregate_patches(shape, patch, stride, z[f"Q{i}"]), z[f"A{i}"])


@pytest.mark.parametrize("kind", ["identity", "row_select", "coded_exposure", "block_average"])
def test_oracle_operators_match_reference(kind):
    z = golden("tensor.npz")
    Y = O.apply_operator(kind, z["X"], rows=z["rows"], mask=z["mask"], windows=2, in_shape=z["in_shape"],
                         factors=z["factors"])
    np.testing.assert_allclose(Y, z[f"Y_{kind}"], rtol=1e-12, atol=1e-12)


def test_layout_validation_matches_reference():
    from paper_1412_0680_b200.patches import PatchLayout
    # pkg/tests/test_tensor.py:55-71
    with pytest.raises(ValueError):
        PatchLayout((4, 4), (2,), (2,))
    with pytest.raises(ValueError):
        PatchLayout((4, 4), (5, 2), (1, 1))
    with pytest.raises(ValueError):
        PatchLayout((8, 8), (2, 2), (3, 3))
    lay = PatchLayout((9, 7), (3, 2), (2, 2))
    assert [list(s) for s in lay.axis_starts] == [[0, 2, 4, 6], [0, 2, 4, 5]]
    assert (lay.num_patches, lay.patch_dim) == (16, 6)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(NCASES))
def test_gpu_extract_aggregate_bitwise(i):
    import torch
    from paper_1412_0680_b200.patches import aggregate_patches, extract_patches
    z = golden("tensor.npz")
    shape, patch, stride = _case(z, i)
    layout, P = extract_patches(z[f"t{i}"], patch, stride)
    np.testing.assert_array_equal(P, z[f"P{i}"])
    np.testing.assert_array_equal(aggregate_patches(layout, z[f"Q{i}"]), z[f"A{i}"])
    # device in, device out; extract -> aggregate round trip is the identity up to f32 rounding
    t = torch.as_tensor(z[f"t{i}"]).cuda()
    layout, Pd = extract_patches(t, patch, stride)
    assert Pd.is_cuda
    back = aggregate_patches(layout, Pd)
    np.testing.assert_allclose(back.cpu().numpy(), z[f"t{i}"], atol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["identity", "row_select", "coded_exposure", "block_average"])
def test_gpu_operators_match_reference(kind):
    from types import SimpleNamespace
    from paper_1412_0680_b200.patches import apply_batch
    z = golden("tensor.npz")
    mask = z["mask"]
    ins, fac = z["in_shape"], z["factors"]
    n_out = {"identity": 72, "row_select": len(z["rows"]), "coded_exposure": 18,
             "block_average": int(np.prod(ins // fac))}[kind]
    op = SimpleNamespace(kind=kind, n_in=72, n_out=n_out, row_indices=z["rows"], mask=mask, windows=2,
                         in_shape=tuple(ins), factors=tuple(fac))
    Y = apply_batch(op, z["X"])
    np.testing.assert_allclose(Y, z[f"Y_{kind}"], rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        apply_batch(op, z["X"][:, :10])
