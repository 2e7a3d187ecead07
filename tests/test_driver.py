"""Batch driver: pipelines._code_patches on the GPU.

The oracle restatement (oracle/stmp_oracle.py code_patches) is pinned against
the reference's own _code_patches output (tests/golden/driver.npz, produced by
tests/golden/make_driver_golden.py); the GPU driver is compared with both.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import stmp_oracle as O

CASES = ("id", "ce")


def _flat(z, pre):
    from paper_1412_0680_b200 import tree as T
    off = z[f"{pre}_t_level_offsets"]
    cc = z[f"{pre}_t_child_count"]
    return T._from_counts(tuple(int(k) for k in z[f"{pre}_branching"]), int(z[f"{pre}_atoms"].shape[1]),
                          int(z[f"{pre}_t_fingerprint"][0]), [cc[off[d]:off[d + 1]] for d in range(len(off) - 1)],
                          z[f"{pre}_t_centroids"], z[f"{pre}_t_leaf_atom"])


def _oracle(z, pre):
    flat = _flat(z, pre)
    a64 = z[f"{pre}_atoms"].astype(np.float64)
    K = int(z[f"{pre}_K"][0])
    alpha = 1.0 / max(int(k) for k in z[f"{pre}_branching"])
    sel = O.tree_selector(O.OracleTree.from_flat(flat), a64, alpha)
    scale = z[f"{pre}_scale"]
    return O.code_patches(sel, a64, z[f"{pre}_base"].astype(np.float64), z[f"{pre}_Y"], z[f"{pre}_dc_meas"], K,
                          "mp", scale=None if np.all(scale == 1.0) else scale, usable=z[f"{pre}_usable"])


@pytest.mark.parametrize("pre", CASES)
def test_oracle_code_patches_matches_reference_golden(pre):
    z = golden("driver.npz")
    out, packed, ips, cips = _oracle(z, pre)
    ref = z[f"{pre}_out"]
    np.testing.assert_allclose(out, ref, rtol=1e-6, atol=1e-6 * np.abs(ref).max())
    assert (ips, cips) == tuple(int(v) for v in z[f"{pre}_ip"])


def test_oracle_dc_split_definition():
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((5, 9)).astype(np.float32)
    dcm = rng.random(9) + 0.5
    Xc, dc = O.dc_split(Y, dcm)
    # the flat component is removed exactly: x . dc_meas == 0
    np.testing.assert_allclose(Xc @ dcm, 0.0, atol=1e-12)
    np.testing.assert_allclose(Xc + dc[:, None] * dcm[None, :], Y.astype(np.float64), atol=1e-12)


def _selector(z, pre):
    import paper_1412_0680_b200 as P
    flat = _flat(z, pre)
    alpha = 1.0 / max(int(k) for k in z[f"{pre}_branching"])
    return P.TreeSelector(flat, z[f"{pre}_atoms"], alpha)


class _PD:
    def __init__(self, z, pre):
        import paper_1412_0680_b200 as P
        self.base = P.Dictionary(z[f"{pre}_base"])
        self.scale = z[f"{pre}_scale"]
        self.usable = z[f"{pre}_usable"].astype(bool)


@pytest.mark.gpu
@pytest.mark.parametrize("pre", CASES)
def test_gpu_code_patches_matches_reference(pre):
    import paper_1412_0680_b200 as P
    from paper_1412_0680_b200.pipelines import code_patches
    z = golden("driver.npz")
    K = int(z[f"{pre}_K"][0])
    params = P.SearchParams(K=K)
    out, counter = code_patches(z[f"{pre}_Y"], z[f"{pre}_dc_meas"], _selector(z, pre), _PD(z, pre), params)
    ref = z[f"{pre}_out"]
    # coefficients within 1e-4 relative (BASELINE parity contract) -> reconstructions likewise
    np.testing.assert_allclose(out, ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max())
    assert (counter.inner_products, counter.centroid_inner_products) == tuple(int(v) for v in z[f"{pre}_ip"])
    # device input gives a device output, same values
    import torch
    out_d, _ = code_patches(torch.as_tensor(z[f"{pre}_Y"]).cuda(), z[f"{pre}_dc_meas"], _selector(z, pre),
                            _PD(z, pre), params)
    assert out_d.is_cuda and out_d.dtype == torch.float64
    np.testing.assert_array_equal(out_d.cpu().numpy(), out)
    # on a side stream: every launch and host read on it, the caller's stream waits
    s = torch.cuda.Stream()
    out_s, counter_s = code_patches(torch.as_tensor(z[f"{pre}_Y"]).cuda(), z[f"{pre}_dc_meas"], _selector(z, pre),
                                    _PD(z, pre), params, stream=s)
    np.testing.assert_array_equal(out_s.cpu().numpy(), out)
    assert counter_s.inner_products == counter.inner_products


@pytest.mark.gpu
def test_gpu_reconstruct_is_exact_f64():
    """stmp_reconstruct on given codes equals the f64 oracle bitwise (same
    entries, same order, separate multiply and add)."""
    import torch
    from paper_1412_0680_b200 import _lib
    import paper_1412_0680_b200 as P
    rng = np.random.default_rng(3)
    base = rng.standard_normal((50, 37)).astype(np.float32)
    N, K = 64, 5
    idx = rng.integers(0, 50, (N, K)).astype(np.int32)
    coef = rng.standard_normal((N, K)).astype(np.float32)
    cnt = rng.integers(0, K + 1, N).astype(np.int32)
    scale = rng.random(50) + 0.5
    dc = rng.standard_normal(N)
    g = P.GpuDictionary(base)
    dev = {k: torch.as_tensor(v).cuda() for k, v in dict(idx=idx, coef=coef, cnt=cnt, scale=scale, dc=dc).items()}
    out = torch.empty((N, 37), dtype=torch.float64, device="cuda")
    lib = _lib.load()
    _lib.check(lib.stmp_reconstruct(g.handle, dev["idx"].data_ptr(), dev["coef"].data_ptr(), dev["cnt"].data_ptr(),
                                    N, K, dev["scale"].data_ptr(), dev["dc"].data_ptr(), out.data_ptr(), 37, None))
    torch.cuda.synchronize()
    ref = O.lift_reconstruct(base.astype(np.float64), idx, coef, cnt, scale, dc)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)


@pytest.mark.gpu
def test_gpu_code_patches_rejects_unusable_atom():
    import paper_1412_0680_b200 as P
    from paper_1412_0680_b200.pipelines import code_patches
    z = golden("driver.npz")
    pd = _PD(z, "id")
    out, _ = code_patches(z["id_Y"], z["id_dc_meas"], _selector(z, "id"), pd, P.SearchParams(K=4))
    pd.usable = np.zeros_like(pd.usable)   # every atom unusable: lift_code raises (operators.py:209-213)
    with pytest.raises(RuntimeError):
        code_patches(z["id_Y"], z["id_dc_meas"], _selector(z, "id"), pd, P.SearchParams(K=4))
    with pytest.raises(ValueError):
        code_patches(z["id_Y"][:, :5], z["id_dc_meas"], _selector(z, "id"), _PD(z, "id"), P.SearchParams(K=4))
