"""CPU-side checks of the C ABI: the in-tree library loads, exports every symbol
include/stmp_b200.h declares, hashes like the reference, and refuses to run
device work without a GPU (no CPU fallback)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_1412_0680_b200 import _lib, build


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "stmp_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(stmp_[a-z0-9_]+)\s*\(", text))


def test_every_declared_symbol_is_exported_and_bound(lib):
    declared = _declared_functions()
    assert declared, "header parse found no functions"
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_version(lib):
    assert b"sm_100a" in lib.stmp_version()


def test_native_fnv_matches_golden(lib):
    z = golden("fnv.npz")
    payload = z["payload"].tobytes()
    pos = 0
    for length, h in zip(z["lengths"], z["hashes"]):
        buf = C.create_string_buffer(payload[pos:pos + length], max(int(length), 1))
        assert lib.stmp_fnv1a64(buf, int(length), _lib.FNV_OFFSET) == int(h)
        pos += length


def test_native_fnv_streams(lib):
    data = np.random.default_rng(0).integers(0, 256, 10_000, dtype=np.uint8)
    whole = lib.stmp_fnv1a64(data.ctypes.data, data.size, _lib.FNV_OFFSET)
    h = _lib.FNV_OFFSET
    for s in range(0, data.size, 777):
        part = np.ascontiguousarray(data[s:s + 777])
        h = lib.stmp_fnv1a64(part.ctypes.data, part.size, h)
    assert h == whole


def test_fingerprint_of_shipped_trees_matches_dictionary(lib):
    """The native FNV over the regenerated config-0/1 dictionaries equals the
    fingerprint the reference stored with the tree (binding check)."""
    from paper_1412_0680_b200 import workloads as W
    from paper_1412_0680_b200.pursuit import fingerprint_atoms
    for cid in (0, 1):
        wl = W.make_dictionary(W.CONFIGS[cid])
        z = np.load(os.path.join(ROOT, "tests", "golden", "trees", f"c{cid}.npz"))
        assert fingerprint_atoms(wl.atoms) == int(z["fingerprint"][0])


def test_device_entry_points_fail_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    atoms = np.eye(4, dtype=np.float32)
    h = C.c_void_p()
    rc = lib.stmp_dict_create(atoms.ctypes.data, 4, 4, 0, 1, None, C.byref(h))
    assert rc == _lib.STMP_ECUDA
    assert h.value is None
    assert lib.stmp_last_error()
    with pytest.raises(RuntimeError):
        _lib.check(rc)


def test_argument_validation_maps_to_value_error(lib):
    h = C.c_void_p()
    rc = lib.stmp_dict_create(None, 0, 4, 0, 1, None, C.byref(h))
    assert rc == _lib.STMP_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc)
    # encode with a NULL dictionary handle is a ValueError, not a crash
    rc = lib.stmp_encode(None, None, None, 0, 4, 3, 1, 1.0, -1.0, None, None, None, None, None,
                         None, None, 0, None)
    assert rc == _lib.STMP_EINVAL


def test_options_and_launch_counter(lib):
    before = _lib.kernel_launches()
    assert before >= 0
    for key, bad in (("path", 3), ("score_kernel", 5), ("score_kernel", 1), ("update_kernel", 2),
                     ("gram", 1), ("score_tma", 1), ("half_scores", 2), ("half_scores", -1)):
        with pytest.raises(ValueError):
            _lib.set_option(key, bad)
    with pytest.raises(ValueError):
        _lib.set_option("no_such_option", 0)
    _lib.set_option("update_kernel", 1)
    _lib.set_option("score_kernel", 2)
    _lib.set_option("half_scores", 1)
    _lib.set_option("path", _lib.PATH_AUTO)
    assert _lib.kernel_launches() == before   # option changes launch nothing


def test_data_format_entry_points_validate_before_touching_the_device(lib):
    """Argument errors of the driver / data-format entry points are ValueErrors
    (STMP_EINVAL) raised before any device work, as in the reference
    (pipelines.py, tensor.py:59-79, operators.py:122-124)."""
    shape = np.array([4, 4], dtype=np.int64)
    patch = np.array([5, 2], dtype=np.int64)   # patch larger than the tensor
    nst = np.array([1, 2], dtype=np.int64)
    dummy = C.c_void_p(16)
    assert lib.stmp_extract_patches(dummy, 2, shape.ctypes.data, patch.ctypes.data, nst.ctypes.data, dummy,
                                    dummy, None) == _lib.STMP_EINVAL
    assert b"exceeds tensor extent" in lib.stmp_last_error()
    assert lib.stmp_aggregate_patches(dummy, 0, shape.ctypes.data, patch.ctypes.data, nst.ctypes.data, dummy,
                                      dummy, None) == _lib.STMP_EINVAL
    assert lib.stmp_apply_operator(99, dummy, 4, 8, None, 0, None, 0, 0, 0, 0, None, None, dummy,
                                   None) == _lib.STMP_EINVAL
    assert lib.stmp_apply_operator(_lib.OP_CODED_EXPOSURE, dummy, 4, 8, None, 0, dummy, 3, 1, 2, 0, None, None,
                                   dummy, None) == _lib.STMP_EINVAL   # 3 x 1 x 2 != 8
    ins = np.array([4, 6], dtype=np.int64)
    fac = np.array([3, 3], dtype=np.int64)                           # 3 does not divide 4
    assert lib.stmp_apply_operator(_lib.OP_BLOCK_AVERAGE, dummy, 4, 24, None, 0, None, 0, 0, 0, 2,
                                   ins.ctypes.data, fac.ctypes.data, dummy, None) == _lib.STMP_EINVAL
    assert lib.stmp_dc_split(dummy, 4, 8, 8, dummy, 0.0, dummy, 8, dummy, None) == _lib.STMP_EINVAL
    assert lib.stmp_dc_split(dummy, -1, 8, 8, dummy, 1.0, dummy, 8, dummy, None) == _lib.STMP_EINVAL
    assert lib.stmp_reconstruct(None, dummy, dummy, dummy, 4, 2, None, None, dummy, 8, None) == _lib.STMP_EINVAL
