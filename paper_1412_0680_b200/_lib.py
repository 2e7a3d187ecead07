"""ctypes binding of the C ABI declared in include/stmp_b200.h.

Loading fails loudly when the in-tree library is missing: there is no CPU
fallback for the encoding path.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import StaleTreeError

HERE = os.path.dirname(os.path.abspath(__file__))
# STMP_LIB_PATH: a kernel-variant build for sweeps (tools/variants.sh); unset normally
LIB_PATH = os.environ.get("STMP_LIB_PATH") or os.path.join(HERE, "_lib", "libstmp_b200.so")

STMP_OK, STMP_EINVAL, STMP_ESTALE, STMP_ECUDA = 0, 1, 2, 3
METHOD_MP, METHOD_OMP, METHOD_SELECT = 0, 1, 2
MAX_K = 128
FNV_OFFSET = 0xCBF29CE484222325

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = {
    "stmp_version": (C.c_char_p, []),
    "stmp_last_error": (C.c_char_p, []),
    "stmp_fnv1a64": (C.c_uint64, [C.c_void_p, C.c_size_t, C.c_uint64]),
    "stmp_dict_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_uint64,
                                   C.c_void_p, C.POINTER(C.c_void_p)]),
    "stmp_dict_free": (None, [C.c_void_p]),
    "stmp_dict_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]),
    "stmp_tree_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64,
                                   C.c_void_p, C.POINTER(C.c_void_p)]),
    "stmp_tree_free": (None, [C.c_void_p]),
    "stmp_encode_workspace": (C.c_size_t, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double]),
    "stmp_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32,
                              C.c_int32, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_size_t, C.c_void_p]),
    "stmp_encode_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                   C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "stmp_stream_sync": (C.c_int, [C.c_void_p]),
    "stmp_set_option": (C.c_int, [C.c_char_p, C.c_int64]),
    "stmp_kernel_launches": (C.c_int, [C.c_void_p]),
    "stmp_kernel_timing": (C.c_int, [C.c_int32]),
    "stmp_kernel_times": (C.c_int, [C.c_int32, C.c_char_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "stmp_dc_split": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_double,
                                C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "stmp_reconstruct": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "stmp_extract_patches": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "stmp_aggregate_patches": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]),
    "stmp_apply_operator": (C.c_int, [C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32,
                                      C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]),
}

PATH_AUTO, PATH_FUSED, PATH_STAGED = 0, 1, 2
OP_ROW_SELECT, OP_CODED_EXPOSURE, OP_BLOCK_AVERAGE = 1, 2, 3


def set_option(key: str, value: int) -> None:
    check(load().stmp_set_option(key.encode(), int(value)))


def kernel_launches() -> int:
    """Cumulative number of kernels the library has launched in this process."""
    v = C.c_int64(0)
    check(load().stmp_kernel_launches(C.byref(v)))
    return int(v.value)


def kernel_timing(enable: bool) -> None:
    """Start (clearing the record) or stop per-kernel CUDA-event timing."""
    check(load().stmp_kernel_timing(1 if enable else 0))


def kernel_times(max_entries: int = 64) -> dict:
    """{kernel name: (launches, total ms)} of the launches recorded since
    kernel_timing(True) (synchronises the recorded events)."""
    import numpy as np
    name_len = 256
    names = C.create_string_buffer(max_entries * name_len)
    launches = np.zeros(max_entries, dtype=np.int64)
    ms = np.zeros(max_entries, dtype=np.float64)
    n = C.c_int32(0)
    check(load().stmp_kernel_times(max_entries, names, name_len, launches.ctypes.data, ms.ctypes.data,
                                   C.byref(n)))
    raw = names.raw
    out = {}
    for i in range(min(n.value, max_entries)):
        nm = raw[i * name_len:(i + 1) * name_len].split(b"\0", 1)[0].decode(errors="replace")
        out[nm] = (int(launches[i]), float(ms[i]))
    return out


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1412_0680_b200.build` "
            "(the encoding path is sm_100a CUDA only; there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == STMP_OK:
        return
    msg = load().stmp_last_error().decode(errors="replace")
    if rc == STMP_EINVAL:
        raise ValueError(msg)
    if rc == STMP_ESTALE:
        raise StaleTreeError(msg)
    raise RuntimeError(msg)
