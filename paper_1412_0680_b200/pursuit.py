"""Drop-in GPU mirror of the reference's sparse-coding API (pkg/src/stmp/pursuit.py).

The reference plugin seam is the selector protocol consumed by
``matching_pursuit`` (pursuit.py:194-221): an object with ``.dictionary`` and
``.select(r, counter=None) -> (index, signed_score)``.  ``ExactSelector`` and
``TreeSelector`` here implement that protocol on the B200 library, so the
reference's own ``matching_pursuit`` runs unchanged with them (one GPU call
per selection), and they also expose the batch entry point ``encode`` that
runs the whole MP / OMP loop for millions of patches in one call.

Error behaviour follows the reference: ``ValueError`` for bad alpha / K /
tolerance / dimensions, ``StaleTreeError`` for a tree built on another
dictionary.  Greedy descent (alpha <= 1/max(k)) runs on the
staged tensor-core pipeline; other alphas run the reference's beam descent on
the warp-per-patch kernel.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field
import math
import os
import weakref

import numpy as np

from . import _lib
from .errors import StaleTreeError
from . import tree as _tree

_CEIL_NUDGE = 1e-9  # pursuit.py:26


def retained_count(alpha: float, k: int) -> int:
    """pursuit.py:29-33."""
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"alpha must lie in (0, 1], got {alpha}")
    return max(1, math.ceil(alpha * k - _CEIL_NUDGE))


def predicted_ip_count(branching, alpha: float) -> int:
    """pursuit.py:36-50."""
    total, branches = 0, 1
    for k in branching:
        total += branches * int(k)
        branches *= retained_count(alpha, int(k))
    return total


@dataclass
class SearchParams:
    """pursuit.py:53-69."""

    K: int
    alpha: float = 1.0
    branching: tuple = ()
    residual_tolerance: float | None = None

    def __post_init__(self):
        if self.K < 1:
            raise ValueError(f"sparsity K must be at least 1, got {self.K}")
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError(f"alpha must lie in (0, 1], got {self.alpha}")
        self.branching = tuple(int(k) for k in self.branching)
        if self.residual_tolerance is not None and self.residual_tolerance < 0:
            raise ValueError(f"residual tolerance must be non-negative, got {self.residual_tolerance}")


@dataclass(eq=False)
class SparseCode:
    """pursuit.py:72-92."""

    m: int
    entries: list = field(default_factory=list)
    ip_count: int = 0

    def combined(self):
        totals: dict = {}
        for index, coefficient in self.entries:
            totals[index] = totals.get(index, 0.0) + coefficient
        return list(totals.items())

    def to_text(self) -> str:
        return "".join(f"{index} {coefficient!r}\n" for index, coefficient in self.entries)


@dataclass(eq=False)
class ScoreCounter:
    """dictionary.py:40-65 (any object with count_atoms/count_centroids works)."""

    inner_products: int = 0
    centroid_inner_products: int = 0

    def count_atoms(self, count: int) -> None:
        self.inner_products += int(count)

    def count_centroids(self, count: int) -> None:
        self.inner_products += int(count)
        self.centroid_inner_products += int(count)

    def merge(self, other) -> None:
        self.inner_products += other.inner_products
        self.centroid_inner_products += other.centroid_inner_products


def fingerprint_atoms(atoms: np.ndarray) -> int:
    """FNV-1a over the f32 little-endian payload (dictionary.py:105-109), native."""
    buf = np.ascontiguousarray(atoms, dtype="<f4")
    lib = _lib.load()
    return int(lib.stmp_fnv1a64(buf.ctypes.data, buf.nbytes, _lib.FNV_OFFSET))


class Dictionary:
    """Minimal mirror of the reference ``Dictionary`` (dictionary.py:68-109) used
    when the caller hands in a bare array."""

    def __init__(self, atoms):
        atoms = np.ascontiguousarray(atoms, dtype=np.float32)
        if atoms.ndim != 2 or atoms.shape[0] == 0 or atoms.shape[1] == 0:
            raise ValueError(f"atoms must form a non-empty 2-D array, got shape {atoms.shape}")
        self.atoms = atoms
        self._fp = None
        self._scoring = None

    @property
    def m(self) -> int:
        return self.atoms.shape[0]

    @property
    def n(self) -> int:
        return self.atoms.shape[1]

    @property
    def scoring_atoms(self) -> np.ndarray:
        if self._scoring is None:
            self._scoring = self.atoms.astype(np.float64)
        return self._scoring

    def fingerprint(self) -> int:
        if self._fp is None:
            self._fp = fingerprint_atoms(self.atoms)
        return self._fp


def _stream_handle(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


class GpuDictionary:
    """Device copy of a dictionary (``stmp_dict_create``)."""

    def __init__(self, dictionary, fingerprint: int | None = None):
        atoms = dictionary.atoms if hasattr(dictionary, "atoms") else dictionary
        atoms = np.ascontiguousarray(atoms, dtype=np.float32)
        if atoms.ndim != 2 or atoms.shape[0] == 0 or atoms.shape[1] == 0:
            raise ValueError(f"atoms must form a non-empty 2-D array, got shape {atoms.shape}")
        if fingerprint is None:
            fingerprint = fingerprint_atoms(atoms)
        self.m, self.n = atoms.shape
        self.fingerprint = int(fingerprint)
        lib = _lib.load()
        h = _lib.C.c_void_p()
        _lib.check(lib.stmp_dict_create(atoms.ctypes.data, self.m, self.n, 0, self.fingerprint,
                                        None, _lib.C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.stmp_dict_free(h)
            self.handle = None


class GpuTree:
    """Device copy of a flattened cluster tree (``stmp_tree_create``)."""

    def __init__(self, tree, gdict: GpuDictionary):
        flat = as_flat_tree(tree)
        if flat.n != gdict.n:
            raise ValueError(f"tree atom dimension {flat.n} != dictionary dimension {gdict.n}")
        self.flat = flat
        self.branching = flat.branching
        self.levels = flat.levels
        lib = _lib.load()
        br = np.asarray(flat.branching, dtype=np.int32)
        off = np.ascontiguousarray(flat.level_offsets, dtype=np.int64)
        cb = np.ascontiguousarray(flat.child_begin, dtype=np.int32)
        cc = np.ascontiguousarray(flat.child_count, dtype=np.int32)
        ce = np.ascontiguousarray(flat.centroids, dtype=np.float32)
        la = np.ascontiguousarray(flat.leaf_atom, dtype=np.int32)
        h = _lib.C.c_void_p()
        _lib.check(lib.stmp_tree_create(gdict.handle, flat.levels, br.ctypes.data, off.ctypes.data,
                                        cb.ctypes.data, cc.ctypes.data, ce.ctypes.data, la.size,
                                        la.ctypes.data, flat.fingerprint, None, _lib.C.byref(h)))
        self.handle = h
        self._keep = gdict

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.stmp_tree_free(h)
            self.handle = None


def as_flat_tree(tree) -> _tree.FlatTree:
    if isinstance(tree, _tree.FlatTree):
        return tree
    if isinstance(tree, (str, os.PathLike)):
        return _tree.read_tree_file(tree)
    if hasattr(tree, "root") and hasattr(tree, "branching"):
        return _tree.from_reference_tree(tree)
    raise TypeError(f"cannot interpret {type(tree).__name__} as a cluster tree")


@dataclass
class EncodeResult:
    """Batch output of ``encode`` (device tensors, or numpy for ``encode_host``)."""

    idx: object        # [N, K] int32, -1 padded, selection order
    coef: object       # [N, K] f32 (MP: step scores, OMP: final refit)
    count: object      # [N] int32
    resnorm: object    # [N] f32
    ip: object         # [N, 2] int32: inner products, centroid inner products
    path: object = None  # [N, K, L] int32 BFS node ids (tree only, optional)
    m: int = 0

    def inner_products(self) -> int:
        ip = self.ip.cpu().numpy() if hasattr(self.ip, "cpu") else np.asarray(self.ip)
        return int(ip[:, 0].astype(np.int64).sum())

    def centroid_inner_products(self) -> int:
        ip = self.ip.cpu().numpy() if hasattr(self.ip, "cpu") else np.asarray(self.ip)
        return int(ip[:, 1].astype(np.int64).sum())

    def to_sparse_codes(self) -> list:
        get = (lambda v: v.cpu().numpy()) if hasattr(self.idx, "cpu") else np.asarray
        idx, coef, cnt, ip = get(self.idx), get(self.coef), get(self.count), get(self.ip)
        return [SparseCode(m=self.m,
                           entries=[(int(idx[p, j]), float(coef[p, j])) for j in range(int(cnt[p]))],
                           ip_count=int(ip[p, 0]))
                for p in range(idx.shape[0])]


class _GpuSelector:
    tree: GpuTree | None = None
    alpha: float = 1.0

    def _select_batch(self, R64: np.ndarray):
        import torch
        R = torch.as_tensor(np.ascontiguousarray(R64, dtype=np.float32)).cuda()
        res = encode(self, R, 1, method="select", paths=self.tree is not None)
        return res

    def select(self, r, counter=None):
        """Selector protocol (pursuit.py:171-172, 190-191)."""
        r = np.asarray(r, dtype=np.float64).ravel()
        if r.shape != (self.gdict.n,):
            raise ValueError(f"query has dimension {r.size}, expected {self.gdict.n}")
        res = self._select_batch(r[None, :])
        idx = int(res.idx[0, 0].item())
        score = float(res.coef[0, 0].item())
        if counter is not None:
            total, cent = (int(v) for v in res.ip[0].tolist())
            if cent:
                counter.count_centroids(cent)
            counter.count_atoms(total - cent)
        return idx, score

    def encode(self, X, K, method="omp", tol=None, paths=False, stream=None) -> EncodeResult:
        return encode(self, X, K, method=method, tol=tol, paths=paths, stream=stream)


# Device copies of dictionaries: weakly keyed by the caller's Dictionary object
# (dropped with it), and a small LRU for bare arrays keyed by content
# (fingerprint, shape), so repeated selectors over the same array share one copy.
_GPU_DICT_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_BARE_CACHE: OrderedDict = OrderedDict()
_BARE_CACHE_SIZE = 4


def _gpu_dict_for(dictionary) -> GpuDictionary:
    try:
        hit = _GPU_DICT_CACHE.get(dictionary)
    except TypeError:          # not weak-referenceable: no cache
        hit = None
    if hit is not None:
        return hit
    fp = dictionary.fingerprint() if hasattr(dictionary, "fingerprint") else None
    g = GpuDictionary(dictionary, fingerprint=fp)
    try:
        _GPU_DICT_CACHE[dictionary] = g
    except TypeError:
        pass
    return g


def _as_dictionary(dictionary):
    """The caller's Dictionary, or a shared wrapper for a bare atom array."""
    if hasattr(dictionary, "atoms"):
        return dictionary
    d = Dictionary(dictionary)
    key = (d.fingerprint(), d.atoms.shape)
    hit = _BARE_CACHE.get(key)
    if hit is not None:
        _BARE_CACHE.move_to_end(key)
        return hit
    _BARE_CACHE[key] = d
    while len(_BARE_CACHE) > _BARE_CACHE_SIZE:
        _BARE_CACHE.popitem(last=False)
    return d


class ExactSelector(_GpuSelector):
    """GPU ``ExactSelector`` (pursuit.py:165-172)."""

    def __init__(self, dictionary):
        dictionary = _as_dictionary(dictionary)
        self.dictionary = dictionary
        self.gdict = _gpu_dict_for(dictionary)
        self.tree = None


class TreeSelector(_GpuSelector):
    """GPU ``TreeSelector`` (pursuit.py:175-191).  Greedy alpha (one child per
    level) runs on the staged tensor-core pipeline for large batches; any other
    alpha is the beam descent of stmp_select (pursuit.py:134-162) on the
    warp-per-patch kernel."""

    def __init__(self, tree, dictionary, alpha: float):
        if not 0.0 < alpha <= 1.0:
            raise ValueError(f"alpha must lie in (0, 1], got {alpha}")
        dictionary = _as_dictionary(dictionary)
        flat = as_flat_tree(tree)
        fp = dictionary.fingerprint() if hasattr(dictionary, "fingerprint") else fingerprint_atoms(dictionary.atoms)
        if flat.fingerprint != fp:
            raise StaleTreeError(
                f"tree fingerprint {flat.fingerprint:#018x} does not match "
                f"dictionary fingerprint {fp:#018x}")
        self.dictionary = dictionary
        self.gdict = _gpu_dict_for(dictionary)
        self.tree = GpuTree(flat, self.gdict)
        self.alpha = float(alpha)


_METHODS = {"mp": _lib.METHOD_MP, "omp": _lib.METHOD_OMP, "select": _lib.METHOD_SELECT}


def encode(selector, X, K: int, method: str = "omp", tol: float | None = None,
           paths: bool = False, stream=None) -> EncodeResult:
    """Encode a batch of patches resident on the GPU.

    ``X`` is a CUDA float32 tensor [N, n] (row stride may exceed n).  Runs the
    reference loop of ``matching_pursuit`` (MP) or its OMP restatement for
    every row in one library call; ``tol`` is the absolute residual tolerance
    (``SearchParams.residual_tolerance``), default ``1e-6 * ||x||``.
    """
    import torch
    if method not in _METHODS:
        raise ValueError(f"unknown method {method!r}")
    if not isinstance(X, torch.Tensor) or not X.is_cuda:
        raise ValueError("encode expects a CUDA tensor; use encode_host for host arrays")
    if X.dtype != torch.float32 or X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be a float32 [N, n] tensor with unit column stride")
    if tol is not None and tol < 0:
        raise ValueError(f"residual tolerance must be non-negative, got {tol}")
    g = selector.gdict
    if X.shape[1] != g.n:
        raise ValueError(f"patches have dimension {X.shape[1]}, dictionary atoms have {g.n}")
    if stream is not None:
        # allocate the outputs and the workspace on the launch stream, so the
        # caching allocator never hands them to another stream while the
        # kernels still run; the stream first waits for the producer of X
        stream.wait_stream(torch.cuda.current_stream(X.device))
        with torch.cuda.stream(stream):
            return _encode_on_stream(selector, X, K, method, tol, paths, stream)
    return _encode_on_stream(selector, X, K, method, tol, paths, None)


def _encode_on_stream(selector, X, K, method, tol, paths, stream) -> EncodeResult:
    import torch
    g = selector.gdict
    N = X.shape[0]
    dev = X.device
    idx = torch.empty((N, K), dtype=torch.int32, device=dev)
    coef = torch.empty((N, K), dtype=torch.float32, device=dev)
    count = torch.empty((N,), dtype=torch.int32, device=dev)
    resn = torch.empty((N,), dtype=torch.float32, device=dev)
    ip = torch.empty((N, 2), dtype=torch.int32, device=dev)
    tree = selector.tree
    path = None
    if paths and tree is not None:
        path = torch.empty((N, K, tree.levels), dtype=torch.int32, device=dev)
    lib = _lib.load()
    th = tree.handle if tree is not None else None
    ws_bytes = int(lib.stmp_encode_workspace(g.handle, th, N, K, _METHODS[method], float(selector.alpha)))
    ws = torch.empty((max(ws_bytes, 1),), dtype=torch.uint8, device=dev)
    _lib.check(lib.stmp_encode(
        g.handle, th, X.data_ptr(), N, X.stride(0) if N > 1 else g.n, K, _METHODS[method],
        float(selector.alpha), -1.0 if tol is None else float(tol),
        idx.data_ptr(), coef.data_ptr(), count.data_ptr(), resn.data_ptr(),
        path.data_ptr() if path is not None else None, ip.data_ptr(),
        ws.data_ptr(), ws_bytes, _stream_handle(stream)))
    return EncodeResult(idx, coef, count, resn, ip, path, m=g.m)


def encode_host(selector, X: np.ndarray, K: int, method: str = "omp", tol: float | None = None,
                chunk: int | None = None, out: dict | None = None) -> EncodeResult:
    """End-to-end encode from host memory (``stmp_encode_host``): chunked H2D,
    encode and D2H overlapped on three streams.  Pass pinned buffers (e.g. torch
    ``pin_memory()`` tensors' numpy views) for full copy bandwidth.

    ``chunk`` (rows per encode) defaults to 2^17 for narrow rows (config 1: 178 M
    patches/s against a 55 GB/s pinned-copy floor of 217 M/s) and to a quarter of
    the batch for rows of >= 256 floats: there every encode also streams the
    deepest level's node tables once per iteration whatever its size, so chunks
    should stay large, but the copy of the first chunk and the encode of the last
    are not overlapped (config 4, 2^19 patches, 55.6 GB/s pinned copies = a
    60.4 ms floor: 71.4 ms in four chunks, 80.8 ms in two, 99.1 ms in one)."""
    if method not in ("mp", "omp"):
        raise ValueError(f"unknown method {method!r}")
    X = np.asarray(X)
    if X.dtype != np.float32 or X.ndim != 2 or X.strides[1] != 4:
        raise ValueError("X must be a float32 [N, n] array with unit column stride")
    g = selector.gdict
    if X.shape[1] != g.n:
        raise ValueError(f"patches have dimension {X.shape[1]}, dictionary atoms have {g.n}")
    N = X.shape[0]
    if chunk is None:
        chunk = 1 << 17 if g.n < 256 else max(4096, -(-N // 4))
    if out is None:
        out = dict(idx=np.empty((N, K), np.int32), coef=np.empty((N, K), np.float32),
                   count=np.empty(N, np.int32), resnorm=np.empty(N, np.float32),
                   ip=np.empty((N, 2), np.int32))
    # the library writes through these pointers: shape, dtype and layout must be exact
    for name, shape, dt in (("idx", (N, K), np.int32), ("coef", (N, K), np.float32),
                            ("count", (N,), np.int32), ("resnorm", (N,), np.float32),
                            ("ip", (N, 2), np.int32)):
        a = out.get(name)
        if not isinstance(a, np.ndarray) or a.shape != shape or a.dtype != dt or not a.flags.c_contiguous \
                or not a.flags.writeable:
            raise ValueError(f"out[{name!r}] must be a writeable C-contiguous {np.dtype(dt).name} array "
                             f"of shape {shape}")
    lib = _lib.load()
    th = selector.tree.handle if selector.tree is not None else None
    _lib.check(lib.stmp_encode_host(
        g.handle, th, X.ctypes.data, N, X.strides[0] // 4, K, _METHODS[method],
        float(selector.alpha), -1.0 if tol is None else float(tol),
        out["idx"].ctypes.data, out["coef"].ctypes.data, out["count"].ctypes.data,
        out["resnorm"].ctypes.data, out["ip"].ctypes.data, int(chunk)))
    return EncodeResult(out["idx"], out["coef"], out["count"], out["resnorm"], out["ip"], None, m=g.m)


def _single(selector, x, params, counter, method):
    import torch
    d = selector.dictionary
    x = np.asarray(x, dtype=np.float64).ravel()
    if x.shape != (d.n,):
        raise ValueError(f"query has dimension {x.size}, expected {d.n}")
    X = torch.as_tensor(x.astype(np.float32)[None, :]).cuda()
    res = encode(selector, X, params.K, method=method, tol=params.residual_tolerance)
    code = res.to_sparse_codes()[0]
    if counter is not None:
        total, cent = (int(v) for v in res.ip[0].tolist())
        if cent:
            counter.count_centroids(cent)
        counter.count_atoms(total - cent)
    return code


def matching_pursuit(selector, x, params: SearchParams, counter=None) -> SparseCode:
    """GPU ``matching_pursuit`` (pursuit.py:194-221) for one patch."""
    return _single(selector, x, params, counter, "mp")


def orthogonal_matching_pursuit(selector, x, params: SearchParams, counter=None) -> SparseCode:
    """GPU OMP for one patch (the SURVEY §8c restatement; coefficients are the final refit)."""
    return _single(selector, x, params, counter, "omp")


# Per-call free functions reuse their selector (device tree tables included)
# for the same (tree, dictionary, alpha): a small LRU holding the arguments.
_SELECTOR_CACHE: OrderedDict = OrderedDict()
_SELECTOR_CACHE_SIZE = 4


def _cached_selector(key, args, make):
    hit = _SELECTOR_CACHE.get(key)
    if hit is not None and all(a is b for a, b in zip(hit[0], args)):
        _SELECTOR_CACHE.move_to_end(key)
        return hit[1]
    sel = make()
    _SELECTOR_CACHE[key] = (args, sel)
    while len(_SELECTOR_CACHE) > _SELECTOR_CACHE_SIZE:
        _SELECTOR_CACHE.popitem(last=False)
    return sel


def exact_select(d, r, counter=None):
    """GPU ``exact_select`` (pursuit.py:102-109)."""
    sel = _cached_selector(("exact", id(d)), (d,), lambda: ExactSelector(d))
    return sel.select(r, counter)


def stmp_select(t, d, r, alpha: float, counter=None):
    """GPU ``stmp_select`` (pursuit.py:112-162)."""
    sel = _cached_selector(("tree", id(t), id(d), float(alpha)), (t, d), lambda: TreeSelector(t, d, alpha))
    return sel.select(r, counter)
