"""Data formats either side of the encoder, on the GPU.

* ``PatchLayout`` / ``extract_patches`` / ``aggregate_patches`` mirror
  pkg/src/stmp/tensor.py:49-136: sliding windows at every multiple of the
  stride with the final valid start forced in; extraction is a bit-exact copy,
  aggregation the f64 mean of the covering patch values summed in origin
  order (bitwise the reference's deterministic result).
* ``apply_batch`` mirrors pkg/src/stmp/operators.py:115-141 for the
  reference's ``ObservationOperator`` kinds (identity, row selection, coded
  exposure, block average): f32 rows in, f64 rows out.

Tensors live on the GPU (torch CUDA tensors, work on torch's current stream);
numpy inputs are copied up and numpy outputs returned, like
``pipelines.code_patches``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

from . import _lib
from .pursuit import _stream_handle


def _as_shape(value, name: str) -> tuple[int, ...]:
    shape = tuple(int(v) for v in value)
    if not shape or any(v <= 0 for v in shape):
        raise ValueError(f"{name} must be a non-empty sequence of positive ints, got {value!r}")
    return shape


def _axis_starts(extent: int, patch: int, stride: int) -> np.ndarray:
    """tensor.py:42-48: starts at multiples of the stride, final valid start forced in."""
    last = extent - patch
    starts = list(range(0, last + 1, stride))
    if starts[-1] != last:
        starts.append(last)
    return np.asarray(starts, dtype=np.int64)


@dataclass
class PatchLayout:
    """tensor.py:51-99 (validation and error behaviour included)."""

    tensor_shape: tuple
    patch_shape: tuple
    stride: tuple
    axis_starts: tuple = field(init=False, repr=False)

    def __post_init__(self):
        self.tensor_shape = _as_shape(self.tensor_shape, "tensor_shape")
        self.patch_shape = _as_shape(self.patch_shape, "patch_shape")
        self.stride = _as_shape(self.stride, "stride")
        rank = len(self.tensor_shape)
        if len(self.patch_shape) != rank or len(self.stride) != rank:
            raise ValueError(f"rank mismatch: tensor rank {rank}, patch rank {len(self.patch_shape)}, "
                             f"stride rank {len(self.stride)}")
        for axis, (extent, patch, step) in enumerate(zip(self.tensor_shape, self.patch_shape, self.stride)):
            if patch > extent:
                raise ValueError(f"patch extent {patch} exceeds tensor extent {extent} on axis {axis}")
            if step > patch:
                raise ValueError(f"stride {step} exceeds patch extent {patch} on axis {axis}")
        self.axis_starts = tuple(_axis_starts(e, p, s)
                                 for e, p, s in zip(self.tensor_shape, self.patch_shape, self.stride))

    @property
    def patch_dim(self) -> int:
        return math.prod(self.patch_shape)

    @property
    def num_patches(self) -> int:
        return math.prod(len(s) for s in self.axis_starts)

    def _device_geometry(self, dev):
        import torch
        rank = len(self.tensor_shape)
        if rank > 8:
            raise ValueError(f"the GPU kernels support ranks up to 8, got {rank}")
        shape = np.asarray(self.tensor_shape, dtype=np.int64)
        patch = np.asarray(self.patch_shape, dtype=np.int64)
        nst = np.asarray([len(s) for s in self.axis_starts], dtype=np.int64)
        starts = torch.as_tensor(np.concatenate(self.axis_starts).astype(np.int64), device=dev)
        return rank, shape, patch, nst, starts


def _to_cuda_f32(a):
    import torch
    on_device = isinstance(a, torch.Tensor) and a.is_cuda
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
    return t.to(device="cuda", dtype=torch.float32).contiguous(), on_device


def extract_patches(t, patch_shape, stride):
    """tensor.py:104-111: every layout window of ``t`` as a row of an (N, n) f32 matrix."""
    T, on_device = _to_cuda_f32(t)
    layout = PatchLayout(tuple(T.shape), patch_shape, stride)
    import torch
    out = torch.empty((layout.num_patches, layout.patch_dim), dtype=torch.float32, device=T.device)
    rank, shape, patch, nst, starts = layout._device_geometry(T.device)
    _lib.check(_lib.load().stmp_extract_patches(T.data_ptr(), rank, shape.ctypes.data, patch.ctypes.data,
                                                nst.ctypes.data, starts.data_ptr(), out.data_ptr(),
                                                _stream_handle()))
    return layout, (out if on_device else out.cpu().numpy())


def aggregate_patches(layout: PatchLayout, patches):
    """tensor.py:114-136: average overlapping patches back into an f32 tensor."""
    P, on_device = _to_cuda_f32(patches)
    if tuple(P.shape) != (layout.num_patches, layout.patch_dim):
        raise ValueError(f"expected {layout.num_patches} patches of dimension {layout.patch_dim}, "
                         f"got array of shape {tuple(P.shape)}")
    import torch
    out = torch.empty(layout.tensor_shape, dtype=torch.float32, device=P.device)
    rank, shape, patch, nst, starts = layout._device_geometry(P.device)
    _lib.check(_lib.load().stmp_aggregate_patches(P.data_ptr(), rank, shape.ctypes.data, patch.ctypes.data,
                                                  nst.ctypes.data, starts.data_ptr(), out.data_ptr(),
                                                  _stream_handle()))
    return out if on_device else out.cpu().numpy()


def apply_batch(op, patches):
    """operators.py:115-141: measure a stack of patch rows (f32 in, f64 out).

    ``op`` is the reference's ``ObservationOperator`` (or any object with its
    fields: kind, n_in, n_out, row_indices, mask, windows, in_shape, factors).
    """
    import torch
    X, on_device = _to_cuda_f32(patches)
    if X.dim() != 2 or X.shape[1] != op.n_in:
        raise ValueError(f"expected patches of dimension {op.n_in}, got array of shape {tuple(X.shape)}")
    N = X.shape[0]
    kind = op.kind
    lib = _lib.load()
    sh = _stream_handle()
    if kind == "identity":
        Y = X.double()
    else:
        Y = torch.empty((N, op.n_out), dtype=torch.float64, device=X.device)
        none = None
        if kind == "row_select":
            rows = torch.as_tensor(np.asarray(op.row_indices, dtype=np.int64), device=X.device)
            _lib.check(lib.stmp_apply_operator(_lib.OP_ROW_SELECT, X.data_ptr(), N, op.n_in, rows.data_ptr(),
                                               rows.numel(), none, 0, 0, 0, 0, none, none, Y.data_ptr(), sh))
        elif kind == "coded_exposure":
            mask = np.ascontiguousarray(op.mask, dtype=np.float32)
            frames = mask.shape[-1]
            pixels = mask.size // frames
            m = torch.as_tensor(mask.reshape(pixels, frames), device=X.device)
            _lib.check(lib.stmp_apply_operator(_lib.OP_CODED_EXPOSURE, X.data_ptr(), N, op.n_in, none, 0,
                                               m.data_ptr(), pixels, int(op.windows), frames, 0, none, none,
                                               Y.data_ptr(), sh))
        elif kind == "block_average":
            ins = np.asarray(op.in_shape, dtype=np.int64)
            fac = np.asarray(op.factors, dtype=np.int64)
            _lib.check(lib.stmp_apply_operator(_lib.OP_BLOCK_AVERAGE, X.data_ptr(), N, op.n_in, none, 0, none,
                                               0, 0, 0, len(ins), ins.ctypes.data, fac.ctypes.data,
                                               Y.data_ptr(), sh))
        else:
            raise ValueError(f"unknown operator kind {kind!r}")
    return Y if on_device else Y.cpu().numpy()
