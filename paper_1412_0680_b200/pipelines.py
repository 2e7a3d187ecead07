"""GPU batch driver around the encoder.

``code_patches`` mirrors ``pipelines._code_patches`` (pkg/src/stmp/pipelines.py:180-217),
the direct caller of the hot path in every reference task: for each measured
patch it removes the flat (DC) component, codes the rest with matching
pursuit (or the OMP restatement), lifts the measurement-space code onto the
full-space atoms and reconstructs the full-space patch.  Here the three steps
are device kernels of the same library (``stmp_dc_split``, ``stmp_encode``,
``stmp_reconstruct``) instead of a per-patch Python loop, so a task feeds
millions of patches through one call.

Semantics follow the reference line by line:
  * ``dc = (y . dc_meas) / (dc_meas . dc_meas)``, ``x = y - dc * dc_meas``
    (pipelines.py:196,201-202), f64 arithmetic, ``x`` coded in f32;
  * the code is ``matching_pursuit(selector, x, params)`` (pipelines.py:203;
    ``method="omp"`` runs the SURVEY §8c OMP restatement instead);
  * ``lift_code`` divides each coefficient by ``pd.scale[index]`` and raises
    ``RuntimeError`` when an unusable atom was selected (operators.py:199-215);
  * ``reconstruct(base, lifted) + dc`` accumulates in f64 in selection order
    (pursuit.py:224-232, pipelines.py:204);
  * the merged ``ScoreCounter`` (pipelines.py:199-216) is the sum of the
    per-patch counts.
The output is independent of any chunking, as in the reference (pipelines.py:12-14).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .pursuit import ScoreCounter, SearchParams, _gpu_dict_for, _stream_handle, encode


def _as_cuda_f32(measured):
    import torch
    if isinstance(measured, torch.Tensor):
        t = measured
    else:
        t = torch.as_tensor(np.asarray(measured))
    if t.dim() != 2:
        raise ValueError(f"measured patches must form a 2-D array, got shape {tuple(t.shape)}")
    return t.to(device="cuda", dtype=torch.float32).contiguous()


def code_patches(measured, dc_meas, selector, pd, params: SearchParams, threads: int | None = None,
                 method: str = "mp", stream=None):
    """Code measured patches and synthesize full-space patches on the GPU.

    ``measured`` is [N, n_meas] (numpy or a torch tensor), ``dc_meas`` the
    measurement-space image of the flat patch, ``selector`` a GPU
    ``TreeSelector`` / ``ExactSelector`` over ``pd.dictionary``, ``pd`` a
    ``ProjectedDictionary`` (reference ``stmp.project_dictionary`` output or any
    object with ``base``, ``scale`` and ``usable``).  ``threads`` is accepted for
    signature parity and ignored (the output never depends on it).

    Returns ``(out, counter)``: ``out`` [N, base.n] float64 -- a CUDA tensor when
    ``measured`` is one, else a numpy array -- and the merged ``ScoreCounter``.
    """
    import torch
    del threads
    if stream is not None:
        # every allocation, launch and host read runs on `stream`; the caller's
        # stream then waits for it before the outputs are used
        cur = torch.cuda.current_stream()
        stream.wait_stream(cur)
        with torch.cuda.stream(stream):
            out = _code_patches(measured, dc_meas, selector, pd, params, method)
        cur.wait_stream(stream)
        return out
    return _code_patches(measured, dc_meas, selector, pd, params, method)


def _code_patches(measured, dc_meas, selector, pd, params, method):
    import torch
    stream = None   # the current stream (set by code_patches)
    on_device = isinstance(measured, torch.Tensor) and measured.is_cuda
    Y = _as_cuda_f32(measured)
    N, n_meas = Y.shape
    dcm = np.asarray(dc_meas, dtype=np.float64).ravel()
    if dcm.shape != (n_meas,):
        raise ValueError(f"dc_meas has {dcm.size} entries, patches have dimension {n_meas}")
    if selector.gdict.n != n_meas:
        raise ValueError(f"patches have dimension {n_meas}, selector atoms have {selector.gdict.n}")
    denom = float(dcm @ dcm)   # pipelines.py:196
    if not denom > 0.0:
        raise ValueError("dc_meas must be non-zero")
    base = pd.base
    gbase = _gpu_dict_for(base)
    if gbase.m != selector.gdict.m:
        raise ValueError(f"base dictionary has {gbase.m} atoms, the coding dictionary {selector.gdict.m}")
    dev = Y.device
    lib = _lib.load()
    sh = _stream_handle(stream)
    dcm_d = torch.as_tensor(dcm, device=dev)
    Yc = torch.empty_like(Y)
    dc = torch.empty((N,), dtype=torch.float64, device=dev)
    _lib.check(lib.stmp_dc_split(Y.data_ptr(), N, n_meas, n_meas, dcm_d.data_ptr(), denom,
                                 Yc.data_ptr(), n_meas, dc.data_ptr(), sh))
    res = encode(selector, Yc, params.K, method=method, tol=params.residual_tolerance, stream=stream)
    usable = np.asarray(pd.usable, dtype=bool)
    if not usable.all():
        # lift_code (operators.py:209-213): a selected unusable atom is an error
        u = torch.as_tensor(usable, device=dev)
        sel = res.idx.long()
        bad = (sel >= 0) & ~u[sel.clamp_min(0)]
        if bool(bad.any()):
            atom = int(sel[bad][0])
            kind = getattr(getattr(pd, 'operator', None), 'kind', '?')
            raise RuntimeError(f"atom {atom} is unusable under the {kind} "
                               "operator; the selector should never have produced it")
    scale = np.asarray(pd.scale, dtype=np.float64)
    scale_d = None if np.all(scale == 1.0) else torch.as_tensor(scale, device=dev)
    out = torch.empty((N, gbase.n), dtype=torch.float64, device=dev)
    _lib.check(lib.stmp_reconstruct(gbase.handle, res.idx.data_ptr(), res.coef.data_ptr(),
                                    res.count.data_ptr(), N, params.K,
                                    scale_d.data_ptr() if scale_d is not None else None,
                                    dc.data_ptr(), out.data_ptr(), gbase.n, sh))
    counter = ScoreCounter()
    ip = res.ip.to(torch.int64).sum(0).tolist() if N else [0, 0]
    counter.inner_products = int(ip[0])
    counter.centroid_inner_products = int(ip[1])
    if on_device:
        return out, counter
    return out.cpu().numpy(), counter
