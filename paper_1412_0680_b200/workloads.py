"""Seeded synthetic workloads for the five BASELINE.json configurations.

No public dataset is named for this path, so every config is a seeded
synthetic stand-in with the shapes, sizes and value distributions that
BASELINE.json states.  Seeds follow the SURVEY recipe:
``SeedSequence(entropy=0, spawn_key=(cfg, role))`` with roles
0 = dictionary draw, 1 = tree seed, 2 = supports, 3 = coefficients,
4 = noise, 5 = exposure mask.  Patch roles add a chunk index to the spawn
key so that the first ``N'`` patches of a config do not depend on how many
patches are requested (a bounded CPU sample is a prefix of the GPU batch).

The dictionary recipe restates the reference's ``normalize_columns``
(``pkg/src/stmp/dictionary.py:122-131``) applied to a
``default_rng(...).standard_normal((m, n))`` draw, which is the recipe the
reference's own ``benchmark`` command uses (``pkg/src/stmp/cli.py:363-366``).
The compressive-video config restates ``coded_exposure_operator``,
``apply_batch`` and ``project_dictionary`` (``pkg/src/stmp/operators.py:67-93,
115-141, 169-196``).  Both restatements are checked bitwise against the
reference in ``tests/test_workloads.py`` (where the reference is importable)
and by the dictionary fingerprint stored with every shipped tree.
"""

from __future__ import annotations

from dataclasses import dataclass
import math

import numpy as np

UNUSABLE_NORM = 1e-6  # pkg/src/stmp/operators.py:26


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    m: int
    n: int
    N: int
    K: int
    branching: tuple
    coef: str          # "normal" | "laplace"
    sigma: float
    sparsity: int      # planted atoms per patch
    n_base: int = 0    # c3: full-space atom dimension before projection
    mask_shape: tuple = ()

    @property
    def alpha(self) -> float:
        """Greedy retention alpha = 1/max(k)."""
        return 1.0 / max(self.branching)

    @property
    def chunk(self) -> int:
        return 65536 if self.n <= 256 else 4096


CONFIGS = {
    0: Config(0, "c0-oracle-4096x64", 4096, 64, 10_000, 5, (16, 16, 16), "normal", 0.05, 5),
    1: Config(1, "c1-denoise-16384x64", 16384, 64, 1_048_576, 8, (32, 32, 16), "laplace", 0.1, 8),
    2: Config(2, "c2-superres-65536x144", 65536, 144, 2_097_152, 6, (256, 256), "laplace", 0.05, 6),
    3: Config(3, "c3-cvideo-100000x49", 100_000, 49, 262_144, 10, (64, 40, 40), "normal", 0.01, 10,
              n_base=1764, mask_shape=(7, 7, 36)),
    4: Config(4, "c4-lightfield-131072x1600", 131_072, 1600, 524_288, 12, (64, 64, 32), "laplace", 0.05, 12),
}


def seed_sequence(cid: int, role: int, *extra: int) -> np.random.SeedSequence:
    return np.random.SeedSequence(entropy=0, spawn_key=(cid, role) + tuple(extra))


def tree_seed(cid: int) -> int:
    """64-bit tree seed, derived like ``cli._spawn_seed`` (pkg/src/stmp/cli.py:219-221)."""
    return int(seed_sequence(cid, 1).generate_state(1, np.uint64)[0])


def normalize_columns(raw) -> np.ndarray:
    """Restates ``normalize_columns`` (pkg/src/stmp/dictionary.py:122-131); returns f32 atoms."""
    raw = np.asarray(raw, dtype=np.float64)
    if raw.ndim != 2:
        raise ValueError(f"expected a 2-D atom array, got shape {raw.shape}")
    norms = np.linalg.norm(raw, axis=1)
    zero = np.flatnonzero(norms == 0.0)
    if zero.size:
        raise ValueError(f"atom {int(zero[0])} is the zero vector and cannot be normalized")
    return np.ascontiguousarray((raw / norms[:, None]).astype(np.float32))


def exposure_mask(cfg: Config) -> np.ndarray:
    """Per-pixel Bernoulli(0.5) binary mask, redrawn until every pixel opens once
    (the precondition of pkg/src/stmp/operators.py:79-80)."""
    rng = np.random.default_rng(seed_sequence(cfg.cid, 5))
    while True:
        mask = (rng.random(cfg.mask_shape) < 0.5).astype(np.float32)
        if (mask.sum(axis=-1) >= 1).all():
            return mask


def coded_exposure_apply(mask: np.ndarray, patches) -> np.ndarray:
    """Restates ``apply_batch`` for a one-window coded-exposure operator
    (pkg/src/stmp/operators.py:127-132): rows in, f64 rows out."""
    patches = np.asarray(patches, dtype=np.float64)
    count = patches.shape[0]
    spatial = mask.shape[:-1]
    frames = mask.shape[-1]
    cube = patches.reshape((count,) + spatial + (1, frames))
    meas = (cube * mask[np.newaxis, ..., np.newaxis, :]).sum(axis=-1)
    return meas.reshape(count, math.prod(spatial))


@dataclass
class Workload:
    cfg: Config
    atoms: np.ndarray              # coding dictionary, f32 [m, n]
    synth: np.ndarray | None = None  # f64 rows used to synthesise patches (c3: Phi·a)
    mask: np.ndarray | None = None
    scale: np.ndarray | None = None
    usable: np.ndarray | None = None


def make_dictionary(cfg: Config) -> Workload:
    rng = np.random.default_rng(seed_sequence(cfg.cid, 0))
    if cfg.n_base == 0:
        atoms = normalize_columns(rng.standard_normal((cfg.m, cfg.n)))
        return Workload(cfg, atoms)
    # c3: base dictionary in full space, projected through the exposure mask
    base = normalize_columns(rng.standard_normal((cfg.m, cfg.n_base)))
    mask = exposure_mask(cfg)
    projected = np.empty((cfg.m, cfg.n), dtype=np.float64)
    step = 8192
    for s in range(0, cfg.m, step):
        projected[s:s + step] = coded_exposure_apply(mask, base[s:s + step])
    del base
    # restates project_dictionary (pkg/src/stmp/operators.py:181-196)
    scale = np.linalg.norm(projected, axis=1)
    usable = scale >= UNUSABLE_NORM
    out = np.zeros_like(projected)
    out[usable] = projected[usable] / scale[usable, None]
    return Workload(cfg, np.ascontiguousarray(out.astype(np.float32)), synth=projected,
                    mask=mask, scale=scale, usable=usable)


def _distinct_supports(rng: np.random.Generator, rows: int, m: int, s: int) -> np.ndarray:
    sup = rng.integers(0, m, size=(rows, s))
    while True:
        srt = np.sort(sup, axis=1)
        dup = np.flatnonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1)) if s > 1 else np.empty(0, int)
        if dup.size == 0:
            return sup
        sup[dup] = rng.integers(0, m, size=(dup.size, s))


def _fill_chunks(wl: Workload, out: np.ndarray, start: int, chunk_ids) -> None:
    cfg = wl.cfg
    src = wl.synth if wl.synth is not None else wl.atoms
    count = out.shape[0]
    c_first = start // cfg.chunk
    for ci in chunk_ids:
        pos = (ci - c_first) * cfg.chunk
        rows = min(cfg.chunk, count - pos)
        full = cfg.chunk  # draw whole chunks so prefixes are stable
        rs = np.random.default_rng(seed_sequence(cfg.cid, 2, ci))
        rc = np.random.default_rng(seed_sequence(cfg.cid, 3, ci))
        rn = np.random.default_rng(seed_sequence(cfg.cid, 4, ci))
        sup = _distinct_supports(rs, full, cfg.m, cfg.sparsity)[:rows]
        if cfg.coef == "normal":
            coef = rc.standard_normal((full, cfg.sparsity))[:rows]
        else:
            coef = rc.laplace(0.0, 1.0, (full, cfg.sparsity))[:rows]
        x = rn.standard_normal((full, cfg.n))[:rows] * cfg.sigma
        for j in range(cfg.sparsity):
            x += coef[:, j:j + 1] * np.asarray(src[sup[:, j]], dtype=np.float64)
        out[pos:pos + rows] = x


_FILL = {}


def _fill_worker(args):
    name, shape, start, ids = args
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(name=name)
    try:
        _fill_chunks(_FILL["wl"], np.ndarray(shape, dtype=np.float32, buffer=shm.buf), start, ids)
    finally:
        shm.close()
    return len(ids)


def make_patches(wl: Workload, count: int | None = None, start: int = 0, procs: int | None = None) -> np.ndarray:
    """Patches ``[start, start + count)`` (default: the first N) as f32 [count, n];
    ``start`` must be a multiple of the config's chunk size.

    Each patch is ``sum_j c_j a_{s_j} + sigma * N(0,1)^n`` over ``sparsity``
    distinct atoms, computed in f64 and cast to f32; c3 synthesises in
    measurement space, ``y = Phi x + sigma * noise`` with x sparse in the base
    dictionary (``Phi a`` rows kept from the projection).
    """
    cfg = wl.cfg
    count = cfg.N if count is None else int(count)
    if start % cfg.chunk:
        raise ValueError(f"start {start} is not a multiple of the chunk size {cfg.chunk}")
    c_first = start // cfg.chunk
    ids = list(range(c_first, c_first + -(-count // cfg.chunk)))
    import os
    procs = procs if procs is not None else min(len(ids), len(os.sched_getaffinity(0)), 32)
    if procs <= 1 or count * cfg.n < (1 << 26):
        out = np.empty((count, cfg.n), dtype=np.float32)
        _fill_chunks(wl, out, start, ids)
        return out
    # large batches: chunks are independent draws, so a fork pool fills disjoint
    # row ranges of one shared buffer (same bytes as the serial loop)
    import multiprocessing as mp
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(create=True, size=count * cfg.n * 4)
    try:
        _FILL["wl"] = wl
        jobs = [(shm.name, (count, cfg.n), start, ids[i::procs]) for i in range(procs)]
        with mp.get_context("fork").Pool(procs) as pool:
            pool.map(_fill_worker, jobs)
        out = np.array(np.ndarray((count, cfg.n), dtype=np.float32, buffer=shm.buf))
    finally:
        _FILL.clear()
        shm.close()
        shm.unlink()
    return out
