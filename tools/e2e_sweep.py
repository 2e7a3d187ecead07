"""End-to-end (host buffers) throughput of stmp_encode_host on a config (CFG,
default 1) for a few chunk sizes, next to the raw pinned H2D / D2H copy
bandwidth of the box and the device-resident encode time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0680_b200 as P  # noqa: E402
from paper_1412_0680_b200 import tree as T, workloads as W  # noqa: E402

cfg = W.CONFIGS[int(os.environ.get("CFG", "1"))]
wl = W.make_dictionary(cfg)
flat = T.load_structure(f"tests/golden/trees/c{cfg.cid}.npz", wl.atoms)
N = cfg.N
sel = P.TreeSelector(flat, wl.atoms, cfg.alpha)
Xp = torch.empty((N, cfg.n), dtype=torch.float32).pin_memory()
Xp.numpy()[:] = W.make_patches(wl, N)
dev = torch.empty_like(Xp, device="cuda")
for name, src, dst in (("H2D", Xp, dev), ("D2H", dev, Xp)):
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(f"{name} pinned copy: {10 * Xp.numel() * 4 / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
Xn = Xp.numpy()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        P.encode(sel, dev, cfg.K, "omp")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        P.encode(sel, dev, cfg.K, "omp")
    torch.cuda.synchronize()
print(f"device-resident encode: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
outs = dict(idx=torch.empty((N, cfg.K), dtype=torch.int32).pin_memory().numpy(),
            coef=torch.empty((N, cfg.K), dtype=torch.float32).pin_memory().numpy(),
            count=torch.empty(N, dtype=torch.int32).pin_memory().numpy(),
            resnorm=torch.empty(N, dtype=torch.float32).pin_memory().numpy(),
            ip=torch.empty((N, 2), dtype=torch.int32).pin_memory().numpy())
for chunk in [int(c) for c in (sys.argv[1:] or [65536, 131072, 262144, 524288])]:
    for _ in range(2):
        P.encode_host(sel, Xn, cfg.K, "omp", chunk=chunk, out=outs)
    t0 = time.perf_counter()
    for _ in range(5):
        P.encode_host(sel, Xn, cfg.K, "omp", chunk=chunk, out=outs)
    dt = (time.perf_counter() - t0) / 5
    print(f"chunk {chunk:7d}: {dt * 1e3:.2f} ms per {N} patches = {N / dt / 1e6:.2f} M patches/s", flush=True)
