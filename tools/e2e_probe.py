"""Time the host-buffer entry point (stmp_encode_host) for several chunk sizes on config 1."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0680_b200 as P  # noqa: E402
from paper_1412_0680_b200 import tree as T, workloads as W  # noqa: E402

cfg = W.CONFIGS[1]
wl = W.make_dictionary(cfg)
flat = T.load_structure("tests/golden/trees/c1.npz", wl.atoms)
X = W.make_patches(wl)
sel = P.TreeSelector(flat, wl.atoms, cfg.alpha)
Xp = torch.from_numpy(X).pin_memory().numpy()
N = len(X)
outs = dict(idx=torch.empty((N, cfg.K), dtype=torch.int32).pin_memory().numpy(),
            coef=torch.empty((N, cfg.K), dtype=torch.float32).pin_memory().numpy(),
            count=torch.empty(N, dtype=torch.int32).pin_memory().numpy(),
            resnorm=torch.empty(N, dtype=torch.float32).pin_memory().numpy(),
            ip=torch.empty((N, 2), dtype=torch.int32).pin_memory().numpy())
Xd = torch.as_tensor(X).cuda()
ref = P.encode(sel, Xd, cfg.K, method="omp")
torch.cuda.synchronize()
for chunk in (131072, 262144, 524288, 1048576):
    P.encode_host(sel, Xp, cfg.K, "omp", chunk=chunk, out=outs)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        P.encode_host(sel, Xp, cfg.K, "omp", chunk=chunk, out=outs)
    dt = (time.perf_counter() - t0) / reps
    same = np.array_equal(outs["idx"], ref.idx.cpu().numpy())
    print(f"chunk {chunk}: {dt * 1e3:.2f} ms/step  {N / dt / 1e6:.1f} M patches/s  idx==device: {same}", flush=True)
t0 = time.perf_counter()
for _ in range(3):
    xd = torch.from_numpy(Xp).cuda(non_blocking=True)
    torch.cuda.synchronize()
print(f"H2D alone: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms for {X.nbytes / 1e6:.0f} MB")
