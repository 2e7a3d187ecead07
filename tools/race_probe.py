"""Repeatability of the staged encoder per (score kernel, update kernel) on 262144 config-1 patches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0680_b200 as P  # noqa: E402
from paper_1412_0680_b200 import _lib, tree as T, workloads as W  # noqa: E402

cfg = W.CONFIGS[int(os.environ.get("CFG", "1"))]
wl = W.make_dictionary(cfg)
path = "tests/golden/trees/c%d.npz" % cfg.cid
flat = T.load_structure(path, wl.atoms)
N = int(os.environ.get("NP", "262144"))
X = W.make_patches(wl, N)
sel = P.TreeSelector(flat, wl.atoms, cfg.alpha)
Xd = torch.as_tensor(X).cuda()
_lib.set_option("path", 2)
ref = None
for upd in (2, 1, 0):
    for sk in (2, 0, 1):
        _lib.set_option("score_kernel", sk)
        _lib.set_option("update_kernel", upd)
        runs = [P.encode(sel, Xd, cfg.K, method=os.environ.get("METHOD", "omp")).idx.cpu().numpy() for _ in range(3)]
        small = np.concatenate([P.encode(sel, Xd[s:s + 8192], cfg.K, method=os.environ.get("METHOD", "omp")).idx.cpu().numpy()
                                for s in range(0, N, 8192)])
        d01 = int((runs[0] != runs[1]).any(1).sum())
        d02 = int((runs[0] != runs[2]).any(1).sum())
        ds = int((runs[0] != small).any(1).sum())
        if ref is None:
            ref = runs[0]
        dr = int((runs[0] != ref).any(1).sum())
        print(f"update={upd} score={sk}: run0 vs run1 {d01} rows, run0 vs run2 {d02}, run0 vs 8192-chunks {ds}, "
              f"vs update=2/score=2 {dr}", flush=True)
