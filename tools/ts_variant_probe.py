"""Determinism of the TS score pass under debug variants (config 1, 262144 patches)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0680_b200 as P  # noqa: E402
from paper_1412_0680_b200 import _lib, tree as T, workloads as W  # noqa: E402

cfg = W.CONFIGS[1]
wl = W.make_dictionary(cfg)
flat = T.load_structure("tests/golden/trees/c1.npz", wl.atoms)
X = torch.as_tensor(W.make_patches(wl, 262144)).cuda()
sel = P.TreeSelector(flat, wl.atoms, cfg.alpha)
_lib.set_option("path", 2)
_lib.set_option("score_kernel", 0)
ref = P.encode(sel, X, cfg.K, method="omp").idx.cpu().numpy()
_lib.set_option("score_kernel", 2)
for v in [0, 1, 2, 4, 3, 7]:
    _lib.set_option("ts_variant", v)
    bad = [int((P.encode(sel, X, cfg.K, method="omp").idx.cpu().numpy() != ref).any(1).sum()) for _ in range(3)]
    print(f"variant {v}: rows differing from the single-role pass over 3 runs: {bad}", flush=True)
