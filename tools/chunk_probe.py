"""Diagnose batch-composition dependence: full-batch device encode vs sub-batches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0680_b200 as P  # noqa: E402
from paper_1412_0680_b200 import tree as T, workloads as W  # noqa: E402
sys.path.insert(0, "tests")
from oracle import stmp_oracle as O  # noqa: E402

cfg = W.CONFIGS[1]
wl = W.make_dictionary(cfg)
flat = T.load_structure("tests/golden/trees/c1.npz", wl.atoms)
X = W.make_patches(wl, 262144)
sel = P.TreeSelector(flat, wl.atoms, cfg.alpha)
Xd = torch.as_tensor(X).cuda()
full = P.encode(sel, Xd, cfg.K, method="omp")
fi = full.idx.cpu().numpy()
for cs in (131072, 65536):
    parts = [P.encode(sel, Xd[s:s + cs], cfg.K, method="omp").idx.cpu().numpy() for s in range(0, len(X), cs)]
    pi = np.concatenate(parts)
    bad = np.flatnonzero((pi != fi).any(1))
    print(f"device sub-batches of {cs}: {bad.size} rows differ; first {bad[:5]}", flush=True)
full2 = P.encode(sel, Xd, cfg.K, method="omp").idx.cpu().numpy()
print("repeat full run identical:", np.array_equal(full2, fi))
h = P.encode_host(sel, X, cfg.K, "omp", chunk=65536)
bad = np.flatnonzero((h.idx != fi).any(1))
print(f"host chunks 65536: {bad.size} rows differ; first {bad[:5]}")
if bad.size:
    a64 = wl.atoms.astype(np.float64)
    sel_o = O.tree_selector(O.OracleTree.from_flat(flat), a64, cfg.alpha)
    for p in bad[:3]:
        r = O.encode_one(sel_o, a64, X[p], cfg.K, "omp")
        print(p, "full", fi[p].tolist(), "host", h.idx[p].tolist(), "oracle", r["indices"], "gaps", np.round(r["gaps"], 7).tolist())
