"""Accuracy of the Gram path's ingredients on config 4 (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1412_0680_b200 as P
from paper_1412_0680_b200 import _lib, tree as T, workloads as W
cfg = W.CONFIGS[4]
wl = W.make_dictionary(cfg)
flat = T.load_structure("tests/golden/trees/c4.npz", wl.atoms)
X = W.make_patches(wl, 4096)
sel = P.TreeSelector(flat, wl.atoms, cfg.alpha)
Xd = torch.as_tensor(X).cuda()
_lib.set_option("path", 2)
a64 = wl.atoms.astype(np.float64)
x64 = X.astype(np.float64)
for gp in (0, 2):
    _lib.set_option("gram_path", gp)
    for K in (1, 2, 12):
        r = P.encode(sel, Xd, K, method="omp")
        torch.cuda.synchronize()
        idx, coef, rn = r.idx.cpu().numpy(), r.coef.cpu().numpy(), r.resnorm.cpu().numpy()
        errs, rerrs = [], []
        for p in range(512):
            S = idx[p][idx[p] >= 0]
            A = a64[S]
            c = np.linalg.solve(A @ A.T, A @ x64[p])
            errs.append(np.max(np.abs(coef[p, :len(S)] - c) / np.abs(c)))
            rr = np.linalg.norm(x64[p] - A.T @ c)
            rerrs.append(abs(rn[p] - rr) / rr)
        print(f"gram_path={gp} K={K}: coef rel err median {np.median(errs):.2e} max {np.max(errs):.2e}; "
              f"resnorm rel err median {np.median(rerrs):.2e} max {np.max(rerrs):.2e}", flush=True)
