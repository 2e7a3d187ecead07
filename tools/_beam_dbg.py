import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1412_0680_b200 as P
from paper_1412_0680_b200 import _lib, tree as T, workloads as W
cfg = W.CONFIGS[0]
wl = W.make_dictionary(cfg)
flat = T.load_structure("tests/golden/trees/c0.npz", wl.atoms)
X = torch.as_tensor(W.make_patches(wl, 4096)).cuda()
sel = P.TreeSelector(flat, wl.atoms, 0.2)
_lib.set_option("path", 2)
_lib.set_option("graphs", 0)
r = P.encode(sel, X, cfg.K, "omp")
torch.cuda.synchronize()
print(r.idx[:3].cpu().numpy(), r.count[:3].cpu().numpy())
