"""Warm-cache per-kernel durations of the encoder (CUPTI activity records via
torch.profiler; no replay, no cache flush), for comparing kernel variants in the
conditions bench.py times them in.

usage: python tools/kprof.py [config] [patches] [option=value ...]
"""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0680_b200 as P  # noqa: E402
from paper_1412_0680_b200 import _lib, build, tree as T, workloads as W  # noqa: E402


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
    build.build()
    for kv in sys.argv[3:]:
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    cfg = W.CONFIGS[cid]
    wl = W.make_dictionary(cfg)
    flat = T.load_structure(f"tests/golden/trees/c{cid}.npz", wl.atoms)
    sel = P.ExactSelector(wl.atoms) if os.environ.get("SELECTOR") == "exact" else P.TreeSelector(flat, wl.atoms, cfg.alpha)
    X = torch.as_tensor(W.make_patches(wl, N)).cuda()
    for _ in range(3):
        P.encode(sel, X, cfg.K, method=os.environ.get("METHOD", "omp"))
    torch.cuda.synchronize()
    reps = 5
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            P.encode(sel, X, cfg.K, method=os.environ.get("METHOD", "omp"))
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = e.name.replace("(anonymous namespace)::", "").split("(")[0][-48:]
        agg[name][0] += 1
        agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    if os.environ.get("KPROF_LIST"):   # every launch of the last encode, in launch order
        evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        evs.sort(key=lambda e: e.time_range.start)
        for e in evs[-(len(evs) // reps):]:
            t = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            print(f"    {t:9.1f} us  {e.name.replace('(anonymous namespace)::', '').split('(')[0][-48:]}")
    tot = sum(v[1] for v in agg.values())
    opts = " ".join(sys.argv[3:]) or "defaults"
    print(f"config {cid}, {N} patches, {opts}: {tot / reps / 1e3:.3f} ms of kernels per encode")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c // reps:4d}/encode {t / reps:9.1f} us/encode {t / c:8.1f} us/launch {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
