"""Benchmark: sparse-coded patches/s of the STMP encoding path on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--method omp|mp]
                  [--selector tree|exact] [--impl ours|reference]
One process per GPU (torchrun for N>1).  A step is one encode of the config's
whole patch batch, inputs already resident in HBM.  Default: config 4, the
largest single-GPU BASELINE config (524,288 light-field patches, 131072x1600
dictionary, tree 64x64x32, tree-OMP K=12); the others via --config.  Weak scaling: every
rank encodes its own N patches (independent patch shards, no data-path
collective); timing is the max over ranks of device-event time.

`--impl reference` times the reference's own CPU algorithm (the oracle port in
oracle/, the reference package cannot travel to the GPU box) on all host cores
over a bounded sample of the same workload.
"""

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse
import json
import math
import multiprocessing as mp
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1412_0680_b200 import roofline as RL  # noqa: E402
from paper_1412_0680_b200 import tree as T  # noqa: E402
from paper_1412_0680_b200 import workloads as W  # noqa: E402

METRIC = "sparse-coded patches/sec (tree-MP/OMP) on 1 B200; % of HBM/tensor roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--method", default="omp", choices=["omp", "mp"])
    ap.add_argument("--selector", default="tree", choices=["tree", "exact"])
    ap.add_argument("--patches", type=int, default=0, help="override N per GPU")
    ap.add_argument("--alpha", type=float, default=0.0,
                    help="tree descent alpha (default 1/max(branching): greedy); larger = beam descent")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel-detail", action="store_true",
                    help="add per-kernel launch counts and times of the instrumented encode (sweeps)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile-run", action="store_true",
                    help="under ncu: only the warm-up and timed encodes (no e2e, CPU leg, peak GEMM or "
                         "instrumented encode)")
    ap.add_argument("--score-kernel", type=int, default=2, choices=[2, 3],
                    help="tcgen05 score pass: 2 node table in shared memory where it fits, 3 streamed table")
    ap.add_argument("--update-kernel", type=int, default=1, choices=[0, 1],
                    help="staged OMP update: 0 generic, 1 lockstep (K<=16) / wide-row")
    ap.add_argument("--pdl", type=int, default=1, choices=[0, 1],
                    help="programmatic dependent launch between the staged kernels")
    ap.add_argument("--path", type=int, default=0, choices=[0, 1, 2],
                    help="encoder: 0 auto, 1 fused warp-per-patch, 2 staged tensor-core pipeline")
    ap.add_argument("--gram", type=int, default=1, choices=[0, 1, 2],
                    help="Gram path (tree OMP without a residual): 0 off, 1 auto, 2 whenever supported")
    ap.add_argument("--graphs", type=int, default=1, choices=[0, 1],
                    help="replay repeated staged encodes as CUDA graphs")
    return ap.parse_args()


def tree_path(cid):
    for p in (os.path.join(ROOT, "tests", "golden", "trees", f"c{cid}.npz"),):
        if os.path.exists(p):
            return p
    raise FileNotFoundError(f"no shipped tree structure for config {cid}")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks sampler

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.rows = []
        self.proc = None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU baseline (oracle port)

_POOL_STATE = {}


def _cpu_worker(args):
    lo, hi = args
    from oracle import stmp_oracle as O
    st = _POOL_STATE
    sel = (O.tree_selector(st["otree"], st["a64"], st["alpha"]) if st["otree"] is not None
           else O.exact_selector(st["a64"]))
    out = []
    for x in st["X"][lo:hi]:
        r = O.encode_one(sel, st["a64"], x, st["K"], st["method"])
        r.pop("residual", None)
        out.append(r)
    return out


def cpu_rate(wl, flat, X, K, method, selector, seconds, cores=None, results=None, alpha=None):
    """Time the reference CPU algorithm (oracle port, f64 NumPy, per-patch loop as
    in pkg/src/stmp/pipelines.py:199-206) on a fork pool of all host cores.
    The per-patch results (rows [0, done) of X) are appended to ``results``."""
    from oracle import stmp_oracle as O
    cores = cores or len(os.sched_getaffinity(0))
    a64 = wl.atoms.astype(np.float64)
    otree = O.OracleTree.from_flat(flat) if selector == "tree" else None
    _POOL_STATE.update(a64=a64, otree=otree, alpha=alpha or wl.cfg.alpha, K=K, method=method, X=X)
    # calibrate on one core
    t0 = time.perf_counter()
    probe = 16 if selector == "tree" else 2
    _cpu_worker((0, probe))
    per = (time.perf_counter() - t0) / probe
    sample = int(min(len(X), max(cores * 4, seconds * cores / per)))
    bounds = [(s, min(s + max(1, sample // (cores * 4)), sample)) for s in
              range(0, sample, max(1, sample // (cores * 4)))]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_worker, [(0, 1)] * cores)  # warm the workers
        t0 = time.perf_counter()
        parts = pool.map(_cpu_worker, bounds)
        wall = time.perf_counter() - t0
    done = sum(len(p) for p in parts)
    if results is not None:
        results.extend(r for p in parts for r in p)
    return done / wall, cores, done, wall


def measure_tf32_tflops(n=8192, reps=10):
    """Dense TF32 tensor-core rate of this GPU (cuBLAS fp32 GEMM with TF32),
    measured live: the denominator of the 3xTF32 score passes' roofline."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        for _ in range(3):
            torch.matmul(a, b, out=c)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        del a, b, c
        return 2 * n ** 3 / statistics.median(ts) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def demangle(name: str) -> str:
    """Readable kernel name from a mangled one (the template arguments kept)."""
    try:
        out = subprocess.run(["c++filt", name], capture_output=True, text=True, timeout=5).stdout.strip()
        return out.replace("stmp::", "").replace("(anonymous namespace)::", "") or name
    except (OSError, subprocess.SubprocessError):
        return name


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ main

def main():
    args = parse()
    rank, world, local = dist_env()
    cfg = W.CONFIGS[args.config]
    exhaustive = args.selector == "exact"
    N = args.patches or cfg.N
    alpha = args.alpha or cfg.alpha
    workload = f"{cfg.name}/{'tree' if not exhaustive else 'exhaustive'}-{args.method.upper()}"
    if args.alpha and not exhaustive:
        workload += f"-alpha{args.alpha:g}"

    if args.impl == "reference":
        if rank != 0:
            return
        wl = W.make_dictionary(cfg)
        flat = T.load_structure(tree_path(cfg.cid), wl.atoms) if not exhaustive else None
        sample_rows = min(N, 65536)
        X = W.make_patches(wl, sample_rows)
        # size each step to ~3 s of the whole CPU so the run ends within minutes
        rate0, cores, _, _ = cpu_rate(wl, flat, X, cfg.K, args.method, args.selector, 3.0, alpha=alpha)
        per_step = int(max(cores, min(len(X), rate0 * 3.0)))
        times = []
        for step in range(args.warmup + args.steps):
            r, cores, done, wall = cpu_rate(wl, flat, X[:per_step], cfg.K, args.method,
                                            args.selector, 1e9, alpha=alpha)
            if step >= args.warmup:
                times.append((done, wall))
        done = sum(d for d, _ in times)
        wall = sum(w for _, w in times)
        value = done / wall
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "patches/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(1, len(times)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "patches_per_step": per_step, "K": cfg.K,
                       "dictionary": [cfg.m, cfg.n], "branching": list(cfg.branching)},
            "cpu_baseline": {"value": value, "unit": "patches/s", "cores": cores, "kind": "port",
                             "sample": f"{per_step} patches per step (prefix of the config batch), "
                                       f"oracle port of the reference (f64 NumPy per-patch loop), "
                                       f"{cores}-process fork pool on {cpu_model()}"},
            "e2e": {"value": value, "unit": "patches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_1412_0680_b200 as P
    from paper_1412_0680_b200 import build
    build.build()
    from paper_1412_0680_b200 import _lib
    _lib.set_option("score_kernel", args.score_kernel)
    _lib.set_option("update_kernel", args.update_kernel)
    _lib.set_option("pdl", args.pdl)
    _lib.set_option("graphs", args.graphs)
    _lib.set_option("path", args.path)
    _lib.set_option("gram_path", args.gram)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    wl = W.make_dictionary(cfg)
    flat = T.load_structure(tree_path(cfg.cid), wl.atoms) if not exhaustive else None
    chunk_start = rank * (-(-N // cfg.chunk) * cfg.chunk)  # distinct patch shard per rank
    X_host = W.make_patches(wl, N, start=chunk_start)
    sel = P.ExactSelector(wl.atoms) if exhaustive else P.TreeSelector(flat, wl.atoms, alpha)
    Xd = torch.as_tensor(X_host).cuda()
    # a dedicated stream: the library replays repeated encodes on it as CUDA graphs
    # (the legacy default stream cannot be captured)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()

    def step():
        with torch.cuda.stream(stream):
            return P.encode(sel, Xd, cfg.K, method=args.method)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    lc0 = _lib.kernel_launches()
    e0.record(stream)
    res = None
    for i in range(args.steps):
        ev[i][0].record(stream)
        if i + 1 < args.steps:
            step()      # outputs freed at once: every step reuses the same buffers (one cached graph)
        else:
            res = step()
        ev[i][1].record(stream)
    e1.record(stream)
    launches = _lib.kernel_launches() - lc0   # counted by the library at each launch site
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    # keep sampling a little longer if the timed region was short
    total_ms = e0.elapsed_time(e1)
    per_launch_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([total_ms], device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    clocks = sampler.stop()

    # end-to-end through the host-buffer C ABI (pinned host memory)
    e2e = None
    if not args.no_e2e and not args.profile_run:
        Xp = torch.from_numpy(X_host).pin_memory()
        outs = dict(idx=torch.empty((N, cfg.K), dtype=torch.int32).pin_memory().numpy(),
                    coef=torch.empty((N, cfg.K), dtype=torch.float32).pin_memory().numpy(),
                    count=torch.empty(N, dtype=torch.int32).pin_memory().numpy(),
                    resnorm=torch.empty(N, dtype=torch.float32).pin_memory().numpy(),
                    ip=torch.empty((N, 2), dtype=torch.int32).pin_memory().numpy())
        Xn = Xp.numpy()
        for _ in range(max(3, args.warmup)):
            P.encode_host(sel, Xn, cfg.K, args.method, out=outs)
        e2e_steps = max(5, min(args.steps, 20))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            P.encode_host(sel, Xn, cfg.K, args.method, out=outs)
        el = torch.tensor([time.perf_counter() - t0], device="cuda")
        if dist:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        h2d = N * cfg.n * 4
        d2h = N * (cfg.K * 8 + 4 + 4 + 8)
        e2e = {"value": world * N * e2e_steps / float(el.item()), "unit": "patches/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "stmp_encode_host (C ABI, pinned host buffers, chunked H2D/encode/D2H)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    value = world * N * args.steps / (total_ms / 1e3)
    launch_ms = statistics.mean(per_launch_ms)
    per_step = launches / max(1, args.steps)
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    bf16 = float(peaks.get("bf16_tflops", 1590.0))
    tf32 = 0.0 if args.profile_run else measure_tf32_tflops()
    rm = RL.model(cfg, N=N, method=args.method, exhaustive=exhaustive, hbm_gbs=hbm,
                  tensor_tflops=(tf32 or 776.3) / 3)

    # per-kernel device time: one more encode, eager, with CUDA events around
    # every launch on the encode stream (outside the timed region: events between
    # launches stop programmatic dependent launch and graph replay)
    ktimes = {}
    if not args.profile_run:
        _lib.kernel_timing(True)
        step()
        torch.cuda.synchronize()
        ktimes = _lib.kernel_times()
        _lib.kernel_timing(False)
    fams = {}
    for name, (cnt, ms) in ktimes.items():
        f = fams.setdefault(RL.family_of(name), {"launches": 0, "ms": 0.0, "kernels": []})
        f["launches"] += cnt
        f["ms"] += ms
        f["kernels"].append(demangle(name))
    timed_ms = sum(f["ms"] for f in fams.values()) or 1.0
    dom = max(fams, key=lambda f: fams[f]["ms"]) if fams else "other"
    gram = any("update_gram_kernel" in k for k in ktimes)
    half = any("score_sh_kernel" in k for k in ktimes)   # Gram-path level passes on fp16 rows
    # tensor-core scores with the 3xFP16 split (score_s16.cu, exact_scan F16 mode): three fp16 products
    # per k-step, so the tensor ceiling of the step model is the dense 16-bit rate / 3, not TF32 / 3
    s16 = any("score_s16_kernel" in k or ("exact_scan_kernel" in k and ("Lb1E" in k or "true" in k))
              for k in ktimes)
    if s16 and not gram:
        rm = RL.model(cfg, N=N, method=args.method, exhaustive=exhaustive, hbm_gbs=hbm, tensor_tflops=bf16 / 3)
    staged_beam = any("beam_resolve_kernel" in k for k in ktimes)
    if dom == "fused":
        work = RL.fused_work(cfg, N, alpha, args.method)
    elif staged_beam:
        work = RL.family_work(cfg, dom, N, args.method, exhaustive, alpha=alpha)
    elif gram:
        work = RL.gram_family_work(cfg, dom, N, half)
    else:
        work = RL.family_work(cfg, dom, N, args.method, exhaustive)
    if gram:   # the step model of the path that ran (Gram path: no residual traffic)
        rm = RL.gram_model(cfg, N, hbm_gbs=hbm, half=half)
    dom_ms = fams[dom]["ms"] if fams else launch_ms
    dom_launches = fams[dom]["launches"] if fams else 1
    avg_s = dom_ms / dom_launches / 1e3
    if work["bound"] == "fp32":
        achieved = work["flops"] / dom_launches / avg_s / 1e12
        roof = {"bound": "fp32 (SIMT FFMA)", "achieved": achieved, "peak": RL.FP32_SIMT_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / RL.FP32_SIMT_TFLOPS, "traffic": None}
    elif work["bound"] == "hbm":
        achieved = work["bytes"] / dom_launches / avg_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": None}
    else:
        achieved = work["flops"] / dom_launches / avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s", "frac": achieved / bf16,
                "traffic": None,
                # the scores are fp32-accurate 3xTF32 (three tf32 products per k-step): against the
                # dense TF32 rate measured live in this run, divided by 3
                "peak_3xtf32": tf32 / 3, "frac_3xtf32": achieved / (tf32 / 3) if tf32 else None,
                # passes that ran the 3xFP16 split (score_s16.cu) spend three fp16 products per k-step:
                # their ceiling is the dense 16-bit rate / 3
                "peak_3xfp16": bf16 / 3 if s16 else None, "frac_3xfp16": achieved / (bf16 / 3) if s16 else None,
                "hbm_frac": work["bytes"] / dom_launches / avg_s / 1e9 / hbm}
    roof.update({
        "kernel": f"{dom}: {', '.join(sorted(set(fams[dom]['kernels'])))}" if fams else "?",
        "launches_per_step": dom_launches, "avg_launch_ms": dom_ms / dom_launches,
        "share_of_step": dom_ms / timed_ms,
        "peak_source": ("MEASURED_PEAKS.json" if peaks else "B200_PROFILING.md fallback") +
                       (f"; TF32 {tf32:.0f} TFLOP/s measured live (cuBLAS 8192^3)" if tf32 else ""),
        "model": ("algorithmic bytes/FLOPs of the dominant kernel family (roofline." +
                  ("gram_family_work, Gram path" if gram else "family_work, SURVEY §8d") +
                  ") per launch / its mean launch time (CUDA events on the encode stream, one instrumented encode)"),
        "families": {f: {"launches": v["launches"], "ms": round(v["ms"], 4), "share": round(v["ms"] / timed_ms, 4)}
                     for f, v in sorted(fams.items(), key=lambda kv: -kv[1]["ms"])},
        # the whole staged step against the §8d per-patch model (the pipeline as one unit)
        "step": {"path": ("gram (no residual; pair tables" + ("; fp16 rows in the level passes)" if half else ")")) if gram
                 else "residual (SURVEY §8d staged design)",
                 "bound": rm["bound"], "bytes_per_patch": rm["bytes_per_patch"],
                 "flops_per_patch": rm["flops_per_patch"], "launch_ms": launch_ms,
                 "launches": per_step, "model_patches_per_s": rm["patches_per_s_roof"],
                 "frac": rm["patches_per_s_roof"] and (N / (launch_ms / 1e3)) / rm["patches_per_s_roof"]},
    })
    if args.kernel_detail:
        roof["kernel_detail"] = {demangle(k)[:70]: [c, round(ms, 4)] for k, (c, ms) in
                                 sorted(ktimes.items(), key=lambda kv: -kv[1][1])}
    traffic_file = os.path.join(ROOT, "profiles", f"r02_traffic_c{cfg.cid}.json")
    if os.path.exists(traffic_file):
        tr = json.load(open(traffic_file))
        key = f"{'exact' if exhaustive else 'tree'}-{args.method}-{N}"
        if key in tr and dom in tr[key]:
            roof["traffic"] = tr[key][dom]   # ncu dram bytes per launch of this family

    cpu = None
    parity = None
    if not args.no_cpu_baseline and not args.profile_run and world == 1:
        from oracle import stmp_oracle as O
        from oracle.parity import compare
        oracle_res = []
        rate, cores, done, wall = cpu_rate(wl, flat, X_host[:65536], cfg.K, args.method, args.selector,
                                           args.cpu_seconds, results=oracle_res, alpha=alpha)
        cpu = {"value": rate, "unit": "patches/s", "cores": cores, "kind": "port",
               "sample": f"{done} patches (prefix of the batch) in {wall:.1f}s, oracle port of the "
                         f"reference (f64 NumPy per-patch loop), {cores}-process pool on {cpu_model()}"}
        # parity of the last timed step's outputs on the same prefix (SURVEY §8c contract)
        ref = O.pack(oracle_res, cfg.K)
        gpu = {k: getattr(res, k)[:done].cpu().numpy() for k in ("idx", "coef", "count", "resnorm", "ip")}
        rep = compare(gpu, ref, X_host[:done], check_path=False)
        parity = rep.as_dict()
        parity["reference"] = "f64 oracle (the cpu_baseline run) on the same prefix; near ties = top-2 gap < 1e-5"
        if half:
            # size-independent check over the whole batch: the fp16 row copies only pre-rank the
            # children, so the encode must equal the one on f32 rows (half_scores = 0) patch for patch
            _lib.set_option("half_scores", 0)
            try:
                ref32 = step()
                torch.cuda.synchronize()
            finally:
                _lib.set_option("half_scores", 1)
            parity["f32_rows_full_batch"] = {
                "patches": N,
                "patches_with_different_support": int((res.idx != ref32.idx).any(1).sum()),
                "coef_bitwise_equal": bool(torch.equal(res.coef, ref32.coef)),
                "resnorm_bitwise_equal": bool(torch.equal(res.resnorm, ref32.resnorm))}
            del ref32

    line = {
        "metric": METRIC, "value": value, "unit": "patches/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded, BASELINE.json config shapes/distributions)",
        "config": {"workload": workload, "patches_per_gpu": N, "dictionary": [cfg.m, cfg.n],
                   "branching": list(cfg.branching), "K": cfg.K, "method": args.method,
                   "parallelism": f"patch shards x{world}",
                   "l2": f"inputs {N * cfg.n * 4 / 1e6:.0f} MB vs 126 MB L2 (no explicit flush)",
                   # every selection, coefficient and norm is an f32 result (3xTF32 / FFMA); where the
                   # level passes read fp16 row copies they only pre-rank the children: decisions within
                   # the copies' noise window are re-taken with exact f32 dots (same outputs as half_scores=0)
                   "arithmetic": ("f32 results; level passes pre-rank on fp16 row copies with exact f32 re-checks"
                                  if half else "f32 (3xTF32 tensor-core scores, FFMA updates)")},
        "roofline": roof,
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline_model_patches_per_s": rm["patches_per_s_roof"],
        "peaks": {"tf32_tflops_live": tf32},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
