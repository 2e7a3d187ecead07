"""Measured dense tensor peaks on this GPU (the roofline denominators for the
3xTF32 score passes): cuBLAS fp32 GEMM with TF32 tensor cores, bf16, and plain
fp32 (SIMT) for comparison.  CUDA-event timing, warm-up, median of repeats.
Writes one JSON line (stdout)."""
import json
import statistics
import sys

import torch


def rate(dtype, tf32, n=8192, reps=20):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(5):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.median(ts)
    return 2 * n ** 3 / t / 1e12


if __name__ == "__main__":
    out = {"tf32_tflops": rate(torch.float32, True), "bf16_tflops": rate(torch.bfloat16, False),
           "fp32_simt_tflops": rate(torch.float32, False, reps=5),
           "gemm": "torch.matmul 8192^3, cuBLAS, median of CUDA-event timings",
           "device": torch.cuda.get_device_name(0)}
    out["tf32x3_tflops"] = out["tf32_tflops"] / 3
    print(json.dumps(out))
    sys.stdout.flush()
