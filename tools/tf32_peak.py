#!/usr/bin/env python
"""TF32 tensor-core peak on this B200 (cuBLAS via torch.matmul, fp32 inputs with TF32 math),
the roofline denominator for the 3xTF32 kernels (CNN layer 2, gemm_tc): their algorithmic
ceiling is TF32 / 3.  Same method as MEASURED_PEAKS.json's bf16 numbers: 8192^3,
best of 10 (burst) and back to back for 4 s (sustained), CUDA events.

    python tools/tf32_peak.py [--out profiles/r02/tf32_peak.json]
"""
import argparse
import json
import os
import time

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/tf32_peak.json")
    ap.add_argument("--n", type=int, default=8192)
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = True
    n = args.n
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    flop = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    reps = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        reps += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sustained = flop * reps / (s.elapsed_time(e) / 1e3) / 1e12
    res = {"tf32_tflops": flop / best / 1e12, "tf32_tflops_sustained": sustained,
           "how": f"torch.matmul fp32 with allow_tf32 (cuBLAS TF32), {n}^3, best of 10 (burst) and "
                  "back to back for 4 s (sustained), CUDA events",
           "gpu": torch.cuda.get_device_name(0), "torch": torch.__version__}
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
