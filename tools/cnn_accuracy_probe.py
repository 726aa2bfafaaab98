"""Probe: accuracy of the fused CNN forecast kernel (widths 2-32-32-1) against the fp64 torch
restatement, for 128 / 64 / 32-wide fields and inputs over several magnitudes; prints the max
error relative to max |out| and the max elementwise error relative to atol 2e-6 + rtol 1e-5 (the
kernel tests' bar).  Also times the C3-shaped forecast (N = 1024, 128 x 128).

    python tools/cnn_accuracy_probe.py [--members 16]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import problems  # noqa: E402
from oracle.models import cnn_step_torch  # noqa: E402
from paper_2410_09663_b200.engine import Forecaster  # noqa: E402
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--members", type=int, default=16)
a = ap.parse_args()
ops = DeviceOps()
pm = problems.product_modules()
worst = 0.0
for size in (128, 64, 32):
    for seed, mag in ((0, 1.0), (1, 10.0), (2, 0.01), (3, 100.0)):
        model = pm.dynamics.CNNDynamics(rows=size, cols=size, widths=(2, 32, 32, 1), seed=seed)
        N = a.members
        rng = np.random.default_rng(seed)
        x = mag * rng.standard_normal((N, size, size))
        u = mag * rng.standard_normal((N, size, size))
        ref = cnn_step_torch(x, u, model.weights, model.biases, model.alpha)
        last = ops.to_device(np.concatenate([x, u], axis=1).transpose(1, 0, 2).reshape(2 * size, -1))
        out = ops.zeros(size, N * size)
        Forecaster(model, ops, size, size)(ops, last, out, size, N)
        got = out.cpu().double().numpy().reshape(size, N, size).transpose(1, 0, 2)
        err = np.abs(got - ref)
        # the residual x dominates |out|: report the error of the CNN increment too
        inc = np.abs(ref - x).max()
        bar = (err / (2e-6 + 1e-5 * np.abs(ref))).max()
        worst = max(worst, bar)
        print(f"size {size:3d} |in| ~ {mag:6.2f}: max err {err.max():.3e}  / max|out| "
              f"{err.max() / np.abs(ref).max():.3e}  / max|increment| {err.max() / inc:.3e}  "
              f"test-bar fraction {bar:.3f}", flush=True)
print(f"worst test-bar fraction {worst:.3f}")

model = pm.dynamics.CNNDynamics(rows=128, cols=128, widths=(2, 32, 32, 1), seed=0)
N = 1024
last = torch.randn(256, N * 128, device="cuda")
out = torch.empty(128, N * 128, device="cuda")
fc = Forecaster(model, ops, 128, 128)
for _ in range(3):
    fc(ops, last, out, 128, N)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    fc(ops, last, out, 128, N)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"C3 forecast N = {N}: {ms:.3f} ms/step, "
      f"{N * model.flops_per_member_step() / ms / 1e9:.1f} TFLOP/s algorithmic", flush=True)
