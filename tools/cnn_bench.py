"""Time the CNN forecast kernel alone at C3 shapes (N members of 128x128, widths 2-32-32-1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import problems  # noqa: E402
from paper_2410_09663_b200.engine import Forecaster  # noqa: E402
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ops = DeviceOps()
pm = problems.product_modules()
model = pm.dynamics.CNNDynamics(rows=128, cols=128, widths=(2, 32, 32, 1), seed=0)
last = torch.randn(256, N * 128, device="cuda")
out = torch.empty(128, N * 128, device="cuda")
fc = Forecaster(model, ops, 128, 128)
for _ in range(2):
    fc(ops, last, out, 128, N)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    fc(ops, last, out, 128, N)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
flops = N * model.flops_per_member_step()
print(f"cnn N={N} debug={os.environ.get('ENKS_CNN_DEBUG', '0')}: {ms:.3f} ms/step, "
      f"{flops / ms / 1e9:.1f} TFLOP/s algorithmic")
