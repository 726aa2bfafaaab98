"""Time the fused W/V_X/V_U noise launch alone at a BASELINE shape (default C3: N=1024, 128x128).

    python tools/noise_bench.py [--members 1024] [--n 128]
"""
import argparse
import os
import sys

import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_09663_b200 import ops as _ops  # noqa: E402
from paper_2410_09663_b200.matvar import entropy_head  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--members", type=int, default=1024)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
ops = _ops.DeviceOps(torch.device("cuda:0"))
N, n = a.members, a.n
K = N * n
diag = torch.ones(n, dtype=torch.float64, device="cuda")
base = torch.randn(n, K, device="cuda")
outs = [torch.empty(n, K, device="cuda") for _ in range(4)]
head = entropy_head(0, ())
jobs = lambda t: [dict(t=t, ch=0, rows=n, diag=diag, out=outs[0], base=base, out_plus=outs[1]),  # noqa
                  dict(t=t, ch=1, rows=n, diag=diag, out=outs[2]),
                  dict(t=t, ch=2, rows=n, diag=diag, out=outs[3])]
for t in range(3):
    ops.noise_fill_multi(head, 0, N, n, jobs(t + 1))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(a.reps):
    ops.noise_fill_multi(head, 0, N, n, jobs(t + 10))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
normals = 3 * N * n * n
print(f"noise N={N} {n}x{n}: {ms * 1e3:.1f} us per step launch, {normals / ms / 1e6:.2f} G normals/s")
