"""Probe: the C3 forecast and the step's noise launch alone, back to back, and concurrently on two
streams (forecast first), with CUDA events -- does the compact forecast layout let the noise blocks
share the SMs (cnn_tc.cu Roles<true>)?

    python tools/corun_probe.py [--members 1024] [--reps 20]
"""
import argparse
import os
import sys

import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import problems  # noqa: E402
from paper_2410_09663_b200.engine import Forecaster  # noqa: E402
from paper_2410_09663_b200.matvar import entropy_head  # noqa: E402
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--members", type=int, default=1024)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
ops = DeviceOps()
pm = problems.product_modules()
n = m = 128
N = a.members
K = N * m
model = pm.dynamics.CNNDynamics(rows=n, cols=m, widths=(2, 32, 32, 1), seed=0)
fc = Forecaster(model, ops, n, n)
last = torch.randn(2 * n, K, device="cuda")
out = torch.empty(n, K, device="cuda")
w, u, vx, vu = (torch.empty(n, K, device="cuda") for _ in range(4))
diag = [torch.rand(n, dtype=torch.float64, device="cuda") + 0.5 for _ in range(3)]
head = entropy_head(4, (2,))
jobs = [dict(t=3, ch=0, rows=n, diag=diag[0], out=w, base=last[n:], out_plus=u),
        dict(t=3, ch=1, rows=n, diag=diag[1], out=vx), dict(t=3, ch=2, rows=n, diag=diag[2], out=vu)]
side = torch.cuda.Stream()
main = torch.cuda.current_stream()


def cnn():
    fc(ops, last, out, n, N)


def noise():
    ops.noise_fill_multi(head, 0, N, m, jobs)


def both():
    ev = torch.cuda.Event()
    ev.record(main)
    cnn()
    side.wait_event(ev)
    with torch.cuda.stream(side):
        noise()
    main.wait_stream(side)


def serial():
    cnn()
    noise()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / a.reps


tag = os.environ.get("ENKS_CNN_COMPACT", "1")
print(f"compact={tag} N={N}: forecast {timed(cnn):.3f} ms, noise {timed(noise):.3f} ms, "
      f"back to back {timed(serial):.3f} ms, concurrent {timed(both):.3f} ms", flush=True)
