"""Time the member-statistics launches (stats.cu) alone at a BASELINE shape (default C3).

    python tools/stats_bench.py [--members 1024] [--n 128]

slice sum (d = 3n rows), slice centring into the pair basis (v4), observation sum (x + v on the
fly, p = 2n rows) and the observation centring with the transposed planes.  Algorithmic bytes as
in DESIGN.md section 4.  ENKS_SUM_SCALAR=1 selects the scalar member-sum kernel.
"""
import argparse
import os
import sys

import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_09663_b200 import ops as _ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--members", type=int, default=1024)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
ops = _ops.DeviceOps(torch.device("cuda:0"))
N, n = a.members, a.n
m, K = n, N * n
d, p = 3 * n, 2 * n
dev = "cuda"
sl = torch.randn(d, K, device=dev)
ob, v = torch.randn(p, K, device=dev), torch.randn(p, K, device=dev)
acc_s, amax_s = torch.empty(d * m, dtype=torch.float64, device=dev), torch.empty(d * m, device=dev)
acc_o, amax_o = torch.empty(p * m, dtype=torch.float64, device=dev), torch.empty(p * m, device=dev)
mean_s, mean_o = torch.empty(d, m, device=dev), torch.empty(p, m, device=dev)
Ah, Al = (torch.empty(2 * n, K, dtype=torch.float16, device=dev) for _ in range(2))
Yh, Yl = (torch.empty(p, K, dtype=torch.float16, device=dev) for _ in range(2))
th, tl = (torch.empty(K, p, dtype=torch.float16, device=dev) for _ in range(2))
a_inv, y_inv, t_inv = (torch.empty(x, device=dev) for x in (d, p, K))
A_new = torch.empty(2 * n, K, device=dev)

cases = {
    "slice_sum": (lambda: ops.member_sum(sl, N, m, None, acc_s, amax_s), 4 * d * K),
    "slice_center": (lambda: ops.member_center_f16pair(sl, N, m, None, acc_s, amax_s, N, mean_s, Ah,
                                                       Al, a_inv, f32=A_new, rows_f32=2 * n,
                                                       skip=(n, 2 * n)),
                     4 * d * K + 4 * 2 * n * K + 4 * 2 * n * K),
    "obs_sum": (lambda: ops.member_sum(ob, N, m, None, acc_o, amax_o, src2=v), 8 * p * K),
    "obs_center_t": (lambda: ops.member_center_f16pair_t(ob, v, N, m, None, acc_o, amax_o, N,
                                                         mean_o, Yh, Yl, y_inv, th, tl, t_inv),
                     8 * p * K + 4 * p * K + 4 * p * K),
}
for name, (fn, nbytes) in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{name:14s} N={N} {n}x{n}: {ms * 1e3:7.1f} us  {nbytes / ms / 1e6:7.0f} GB/s algorithmic")
