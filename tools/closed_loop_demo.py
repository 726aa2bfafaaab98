"""SPEC controller example (SPEC.md controller.run_closed_loop): Burgers boundary control on a
2 x 32 x 32 grid, H = 5, N = 100, x_ref = 1 -- rmse trajectory and per-step wall time."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--mode", default="boundary")
args = ap.parse_args()

pm = problems.product_modules()
from paper_2410_09663_b200.controller import ControllerConfig, run_closed_loop  # noqa: E402

from paper_2410_09663_b200.controller import DeviceClosedLoop  # noqa: E402
import torch  # noqa: E402

pr = problems.make_burgers_problem(pm, args.mode)
cfg = ControllerConfig(horizon_h=5, ensemble_n=100, weights=pr.vs.weights, seed=0)
for graph in (False, True):
    loop = DeviceClosedLoop(pr.model, pr.model, cfg, pr.x0.x)
    loop.run(2, graph=graph)  # warm-up / capture
    loop = DeviceClosedLoop(pr.model, pr.model, cfg, pr.x0.x)
    if graph:
        loop.run(0, graph=True)  # capture outside the timed loop
    torch.cuda.synchronize()
    t0 = time.time()
    tr = loop.run(args.steps, graph=graph)
    dt = time.time() - t0
    print(f"graph={graph}: {args.steps} control steps in {dt:.2f} s ({dt / args.steps * 1e3:.2f} "
          f"ms/step)")
print(f"rmse0 {tr.rmse0:.4f}  rmse[10] {tr.rmse[min(9, len(tr) - 1)]:.4f}  "
      f"rmse[-1] {tr.rmse[-1]:.4f}  ratio {tr.rmse[-1] / tr.rmse0:.4f}")
print(f"device time per control step {np.mean(tr.smoother_time) * 1e3:.2f} ms")
print("rmse every 20:", np.round(tr.rmse[::20], 4).tolist())
