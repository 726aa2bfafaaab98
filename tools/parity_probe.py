"""Probe: device smoother vs the fp64 oracle at larger sizes, tcgen05 vs SIMT cross moments.

    python tools/parity_probe.py --n 64 --members 512 --horizon 6 [--linear]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import enks_oracle, problems  # noqa: E402
from oracle.models import OracleCNN  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--members", type=int, default=512)
ap.add_argument("--horizon", type=int, default=6)
ap.add_argument("--linear", action="store_true")
args = ap.parse_args()

pm = problems.product_modules()
pr = problems.make_cnn_problem(pm, "C2", size=args.n, n_members=args.members, horizon=args.horizon)
if args.linear:
    rng = np.random.default_rng(0)
    a = rng.standard_normal((args.n, args.n))
    a *= 0.9 / np.abs(np.linalg.eigvals(a)).max()
    model = pm.dynamics.LinearDynamics(a, rng.standard_normal((args.n, args.n)), state_cols=args.n)
    pr = problems.make_cnn_problem(pm, "C2", size=args.n, n_members=args.members,
                                   horizon=args.horizon, model=model)
    ovs = pr.vs
else:
    import torch
    torch.set_num_threads(os.cpu_count())
    ovs = pm.virtualsys.build_virtual_system(pr.model, pr.vs.weights)  # fp64 torch-CPU host step
t0 = time.time()
ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=0, backend="c")
print(f"oracle {time.time() - t0:.1f}s", flush=True)
from paper_2410_09663_b200 import enks  # noqa: E402

n, l = pr.n, pr.l
for tc, prod in (("1", "3"), ("1", "2"), ("0", "3")):
    os.environ["ENKS_TC"] = tc
    os.environ["ENKS_F16P_PRODUCTS"] = prod
    got, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, pm.matvar.NoiseStreams(seed=0))
    sc = np.abs(ref).max()
    print(f"ENKS_TC={tc} products={prod} rel all {np.abs(got - ref).max() / sc:.3e}  X {np.abs(got[:, :n] - ref[:, :n]).max() / sc:.3e}"
          f"  U {np.abs(got[:, n:n + l] - ref[:, n:n + l]).max() / np.abs(ref[:, n:n + l]).max():.3e}", flush=True)
