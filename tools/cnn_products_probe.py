"""Probe: accuracy of the fused CNN forecast with 3 vs 2 tf32 products (ENKS_CNN_PRODUCTS) on a
whole smoothed horizon against the fp64 oracle (C3-shaped fields, fewer members).

    python tools/cnn_products_probe.py [--n 128] [--members 256] [--horizon 20]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import enks_oracle, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--members", type=int, default=256)
ap.add_argument("--horizon", type=int, default=20)
a = ap.parse_args()
torch.set_num_threads(os.cpu_count())
pm = problems.product_modules()
pr = problems.make_cnn_problem(pm, "C3", size=a.n, n_members=a.members, horizon=a.horizon)
ovs = pm.virtualsys.build_virtual_system(pr.model, pr.vs.weights)  # fp64 torch-CPU host step
t0 = time.time()
ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=0, backend="c")
print(f"oracle {time.time() - t0:.1f}s", flush=True)
from paper_2410_09663_b200 import enks  # noqa: E402

n, l = pr.n, pr.l
sc = np.abs(ref).max()
for prod in ("3", "2"):
    os.environ["ENKS_CNN_PRODUCTS"] = prod
    got, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, pm.matvar.NoiseStreams(seed=0))
    err = np.abs(got - ref)
    per_t = err.reshape(err.shape[0], -1).max(axis=1) / sc
    print(f"cnn products={prod}: rel all {err.max() / sc:.3e}  X {err[:, :n].max() / sc:.3e}  "
          f"U {err[:, n:n + l].max() / np.abs(ref[:, n:n + l]).max():.3e}  "
          f"per-step max {' '.join(f'{v:.1e}' for v in per_t[::max(1, len(per_t) // 8)])}",
          flush=True)
