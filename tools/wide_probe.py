"""Parity vs the fp64 oracle as the observation dimension p approaches K = N m (conditioning of
Sigma_y) and across the one-CTA (p <= 288) / Schur (p > 288) gain solves."""
import os
import sys

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import enks_oracle, problems  # noqa: E402
from paper_2410_09663_b200 import enks  # noqa: E402

pm = problems.product_modules()
cases = [(150, 100, 312, 4), (200, 120, 400, 4), (100, 60, 200, 4), (50, 30, 100, 4)]
for n, l, N, m in cases:
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(31), n=n, l=l, m=m,
                                           identity_weights=True)
    y = vs.reference_observation()
    ref, _, _ = enks_oracle.oracle_smooth(x0, y, vs, 3, N, seed=5, backend="c")
    got, _ = enks.smooth_horizon(x0, y, vs, 3, N, pm.matvar.NoiseStreams(seed=5))
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    print(f"p={n + l} K={N * m} K/p={N * m / (n + l):.2f} rel={rel:.2e}", flush=True)
