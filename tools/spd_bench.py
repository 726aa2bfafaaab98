"""Time the gain solve (Sigma_y^-1 via blocked Cholesky, chol.cu) at p = 64..288."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

ops = DeviceOps()
for p in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("64", "128", "256", "288", "512"))]:
    rng = np.random.default_rng(p)
    a = rng.standard_normal((p, 2 * p))
    s = ops.to_device(a @ a.T / (2 * p) + 0.1 * np.eye(p))
    inv = ops.zeros(p, p)
    st, jt = ops.zeros(1, dtype=torch.int32), ops.zeros(1, dtype=torch.int32)
    for _ in range(3):
        ops.spd_inverse(s, 1.0, inv, st, jt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ops.spd_inverse(s, 1.0, inv, st, jt)
    e1.record()
    torch.cuda.synchronize()
    err = np.abs(inv.double().cpu().numpy() @ s.double().cpu().numpy() - np.eye(p)).max()
    print(f"p={p}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/solve  |inv*S - I| = {err:.2e}", flush=True)
