"""Debug probe: fused CNN at 128-pixel images with a given unit split vs the fp64 oracle, per row."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import problems  # noqa: E402
from oracle.models import cnn_step_torch  # noqa: E402
from paper_2410_09663_b200.engine import Forecaster  # noqa: E402
from paper_2410_09663_b200.ops import DeviceOps  # noqa: E402

N, rows = int(sys.argv[1]), int(sys.argv[2])
ops = DeviceOps()
pm = problems.product_modules()
model = pm.dynamics.CNNDynamics(rows=rows, cols=128, widths=(2, 32, 32, 1), seed=1)
model.state_rows = model.input_rows = rows
rng = np.random.default_rng(0)
x = rng.standard_normal((N, rows, 128))
u = rng.standard_normal((N, rows, 128))
ref = cnn_step_torch(x, u, model.weights, model.biases, model.alpha)
last = ops.to_device(np.concatenate([x, u], axis=1).transpose(1, 0, 2).reshape(2 * rows, -1))
out = ops.zeros(rows, N * 128)
Forecaster(model, ops, rows, rows)(ops, last, out, rows, N)
got = out.double().cpu().numpy().reshape(rows, N, 128).transpose(1, 0, 2)
err = np.abs(got - ref).max(axis=(0, 2))
bad = np.where(~(err < 1e-4))[0]
nanpos = np.argwhere(np.isnan(got))
imgs = sorted(set(int(i) for i in nanpos[:, 0])) if len(nanpos) else []
cols = sorted(set(int(i) for i in nanpos[:, 2])) if len(nanpos) else []
print("nan images", imgs[:10], "cols", cols[:5], "...", cols[-5:] if cols else [])
print(f"N={N} rows={rows} parts={os.environ.get('ENKS_CNN_PARTS', 'auto')}: max err {np.nanmax(err):.2e}, "
      f"nan {int(np.isnan(got).sum())}, bad rows {bad[:20].tolist()}")
