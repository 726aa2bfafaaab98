"""Vector-EnKS comparator on the device (reference baselines.py:44-197).

The paper's Table 1 contrasts the matrix-variate smoother with the same single-pass
stochastic EnKS on the vectorised virtual system, whose observation covariance has
(obs_rows * m)^2 entries instead of obs_rows^2.  This module runs that comparator on
the GPU with the same noise substreams (bit-identical draws), the same jitter rule and
the reference's memory projection: before the covariances of a step are formed it
projects the bytes they need (``_predicted_update_bytes``, baselines.py:84-92, here
for fp32 storage) and raises ``MemoryBudgetError`` when they exceed the budget (by
default the device's free memory) -- the "memory outage" the matrix form avoids.

Layout: members in member-row form (N x T*d*m, each slice a row-major d x m block,
baselines.py:57-73); the model forecast, noise and reductions reuse the product's
device kernels (``engine.Forecaster``, ``ops.noise_fill``, ``ops.gemm``,
``ops.spd_inverse``).  Single-column states (m = 1) coincide with the matrix smoother
(reference test_enks.py:147-157).  The gain solve uses the shared-memory Cholesky, so
obs_len = (n + l) m is limited to ``spd_max_p`` (288); larger problems are the ones
this comparator exists to reject.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .engine import CH_VU, CH_VX, CH_W, Forecaster
from .matvar import entropy_head

__all__ = ["MemoryBudgetError", "VectorSmootherReport", "covariance_entry_counts",
           "vector_enks_smooth"]

_FP32 = 4


class MemoryBudgetError(MemoryError):
    """Predicted covariance storage exceeds the configured budget (baselines.py:44-45)."""


@dataclass
class VectorSmootherReport:
    obs_cov_entries: int
    cross_cov_entries: int
    peak_tracked_bytes: int
    jitter_events: int


def covariance_entry_counts(obs_rows: int, m: int) -> dict:
    """Observation-covariance entries of the two formulations (baselines.py:48-50)."""
    return {"vector": (obs_rows * m) ** 2, "matrix": obs_rows ** 2}


def _predicted_update_bytes(n_members: int, traj_len: int, obs_len: int,
                            elem: int = _FP32) -> int:
    """Observation covariance + cross covariance + gain + members + observations."""
    return elem * (obs_len * obs_len + 2 * traj_len * obs_len
                   + n_members * (traj_len + 2 * obs_len))


def _noise_rows(ops, params, head, t, ch, N, rows, m):
    """Coloured draws of substreams (i, t, ch) as (N, rows, m) (enks.py:131-145)."""
    if params is None:
        return ops.zeros(N, rows, m)
    L = np.asarray(params.row_chol, float)
    if not np.array_equal(np.asarray(params.col_chol), np.eye(m)) or np.any(params.mean != 0):
        raise NotImplementedError("device noise supports zero-mean channels with I_m columns")
    z = ops.empty(rows, N * m)
    if np.array_equal(L, np.diag(np.diag(L))):
        ops.noise_fill(head, t, ch, 0, N, rows, m,
                       diag=ops.to_device(np.diag(L).copy(), dtype=torch.float64), out=z)
    else:
        zr = ops.empty(rows, N * m)
        ops.noise_fill(head, t, ch, 0, N, rows, m, out=zr)
        ops.gemm(ops.to_device(L), zr, z)
    return z.view(rows, N, m).permute(1, 0, 2)


def vector_enks_smooth(x0, y_refs, vs, h: int, n_members: int, streams,
                       memory_budget_bytes: Optional[int] = None, ops=None):
    """Single-pass stochastic EnKS on the vectorised virtual system (baselines.py:95-197).

    Returns (mean (h+1, d, m) fp64 ndarray, VectorSmootherReport); raises MemoryBudgetError
    before allocating covariances that would exceed the budget."""
    if vs.constraint is not None:
        raise NotImplementedError("vector baseline does not support constraints")
    if n_members < 2:
        raise ValueError("need at least 2 ensemble members")
    if ops is None:
        from . import enks

        ops = enks._ops()
    y_refs = np.asarray(y_refs, dtype=float)
    if y_refs.ndim == 2:
        y_refs = np.broadcast_to(y_refs, (h, *y_refs.shape))
    n, l, m = x0.n, x0.l, x0.m
    d, N = n + 2 * l, int(n_members)
    obs_len = (n + l) * m
    if memory_budget_bytes is None and ops.device.type == "cuda":
        memory_budget_bytes = int(torch.cuda.mem_get_info(ops.device)[0])
    # the whole horizon's projection first: the outage is reported before any work
    for step in range(1, h + 1):
        need = _predicted_update_bytes(N, (step + 1) * d * m, obs_len)
        if memory_budget_bytes is not None and need > memory_budget_bytes:
            raise MemoryBudgetError(
                f"vector smoother needs ~{need / 1e9:.2f} GB at step {step}, "
                f"budget is {memory_budget_bytes / 1e9:.2f} GB")
    if obs_len > ops.spd_max_p():
        raise NotImplementedError(f"device vector smoother: obs_len {obs_len} > "
                                  f"{ops.spd_max_p()} (shared-memory gain solve)")
    fc = Forecaster(vs.model, ops, n, l)
    head = entropy_head(streams.seed, tuple(streams.prefix))
    traj = (h + 1) * d * m
    members = ops.zeros(N, traj)
    members[:, :d * m] = ops.to_device(np.asarray(x0.packed, float).ravel())[None, :]
    ones = ops.zeros(1, N)
    ones.fill_(1.0 / N)
    status, jitter = ops.zeros(1, dtype=torch.int32), ops.zeros(1, dtype=torch.int32)
    sinv = ops.empty(obs_len, obs_len)
    peak = 0
    for step in range(1, h + 1):
        L0 = step * d * m            # columns before the new slice
        L1 = L0 + d * m
        tail = members[:, L0 - d * m:L0].view(N, d, m)
        # predict: [f(x, u); u + w; w]  (baselines.py:137-149, enks.py:156-171)
        w = _noise_rows(ops, vs.process_noise, head, step, CH_W, N, l, m)
        last = tail[:, :n + l].permute(1, 0, 2).reshape(n + l, N * m).contiguous()
        xn = ops.empty(n, N * m)
        fc(ops, last, xn, n, N)
        new = members[:, L0:L1].view(N, d, m)
        new[:, :n] = xn.view(n, N, m).permute(1, 0, 2)
        new[:, n:n + l] = tail[:, n:n + l] + w
        new[:, n + l:] = w
        # perturbed flattened observation (baselines.py:151-166)
        vx = _noise_rows(ops, vs.obs_noise_x, head, step, CH_VX, N, n, m)
        vu = _noise_rows(ops, vs.obs_noise_u, head, step, CH_VU, N, l, m)
        obs = torch.cat([new[:, :n] + vx, new[:, n:n + l] + vu], dim=1).reshape(N, obs_len)
        peak = max(peak, _predicted_update_bytes(N, L1, obs_len))
        # centred members / observations: column means by a (1 x N) GEMM
        mobs, mtr = ops.empty(1, obs_len), ops.empty(1, L1)
        ops.gemm(ones, obs, mobs)
        ops.gemm(ones, members[:, :L1], mtr)
        dy, dx = ops.empty(N, obs_len), ops.empty(N, L1)
        ops.sub(obs, mobs.expand(N, obs_len), dy)
        ops.sub(members[:, :L1], mtr.expand(N, L1), dx)
        # Sigma_y = dy^T dy / N, Sigma_xy = dx^T dy / N  (baselines.py:176-180)
        sy, sxy = ops.empty(obs_len, obs_len), ops.empty(L1, obs_len)
        ops.gemm(dy, dy, sy, trans_a=True, alpha=1.0 / N)
        ops.gemm(dx, dy, sxy, trans_a=True, alpha=1.0 / N)
        # gain = Sigma_xy Sigma_y^{-1} with the reference's jitter rule (181-187)
        ops.spd_inverse(sy, 1.0, sinv, status, jitter)
        gain = ops.empty(L1, obs_len)
        ops.gemm(sxy, sinv, gain)
        # members += (y_target - obs) gain^T  (188-190)
        innov = ops.empty(N, obs_len)
        yt = ops.to_device(y_refs[step - 1].ravel())[None, :]
        ops.sub(yt.expand(N, obs_len), obs, innov)
        upd = members[:, :L1]
        ops.gemm(innov, gain, upd, trans_b=True, beta=1.0, C0=upd)
    if int(status.item()) != 0:
        raise np.linalg.LinAlgError("observation covariance not positive definite even "
                                    "after jitter")
    mean = ops.empty(1, traj)
    ops.gemm(ones, members, mean)
    report = VectorSmootherReport(obs_cov_entries=obs_len ** 2,
                                  cross_cov_entries=(h + 1) * d * m * obs_len,
                                  peak_tracked_bytes=peak, jitter_events=int(jitter.item()))
    return mean.double().cpu().numpy().reshape(h + 1, d, m), report
