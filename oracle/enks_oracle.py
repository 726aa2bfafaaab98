"""ORACLE (test infrastructure only) — fp64 NumPy restatement of the reference smoother.

Restates reference pkg/src/enksmpc/enks.py step by step, in the reference's
own data layout (members (N, (t+1) d, m), fp64, BLAS GEMMs, LAPACK Cholesky):

  OracleEnsemble      enks.py:56-93   (members, mean, t, lam, jitter_events)
  oracle_init         enks.py:105-128 (N identical copies, lam = 1/tr(Psi))
  _draw               enks.py:131-145 (per-member substream draws, coloured)
  _pair_cov           enks.py:148-153 ((lam/N) A B^T over (member, column) pairs)
  oracle_predict      enks.py:156-186 (W draw, [f(x,u); u+w; w], append, mean, optional cov)
  _barrier_rows       enks.py:201-208 + virtualsys.py:289-302 (constraint barrier row)
  oracle_update       enks.py:189-253 (perturbed obs, Sigma_y, Sigma_xy, jittered Cholesky gain,
                                       whole-trajectory shift, mean, optional cov)
  oracle_smooth       enks.py:256-284 (h x (predict, update))

It is also the CPU baseline that bench.py times (``kind: "port"``): the
reference is pure Python and cannot travel to the GPU box, so this port, which
performs the same fp64 operations in the same order, stands in for it.
Parity of this restatement with the reference itself is pinned by
tests/golden/make_golden.py (run here, where /root/reference is importable)
and re-checked on every box by tests/test_oracle_golden.py.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
from scipy.linalg import cho_factor, cho_solve

from . import noise as _noise

CH_W, CH_VX, CH_VU, CH_EPS = 0, 1, 2, 3
JITTER_REL, JITTER_FLOOR = 1e-9, 1e-30


@dataclass
class OracleEnsemble:
    members: np.ndarray          # (N, (t+1) d, m)
    mean: np.ndarray             # ((t+1) d, m)
    t: int
    lam: float
    n_x: int
    n_u: int
    jitter_events: int = 0

    @property
    def d(self) -> int:
        return self.n_x + 2 * self.n_u

    @property
    def N(self) -> int:
        return self.members.shape[0]

    def tail(self):
        d, n, l = self.d, self.n_x, self.n_u
        last = self.members[:, -d:, :]
        return last[:, :n], last[:, n:n + l], last[:, n + l:]


@dataclass
class OracleCov:
    sigma_traj: np.ndarray
    sigma_pred: Optional[np.ndarray] = None
    sigma_cross: Optional[np.ndarray] = None


@dataclass
class OracleTimers:
    """Wall-clock split of the CPU run (for the baseline report)."""

    noise: float = 0.0
    model: float = 0.0
    other: float = 0.0
    per_step: list = field(default_factory=list)


def oracle_init(x0_packed: np.ndarray, n: int, l: int, n_members: int,
                shared_col_cov: Optional[np.ndarray] = None) -> OracleEnsemble:
    if n_members < 2:
        raise ValueError("need at least 2 ensemble members")
    packed = np.asarray(x0_packed, dtype=float)
    lam = 1.0 / packed.shape[1] if shared_col_cov is None else 1.0 / float(np.trace(shared_col_cov))
    return OracleEnsemble(members=np.repeat(packed[None], n_members, axis=0), mean=packed.copy(),
                          t=0, lam=lam, n_x=n, n_u=l)


def _draw(params, seed, prefix, t, ch, n_members, shape, backend):
    if params is None:
        return np.zeros((n_members, *shape))
    z = _noise.member_normals(seed, prefix, t, ch, n_members, shape, backend=backend)
    return params.mean + params.row_chol @ z @ params.col_chol.T


def _barrier_rows(spec, x, u, du, seed, prefix, t, backend):
    """One row per member: softplus(g(slice_i)) + sqrt(var) * (first draw of (i, t, CH_EPS))."""
    import math
    from types import SimpleNamespace

    N, m = x.shape[0], x.shape[2]
    eps = _noise.member_normals(seed, prefix, t, CH_EPS, N, (1, 1), backend=backend)[:, 0, 0]
    rows = np.empty((N, 1, m))
    for i in range(N):
        g = float(spec.g(SimpleNamespace(x=x[i], u=u[i], du=du[i])))
        z = spec.beta * g
        clean = z / spec.alpha if z > 30.0 else math.log1p(math.exp(z)) / spec.alpha
        rows[i, 0, :] = clean + math.sqrt(spec.noise_var) * eps[i]
    return rows


def _pair_cov(a: np.ndarray, b: np.ndarray, lam: float) -> np.ndarray:
    N = a.shape[0]
    am = np.swapaxes(a, 0, 1).reshape(a.shape[1], -1)
    bm = np.swapaxes(b, 0, 1).reshape(b.shape[1], -1)
    return (lam / N) * (am @ bm.T)


def oracle_predict(ens: OracleEnsemble, vs, seed: int, prefix=(), cov: Optional[OracleCov] = None,
                   backend: str = "numpy", timers: Optional[OracleTimers] = None) -> OracleEnsemble:
    import time

    t0 = time.perf_counter()
    tn = ens.t + 1
    x, u, _ = ens.tail()
    w = _draw(vs.process_noise, seed, prefix, tn, CH_W, ens.N, (ens.n_u, x.shape[2]), backend)
    t1 = time.perf_counter()
    xn = vs.model.step(x, u)
    t2 = time.perf_counter()
    ens.members = np.concatenate([ens.members, np.concatenate([xn, u + w, w], axis=1)], axis=1)
    ens.t = tn
    ens.mean = ens.members.mean(axis=0)
    if cov is not None:
        new = ens.members[:, -ens.d:]
        dev_new = new - new.mean(axis=0)
        dev_traj = ens.members - ens.mean
        cov.sigma_pred = _pair_cov(dev_new, dev_new, ens.lam)
        cov.sigma_cross = _pair_cov(dev_traj, dev_new, ens.lam)
        old = cov.sigma_traj.shape[0]
        grown = np.zeros((old + ens.d, old + ens.d))
        grown[:old, :old] = cov.sigma_traj
        grown[:old, old:] = cov.sigma_cross[:old]
        grown[old:, :old] = cov.sigma_cross[:old].T
        grown[old:, old:] = cov.sigma_pred
        cov.sigma_traj = grown
    if timers is not None:
        timers.noise += t1 - t0
        timers.model += t2 - t1
        timers.other += time.perf_counter() - t2
    return ens


def oracle_update(ens: OracleEnsemble, y_ref: np.ndarray, vs, seed: int, prefix=(),
                  cov: Optional[OracleCov] = None, backend: str = "numpy",
                  timers: Optional[OracleTimers] = None, record: Optional[dict] = None
                  ) -> OracleEnsemble:
    import time

    t0 = time.perf_counter()
    y_ref = np.asarray(y_ref, dtype=float)
    x, u, du = ens.tail()
    m = x.shape[2]
    vx = _draw(vs.obs_noise_x, seed, prefix, ens.t, CH_VX, ens.N, (ens.n_x, m), backend)
    vu = _draw(vs.obs_noise_u, seed, prefix, ens.t, CH_VU, ens.N, (ens.n_u, m), backend)
    obs = np.concatenate([x + vx, u + vu], axis=1)
    if getattr(vs, "constraint", None) is not None:
        obs = np.concatenate([obs, _barrier_rows(vs.constraint, x, u, du, seed, prefix, ens.t,
                                                 backend)], axis=1)
    t1 = time.perf_counter()
    if y_ref.shape != obs.shape[1:]:
        raise ValueError(f"y_ref shape {y_ref.shape} != observation {obs.shape[1:]}")
    ybar = obs.mean(axis=0)
    dy = obs - ybar
    dtraj = ens.members - ens.mean
    sy = _pair_cov(dy, dy, ens.lam)
    sy = 0.5 * (sy + sy.T)
    sxy = _pair_cov(dtraj, dy, ens.lam)
    try:
        fac = cho_factor(sy, lower=True)
    except np.linalg.LinAlgError:
        p = sy.shape[0]
        fac = cho_factor(sy + (JITTER_REL * np.trace(sy) / p + JITTER_FLOOR) * np.eye(p),
                         lower=True)
        ens.jitter_events += 1
    gain = cho_solve(fac, sxy.T).T
    ens.members = ens.members + gain @ (y_ref - obs)
    ens.mean = ens.members.mean(axis=0)
    if record is not None:
        record.setdefault("sigma_y", []).append(sy)
        record.setdefault("sigma_xy", []).append(sxy)
        record.setdefault("gain", []).append(gain)
    if cov is not None:
        dev = ens.members - ens.mean
        cov.sigma_traj = _pair_cov(dev, dev, ens.lam)
    if timers is not None:
        timers.noise += t1 - t0
        timers.other += time.perf_counter() - t1
    return ens


def oracle_smooth(x0, y_refs, vs, h: int, n_members: int, seed: int, prefix=(),
                  track_cov: bool = False, backend: str = "numpy",
                  timers: Optional[OracleTimers] = None, record: Optional[dict] = None):
    """enks.py:256-284.  Returns (mean slices (h+1, d, m), OracleCov | None, ensemble)."""
    import time

    if h < 1:
        raise ValueError("horizon must be at least 1")
    y_refs = np.asarray(y_refs, dtype=float)
    if y_refs.ndim == 2:
        y_refs = np.broadcast_to(y_refs, (h, *y_refs.shape))
    elif y_refs.shape[0] != h:
        raise ValueError(f"need {h} reference observations, got {y_refs.shape[0]}")
    ens = oracle_init(x0.packed, x0.n, x0.l, n_members, shared_col_cov=vs.shared_col_cov)
    cov = OracleCov(sigma_traj=np.zeros((ens.d, ens.d))) if track_cov else None
    for k in range(h):
        ts = time.perf_counter()
        oracle_predict(ens, vs, seed, prefix, cov=cov, backend=backend, timers=timers)
        oracle_update(ens, y_refs[k], vs, seed, prefix, cov=cov, backend=backend, timers=timers,
                      record=record)
        if timers is not None:
            timers.per_step.append(time.perf_counter() - ts)
    return ens.mean.reshape(ens.t + 1, ens.d, -1), cov, ens
