"""Closed-loop receding-horizon driver on the device.

The reference ships the smoother but not the controller: SPEC.md:365-428 (module
``controller``: ``mpc_step``, ``run_closed_loop``, ``rmse``) describes it, and
the reference provides its pieces -- ``stage_cost`` (virtualsys.py:279-286),
``tracking_cost`` (baselines.py:268-278) and ``NoiseStreams.child``
(matvar.py:153-154).  This module is that loop with everything resident on the
GPU: per MPC step it re-centres the smoother on the plant state
(``DeviceSmoother.reset``, no reallocation), smooths H steps with the noise
substreams ``NoiseStreams(seed).child(k)``, extracts the control from the mean
trajectory on the device, advances the plant with its device forecast kernel,
and folds rmse and stage cost into device buffers.  The host synchronises once,
when the trace is read.

Semantics (SPEC controller, with the choices the SPEC leaves open stated here):
  * x0 = (plant_state, prev_u, dU0) with dU0 = 0 (cold start, the default) or, with
    ``warm_start``, the previous plan's slice-1 dU -- the only part of the shifted
    previous mean trajectory that a smoother started from identical copies can use.
  * The applied control is the U block of mean slice 1 (slice 0 holds prev_u, which
    no update can move: its anomalies are zero).  ``full_horizon`` applies the U
    blocks of slices 1..H on the next H plant steps and re-plans after them.
  * rmse = ||phi - phi_ref||_F^2 / points (SPEC's printed formula, no square root),
    recorded after every plant step; ``rmse0`` is the initial state's value.
  * stage cost of the applied slice (x_next, u, u - prev_u) under the inverse-weight
    metrics (virtualsys.py:279-286).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from .engine import DeviceSmoother, Forecaster, LocalComm
from .matvar import NoiseStreams, entropy_head
from .virtualsys import AugmentedState, MpcWeights, build_virtual_system

__all__ = ["ControllerConfig", "ClosedLoopTrace", "rmse", "mpc_step", "run_closed_loop",
           "DeviceClosedLoop"]


@dataclass
class ControllerConfig:
    """SPEC ControllerConfig: H, N, weights, optional constraint, apply mode, warm start, seed."""

    horizon_h: int = 5
    ensemble_n: int = 100
    weights: Optional[MpcWeights] = None
    constraint: object = None
    apply_mode: str = "first_action"
    warm_start: bool = False
    seed: int = 0

    def __post_init__(self) -> None:
        if self.horizon_h < 1:
            raise ValueError("horizon_h must be at least 1")
        if self.ensemble_n < 2:
            raise ValueError("ensemble_n must be at least 2")
        if self.apply_mode not in ("first_action", "full_horizon"):
            raise ValueError(f"unknown apply_mode {self.apply_mode!r}")


@dataclass
class ClosedLoopTrace:
    """Per plant step: applied control, rmse, stage cost; per MPC solve: smoother time (s)."""

    controls: np.ndarray
    rmse: np.ndarray
    cost: np.ndarray
    smoother_time: np.ndarray
    rmse0: float = 0.0
    fields: list = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.rmse)


def rmse(fld: np.ndarray, ref: np.ndarray) -> float:
    """||fld - ref||_F^2 / number of entries (SPEC controller.rmse)."""
    fld, ref = np.asarray(fld, float), np.asarray(ref, float)
    if fld.shape != ref.shape:
        raise ValueError(f"shape mismatch {fld.shape} vs {ref.shape}")
    return float(np.sum((fld - ref) ** 2) / fld.size)


def mpc_step(plant_state: np.ndarray, prev_u: np.ndarray, cfg: ControllerConfig, vs, streams):
    """One receding-horizon solve through the drop-in smoother API (SPEC mpc_step).

    Returns (control, mean trajectory (H+1, d, m)); control is the slice-1 U block, or the
    U blocks of slices 1..H (shape (H, l, m)) with apply_mode='full_horizon'."""
    from . import enks

    n, l = vs.n, vs.l
    x0 = AugmentedState(np.asarray(plant_state, float), np.asarray(prev_u, float),
                        np.zeros_like(prev_u, dtype=float))
    traj, _ = enks.smooth_horizon(x0, vs.reference_observation(), vs, cfg.horizon_h,
                                  cfg.ensemble_n, streams)
    u = traj[1:, n:n + l] if cfg.apply_mode == "full_horizon" else traj[1, n:n + l]
    if not np.all(np.isfinite(u)):
        raise FloatingPointError("non-finite control from the smoother")
    return u, traj


class DeviceClosedLoop:
    """Device-resident closed loop: smoother (model) + plant forecast + metrics on one stream."""

    def __init__(self, plant, model, cfg: ControllerConfig, x_init, u_init=None, ops=None,
                 comm=None):
        from .ops import DeviceOps

        if cfg.weights is None:
            raise ValueError("ControllerConfig.weights is required")
        self.cfg = cfg
        self.ops = ops or DeviceOps()
        ops = self.ops
        self.vs = build_virtual_system(model, cfg.weights, cfg.constraint)
        vs = self.vs
        self.n, self.l, self.m = vs.n, vs.l, vs.m
        n, l, m = self.n, self.l, self.m
        if (plant.state_rows, plant.input_rows, plant.state_cols) != (n, l, m):
            raise ValueError("plant and model shapes differ")
        self.d, self.p = n + 2 * l, n + l
        lam = 1.0 / float(np.trace(vs.shared_col_cov))
        x0 = np.vstack([np.asarray(x_init, float), np.zeros((2 * l, m)) if u_init is None else
                        np.vstack([np.asarray(u_init, float), np.zeros((l, m))])])
        self.eng = DeviceSmoother(ops, x0, n, l, cfg.ensemble_n, lam, capacity=cfg.horizon_h,
                                  comm=comm or LocalComm())
        self.eng.bind(vs)
        self.plant_fc = Forecaster(plant, ops, n, l)
        self.yref = ops.to_device(vs.reference_observation())
        self.plant = ops.empty(self.p, m)           # [x; u] fed to the plant forecast
        self.plant[:n] = ops.to_device(np.asarray(x_init, float))
        self.plant[n:] = ops.to_device(np.zeros((l, m)) if u_init is None else
                                       np.asarray(u_init, float))
        self.x0 = ops.zeros(self.d, m)
        self.xnext = ops.empty(n, m)
        self.err = ops.empty(max(n, l), m)
        self.werr = ops.empty(max(n, l), m)
        self.du = ops.empty(l, m)
        self.plan = ops.zeros(cfg.horizon_h, l, m)   # U blocks of the newest plan
        self.plan_du = ops.zeros(l, m)               # slice-1 dU of the newest plan
        w = cfg.weights
        self.x_ref = ops.to_device(w.x_ref)
        self.u_ref = ops.to_device(w.u_ref)
        self.winv = {}
        for key, mat in (("x", w.r), ("u", w.q_u), ("du", w.q_du)):
            mat = np.asarray(mat, float)
            self.winv[key] = None if np.array_equal(mat, np.eye(mat.shape[0])) else \
                ops.to_device(np.linalg.inv(mat))

    # ------------------------------------------------------------ pieces
    def _quad(self, e, key, out, accumulate):
        """out (+)= sum(e * W^-1 e)."""
        winv = self.winv[key]
        if winv is None:
            self.ops.quad_form(e, e, out, accumulate=accumulate)
        else:
            we = self.werr[:e.shape[0]]
            self.ops.gemm(winv, e, we)
            self.ops.quad_form(e, we, out, accumulate=accumulate)

    def _plan(self, k: int, set_head: bool = True) -> None:
        """Smooth H steps from (plant x, prev u, dU0) with streams child(k); keep the U plan."""
        eng, n, l, d, H = self.eng, self.n, self.l, self.d, self.cfg.horizon_h
        if set_head and eng.dev_head is not None:
            eng.dev_head.set(entropy_head(self.cfg.seed, (k,)))
        self.x0[:n + l].copy_(self.plant)
        if self.cfg.warm_start:
            self.x0[n + l:].copy_(self.plan_du)
        else:
            self.x0[n + l:].zero_()
        eng.reset(self.x0)
        streams = NoiseStreams(self.cfg.seed).child(k)
        for _ in range(H):
            eng.predict(self.vs, streams)
            eng.update(self.yref, streams)
        mean = eng.mean[:(H + 1) * d].view(H + 1, d, self.m)
        self.plan.copy_(mean[1:, n:n + l])
        self.plan_du.copy_(mean[1, n + l:])

    def _plant_step(self, u, rm_out, cost_out) -> None:
        ops, n, l = self.ops, self.n, self.l
        ops.sub(u, self.plant[n:], self.du)          # applied dU = u - prev u
        self.plant[n:].copy_(u)
        self.plant_fc(ops, self.plant, self.xnext, n, 1)
        self.plant[:n].copy_(self.xnext)
        ex = self.err[:n]
        ops.sub(self.xnext, self.x_ref, ex)
        ops.quad_form(ex, ex, rm_out, scale=1.0 / ex.numel())
        self._quad(ex, "x", cost_out, False)
        eu = self.err[:l]
        ops.sub(u, self.u_ref, eu)
        self._quad(eu, "u", cost_out, True)
        self._quad(self.du, "du", cost_out, True)

    # ------------------------------------------------------------ CUDA graph of one MPC step
    def _graph_body(self) -> None:
        """plan (smoother with the device-resident noise head) + plant step + metrics into fixed
        buffers; captured once, replayed per control step with the head of child(k)."""
        self._plan(0, set_head=False)
        u = self.plan[0]
        self.ctl_cur.copy_(u)
        self._plant_step(u, self.rm_cur, self.cost_cur)

    def _ensure_graph(self) -> None:
        if getattr(self, "graph", None) is not None:
            return
        from .ops import DeviceHead

        ops = self.ops
        words = entropy_head(self.cfg.seed, (0,))
        self.dev_head = DeviceHead(ops.zeros(32, dtype=torch.int32), len(words))
        self.dev_head.set(words)
        self.eng.dev_head = self.dev_head
        self.ctl_cur = ops.zeros(self.l, self.m)
        self.rm_cur = ops.zeros(1, dtype=torch.float64)
        self.cost_cur = ops.zeros(1, dtype=torch.float64)
        saved = (self.plant.clone(), self.plan.clone(), self.plan_du.clone())
        self._graph_body()  # warm-up (kernel attributes, workspaces); the state is restored
        torch.cuda.synchronize()
        self.plant.copy_(saved[0])
        self.plan.copy_(saved[1])
        self.plan_du.copy_(saved[2])
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._graph_body()

    # ------------------------------------------------------------ run
    def run(self, steps: int, record_every: int = 0, graph: bool | None = None) -> ClosedLoopTrace:
        """``graph`` (default: on a CUDA device with apply_mode='first_action') replays one
        captured MPC step per control step; the noise head of child(k) is rewritten in device
        memory before each replay.  Same kernels and results as the eager loop."""
        ops, n, l, m, H = self.ops, self.n, self.l, self.m, self.cfg.horizon_h
        if graph is None:
            graph = ops.device.type == "cuda" and self.cfg.apply_mode == "first_action"
        if graph:
            if self.cfg.apply_mode != "first_action":
                raise ValueError("graph replay supports apply_mode='first_action' only")
            return self._run_graph(steps, record_every)
        rm = ops.zeros(max(steps, 1), dtype=torch.float64)
        cost = ops.zeros(max(steps, 1), dtype=torch.float64)
        controls = ops.zeros(max(steps, 1), l, m)
        r0 = ops.zeros(1, dtype=torch.float64)
        ex0 = self.err[:n]
        ops.sub(self.plant[:n], self.x_ref, ex0)
        ops.quad_form(ex0, ex0, r0, scale=1.0 / ex0.numel())
        events, fields = [], []
        k = 0   # plan index (noise child id)
        j = H   # position inside the current plan
        for s in range(steps):
            if self.cfg.apply_mode == "first_action" or j >= H:
                timed = ops.device.type == "cuda"
                if timed:
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev1 = torch.cuda.Event(enable_timing=True)
                    ev0.record()
                self._plan(k)
                if timed:
                    ev1.record()
                    events.append((ev0, ev1))
                k += 1
                j = 0
            u = self.plan[j]
            controls[s].copy_(u)
            self._plant_step(u, rm[s:s + 1], cost[s:s + 1])
            j += 1
            if record_every and (s + 1) % record_every == 0:
                fields.append(self.plant[:n].clone())
        self.eng.check_status()
        if self.plant_fc.kind == "burgers":
            self.plant_fc.check_cfl()
        ctl = controls[:steps].double().cpu().numpy()
        if not np.all(np.isfinite(ctl)):
            raise FloatingPointError("non-finite control in the closed loop")
        times = np.array([a.elapsed_time(b) * 1e-3 for a, b in events]) if events else \
            np.zeros(0)
        return ClosedLoopTrace(controls=ctl, rmse=rm[:steps].cpu().numpy(),
                               cost=cost[:steps].cpu().numpy(), smoother_time=times,
                               rmse0=float(r0.item()),
                               fields=[f.double().cpu().numpy() for f in fields])


def _run_graph_impl(self, steps: int, record_every: int) -> ClosedLoopTrace:
    ops, n, l, m = self.ops, self.n, self.l, self.m
    rm = ops.zeros(max(steps, 1), dtype=torch.float64)
    cost = ops.zeros(max(steps, 1), dtype=torch.float64)
    controls = ops.zeros(max(steps, 1), l, m)
    r0 = ops.zeros(1, dtype=torch.float64)
    ex0 = self.err[:n]
    ops.sub(self.plant[:n], self.x_ref, ex0)
    ops.quad_form(ex0, ex0, r0, scale=1.0 / ex0.numel())
    self._ensure_graph()
    # the heads of child(0 .. steps-1), uploaded once; per step a device-to-device copy (async)
    heads = np.zeros((max(steps, 1), 32), dtype=np.uint32)
    for s in range(steps):
        w = entropy_head(self.cfg.seed, (s,))
        if len(w) != self.dev_head.n:
            raise ValueError("noise head length changed across control steps")
        heads[s, :len(w)] = w
    heads_dev = ops.to_device(heads.view(np.int32), dtype=torch.int32)
    events, fields = [], []
    for s in range(steps):
        self.dev_head.words.copy_(heads_dev[s])
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        self.graph.replay()
        ev1.record()
        events.append((ev0, ev1))
        controls[s].copy_(self.ctl_cur)
        rm[s:s + 1].copy_(self.rm_cur)
        cost[s:s + 1].copy_(self.cost_cur)
        if record_every and (s + 1) % record_every == 0:
            fields.append(self.plant[:n].clone())
    self.eng.t = self.cfg.horizon_h
    self.eng.check_status()
    if self.plant_fc.kind == "burgers":
        self.plant_fc.check_cfl()
    ctl = controls[:steps].double().cpu().numpy()
    if not np.all(np.isfinite(ctl)):
        raise FloatingPointError("non-finite control in the closed loop")
    times = np.array([a.elapsed_time(b) * 1e-3 for a, b in events]) if events else np.zeros(0)
    return ClosedLoopTrace(controls=ctl, rmse=rm[:steps].cpu().numpy(),
                           cost=cost[:steps].cpu().numpy(), smoother_time=times,
                           rmse0=float(r0.item()),
                           fields=[f.double().cpu().numpy() for f in fields])


DeviceClosedLoop._run_graph = _run_graph_impl


def run_closed_loop(plant, model, cfg: ControllerConfig, steps: int, x_init, u_init=None,
                    record_every: int = 0) -> ClosedLoopTrace:
    """SPEC run_closed_loop: alternate mpc solves (smoother on `model`) and plant steps."""
    if steps < 0:
        raise ValueError("steps must be >= 0")
    loop = DeviceClosedLoop(plant, model, cfg, x_init, u_init)
    return loop.run(steps, record_every)
