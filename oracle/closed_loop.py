"""ORACLE (test infrastructure only) — fp64 closed-loop receding-horizon driver.

Restates the SPEC controller (the reference does not ship it) on top
of the fp64 oracle smoother (oracle/enks_oracle.py, = reference enks.py:256-284) with
the same semantics as paper_2410_09663_b200/controller.py: per plan k the smoother runs
from (plant x, prev u, dU0) with NoiseStreams(seed).child(k) (matvar.py:153-154), the
applied control is the U block of mean slice 1 (or slices 1..H for full_horizon), the
plant is stepped in fp64, rmse = ||x - x_ref||_F^2 / points and the stage cost follows
virtualsys.py:279-286.
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from .enks_oracle import oracle_smooth


def _stage_cost(x, u, du, w) -> float:
    ex, eu = x - w.x_ref, u - w.u_ref
    return float(np.sum(ex * np.linalg.solve(w.r, ex)) + np.sum(eu * np.linalg.solve(w.q_u, eu))
                 + np.sum(du * np.linalg.solve(w.q_du, du)))


def oracle_closed_loop(plant_step, vs, x_init, H: int, N: int, seed: int, steps: int,
                       u_init=None, apply_mode: str = "first_action", warm_start: bool = False):
    n, l, m = vs.n, vs.l, vs.m
    w = vs.weights
    x = np.asarray(x_init, float)
    u = np.zeros((l, m)) if u_init is None else np.asarray(u_init, float)
    du0 = np.zeros((l, m))
    y = vs.reference_observation()
    controls, rm, cost = [], [], []
    plan, j, k = None, H, 0
    for _ in range(steps):
        if apply_mode == "first_action" or j >= H:
            x0 = SimpleNamespace(packed=np.vstack([x, u, du0 if warm_start else np.zeros((l, m))]),
                                 n=n, l=l, m=m)
            mean, _, _ = oracle_smooth(x0, y, vs, H, N, seed=seed, prefix=(k,), backend="c")
            plan = mean[1:, n:n + l].copy()
            du0 = mean[1, n + l:].copy()
            k += 1
            j = 0
        u_new = plan[j]
        du = u_new - u
        x = plant_step(x, u_new)
        u = u_new
        controls.append(u_new)
        rm.append(float(np.sum((x - w.x_ref) ** 2) / x.size))
        cost.append(_stage_cost(x, u_new, du, w))
        j += 1
    return np.array(controls), np.array(rm), np.array(cost)
