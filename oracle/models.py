"""ORACLE (test infrastructure only) — fp64 dynamics restated in NumPy.

* ``cnn_step``     the CNN surrogate (not in the reference) as an
                   explicit fp64 zero-padded 3x3 cross-correlation stack with tanh
                   between layers and the residual x + alpha * y.  Used to pin the
                   device conv kernel and the product's host ``CNNDynamics.step``.
* ``OracleCNN``    MatrixDynamics wrapper around ``cnn_step`` (plugs into the
                   oracle smoother and into the reference's own smooth_horizon).
* ``linear_step``  reference dynamics.py:53-63.
* ``burgers_step`` reference dynamics.py:156-216 (_neighbor_slices, _cfl_check,
                   _step_packed), restated with explicit padded-array shifts; one
                   call = ``substeps`` solver steps (BurgersDynamics.step 264-270).
                   Pinned bit-for-bit against the reference (tests/golden/burgers_*.npz).
* ``OracleBurgers`` MatrixDynamics wrapper around ``burgers_step``.
"""
from __future__ import annotations

import numpy as np


def _conv3x3_same(h: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """h (B, Cin, H, W), w (Cout, Cin, 3, 3), b (Cout,) -> (B, Cout, H, W); zero padding 1."""
    B, cin, H, W = h.shape
    hp = np.zeros((B, cin, H + 2, W + 2))
    hp[:, :, 1:-1, 1:-1] = h
    out = np.broadcast_to(b[None, :, None, None], (B, w.shape[0], H, W)).copy()
    for ky in range(3):
        for kx in range(3):
            patch = hp[:, :, ky:ky + H, kx:kx + W]          # (B, Cin, H, W)
            out += np.einsum("oc,bchw->bohw", w[:, :, ky, kx], patch, optimize=True)
    return out


def cnn_step(x: np.ndarray, u: np.ndarray, weights, biases, alpha: float) -> np.ndarray:
    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    lead = np.broadcast_shapes(x.shape[:-2], u.shape[:-2])
    H, W = x.shape[-2:]
    xb = np.broadcast_to(x, lead + (H, W)).reshape(-1, H, W)
    ub = np.broadcast_to(u, lead + (H, W)).reshape(-1, H, W)
    h = np.stack([xb, ub], axis=1)
    L = len(weights)
    for k, (w, b) in enumerate(zip(weights, biases)):
        h = _conv3x3_same(h, np.asarray(w, float), np.asarray(b, float))
        if k < L - 1:
            h = np.tanh(h)
    return (xb + alpha * h[:, 0]).reshape(lead + (H, W))


def cnn_step_torch(x: np.ndarray, u: np.ndarray, weights, biases, alpha: float,
                   chunk: int = 64) -> np.ndarray:
    """The same fp64 stack as ``cnn_step`` through torch-CPU conv2d, in member chunks (bounded
    memory), for oracle runs at the benchmarked sizes (C2/C3/C5: 10^2..10^4 members of
    64x64..128x128).  Pinned to ``cnn_step`` at 1e-12 by tests/test_oracle_golden.py."""
    import torch
    import torch.nn.functional as F

    x = np.asarray(x, dtype=float)
    u = np.asarray(u, dtype=float)
    lead = np.broadcast_shapes(x.shape[:-2], u.shape[:-2])
    H, W = x.shape[-2:]
    xb = np.broadcast_to(x, lead + (H, W)).reshape(-1, H, W)
    ub = np.broadcast_to(u, lead + (H, W)).reshape(-1, H, W)
    ws = [torch.from_numpy(np.asarray(w, float)) for w in weights]
    bs = [torch.from_numpy(np.asarray(b, float)) for b in biases]
    out = np.empty_like(xb)
    for i0 in range(0, xb.shape[0], chunk):
        h = torch.from_numpy(np.stack([xb[i0:i0 + chunk], ub[i0:i0 + chunk]], axis=1))
        for k, (w, b) in enumerate(zip(ws, bs)):
            h = F.conv2d(h, w, b, padding=1)
            if k < len(ws) - 1:
                h = torch.tanh(h)
        out[i0:i0 + chunk] = xb[i0:i0 + chunk] + alpha * h[:, 0].numpy()
    return out.reshape(lead + (H, W))


def cnn_init(widths, seed: int = 0):
    """The CNN surrogate's seeded random init (w ~ N(0,1)/sqrt(9 C_in), bias ~
    0.01 N(0,1), numpy default_rng(seed), layer by layer), restated so the reference arm builds
    its model without the product package.  Equal to dynamics.CNNDynamics's init (test)."""
    rng = np.random.default_rng(seed)
    weights, biases = [], []
    for cin, cout in zip(widths[:-1], widths[1:]):
        weights.append(rng.standard_normal((cout, cin, 3, 3)) / np.sqrt(9.0 * cin))
        biases.append(0.01 * rng.standard_normal(cout))
    return weights, biases


class CnnSpec:
    """Minimal CNNDynamics-like spec (weights, biases, alpha, shapes) for OracleCNN."""

    def __init__(self, rows, cols, widths, alpha=0.1, seed=0):
        self.widths = tuple(widths)
        self.weights, self.biases = cnn_init(self.widths, seed)
        self.alpha = float(alpha)
        self.state_rows = self.input_rows = int(rows)
        self.state_cols = int(cols)

    def flops_per_member_step(self) -> int:
        return self.state_rows * self.state_cols * sum(
            18 * ci * co for ci, co in zip(self.widths[:-1], self.widths[1:]))


class OracleCNN:
    """fp64 MatrixDynamics for the CNN surrogate, from a CNNDynamics-like spec.

    backend "numpy": explicit einsum taps (``cnn_step``); "torch": torch-CPU fp64 conv2d
    (``cnn_step_torch``), for the large configurations."""

    def __init__(self, spec, backend: str = "numpy"):
        self.weights = [np.asarray(w, float) for w in spec.weights]
        self.biases = [np.asarray(b, float) for b in spec.biases]
        self.alpha = float(spec.alpha)
        self.state_rows = spec.state_rows
        self.state_cols = spec.state_cols
        self.input_rows = spec.input_rows
        self.backend = backend

    def step(self, x, u):
        if self.backend == "torch":
            return cnn_step_torch(x, u, self.weights, self.biases, self.alpha)
        return cnn_step(x, u, self.weights, self.biases, self.alpha)


def linear_step(x, u, a, b):
    return np.asarray(a, float) @ np.asarray(x, float) + np.asarray(b, float) @ np.asarray(u, float)


class OracleCflError(RuntimeError):
    pass


def burgers_step(packed, force, grid_n: int, nu: float, dt: float, mode: str = "boundary",
                 substeps: int = 1):
    """fp64 Burgers forecast on (..., 2g, g) packed fields (dynamics.py:183-216, 264-270).

    Edge-copy ghost cells (dynamics.py:156-165): pad by one with the edge value, read the
    four shifted interior windows.  Returns (out, max|phi| over every substep input)."""
    g = grid_n
    dx = 1.0 / (g - 1)
    out = np.asarray(packed, dtype=float)
    vmax_all = 0.0
    for _ in range(substeps):
        vx, vy = out[..., :g, :], out[..., g:, :]
        vmax = max(float(np.max(np.abs(vx))), float(np.max(np.abs(vy))))
        if not np.isfinite(vmax):
            raise OracleCflError("non-finite field")
        if nu * dt / dx ** 2 > 0.25 or vmax * dt / dx > 1.0:
            raise OracleCflError("CFL violated")
        vmax_all = max(vmax_all, vmax)
        new = []
        for q in (vx, vy):
            pad = [(0, 0)] * (q.ndim - 2) + [(1, 1), (1, 1)]
            qp = np.pad(q, pad, mode="edge")
            up, down = qp[..., :-2, 1:-1], qp[..., 2:, 1:-1]
            left, right = qp[..., 1:-1, :-2], qp[..., 1:-1, 2:]
            lap = (up + down + left + right - 4.0 * q) / dx ** 2
            ddx = np.where(vx > 0, q - left, right - q) / dx
            ddy = np.where(vy > 0, q - up, down - q) / dx
            new.append(q + dt * (nu * lap - vx * ddx - vy * ddy))
        out = np.concatenate(new, axis=-2)
        if force is not None:
            f = np.asarray(force, dtype=float)
            if mode == "pointwise":
                out = out + dt * f
            else:
                out[..., g - 1, :] += dt * f[..., 0, :]
                out[..., 2 * g - 1, :] += dt * f[..., 1, :]
    return out, vmax_all


class OracleBurgers:
    """fp64 MatrixDynamics for the Burgers model, from a BurgersDynamics-like spec."""

    def __init__(self, spec):
        cfg = spec.cfg
        self.g, self.nu, self.dt = int(cfg.grid_n), float(cfg.nu), float(cfg.dt)
        self.mode, self.substeps = cfg.control_mode, int(cfg.substeps)
        self.state_rows = spec.state_rows
        self.state_cols = spec.state_cols
        self.input_rows = spec.input_rows

    def step(self, x, u):
        return burgers_step(x, u, self.g, self.nu, self.dt, self.mode, self.substeps)[0]
