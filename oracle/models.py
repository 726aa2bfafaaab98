"""ORACLE (test infrastructure only) — fp64 dynamics restated in NumPy.

* ``cnn_step``     the CNN surrogate (not in the reference) as an
                   explicit fp64 zero-padded 3x3 cross-correlation stack with tanh
                   between layers and the residual x + alpha * y.  Used to pin the
                   device conv kernel and the product's host ``CNNDynamics.step``.
* ``OracleCNN``    MatrixDynamics wrapper around ``cnn_step`` (plugs into the
                   oracle smoother and into the reference's own smooth_horizon).
* ``linear_step``  reference dynamics.py:53-63.
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


class OracleCNN:
    """fp64 MatrixDynamics for the CNN surrogate, from a CNNDynamics-like spec."""

    def __init__(self, spec):
        self.weights = [np.asarray(w, float) for w in spec.weights]
        self.biases = [np.asarray(b, float) for b in spec.biases]
        self.alpha = float(spec.alpha)
        self.state_rows = spec.state_rows
        self.state_cols = spec.state_cols
        self.input_rows = spec.input_rows

    def step(self, x, u):
        return cnn_step(x, u, self.weights, self.biases, self.alpha)


def linear_step(x, u, a, b):
    return np.asarray(a, float) @ np.asarray(x, float) + np.asarray(b, float) @ np.asarray(u, float)
