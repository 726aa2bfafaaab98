"""Synthetic problem builders for the benchmark configurations and the tests.

Input construction only (host NumPy, outside every timed region); nothing here computes on
the smoother path.

``make_linear_setup`` mirrors the reference test fixture make_setup
(pkg/tests/test_enks.py:19-43): random stable linear dynamics, random SPD (or
identity) weights, random references and x0, drawn from
``np.random.default_rng(seed)`` in the same order, so the same seed gives the
same problem as the reference tests.

``make_cnn_problem`` builds the bench configurations: single-channel field
X (n x m), pointwise control U (l = n), identity weights, scale 1,
x_ref = 1, u_ref = 0, x0 = 4-mode smooth sine field with seeded amplitudes
(as reference dynamics.py:227-243, one channel), CNN widths per config.

Both take the module providing the host types (``paper_2410_09663_b200`` or the
reference ``enksmpc``) so the same problem can be handed to either side.
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np

CONFIGS = {
    # name: (n = m = l, N, H, widths)
    "C1": (32, 100, 5, (2, 16, 16, 1)),
    "C2": (64, 512, 20, (2, 32, 32, 1)),
    "C3": (128, 1024, 50, (2, 32, 32, 1)),
    # C4: 256 x 256 control field, deep CNN (SURVEY.md §8d proposal: 6 layers), N = 4096, H = 20
    "C4": (256, 4096, 20, (2, 32, 32, 32, 32, 32, 1)),
    "C5": (128, 16384, 10, (2, 32, 32, 1)),
}


def _spd(rng, k):
    a = rng.standard_normal((k, k))
    return a @ a.T + k * np.eye(k)


def make_linear_setup(mods, rng, n=4, l=2, m=3, scale=1.0, stable=0.9, identity_weights=False):
    """Same draws, same order as reference pkg/tests/test_enks.py:24-43."""
    a = rng.standard_normal((n, n))
    a *= stable / np.abs(np.linalg.eigvals(a)).max()
    b = rng.standard_normal((n, l))
    model = mods.dynamics.LinearDynamics(a, b, state_cols=m)
    if identity_weights:
        r, q_u, q_du = np.eye(n), np.eye(l), np.eye(l)
    else:
        r, q_u, q_du = _spd(rng, n), _spd(rng, l), _spd(rng, l)
    weights = mods.virtualsys.MpcWeights(r=r, q_u=q_u, q_du=q_du,
                                         x_ref=rng.standard_normal((n, m)),
                                         u_ref=rng.standard_normal((l, m)), scale=scale)
    vs = mods.virtualsys.build_virtual_system(model, weights)
    x0 = mods.virtualsys.AugmentedState(rng.standard_normal((n, m)), rng.standard_normal((l, m)),
                                        np.zeros((l, m)))
    return model, vs, x0


def sine_field(n: int, m: int, seed: int) -> np.ndarray:
    """One channel of reference make_initial_field (dynamics.py:227-243) on an n x m grid."""
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.linspace(0.0, 1.0, n), np.linspace(0.0, 1.0, m), indexing="ij")
    amps = rng.uniform(-0.5, 0.5, size=4)
    q = np.zeros((n, m))
    for a, (kx, ky) in zip(amps, [(1, 1), (1, 2), (2, 1), (2, 2)]):
        q += a * np.sin(np.pi * kx * xx) * np.sin(np.pi * ky * yy)
    return q


def make_cnn_problem(mods, config: str = "C1", seed: int = 0, size=None, n_members=None,
                     horizon=None, widths=None, model=None):
    n, N, H, w = CONFIGS[config]
    n = size or n
    N = n_members or N
    H = horizon or H
    w = widths or w
    m = l = n
    if model is None:
        model = mods.dynamics.CNNDynamics(rows=n, cols=m, widths=w, alpha=0.1, seed=0)
    weights = mods.virtualsys.MpcWeights(r=np.eye(n), q_u=np.eye(l), q_du=np.eye(l),
                                         x_ref=np.ones((n, m)), u_ref=np.zeros((l, m)), scale=1.0)
    vs = mods.virtualsys.build_virtual_system(model, weights)
    x0 = mods.virtualsys.AugmentedState(sine_field(n, m, seed), np.zeros((l, m)), np.zeros((l, m)))
    return SimpleNamespace(model=model, vs=vs, x0=x0, n=n, l=l, m=m, N=N, H=H, widths=tuple(w),
                           y_ref=vs.reference_observation())


def make_burgers_problem(mods, mode: str = "boundary", grid_n: int = 32, n_members: int = 100,
                         horizon: int = 5, seed: int = 0, substeps: int = 1, model=None):
    """C1a: reference Burgers FD, grid 32 -> X 64 x 32, boundary (l = 2) or
    pointwise (l = 64) control, N = 100, H = 5, x0 = make_initial_field(cfg, seed), u0 = dU0 = 0,
    identity weights, x_ref = 1, u_ref = 0."""
    cfg = mods.dynamics.BurgersConfig(grid_n=grid_n, control_mode=mode, substeps=substeps)
    if model is None:
        model = mods.dynamics.BurgersDynamics(cfg)
    n, m, l = 2 * grid_n, grid_n, model.input_rows
    weights = mods.virtualsys.MpcWeights(r=np.eye(n), q_u=np.eye(l), q_du=np.eye(l),
                                         x_ref=np.ones((n, m)), u_ref=np.zeros((l, m)), scale=1.0)
    vs = mods.virtualsys.build_virtual_system(model, weights)
    x = mods.dynamics.make_initial_field(cfg, seed).packed
    x0 = mods.virtualsys.AugmentedState(x, np.zeros((l, m)), np.zeros((l, m)))
    return SimpleNamespace(model=model, vs=vs, x0=x0, n=n, l=l, m=m, N=n_members, H=horizon,
                           cfg=cfg, y_ref=vs.reference_observation())


def make_constraint(mods, kind: str, n: int, l: int, m: int):
    """ConstraintSpec with a device-expressible g (product virtualsys Linear/BoxConstraint),
    built from the given module's ConstraintSpec so it plugs into either side."""
    from paper_2410_09663_b200.virtualsys import BoxConstraint, LinearConstraint

    if kind == "linear":
        g = LinearConstraint(cu=0.3 * np.ones((l, m)), cx=0.05 * np.ones((n, m)), c0=-0.5)
    elif kind == "box":
        g = BoxConstraint(1.0, "u")
    else:
        raise ValueError(kind)
    return mods.virtualsys.ConstraintSpec(g=g, alpha=10.0, beta=5.0, noise_var=1e-2)
