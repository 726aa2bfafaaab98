"""The reference's Burgers solver tests (pkg/tests/test_dynamics.py:76-216) on the device kernel.

Each property of the reference's own suite is checked on ``csrc/burgers.cu`` through the
engine's forecast seam (many members per launch, member-column layout), with fp32
tolerances where the reference compares fp64 results exactly.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _forecast(dev_ops, pm, fields, force, **cfg_kw):
    """fields (N, 2g, g), force (N, u_rows, g) -> device forecast (N, 2g, g) and forecaster."""
    from paper_2410_09663_b200.engine import Forecaster

    cfg = pm.dynamics.BurgersConfig(**cfg_kw)
    model = pm.dynamics.BurgersDynamics(cfg)
    g = cfg.grid_n
    N = fields.shape[0]
    if force is None:
        force = np.zeros((N, model.input_rows, g))
    fc = Forecaster(model, dev_ops, 2 * g, model.input_rows)
    last = np.concatenate([fields, force], axis=1).transpose(1, 0, 2).reshape(-1, N * g)
    out = dev_ops.zeros(2 * g, N * g)
    fc(dev_ops, dev_ops.to_device(last), out, 2 * g, N)
    return out.double().cpu().numpy().reshape(2 * g, N, g).transpose(1, 0, 2), fc, model


def test_zero_is_equilibrium(dev_ops, pm):  # test_dynamics.py:79-83
    out, _, _ = _forecast(dev_ops, pm, np.zeros((3, 32, 16)), None, grid_n=16)
    assert not out.any()


def test_uniform_one_is_equilibrium(dev_ops, pm):  # test_dynamics.py:85-91 (50 steps)
    out, _, _ = _forecast(dev_ops, pm, np.ones((2, 32, 16)), None, grid_n=16, substeps=50)
    assert np.allclose(out, 1.0, atol=1e-6)


def test_spike_diffuses_and_matches_substep_refinement(dev_ops, pm):  # 93-110
    n = 16
    phi = np.zeros((1, 2 * n, n))
    phi[0, n // 2, n // 2] = 1.0
    coarse, _, _ = _forecast(dev_ops, pm, phi, None, grid_n=n, nu=0.005, dt=0.001)
    c = n // 2
    assert coarse[0, c, c] < 1.0
    for di, dj in [(-1, 0), (1, 0), (0, -1), (0, 1)]:
        assert coarse[0, c + di, c + dj] > 0.0
    fine, _, _ = _forecast(dev_ops, pm, phi, None, grid_n=n, nu=0.005, dt=0.0001, substeps=10)
    assert np.abs(coarse - fine).max() < 5 * 0.001 * np.abs(fine).max()


def test_row_uniform_profile_matches_1d_upwind(dev_ops, pm):  # 112-129
    n = 16
    cfg = pm.dynamics.BurgersConfig(grid_n=n, nu=1e-12, dt=0.001)
    profile = np.random.default_rng(5).uniform(-0.5, 0.5, size=n)
    phi = np.zeros((1, 2 * n, n))
    phi[0, :n] = np.tile(profile, (n, 1))
    out, _, _ = _forecast(dev_ops, pm, phi, None, grid_n=n, nu=1e-12, dt=0.001)
    dx = cfg.dx
    left = np.concatenate([[profile[0]], profile[:-1]])
    right = np.concatenate([profile[1:], [profile[-1]]])
    lap1d = (left + right - 2 * profile) / dx ** 2
    ddx = np.where(profile > 0, profile - left, right - profile) / dx
    expect = profile + cfg.dt * (cfg.nu * lap1d - profile * ddx)
    for i in range(n):
        np.testing.assert_allclose(out[0, i], expect, rtol=0, atol=1e-6)


def test_grid_refinement_first_order(dev_ops, pm):  # 131-139
    n = 16
    f0 = pm.dynamics.make_initial_field(pm.dynamics.BurgersConfig(grid_n=n), 3).packed[None]
    one, _, _ = _forecast(dev_ops, pm, f0, None, grid_n=n, dt=0.002)
    two, _, _ = _forecast(dev_ops, pm, f0, None, grid_n=n, dt=0.001, substeps=2)
    assert np.abs(one - two).max() < 10 * 0.002


def test_boundary_force_hits_y1_row_only(dev_ops, pm):  # 141-149
    n = 16
    force = np.vstack([np.ones(n), 2 * np.ones(n)])[None]
    out, _, _ = _forecast(dev_ops, pm, np.zeros((1, 2 * n, n)), force, grid_n=n)
    assert np.allclose(out[0, n - 1], 0.001)
    assert np.allclose(out[0, 2 * n - 1], 0.002)
    assert not out[0, :n - 1].any() and not out[0, n:2 * n - 1].any()


def test_pointwise_force_adds_source(dev_ops, pm):  # 151-157
    n = 16
    force = np.random.default_rng(6).standard_normal((2, 2 * n, n))
    out, _, _ = _forecast(dev_ops, pm, np.zeros((2, 2 * n, n)), force, grid_n=n,
                          control_mode="pointwise")
    np.testing.assert_allclose(out, 0.001 * force, rtol=1e-6, atol=1e-9)


def test_cfl_violation_raises(dev_ops, pm):  # 159-164 (diffusion) + advection limit
    from paper_2410_09663_b200.dynamics import CflError

    with pytest.raises(CflError, match="nu"):
        _forecast(dev_ops, pm, np.ones((1, 32, 16)), None, grid_n=16, nu=0.005, dt=0.5)
    _, fc, _ = _forecast(dev_ops, pm, 20.0 * np.ones((2, 32, 16)), None, grid_n=16, dt=0.01)
    with pytest.raises(CflError, match="max"):
        fc.check_cfl()


def test_nonfinite_field_raises(dev_ops, pm):  # 166-171
    from paper_2410_09663_b200.dynamics import CflError

    bad = np.zeros((2, 32, 16))
    bad[1, 0, 0] = np.inf
    _, fc, _ = _forecast(dev_ops, pm, bad, None, grid_n=16)
    with pytest.raises(CflError, match="non-finite"):
        fc.check_cfl()


def test_diagnostics_recorded(dev_ops, pm):  # 173-181
    n = 16
    f = np.zeros((1, 2 * n, n))
    f[0, :n] = 1.0
    _, fc, model = _forecast(dev_ops, pm, f, None, grid_n=n)
    assert fc.advection_number == pytest.approx(model.cfg.dt / model.cfg.dx, rel=1e-6)
    assert fc.nu * fc.dt / fc.dx ** 2 == pytest.approx(model.cfg.diffusion_number)


def test_adapter_batches_and_substeps(dev_ops, pm):  # 183-197
    from oracle.models import burgers_step

    cfg = pm.dynamics.BurgersConfig(grid_n=12, substeps=3)
    f0 = pm.dynamics.make_initial_field(cfg, 1).packed
    batch = np.stack([f0, 0.5 * f0])
    u = np.zeros((2, 2, 12))
    out, _, _ = _forecast(dev_ops, pm, batch, u, grid_n=12, substeps=3)
    ref = burgers_step(batch, u, 12, cfg.nu, cfg.dt, "boundary", 3)[0]
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-6)
