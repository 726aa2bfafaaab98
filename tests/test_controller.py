"""Closed-loop driver: device loop vs the fp64 oracle loop.

CPU: the product's DeviceClosedLoop orchestration on the fp64 CPU operator set
(tests/cpu_ops.py) must equal the oracle closed loop to rounding.  GPU: the same
loop on the B200 matches the oracle within the north_star tolerance (1e-4
relative on controls and on the closed-loop cost).
"""
import numpy as np
import pytest

from cpu_ops import CpuOps
from oracle import problems
from oracle.closed_loop import oracle_closed_loop
from oracle.models import OracleBurgers, linear_step


def _linear(pm, seed=3):
    model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(seed), n=4, l=2, m=3)
    return model, vs, x0


def _cfg(pm, vs, **kw):
    from paper_2410_09663_b200.controller import ControllerConfig

    return ControllerConfig(weights=vs.weights, **kw)


def test_rmse_formula():
    from paper_2410_09663_b200.controller import rmse

    assert rmse(np.ones((3, 3)), np.ones((3, 3))) == 0.0
    assert rmse(np.zeros((4, 5)), np.ones((4, 5))) == 1.0
    assert rmse(np.array([[1.0, 0.0], [0.0, 1.0]]), np.zeros((2, 2))) == 0.5
    with pytest.raises(ValueError):
        rmse(np.zeros((2, 2)), np.zeros((2, 3)))


def test_config_validation(pm):
    from paper_2410_09663_b200.controller import ControllerConfig

    with pytest.raises(ValueError):
        ControllerConfig(horizon_h=0)
    with pytest.raises(ValueError):
        ControllerConfig(ensemble_n=1)
    with pytest.raises(ValueError):
        ControllerConfig(apply_mode="all")


@pytest.mark.parametrize("mode,warm", [("first_action", False), ("full_horizon", False),
                                       ("first_action", True)])
def test_closed_loop_linear_cpu_equals_oracle(pm, mode, warm):
    from paper_2410_09663_b200.controller import DeviceClosedLoop

    model, vs, x0 = _linear(pm)
    cfg = _cfg(pm, vs, horizon_h=3, ensemble_n=12, apply_mode=mode, warm_start=warm, seed=5)
    loop = DeviceClosedLoop(model, model, cfg, x0.x, ops=CpuOps())
    tr = loop.run(7)
    ctl, rm, cost = oracle_closed_loop(lambda x, u: linear_step(x, u, model.a, model.b), vs, x0.x,
                                       3, 12, 5, 7, apply_mode=mode, warm_start=warm)
    assert len(tr) == 7 and tr.controls.shape == ctl.shape
    np.testing.assert_allclose(tr.controls, ctl, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(tr.rmse, rm, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(tr.cost, cost, rtol=1e-9, atol=1e-12)


def test_closed_loop_burgers_cpu_equals_oracle(pm):
    from paper_2410_09663_b200.controller import DeviceClosedLoop

    pr = problems.make_burgers_problem(pm, "boundary", grid_n=8, n_members=10, horizon=2)
    cfg = _cfg(pm, pr.vs, horizon_h=2, ensemble_n=10, seed=1)
    loop = DeviceClosedLoop(pr.model, pr.model, cfg, pr.x0.x, ops=CpuOps())
    tr = loop.run(4, record_every=2)
    ob = OracleBurgers(pr.model)
    ctl, rm, cost = oracle_closed_loop(ob.step, pr.vs, pr.x0.x, 2, 10, 1, 4)
    np.testing.assert_allclose(tr.controls, ctl, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(tr.cost, cost, rtol=1e-9)
    assert len(tr.fields) == 2 and tr.fields[0].shape == pr.x0.x.shape


def test_zero_steps_empty_trace(pm):
    from paper_2410_09663_b200.controller import DeviceClosedLoop

    model, vs, x0 = _linear(pm)
    tr = DeviceClosedLoop(model, model, _cfg(pm, vs), x0.x, ops=CpuOps()).run(0)
    assert len(tr) == 0 and tr.controls.shape[0] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["first_action", "full_horizon"])
def test_closed_loop_burgers_gpu_matches_oracle(pm, mode):
    """C1a Burgers boundary control, H=5, N=100: 6 plant steps on the B200 vs fp64 oracle."""
    from paper_2410_09663_b200.controller import run_closed_loop

    pr = problems.make_burgers_problem(pm, "boundary")
    cfg = _cfg(pm, pr.vs, horizon_h=5, ensemble_n=100, apply_mode=mode, seed=3)
    tr = run_closed_loop(pr.model, pr.model, cfg, 6, pr.x0.x)
    ctl, rm, cost = oracle_closed_loop(OracleBurgers(pr.model).step, pr.vs, pr.x0.x, 5, 100, 3, 6,
                                       apply_mode=mode)
    rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())  # noqa: E731
    assert rel(tr.controls, ctl) < 1e-4
    assert rel(tr.cost, cost) < 1e-4
    assert rel(tr.rmse, rm) < 1e-4
    assert tr.smoother_time.shape == ((6,) if mode == "first_action" else (2,))


@pytest.mark.gpu
def test_mpc_step_host_api_and_determinism(pm):
    from paper_2410_09663_b200.controller import mpc_step
    from oracle.enks_oracle import oracle_smooth

    model, vs, x0 = _linear(pm, 8)
    cfg = _cfg(pm, vs, horizon_h=4, ensemble_n=32)
    st = pm.matvar.NoiseStreams(seed=2).child(0)
    u1, traj = mpc_step(x0.x, x0.u, cfg, vs, st)
    u2, _ = mpc_step(x0.x, x0.u, cfg, vs, st)
    assert np.array_equal(u1, u2)
    ref, _, _ = oracle_smooth(x0.__class__(x0.x, x0.u, np.zeros_like(x0.u)), vs.reference_observation(),
                              vs, 4, 32, seed=2, prefix=(0,), backend="c")
    assert np.abs(traj - ref).max() < 1e-4 * np.abs(ref).max()
    assert np.abs(u1 - ref[1, 4:6]).max() < 1e-4 * np.abs(ref).max()


@pytest.mark.gpu
def test_closed_loop_graph_replay_equals_eager(pm):
    """One captured MPC step replayed per control step (device-resident noise head of
    child(k)) gives exactly the eager loop's trace."""
    from paper_2410_09663_b200.controller import DeviceClosedLoop

    pr = problems.make_burgers_problem(pm, "boundary")
    cfg = _cfg(pm, pr.vs, horizon_h=5, ensemble_n=100, seed=4)
    eager = DeviceClosedLoop(pr.model, pr.model, cfg, pr.x0.x).run(8, graph=False)
    g = DeviceClosedLoop(pr.model, pr.model, cfg, pr.x0.x).run(8, graph=True)
    assert np.array_equal(g.controls, eager.controls)
    assert np.array_equal(g.rmse, eager.rmse) and np.array_equal(g.cost, eager.cost)
