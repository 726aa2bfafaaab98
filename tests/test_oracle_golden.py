"""The oracle restatement reproduces the reference's own outputs (golden fixtures).

Fixtures come from the unmodified reference run in the build container
(tests/golden/make_golden.py); this check runs anywhere, without /root/reference.
"""
import os

import numpy as np
import pytest

from oracle import enks_oracle, noise, problems
from oracle.models import OracleCNN

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def _case(pm, name):
    from golden.make_golden import LINEAR_CASES

    for cname, kw, seed, N, h, sseed, extra in LINEAR_CASES:
        if cname == name:
            model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(seed), **kw)
            if "col_cov" in extra:
                vs = pm.virtualsys.build_virtual_system(
                    model, vs.weights, shared_col_cov=extra["col_cov"] * np.eye(x0.m))
            if "constraint" in extra:
                con = problems.make_constraint(pm, extra["constraint"], x0.n, x0.l, x0.m)
                vs = pm.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
            return model, vs, x0, N, h, sseed, extra
    raise KeyError(name)


NAMES = ["lin_spd_4x2x3", "lin_id_8x4x8", "lin_m1", "lin_scale0_N4", "lin_trackcov", "lin_colcov7",
         "lin_yref_stack", "lin_con_linear", "lin_con_box"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("backend", ["numpy", "c"])
def test_oracle_matches_reference_golden(pm, name, backend):
    gold = _load(name)
    model, vs, x0, N, h, sseed, extra = _case(pm, name)
    assert np.array_equal(x0.packed, gold["x0"])  # same problem as the reference run
    out, cov, _ = enks_oracle.oracle_smooth(x0, gold["y"], vs, h, N, seed=sseed,
                                            track_cov=bool(extra.get("track_cov")),
                                            backend=backend)
    np.testing.assert_allclose(out, gold["mean"], rtol=1e-12, atol=1e-12)
    if extra.get("track_cov"):
        for k in ("sigma_traj", "sigma_pred", "sigma_cross"):
            np.testing.assert_allclose(getattr(cov, k), gold[k], rtol=1e-12, atol=1e-12)


def test_oracle_cnn_matches_reference_golden(pm):
    gold = _load("cnn_c1_16")
    pr = problems.make_cnn_problem(pm, "C1", size=16, n_members=24, horizon=3)
    assert np.array_equal(pr.x0.packed, gold["x0"])
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model), pr.vs.weights)
    out, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=1, backend="c")
    np.testing.assert_allclose(out, gold["mean"], rtol=1e-12, atol=1e-12)


def test_c_noise_matches_reference_golden():
    from golden.make_golden import NOISE_CASES

    gold = _load("noise")
    for k, (seed, prefix, ids, shape) in enumerate(NOISE_CASES):
        z = noise.c_standard_normal(seed, tuple(prefix) + tuple(ids), int(np.prod(shape)))
        assert np.array_equal(z.reshape(shape), gold[f"z{k}"])


def test_oracle_burgers_step_matches_reference_golden():
    from golden.make_golden import BURGERS_STEP_CASES
    from oracle.models import burgers_step

    gold = _load("burgers_steps")
    for k, (g, mode, sub) in enumerate(BURGERS_STEP_CASES):
        y, _ = burgers_step(gold[f"x{k}"], gold[f"u{k}"], g, 0.005, 0.001, mode, sub)
        assert np.array_equal(y, gold[f"y{k}"]), (g, mode, sub)


def test_product_host_burgers_step_matches_reference_golden(pm):
    from golden.make_golden import BURGERS_STEP_CASES

    gold = _load("burgers_steps")
    for k, (g, mode, sub) in enumerate(BURGERS_STEP_CASES):
        model = pm.dynamics.BurgersDynamics(pm.dynamics.BurgersConfig(grid_n=g, control_mode=mode,
                                                                      substeps=sub))
        assert np.array_equal(model.step(gold[f"x{k}"], gold[f"u{k}"]), gold[f"y{k}"])


@pytest.mark.parametrize("mode", ["boundary", "pointwise"])
def test_oracle_burgers_horizon_matches_reference_golden(pm, mode):
    from oracle.models import OracleBurgers

    gold = _load(f"burgers_c1a_{mode}")
    pr = problems.make_burgers_problem(pm, mode)
    assert np.array_equal(pr.x0.packed, gold["x0"])
    ovs = pm.virtualsys.build_virtual_system(OracleBurgers(pr.model), pr.vs.weights)
    out, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=2, backend="c")
    np.testing.assert_allclose(out, gold["mean"], rtol=1e-12, atol=1e-12)


def test_oracle_cnn_torch_backend_matches_einsum(pm):
    """The torch-CPU fp64 conv backend (used for oracle runs at C2/C3/C5 sizes) equals the
    explicit-tap restatement, including member chunking."""
    from oracle.models import cnn_step, cnn_step_torch

    pr = problems.make_cnn_problem(pm, "C1", size=24, widths=(2, 32, 32, 1))
    rng = np.random.default_rng(3)
    x = rng.standard_normal((70, 24, 24))
    u = rng.standard_normal((70, 24, 24))
    ref = cnn_step(x, u, pr.model.weights, pr.model.biases, pr.model.alpha)
    got = cnn_step_torch(x, u, pr.model.weights, pr.model.biases, pr.model.alpha, chunk=16)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    gold = _load("cnn_c1_16")
    pr = problems.make_cnn_problem(pm, "C1", size=16, n_members=24, horizon=3)
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model, backend="torch"), pr.vs.weights)
    out, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=1, backend="c")
    np.testing.assert_allclose(out, gold["mean"], rtol=1e-12, atol=1e-12)


def test_oracle_cnn_init_equals_product_init(pm):
    from oracle.models import CnnSpec

    prod = pm.dynamics.CNNDynamics(rows=8, cols=8, widths=(2, 32, 32, 1), alpha=0.1, seed=0)
    spec = CnnSpec(8, 8, (2, 32, 32, 1))
    for a, b in zip(prod.weights + prod.biases, spec.weights + spec.biases):
        assert np.array_equal(a, b)
    assert spec.flops_per_member_step() == prod.flops_per_member_step()
