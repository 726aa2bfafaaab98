"""The reference's own smoother tests (pkg/tests/test_enks.py) run against the B200 path.

Each test mirrors the reference test of the same name (file:line cited); the
arithmetic is fp32 on device, so 1e-12 / array_equal bounds on fp64 values
become fp32 bounds, while determinism stays bitwise.
"""
import os

import numpy as np
import pytest

from oracle import problems

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F32 = 2e-6  # relative fp32 tolerance for consistency checks


def setup(pm, seed, **kw):
    return problems.make_linear_setup(pm, np.random.default_rng(seed), **kw)


def assert_mean_consistent(ens):
    mem = ens.members
    assert np.abs(ens.mean - mem.mean(axis=0)).max() < F32 * max(1.0, np.abs(mem).max())


def test_identical_copies(pm):  # test_enks.py:51-58
    from paper_2410_09663_b200 import enks

    _, _, x0 = setup(pm, 0)
    ens = enks.init_ensemble(x0, 3)
    assert ens.members.shape == (3, 8, 3)
    for i in range(3):
        assert np.allclose(ens.members[i], x0.packed, atol=1e-6)
    assert_mean_consistent(ens)


def test_lambda_is_inverse_column_count(pm):  # test_enks.py:60-63
    from paper_2410_09663_b200 import enks

    _, _, x0 = setup(pm, 1, m=3)
    assert enks.init_ensemble(x0, 4).lam == pytest.approx(1.0 / 3.0)


def test_zero_noise_keeps_members_identical(pm):  # test_enks.py:73-82
    from paper_2410_09663_b200 import enks

    model, vs, x0 = setup(pm, 3, scale=0.0)
    ens = enks.init_ensemble(x0, 5)
    enks.predict(ens, vs, pm.matvar.NoiseStreams(seed=0))
    expected = np.vstack([model.step(x0.x, x0.u), x0.u, np.zeros_like(x0.u)])
    for i in range(5):
        assert np.allclose(ens.members[i, 8:, :], expected, atol=1e-5)
    assert_mean_consistent(ens)


def test_shapes_grow_by_one_slice(pm):  # test_enks.py:84-91
    from paper_2410_09663_b200 import enks

    _, vs, x0 = setup(pm, 4)
    ens = enks.init_ensemble(x0, 6)
    enks.predict(ens, vs, pm.matvar.NoiseStreams(seed=1))
    assert ens.members.shape == (6, 16, 3)
    assert ens.t == 1
    assert_mean_consistent(ens)


def test_u_block_covariance_matches_process_noise(pm):  # test_enks.py:93-102
    from paper_2410_09663_b200 import enks

    _, vs, x0 = setup(pm, 5, n=3, l=2, m=1)
    ens = enks.init_ensemble(x0, 100_000)
    enks.predict(ens, vs, pm.matvar.NoiseStreams(seed=2))
    u_next = ens.members[:, ens.slice_rows + 3:ens.slice_rows + 5, 0]
    emp = np.cov(u_next.T, bias=True)
    expect = vs.weights.scale * vs.weights.q_du
    assert np.allclose(emp, expect, atol=0.05 * np.abs(expect).max())


def test_zero_innovation_leaves_ensemble_unchanged(pm):  # test_enks.py:106-117
    from paper_2410_09663_b200 import enks

    model, vs, x0 = setup(pm, 6, scale=0.0)
    ens = enks.init_ensemble(x0, 4)
    enks.predict(ens, vs, pm.matvar.NoiseStreams(seed=3))
    before = ens.members.copy()
    y_ref = np.vstack([model.step(x0.x, x0.u), x0.u])
    enks.update(ens, y_ref, vs, pm.matvar.NoiseStreams(seed=3))
    assert np.allclose(ens.members, before, atol=1e-6)


def test_mean_consistency_through_sweep(pm):  # test_enks.py:133-143
    from paper_2410_09663_b200 import enks

    _, vs, x0 = setup(pm, 8)
    ens = enks.init_ensemble(x0, 12)
    st = pm.matvar.NoiseStreams(seed=5)
    y = np.vstack([vs.weights.x_ref, vs.weights.u_ref])
    for _ in range(4):
        enks.predict(ens, vs, st)
        assert_mean_consistent(ens)
        enks.update(ens, y, vs, st)
        assert_mean_consistent(ens)


def test_matrix_equals_vector_for_single_column(pm):  # test_enks.py:147-157
    """m = 1: the reference's matrix smoother equals its vector EnKS to 1e-10; both are
    pinned by the golden fixture lin_m1 (reference output), so match it at fp32."""
    from paper_2410_09663_b200 import enks

    gold = np.load(os.path.join(GOLD, "lin_m1.npz"))
    _, vs, x0 = setup(pm, 9, n=4, l=1, m=1)
    out, _ = enks.smooth_horizon(x0, gold["y"], vs, 3, 8, pm.matvar.NoiseStreams(seed=6))
    assert np.abs(out - gold["mean"]).max() / np.abs(gold["mean"]).max() < 1e-4


def test_mean_converges_to_exact_smoother(pm):  # test_enks.py:177-186
    from paper_2410_09663_b200 import enks

    gold = np.load(os.path.join(GOLD, "exact_lin_4x1x1.npz"))
    _, vs, x0 = setup(pm, 11, n=4, l=1, m=1)
    assert np.array_equal(x0.packed, gold["x0"])
    y = np.vstack([vs.weights.x_ref, vs.weights.u_ref])
    approx, _ = enks.smooth_horizon(x0, y, vs, 3, 4000, pm.matvar.NoiseStreams(seed=7))
    exact = gold["exact"]
    assert np.abs(approx - exact).max() / np.abs(exact).max() < 0.05


def test_shift_equivariance(pm):  # test_enks.py:205-240
    from paper_2410_09663_b200 import enks

    rng = np.random.default_rng(13)
    n, l, m = 3, 2, 2
    model = pm.dynamics.LinearDynamics(np.eye(n), rng.standard_normal((n, l)), state_cols=m)

    def spd(k):
        a = rng.standard_normal((k, k))
        return a @ a.T + k * np.eye(k)

    w = pm.virtualsys.MpcWeights(r=spd(n), q_u=spd(l), q_du=spd(l),
                                 x_ref=rng.standard_normal((n, m)), u_ref=rng.standard_normal((l, m)))
    shift = rng.standard_normal((n, m))
    ws = pm.virtualsys.MpcWeights(r=w.r, q_u=w.q_u, q_du=w.q_du, x_ref=w.x_ref + shift, u_ref=w.u_ref)
    vs = pm.virtualsys.build_virtual_system(model, w)
    vss = pm.virtualsys.build_virtual_system(model, ws)
    x0 = pm.virtualsys.AugmentedState(rng.standard_normal((n, m)), rng.standard_normal((l, m)),
                                      np.zeros((l, m)))
    x0s = pm.virtualsys.AugmentedState(x0.x + shift, x0.u, x0.du)
    base, _ = enks.smooth_horizon(x0, vs.reference_observation(), vs, 3, 32,
                                  pm.matvar.NoiseStreams(seed=8))
    moved, _ = enks.smooth_horizon(x0s, vss.reference_observation(), vss, 3, 32,
                                   pm.matvar.NoiseStreams(seed=8))
    for t in range(4):
        assert np.allclose(moved[t, :n], base[t, :n] + shift, atol=2e-5)
        assert np.allclose(moved[t, n:], base[t, n:], atol=2e-5)


def test_track_cov_does_not_change_mean(pm):  # test_enks.py:253-265
    from paper_2410_09663_b200 import enks

    _, vs, x0 = setup(pm, 15)
    y = np.vstack([vs.weights.x_ref, vs.weights.u_ref])
    plain, off = enks.smooth_horizon(x0, y, vs, 3, 10, pm.matvar.NoiseStreams(seed=10))
    tracked, on = enks.smooth_horizon(x0, y, vs, 3, 10, pm.matvar.NoiseStreams(seed=10),
                                      track_cov=True)
    assert np.array_equal(plain, tracked)
    assert off is None
    assert isinstance(on, enks.SmootherCovariances)


def test_tracked_covariance_is_psd_and_sized(pm):  # test_enks.py:267-277
    from paper_2410_09663_b200 import enks

    _, vs, x0 = setup(pm, 16)
    y = np.vstack([vs.weights.x_ref, vs.weights.u_ref])
    traj, cov = enks.smooth_horizon(x0, y, vs, 5, 16, pm.matvar.NoiseStreams(seed=11),
                                    track_cov=True)
    d = x0.n + 2 * x0.l
    assert cov.sigma_traj.shape == (6 * d, 6 * d)
    eigs = np.linalg.eigvalsh(cov.sigma_traj)
    assert eigs.min() > -1e-5 * np.trace(cov.sigma_traj)


@pytest.mark.parametrize("name", ["lin_spd_4x2x3", "lin_id_8x4x8", "lin_scale0_N4", "lin_colcov7",
                                  "lin_yref_stack", "lin_trackcov"])
def test_golden_reference_outputs(pm, name):
    """Device smoother vs the reference's own stored outputs (fp32 tolerance 1e-4)."""
    from test_oracle_golden import _case, _load

    from paper_2410_09663_b200 import enks

    gold = _load(name)
    _, vs, x0, N, h, sseed, extra = _case(pm, name)
    out, cov = enks.smooth_horizon(x0, gold["y"], vs, h, N, pm.matvar.NoiseStreams(seed=sseed),
                                   track_cov=bool(extra.get("track_cov")))
    assert np.abs(out - gold["mean"]).max() / np.abs(gold["mean"]).max() < 1e-4
    if cov is not None:
        for k in ("sigma_traj", "sigma_pred", "sigma_cross"):
            g = gold[k]
            assert np.abs(getattr(cov, k) - g).max() / np.abs(g).max() < 1e-4


def test_golden_cnn_reference_output(pm):
    from paper_2410_09663_b200 import enks

    gold = np.load(os.path.join(GOLD, "cnn_c1_16.npz"))
    pr = problems.make_cnn_problem(pm, "C1", size=16, n_members=24, horizon=3)
    out, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, pm.matvar.NoiseStreams(seed=1))
    assert np.abs(out - gold["mean"]).max() / np.abs(gold["mean"]).max() < 1e-4
