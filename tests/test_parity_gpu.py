"""End-to-end parity of the device smoother with the fp64 CPU oracle.

Tolerance (north_star): relative error <= 1e-4 on the smoothed state/control
means (max |dev - ref| / max |ref|), and on tracked covariances; noise is
bit-identical, so the only differences are fp32 rounding.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


def _linear_case(pm, seed, **kw):
    from oracle import problems

    return problems.make_linear_setup(pm, np.random.default_rng(seed), **kw)


@pytest.mark.parametrize("seed,kw,N,h", [
    (0, dict(n=4, l=2, m=3), 16, 5),
    (1, dict(n=8, l=4, m=8, identity_weights=True), 32, 6),
    (2, dict(n=16, l=8, m=16), 64, 10),
    (3, dict(n=4, l=1, m=1), 8, 3),
    (4, dict(n=32, l=32, m=32, identity_weights=True), 100, 8),
])
def test_smooth_horizon_linear_matches_oracle(pm, seed, kw, N, h):
    from oracle import enks_oracle
    from paper_2410_09663_b200 import enks

    _, vs, x0 = _linear_case(pm, seed, **kw)
    y = vs.reference_observation()
    ref, _, oens = enks_oracle.oracle_smooth(x0, y, vs, h, N, seed=seed + 10, backend="c")
    got, cov = enks.smooth_horizon(x0, y, vs, h, N, pm.matvar.NoiseStreams(seed=seed + 10))
    assert cov is None
    assert got.shape == ref.shape
    assert _rel(got, ref) < TOL


def test_smooth_horizon_cnn_c1_matches_oracle(pm):
    """C1b: CNN 2-16-16-1 on a 32x32 field, N=100, H=5."""
    from oracle import enks_oracle, problems
    from oracle.models import OracleCNN

    from paper_2410_09663_b200 import enks

    pr = problems.make_cnn_problem(pm, "C1")
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model), pr.vs.weights)
    ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=0, backend="c")
    got, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N,
                                 pm.matvar.NoiseStreams(seed=0))
    n, l = pr.n, pr.l
    assert _rel(got, ref) < TOL
    assert _rel(got[:, n:n + l], ref[:, n:n + l]) < TOL  # control block on its own


def test_track_cov_matches_oracle(pm):
    from oracle import enks_oracle
    from paper_2410_09663_b200 import enks

    _, vs, x0 = _linear_case(pm, 16)
    y = vs.reference_observation()
    ref, rcov, _ = enks_oracle.oracle_smooth(x0, y, vs, 5, 16, seed=11, track_cov=True,
                                             backend="c")
    got, cov = enks.smooth_horizon(x0, y, vs, 5, 16, pm.matvar.NoiseStreams(seed=11),
                                   track_cov=True)
    assert _rel(got, ref) < TOL
    assert cov.sigma_traj.shape == rcov.sigma_traj.shape
    assert _rel(cov.sigma_traj, rcov.sigma_traj) < TOL
    assert _rel(cov.sigma_cross, rcov.sigma_cross) < TOL
    assert _rel(cov.sigma_pred, rcov.sigma_pred) < TOL


def test_members_and_predict_update_api(pm):
    """Bare predict/update (capacity growth) and lazily materialised members."""
    from oracle import enks_oracle
    from paper_2410_09663_b200 import enks

    _, vs, x0 = _linear_case(pm, 8)
    y = vs.reference_observation()
    ens = enks.init_ensemble(x0, 12, capacity=1)
    o = enks_oracle.oracle_init(x0.packed, x0.n, x0.l, 12)
    st = pm.matvar.NoiseStreams(seed=5)
    for _ in range(4):
        enks.predict(ens, vs, st)
        enks_oracle.oracle_predict(o, vs, 5, backend="c")
        assert ens.members.shape == o.members.shape
        assert _rel(ens.members, o.members) < TOL
        enks.update(ens, y, vs, st)
        enks_oracle.oracle_update(o, y, vs, 5, backend="c")
        assert _rel(ens.members, o.members) < TOL
        assert _rel(ens.mean, o.mean) < TOL
        assert np.abs(ens.mean - ens.members.mean(axis=0)).max() < 1e-5 * np.abs(o.mean).max()
    assert ens.t == 4 and ens.jitter_events == 0


def test_degenerate_noise_exact(pm):
    """scale=0: members identical, G = 0 through the 1e-30 jitter path (test_enks.py:244-251)."""
    from paper_2410_09663_b200 import enks

    model, vs, x0 = _linear_case(pm, 14, scale=0.0)
    y = np.vstack([vs.weights.x_ref, vs.weights.u_ref])
    traj, _ = enks.smooth_horizon(x0, y, vs, 1, 4, pm.matvar.NoiseStreams(seed=9))
    assert np.allclose(traj[0], x0.packed)
    expected = np.vstack([model.step(x0.x, x0.u), x0.u, np.zeros_like(x0.u)])
    assert np.allclose(traj[1], expected, atol=1e-6)
    # non-power-of-two N as well: the member-0 shift keeps the spread exactly zero
    traj, _ = enks.smooth_horizon(x0, y, vs, 3, 12, pm.matvar.NoiseStreams(seed=9))
    ens_ref = x0.packed
    for t in range(1, 4):
        ens_ref = np.vstack([model.step(ens_ref[:x0.n], ens_ref[x0.n:x0.n + x0.l]),
                             ens_ref[x0.n:x0.n + x0.l], np.zeros_like(x0.u)])
        assert np.allclose(traj[t], ens_ref, atol=1e-5)


def test_same_streams_bit_identical(pm):
    from paper_2410_09663_b200 import enks

    _, vs, x0 = _linear_case(pm, 17)
    y = vs.reference_observation()
    a, _ = enks.smooth_horizon(x0, y, vs, 3, 64, pm.matvar.NoiseStreams(seed=12))
    b, _ = enks.smooth_horizon(x0, y, vs, 3, 64, pm.matvar.NoiseStreams(seed=12))
    assert np.array_equal(a, b)


def test_lambda_cancellation(pm):
    from paper_2410_09663_b200 import enks

    model, vs, x0 = _linear_case(pm, 7)
    vs7 = pm.virtualsys.build_virtual_system(model, vs.weights, shared_col_cov=7.0 * np.eye(x0.m))
    y = vs.reference_observation()
    a, _ = enks.smooth_horizon(x0, y, vs, 3, 16, pm.matvar.NoiseStreams(seed=4))
    b, _ = enks.smooth_horizon(x0, y, vs7, 3, 16, pm.matvar.NoiseStreams(seed=4))
    assert _rel(a, b) < 1e-5


@pytest.mark.parametrize("mode", ["boundary", "pointwise"])
def test_smooth_horizon_burgers_c1a_matches_reference_golden(pm, mode):
    """C1a: the reference's own Burgers FD problem (grid 32, N=100, H=5), compared with the
    UNMODIFIED reference smooth_horizon output (tests/golden/burgers_c1a_*.npz)."""
    import os

    from oracle import problems
    from paper_2410_09663_b200 import enks

    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", f"burgers_c1a_{mode}.npz"))
    pr = problems.make_burgers_problem(pm, mode)
    assert np.array_equal(pr.x0.packed, gold["x0"])
    got, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N,
                                 pm.matvar.NoiseStreams(seed=2))
    n, l = pr.n, pr.l
    assert _rel(got, gold["mean"]) < TOL
    assert _rel(got[:, n:n + l], gold["mean"][:, n:n + l]) < TOL


@pytest.mark.parametrize("name,kind", [("lin_con_linear", "linear"), ("lin_con_box", "box")])
def test_smooth_horizon_constraint_matches_reference_golden(pm, name, kind):
    """Barrier row on the device (csrc/barrier.cu) vs the UNMODIFIED reference run."""
    import os

    from golden.make_golden import LINEAR_CASES
    from oracle import problems
    from paper_2410_09663_b200 import enks

    _, kw, seed, N, h, sseed, _ = next(c for c in LINEAR_CASES if c[0] == name)
    model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(seed), **kw)
    con = problems.make_constraint(pm, kind, x0.n, x0.l, x0.m)
    vs = pm.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", name + ".npz"))
    got, _ = enks.smooth_horizon(x0, gold["y"], vs, h, N, pm.matvar.NoiseStreams(seed=sseed))
    assert _rel(got, gold["mean"]) < TOL


def test_track_cov_tensor_core_path_matches_oracle(pm):
    """C1b-shaped CNN with track_cov: K = N m = 3200 routes the covariance contractions through
    the fp16-pair tcgen05 kernel in 256-column blocks (T d = 576 > 256)."""
    from oracle import enks_oracle, problems
    from oracle.models import OracleCNN
    from paper_2410_09663_b200 import enks

    pr = problems.make_cnn_problem(pm, "C1", n_members=100, horizon=5)
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model), pr.vs.weights)
    ref, rcov, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=4,
                                             track_cov=True, backend="c")
    got, cov = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N,
                                   pm.matvar.NoiseStreams(seed=4), track_cov=True)
    assert _rel(got, ref) < TOL
    for k in ("sigma_traj", "sigma_cross", "sigma_pred"):
        assert getattr(cov, k).shape == getattr(rcov, k).shape
        assert _rel(getattr(cov, k), getattr(rcov, k)) < TOL, k


def test_cuda_graph_horizon_bit_identical_to_eager(pm):
    """smooth_horizon(graph=True) replays a captured horizon: same kernels, same results."""
    from oracle import problems
    from paper_2410_09663_b200 import enks

    pr = problems.make_cnn_problem(pm, "C1", size=32, n_members=64, horizon=4,
                                   widths=(2, 32, 32, 1))
    st = pm.matvar.NoiseStreams(seed=3)
    eager, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st)
    g1, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st, graph=True)
    g2, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st, graph=True)  # replay
    assert np.array_equal(g1, eager) and np.array_equal(g2, eager)
    # new static inputs through the same graph
    x1 = pm.virtualsys.AugmentedState(pr.x0.x * 0.5, pr.x0.u, pr.x0.du)
    e1, _ = enks.smooth_horizon(x1, pr.y_ref, pr.vs, pr.H, pr.N, st)
    g3, _ = enks.smooth_horizon(x1, pr.y_ref, pr.vs, pr.H, pr.N, st, graph=True)
    assert np.array_equal(g3, e1)
    # other noise streams with the same entropy word count replay the SAME capture (device head)
    n_graphs = len(enks._GRAPHS)
    for st2 in (pm.matvar.NoiseStreams(seed=4), pm.matvar.NoiseStreams(seed=3, prefix=(7,)),
                pm.matvar.NoiseStreams(seed=4, prefix=(8,))):
        e2, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st2)
        g4, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st2, graph=True)
        assert np.array_equal(g4, e2)
        assert not np.array_equal(g4, eager)
    assert len(enks._GRAPHS) == n_graphs + 1  # one extra capture: the prefixed word count


def test_smooth_horizon_wide_observation_schur_gain(pm):
    """p = n + l = 320 > 288: fp16-pair cross moments in 256-column tiles and the two-level
    (Schur complement) gain solve."""
    from oracle import enks_oracle
    from paper_2410_09663_b200 import enks

    # K = N m = 5 p keeps Sigma_y well conditioned (fp32 tolerance; see DESIGN.md §5 for
    # N m ~ p, where the conditioning of the sample covariance amplifies fp32 rounding)
    _, vs, x0 = _linear_case(pm, 31, n=200, l=120, m=4, identity_weights=True)
    y = vs.reference_observation()
    ref, _, _ = enks_oracle.oracle_smooth(x0, y, vs, 3, 400, seed=5, backend="c")
    got, _ = enks.smooth_horizon(x0, y, vs, 3, 400, pm.matvar.NoiseStreams(seed=5))
    assert _rel(got, ref) < TOL


@pytest.mark.parametrize("n,l", [(60, 40), (200, 120)])
def test_rank_deficient_sigma_y_jitter(pm, n, l):
    """(N - 1) m < p: Sigma_y is singular and the reference rescues it with a 1e-9 relative
    jitter in fp64.  That regularisation is below fp32 resolution, so the device escalates the
    jitter (one jitter event per update, as the reference counts) and warns that the fp32 gain
    is not reliable there."""
    from oracle import enks_oracle
    from paper_2410_09663_b200 import enks

    _, vs, x0 = _linear_case(pm, 33, n=n, l=l, m=2, identity_weights=True)
    y = vs.reference_observation()
    N = (n + l) // 4  # N m = p / 2
    _, _, oens = enks_oracle.oracle_smooth(x0, y, vs, 3, N, seed=6, backend="c")
    with pytest.warns(RuntimeWarning, match="rank-deficient"):
        ens = enks.init_ensemble(x0, N, capacity=3)
        st = pm.matvar.NoiseStreams(seed=6)
        try:
            for _ in range(3):
                enks.predict(ens, vs, st)
                enks.update(ens, y, vs, st)
        except np.linalg.LinAlgError:
            # p > 288 (Schur-complement gain solve): the fp32 Schur complement of a jittered
            # singular block may itself fail -- reported, never silently wrong
            assert n + l > 288
            return
    assert ens.jitter_events == oens.jitter_events == 3
    assert np.all(np.isfinite(ens.mean))


def test_smooth_horizon_c4_shape_matches_oracle(pm):
    """BASELINE C4 shapes (256 x 256 field, l = m = 256, 6-layer CNN 2-32-32-32-32-32-1) at a
    small ensemble: deep tcgen05 CNN, p = 512 cross moments in 256-column tiles, Schur gain."""
    from oracle import enks_oracle, problems
    from oracle.models import OracleCNN

    from paper_2410_09663_b200 import enks

    pr = problems.make_cnn_problem(pm, "C4", n_members=8, horizon=2)
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model), pr.vs.weights)
    ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=1, backend="c")
    got, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N,
                                 pm.matvar.NoiseStreams(seed=1))
    n, l = pr.n, pr.l
    assert _rel(got, ref) < TOL
    assert _rel(got[:, n:n + l], ref[:, n:n + l]) < TOL
