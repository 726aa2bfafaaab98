"""The append-only-basis restatement (engine.py) equals the reference algorithm.

Runs the product engine's orchestration against a CPU fp64 operator set
(tests/cpu_ops.py, test-only) and compares with the fp64 oracle: any
difference beyond rounding would be an algebra error in the restructuring.
"""
import numpy as np
import pytest

from cpu_ops import CpuOps
from oracle import enks_oracle, problems
from paper_2410_09663_b200.engine import DeviceSmoother


def _run(pm, x0, y, vs, h, N, seed, cap=2, pair=False):
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, N, 1.0 / np.trace(vs.shared_col_cov),
                         capacity=cap, basis="f16pair" if pair else "fp32")
    st = pm.matvar.NoiseStreams(seed=seed)
    yd = ops.to_device(np.broadcast_to(y, (h,) + y.shape[-2:]).copy() if y.ndim == 2 else y)
    for k in range(h):
        eng.predict(vs, st)
        eng.update(yd[k], st)
    return eng


@pytest.mark.parametrize("kw,N,h,seed", [
    (dict(n=4, l=2, m=3), 16, 5, 0),
    (dict(n=4, l=2, m=3, scale=0.0), 4, 3, 1),
    (dict(n=8, l=4, m=8, identity_weights=True), 32, 6, 2),
    (dict(n=4, l=1, m=1), 8, 3, 3),
    (dict(n=6, l=6, m=5), 13, 7, 4),
])
@pytest.mark.parametrize("pair", [False, True])
def test_engine_equals_oracle_fp64(pm, kw, N, h, seed, pair):
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(seed), **kw)
    y = vs.reference_observation()
    ref, _, oens = enks_oracle.oracle_smooth(x0, y, vs, h, N, seed=seed + 7, backend="c")
    if pair and (N * x0.m) % 8:
        pytest.skip("fp16-pair basis needs N*m % 8 == 0 (16-B aligned fp16 rows)")
    eng = _run(pm, x0, y, vs, h, N, seed + 7, pair=pair)
    assert eng.pair == pair
    assert eng.chain == pair  # the fp16-pair basis keeps [X; dU] only (derived-U chain)
    d, m = x0.n + 2 * x0.l, x0.m
    mean = eng.mean_host().reshape(h + 1, d, m)
    members = eng.members_device().numpy().reshape((h + 1) * d, N, m).transpose(1, 0, 2)
    scale = np.abs(ref).max()
    assert np.abs(mean - ref).max() < 1e-10 * scale
    assert np.abs(members - oens.members).max() < 1e-10 * np.abs(oens.members).max()
    assert eng.jitter.item() == oens.jitter_events


def test_engine_pair_without_uchain(pm, monkeypatch):
    """ENKS_UCHAIN=0: the fp16-pair basis with the full [X; U; dU] rows per slice."""
    monkeypatch.setenv("ENKS_UCHAIN", "0")
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(4), n=6, l=6, m=4)
    y = vs.reference_observation()
    ref, _, oens = enks_oracle.oracle_smooth(x0, y, vs, 5, 12, seed=3, backend="c")
    eng = _run(pm, x0, y, vs, 5, 12, 3, pair=True)
    assert eng.pair and not eng.chain and eng.ds == eng.d
    mean = eng.mean_host().reshape(ref.shape)
    assert np.abs(mean - ref).max() < 1e-10 * np.abs(ref).max()
    members = eng.members_device().numpy().reshape(ref.shape[0] * ref.shape[1], 12, 4)
    assert np.abs(members.transpose(1, 0, 2) - oens.members).max() < 1e-10 * np.abs(ref).max()


def test_engine_cnn_equals_oracle_fp64(pm):
    pr = problems.make_cnn_problem(pm, "C1", size=8, n_members=10, horizon=3)
    ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, seed=0, backend="c")
    eng = _run(pm, pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, 0)
    assert np.abs(eng.mean_host().reshape(ref.shape) - ref).max() < 1e-10 * np.abs(ref).max()


@pytest.mark.parametrize("pair", [False, True])
def test_engine_explicit_members_restart(pm, pair):
    """replace_members (TrajectoryEnsemble(members=...)) then continue == oracle continuing."""
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(5))
    y = vs.reference_observation()
    o = enks_oracle.oracle_init(x0.packed, x0.n, x0.l, 9)
    for _ in range(2):
        enks_oracle.oracle_predict(o, vs, 3, backend="c")
        enks_oracle.oracle_update(o, y, vs, 3, backend="c")
    o.members = o.members + 0.01 * np.random.default_rng(0).standard_normal(o.members.shape)
    o.mean = o.members.mean(axis=0)
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, 9, o.lam, capacity=1,
                         basis="f16pair" if pair else "fp32")
    eng.replace_members(o.members, o.t)
    st = pm.matvar.NoiseStreams(seed=3)
    for _ in range(2):
        enks_oracle.oracle_predict(o, vs, 3, backend="c")
        enks_oracle.oracle_update(o, y, vs, 3, backend="c")
        eng.predict(vs, st)
        eng.update(ops.to_device(y), st)
    got = eng.members_device().numpy().reshape(o.members.shape[1], 9, x0.m).transpose(1, 0, 2)
    assert np.abs(got - o.members).max() < 1e-10 * np.abs(o.members).max()


@pytest.mark.parametrize("mode", ["boundary", "pointwise"])
def test_engine_burgers_equals_oracle_fp64(pm, mode):
    from oracle.models import OracleBurgers

    pr = problems.make_burgers_problem(pm, mode, grid_n=8, n_members=12, horizon=3)
    ovs = pm.virtualsys.build_virtual_system(OracleBurgers(pr.model), pr.vs.weights)
    ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, pr.H, pr.N, seed=2, backend="c")
    eng = _run(pm, pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, 2)
    assert eng.forecast.kind == "burgers"
    assert np.abs(eng.mean_host().reshape(ref.shape) - ref).max() < 1e-10 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["linear", "box"])
@pytest.mark.parametrize("pair", [False, True])
def test_engine_constraint_barrier_equals_oracle_fp64(pm, kind, pair):
    """Barrier observation row (enks.py:201-208): p = n + l + 1 observation rows."""
    model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(2), n=4, l=2, m=4)
    con = problems.make_constraint(pm, kind, x0.n, x0.l, x0.m)
    vs = pm.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
    y = vs.reference_observation()
    ref, _, oens = enks_oracle.oracle_smooth(x0, y, vs, 4, 16, seed=8, backend="c")
    eng = _run(pm, x0, y, vs, 4, 16, 8, pair=pair)
    assert eng.p == x0.n + x0.l + 1 and eng.q == x0.n + x0.l
    mean = eng.mean_host().reshape(ref.shape)
    assert np.abs(mean - ref).max() < 1e-10 * np.abs(ref).max()
    members = eng.members_device().numpy().reshape(ref.shape[0] * ref.shape[1], 16, 4)
    assert np.abs(members.transpose(1, 0, 2) - oens.members).max() < 1e-10 * np.abs(ref).max()


def test_engine_rejects_host_only_constraint(pm):
    model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(2))
    con = pm.virtualsys.ConstraintSpec(g=lambda s: float(s.u.sum()))
    vs = pm.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
    eng = DeviceSmoother(CpuOps(), x0.packed, x0.n, x0.l, 8, 1.0 / x0.m)
    with pytest.raises(TypeError, match="LinearConstraint or BoxConstraint"):
        eng.bind(vs)


@pytest.mark.parametrize("pair", [False, True])
def test_engine_record_equals_oracle_record(pm, pair):
    """The per-update record hook (Sigma_y, Sigma_xy, gain on the reference's full T d rows,
    U rows re-expanded from the derived-U chain) equals the oracle's record= output."""
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(5), n=6, l=3, m=4)
    y = vs.reference_observation()
    h, N, seed = 4, 16, 9
    orec = {}
    enks_oracle.oracle_smooth(x0, y, vs, h, N, seed=seed, backend="c", record=orec)
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, N, 1.0 / np.trace(vs.shared_col_cov),
                         capacity=h, basis="f16pair" if pair else "fp32")
    eng.record = {}
    st = pm.matvar.NoiseStreams(seed=seed)
    yd = ops.to_device(np.broadcast_to(y, (h,) + y.shape).copy())
    for k in range(h):
        eng.predict(vs, st)
        eng.update(yd[k], st)
    assert eng.chain == pair
    for key in ("sigma_y", "sigma_xy", "gain"):
        assert len(eng.record[key]) == h
        for a, b in zip(eng.record[key], orec[key]):
            assert a.shape == b.shape, key
            assert np.abs(a - b).max() < 1e-10 * np.abs(b).max(), key


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("spread", [False, True])
def test_engine_irregular_update_sequences_equal_oracle(pm, pair, spread):
    """update() at t = 0 (before any predict) and a second update at the same t, as the
    reference allows (enks.py:212-253): identical copies (gain exactly zero at t = 0) and
    explicit members with spread at t = 0 (the slice-0 gain moves them)."""
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(21), n=5, l=3, m=4)
    y = vs.reference_observation()
    N, seed = 16, 4
    o = enks_oracle.oracle_init(x0.packed, x0.n, x0.l, N)
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, N, o.lam, capacity=2,
                         basis="f16pair" if pair else "fp32")
    if spread:
        o.members = o.members + 0.3 * np.random.default_rng(1).standard_normal(o.members.shape)
        o.mean = o.members.mean(axis=0)
        eng.replace_members(o.members, 0)
    eng.bind(vs)
    st = pm.matvar.NoiseStreams(seed=seed)
    yd = ops.to_device(y)
    seq = ["u", "p", "u", "u", "p", "u", "p", "p", "u"]
    for op in seq:
        if op == "p":
            enks_oracle.oracle_predict(o, vs, seed, backend="c")
            eng.predict(vs, st)
        else:
            enks_oracle.oracle_update(o, y, vs, seed, backend="c")
            eng.update(yd, st)
        members = eng.members_device().numpy().reshape(eng.t + 1, eng.d, N, x0.m)
        members = members.reshape((eng.t + 1) * eng.d, N, x0.m).transpose(1, 0, 2)
        assert eng.t == o.t
        assert np.abs(members - o.members).max() < 1e-10 * np.abs(o.members).max(), op
        assert np.abs(eng.mean_host() - o.mean).max() < 1e-10 * np.abs(o.mean).max(), op
    assert eng.jitter.item() == o.jitter_events


@pytest.mark.parametrize("pair", [False, True])
def test_device_covariance_tracking_equals_oracle(pm, pair):
    """covariance.py's device tracking (SYRK over 256-blocks, lazy block assembly after predict,
    sigma_pred = last rows of sigma_cross) equals the oracle's track_cov after every call."""
    from paper_2410_09663_b200.covariance import (SmootherCovariances, track_predict,
                                                  track_update)

    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(6), n=60, l=40, m=4)
    y = vs.reference_observation()
    h, N, seed = 4, 40, 3  # T d up to 5 * 140 = 700 rows: three 256-blocks
    o = enks_oracle.oracle_init(x0.packed, x0.n, x0.l, N)
    ocov = enks_oracle.OracleCov(sigma_traj=np.zeros((o.d, o.d)))
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, N, o.lam, capacity=2,
                         basis="f16pair" if pair else "fp32")
    eng.bind(vs)
    cov = SmootherCovariances(sigma_traj=np.zeros((o.d, o.d)))
    st = pm.matvar.NoiseStreams(seed=seed)
    yd = ops.to_device(y)
    for _ in range(h):
        enks_oracle.oracle_predict(o, vs, seed, cov=ocov, backend="c")
        eng.predict(vs, st)
        track_predict(eng, cov)
        for k in ("sigma_traj", "sigma_cross", "sigma_pred"):
            ref = getattr(ocov, k)
            assert np.abs(getattr(cov, k) - ref).max() < 1e-10 * np.abs(ref).max(), k
        enks_oracle.oracle_update(o, y, vs, seed, cov=ocov, backend="c")
        eng.update(yd, st)
        track_update(eng, cov)
        ref = ocov.sigma_traj
        assert cov.sigma_traj.shape == ref.shape
        assert np.abs(cov.sigma_traj - ref).max() < 1e-10 * np.abs(ref).max()
