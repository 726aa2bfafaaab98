"""Covariance tracking at the C2 configuration against the fp64 oracle.

smooth_horizon(track_cov=True) returns the lambda-scaled covariances of the last predict / update
(enks.py:173-185, 250-252).  The oracle side computes exactly those from its fp64 members: after
the last predict, Sigma_cross = (lam/N) D dev_new^T and Sigma_pred = its last d rows; after the
last update, Sigma_traj = (lam/N) D D^T (T d = 21 x 192 = 4032 rows, K = N m = 32768).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


def _pair_cov(a, b, lam):
    N = a.shape[0]
    am = np.swapaxes(a, 0, 1).reshape(a.shape[1], -1)
    bm = np.swapaxes(b, 0, 1).reshape(b.shape[1], -1)
    return (lam / N) * (am @ bm.T)


def test_track_cov_c2_full_horizon(pm):
    from oracle import enks_oracle, problems
    from oracle.models import OracleCNN
    from paper_2410_09663_b200 import enks

    pr = problems.make_cnn_problem(pm, "C2")
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model, backend="torch"), pr.vs.weights)
    o = enks_oracle.oracle_init(pr.x0.packed, pr.n, pr.l, pr.N, shared_col_cov=pr.vs.shared_col_cov)
    seed = 3
    for k in range(pr.H):
        enks_oracle.oracle_predict(o, ovs, seed, backend="c")
        if k == pr.H - 1:
            new = o.members[:, -o.d:]
            dev_new = new - new.mean(axis=0)
            dev_traj = o.members - o.mean
            ref_pred = _pair_cov(dev_new, dev_new, o.lam)
            ref_cross = _pair_cov(dev_traj, dev_new, o.lam)
        enks_oracle.oracle_update(o, pr.y_ref, ovs, seed, backend="c")
    dev = o.members - o.mean
    ref_traj = _pair_cov(dev, dev, o.lam)
    got, cov = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N,
                                   pm.matvar.NoiseStreams(seed=seed), track_cov=True)
    assert _rel(got, o.mean.reshape(pr.H + 1, o.d, -1)) < TOL
    errs = {"traj": _rel(cov.sigma_traj, ref_traj), "cross": _rel(cov.sigma_cross, ref_cross),
            "pred": _rel(cov.sigma_pred, ref_pred)}
    print("C2 track_cov rel errors", {k: f"{v:.2e}" for k, v in errs.items()})
    assert cov.sigma_traj.shape == ref_traj.shape == (4032, 4032)
    assert np.array_equal(cov.sigma_traj, cov.sigma_traj.T)
    assert all(v < TOL for v in errs.values()), errs
