"""Parity at the configurations bench.py measures (BASELINE C2, C3, C5) against the fp64 oracle.

SURVEY.md §8(c): the device smoother's mean trajectory and the per-update Sigma_y, Sigma_xy and
gain are compared with oracle/enks_oracle.py (the reference's enks.py:212-284 restated in fp64,
pinned to the unmodified reference by tests/golden) on identical seeds, inputs and noise draws
(the device noise is bit-identical).  The oracle's CNN is the fp64 torch-CPU conv stack
(oracle.models.cnn_step_torch, pinned to the explicit-tap restatement at 1e-12).

Tolerance (north_star): relative error <= 1e-4, measured as max |dev - ref| / max |ref| over
the whole array, and separately over the X and U blocks of the mean trajectory.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


def _run(pm, config, N, H, seed, taus, graph_check=False):
    from oracle import enks_oracle, problems
    from oracle.models import OracleCNN
    from paper_2410_09663_b200 import enks

    pr = problems.make_cnn_problem(pm, config, n_members=N, horizon=H)
    ovs = pm.virtualsys.build_virtual_system(OracleCNN(pr.model, backend="torch"), pr.vs.weights)
    orec = {}
    ref, _, _ = enks_oracle.oracle_smooth(pr.x0, pr.y_ref, ovs, H, N, seed=seed, backend="c",
                                          record=orec)
    st = pm.matvar.NoiseStreams(seed=seed)
    ens = enks.init_ensemble(pr.x0, N, shared_col_cov=pr.vs.shared_col_cov, capacity=H)
    rec = {}
    for k in range(H):
        enks.predict(ens, pr.vs, st)
        ens.engine.record = rec if (k + 1) in taus else None
        enks.update(ens, pr.y_ref, pr.vs, st)
    ens.engine.record = None
    got = ens.slices()
    n, l = pr.n, pr.l
    errs = {"all": _rel(got, ref), "X": _rel(got[:, :n], ref[:, :n]),
            "U": _rel(got[:, n:n + l], ref[:, n:n + l]),
            "dU": _rel(got[:, n + l:], ref[:, n + l:])}
    for j, tau in enumerate(sorted(taus)):
        for key in ("sigma_y", "sigma_xy", "gain"):
            a, b = rec[key][j], orec[key][tau - 1]
            assert a.shape == b.shape, (key, tau)
            errs[f"{key}@{tau}"] = _rel(a, b)
    if graph_check:  # the bench's default path (CUDA-graph replay) gives the same numbers
        g, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, H, N, st, graph=True)
        errs["graph_vs_eager"] = _rel(g, got)
    print(config, N, H, {k: f"{v:.2e}" for k, v in errs.items()})
    return errs


def _check(errs):
    bad = {k: v for k, v in errs.items() if k != "dU" and not v < TOL}
    assert not bad, bad


def test_c2_full_horizon(pm):
    """C2 as benchmarked: 64 x 64 field, CNN 2-32-32-1, N = 512, H = 20."""
    _check(_run(pm, "C2", 512, 20, seed=0, taus=(1, 10, 20)))


def test_c3_shapes_full_ensemble(pm):
    """C3 shapes at the full ensemble (128 x 128, N = 1024, K = N m = 131072, p = 256), H = 10,
    with Sigma_y / Sigma_xy / gain compared at tau = 1, 5, 10; the CUDA-graph replay (bench.py's
    default timing path) must equal the eager result."""
    errs = _run(pm, "C3", 1024, 10, seed=0, taus=(1, 5, 10), graph_check=True)
    assert errs["graph_vs_eager"] == 0.0
    _check(errs)


@pytest.mark.parametrize("N", [64, 16384])
def test_c5_ensemble_sweep_ends(pm, N):
    """C5's sweep ends: 128 x 128, N = 64 (K = 8192) and N = 16384 (K = 2^21), H = 3."""
    _check(_run(pm, "C5", N, 3, seed=1, taus=(1, 3)))
