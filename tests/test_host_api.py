"""Host-side mirror of the reference API: validation, error behaviour, configuration types."""
import numpy as np
import pytest

from oracle import problems


def test_mirror_types_build_the_same_noise_channels(pm):
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(3))
    assert vs.obs_rows == x0.n + x0.l
    np.testing.assert_allclose(vs.process_noise.row_chol @ vs.process_noise.row_chol.T,
                               vs.weights.scale * vs.weights.q_du)
    assert np.array_equal(vs.process_noise.col_chol, np.eye(x0.m))
    assert np.array_equal(vs.shared_col_cov, np.eye(x0.m))
    assert vs.reference_observation().shape == (x0.n + x0.l, x0.m)


def test_weights_validation(pm):
    vsm = pm.virtualsys
    with pytest.raises(ValueError):
        vsm.MpcWeights(r=np.eye(2), q_u=np.eye(1), q_du=np.eye(1), x_ref=np.zeros((2, 3)),
                       u_ref=np.zeros((1, 3)), scale=-1.0)
    with pytest.raises(np.linalg.LinAlgError):
        vsm.MpcWeights(r=-np.eye(2), q_u=np.eye(1), q_du=np.eye(1), x_ref=np.zeros((2, 3)),
                       u_ref=np.zeros((1, 3)))


def test_scale_zero_has_no_noise_channels(pm):
    _, vs, _ = problems.make_linear_setup(pm, np.random.default_rng(4), scale=0.0)
    assert vs.process_noise is None and vs.obs_noise_x is None and vs.obs_noise_u is None


def test_reference_errors_before_device_work(pm):
    """ValueErrors of enks.py:113-114, 271-277, 228-229 are raised with no GPU touched."""
    from paper_2410_09663_b200 import enks

    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(5))
    y = vs.reference_observation()
    with pytest.raises(ValueError):
        enks.init_ensemble(x0, 1)
    with pytest.raises(ValueError):
        enks.smooth_horizon(x0, y, vs, 0, 8, pm.matvar.NoiseStreams(0))
    with pytest.raises(ValueError):
        enks.smooth_horizon(x0, np.stack([y, y]), vs, 3, 8, pm.matvar.NoiseStreams(0))
    with pytest.raises(ValueError):
        enks.smooth_horizon(x0, y[:-1], vs, 2, 8, pm.matvar.NoiseStreams(0))


def test_noise_streams_mirror_numpy(pm):
    st = pm.matvar.NoiseStreams(seed=7, prefix=(1,))
    a = st.substream(2, 3, 0).standard_normal(5)
    b = np.random.Generator(np.random.Philox(np.random.SeedSequence(7, spawn_key=(1, 2, 3, 0))))
    assert np.array_equal(a, b.standard_normal(5))
    assert st.child(4).prefix == (1, 4)


def test_cnn_dynamics_host_step_matches_oracle(pm):
    from oracle.models import cnn_step

    m = pm.dynamics.CNNDynamics(rows=12, cols=10, widths=(2, 8, 8, 1), seed=2)
    rng = np.random.default_rng(0)
    x, u = rng.standard_normal((3, 12, 10)), rng.standard_normal((3, 12, 10))
    np.testing.assert_allclose(m.step(x, u), cnn_step(x, u, m.weights, m.biases, m.alpha),
                               rtol=1e-12, atol=1e-12)
    assert m.flops_per_member_step() == 12 * 10 * 18 * (2 * 8 + 8 * 8 + 8)


def test_partition_covers_members_once():
    from paper_2410_09663_b200.engine import partition

    for N in (2, 7, 100, 1024):
        for size in (1, 2, 3, 8):
            if N < size:
                continue
            spans = [partition(N, size, r) for r in range(size)]
            assert spans[0][0] == 0
            for (a, c), (b, _) in zip(spans, spans[1:]):
                assert a + c == b
            assert sum(c for _, c in spans) == N
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_forecaster_rejects_unknown_models():
    from paper_2410_09663_b200.engine import Forecaster

    class Weird:
        state_rows = state_cols = input_rows = 2

    with pytest.raises(TypeError):
        Forecaster(Weird(), None, 2, 2)
