"""Generate the golden fixtures that pin the oracle to the reference itself.

Run in the build container, where the reference is importable read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It runs the UNMODIFIED reference smoother (/root/reference/pkg/src/enksmpc,
enks.smooth_horizon, enks.py:256-284) and numpy's own noise substreams
(matvar.py:149-151) on small seeded problems and stores inputs' checksums and
outputs as .npz files next to this script.  tests/test_oracle_golden.py then
checks the oracle restatement (oracle/enks_oracle.py, oracle/npy_noise.c)
against these files on any box, without /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import problems  # noqa: E402
from oracle.models import OracleCNN  # noqa: E402

# (name, make_linear_setup kwargs, seed, N, h, stream seed, extra)
LINEAR_CASES = [
    ("lin_spd_4x2x3", dict(n=4, l=2, m=3), 0, 16, 5, 10, {}),
    ("lin_id_8x4x8", dict(n=8, l=4, m=8, identity_weights=True), 1, 32, 6, 11, {}),
    ("lin_m1", dict(n=4, l=1, m=1), 9, 8, 3, 6, {}),
    ("lin_scale0_N4", dict(n=4, l=2, m=3, scale=0.0), 14, 4, 3, 9, {}),
    ("lin_trackcov", dict(n=4, l=2, m=3), 16, 16, 5, 11, {"track_cov": True}),
    ("lin_colcov7", dict(n=4, l=2, m=3), 7, 16, 3, 4, {"col_cov": 7.0}),
    ("lin_yref_stack", dict(n=5, l=3, m=4), 21, 20, 4, 3, {"yref_stack": True}),
    ("lin_con_linear", dict(n=4, l=2, m=4), 2, 16, 4, 8, {"constraint": "linear"}),
    ("lin_con_box", dict(n=4, l=2, m=4), 4, 24, 5, 9, {"constraint": "box"}),
]
NOISE_CASES = [(0, (), (0, 1, 0), (3, 4)), (3, (), (7, 2, 1), (5, 7)), (12345, (7, 2), (1, 4, 2), (8, 33)),
               (2 ** 40 + 5, (1,), (3, 0, 3), (64, 66))]


def _cnn_case(ref):
    pm = problems.product_modules()
    pr = problems.make_cnn_problem(pm, "C1", size=16, n_members=24, horizon=3)
    model = OracleCNN(pr.model)
    w = ref.virtualsys.MpcWeights(r=np.eye(pr.n), q_u=np.eye(pr.l), q_du=np.eye(pr.l),
                                  x_ref=np.ones((pr.n, pr.m)), u_ref=np.zeros((pr.l, pr.m)))
    vs = ref.virtualsys.build_virtual_system(model, w)
    x0 = ref.virtualsys.AugmentedState(pr.x0.x, pr.x0.u, pr.x0.du)
    out, _ = ref.enks.smooth_horizon(x0, vs.reference_observation(), vs, pr.H, pr.N,
                                     ref.matvar.NoiseStreams(seed=1))
    return dict(mean=out, x0=x0.packed)


BURGERS_STEP_CASES = [(12, "boundary", 1), (12, "pointwise", 3), (32, "boundary", 3),
                      (32, "pointwise", 1)]


def _burgers_steps(ref):
    """Reference BurgersDynamics.step (dynamics.py:264-270) on seeded member batches."""
    out = {}
    for k, (g, mode, sub) in enumerate(BURGERS_STEP_CASES):
        cfg = ref.dynamics.BurgersConfig(grid_n=g, control_mode=mode, substeps=sub)
        model = ref.dynamics.BurgersDynamics(cfg)
        rng = np.random.default_rng(100 + k)
        x = np.stack([ref.dynamics.make_initial_field(cfg, s).packed for s in range(3)])
        x = x + 0.05 * rng.standard_normal(x.shape)
        u = rng.standard_normal((3, model.input_rows, g))
        out[f"x{k}"], out[f"u{k}"], out[f"y{k}"] = x, u, model.step(x, u)
    return out


def _burgers_horizon(ref, mode):
    """Reference smooth_horizon (enks.py:256-284) with the reference Burgers model (C1a)."""
    pr = problems.make_burgers_problem(ref, mode)
    out, _ = ref.enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N,
                                     ref.matvar.NoiseStreams(seed=2))
    return dict(mean=out, x0=pr.x0.packed)


VECTOR_CASES = [("vec_m1", dict(n=4, l=1, m=1), 9, 8, 3, 6), ("vec_m2", dict(n=3, l=2, m=2), 12, 16, 4, 5),
                ("vec_m4", dict(n=6, l=3, m=4), 13, 40, 3, 7)]


def _vector_cases(ref):
    """Reference vector_enks_smooth (baselines.py:95-197) on seeded linear problems."""
    import importlib

    base = importlib.import_module("enksmpc.baselines")
    for name, kw, seed, N, h, sseed in VECTOR_CASES:
        _, vs, x0 = problems.make_linear_setup(ref, np.random.default_rng(seed), **kw)
        y = vs.reference_observation()
        mean, rep = base.vector_enks_smooth(x0, y, vs, h, N, ref.matvar.NoiseStreams(seed=sseed))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), mean=mean, x0=x0.packed,
                            obs_cov_entries=rep.obs_cov_entries,
                            cross_cov_entries=rep.cross_cov_entries,
                            jitter_events=rep.jitter_events)


def main():
    ref = problems.reference_modules()
    for name, kw, seed, N, h, sseed, extra in LINEAR_CASES:
        model, vs, x0 = problems.make_linear_setup(ref, np.random.default_rng(seed), **kw)
        if "col_cov" in extra:
            vs = ref.virtualsys.build_virtual_system(model, vs.weights,
                                                     shared_col_cov=extra["col_cov"] * np.eye(x0.m))
        if "constraint" in extra:
            con = problems.make_constraint(ref, extra["constraint"], x0.n, x0.l, x0.m)
            vs = ref.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
        y = vs.reference_observation()
        if extra.get("yref_stack"):
            y = np.stack([y + 0.1 * k for k in range(h)])
        out, cov = ref.enks.smooth_horizon(x0, y, vs, h, N, ref.matvar.NoiseStreams(seed=sseed),
                                           track_cov=bool(extra.get("track_cov")))
        payload = dict(mean=out, x0=x0.packed, y=np.asarray(y))
        if cov is not None:
            payload.update(sigma_traj=cov.sigma_traj, sigma_pred=cov.sigma_pred,
                           sigma_cross=cov.sigma_cross)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **payload)
    np.savez_compressed(os.path.join(HERE, "cnn_c1_16.npz"), **_cnn_case(ref))
    # closed-form oracle of reference test_enks.py:177-186 (baselines.exact_linear_smoother)
    import importlib

    base = importlib.import_module("enksmpc.baselines")
    _, vs, x0 = problems.make_linear_setup(ref, np.random.default_rng(11), n=4, l=1, m=1)
    np.savez_compressed(os.path.join(HERE, "exact_lin_4x1x1.npz"), x0=x0.packed,
                        exact=base.exact_linear_smoother(x0, vs, h=3))
    np.savez_compressed(os.path.join(HERE, "burgers_steps.npz"), **_burgers_steps(ref))
    for mode in ("boundary", "pointwise"):
        np.savez_compressed(os.path.join(HERE, f"burgers_c1a_{mode}.npz"),
                            **_burgers_horizon(ref, mode))
    _vector_cases(ref)
    noise = {}
    for k, (seed, prefix, ids, shape) in enumerate(NOISE_CASES):
        st = ref.matvar.NoiseStreams(seed=seed, prefix=prefix)
        noise[f"z{k}"] = st.substream(*ids).standard_normal(shape)
    np.savez_compressed(os.path.join(HERE, "noise.npz"), **noise)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
