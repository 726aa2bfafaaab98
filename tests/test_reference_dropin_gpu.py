"""Drop-in proof with the reference's OWN objects and its OWN test file.

The unmodified reference package is installed by __graft_entry__.build() into baseline/_ref
(git-ignored; it travels to the GPU box, /root/reference does not).  Two checks:

* the product's smooth_horizon / init_ensemble / predict / update driven by enksmpc's own
  VirtualSystem, AugmentedState, NoiseStreams (incl. child prefixes), LinearDynamics and
  BurgersDynamics equals enksmpc.enks.smooth_horizon run on the same objects (fp64, CPU);
* /root/reference/pkg/tests/test_enks.py itself, run in a subprocess with the INTEGRATION.md shim
  ``sys.modules["enksmpc.enks"] = paper_2410_09663_b200.enks`` -- so every smoother call in the
  reference's suite lands on the B200 path -- with its fp64 tolerances relaxed to fp32 ones
  (FP32_RELAX below; nothing else in the file is touched).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.reference]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TOL = 1e-4

# fp64 -> fp32 tolerance relaxations applied to the reference's test_enks.py (text substitution).
# The reference asserts 1e-12 / 1e-10 / atol=1e-9 on O(1..10) values computed in fp64; the
# device computes in fp32 (north_star: relative error <= 1e-4), so those become 1e-4 absolute.
# Bit-identity (np.array_equal), shapes, lambda, jitter counts and the 5 % statistical checks
# are unchanged.
# The PSD check's -1e-8 tr(Sigma) floor is below fp32 resolution of a Gram matrix (eigenvalue
# error ~ eps_fp32 * ||Sigma||), so it becomes -1e-6 tr(Sigma).
FP32_RELAX = [("< 1e-12", "< 1e-4"), ("rel < 1e-10", "rel < 1e-4"), ("atol=1e-12", "atol=1e-4"),
              ("atol=1e-9", "atol=1e-4"), ("> -1e-8 * np.trace", "> -1e-6 * np.trace")]


def _ref_mods():
    if not os.path.isdir(os.path.join(REF, "enksmpc")):
        pytest.skip("reference not installed in baseline/_ref (run __graft_entry__.build())")
    from oracle import problems

    return problems.reference_modules(REF)


def _rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("seed,kw,N,h", [
    (0, dict(n=4, l=2, m=3), 16, 5),
    (2, dict(n=16, l=8, m=16), 64, 6),
])
def test_reference_objects_linear(seed, kw, N, h):
    from oracle import problems
    from paper_2410_09663_b200 import enks

    rm = _ref_mods()
    _, vs, x0 = problems.make_linear_setup(rm, np.random.default_rng(seed), **kw)
    y = vs.reference_observation()
    for streams in (rm.matvar.NoiseStreams(seed=seed + 3),
                    rm.matvar.NoiseStreams(seed=seed + 3).child(7)):
        ref, _ = rm.enks.smooth_horizon(x0, y, vs, h, N, streams)
        got, _ = enks.smooth_horizon(x0, y, vs, h, N, streams)
        assert got.shape == ref.shape
        assert _rel(got, ref) < TOL
    # the step-wise API on reference objects, with an update before the first predict
    ens_r = rm.enks.init_ensemble(x0, N, shared_col_cov=vs.shared_col_cov)
    ens_g = enks.init_ensemble(x0, N, shared_col_cov=vs.shared_col_cov)
    st = rm.matvar.NoiseStreams(seed=seed)
    for op in ("u", "p", "u", "p", "p", "u", "u"):
        if op == "p":
            rm.enks.predict(ens_r, vs, st)
            enks.predict(ens_g, vs, st)
        else:
            rm.enks.update(ens_r, y, vs, st)
            enks.update(ens_g, y, vs, st)
        assert ens_g.t == ens_r.t
        assert _rel(ens_g.members, ens_r.members) < TOL, op
        assert _rel(ens_g.mean, ens_r.mean) < TOL, op
    assert ens_g.jitter_events == ens_r.jitter_events


@pytest.mark.parametrize("mode", ["boundary", "pointwise"])
def test_reference_objects_burgers(mode):
    """The SPEC reference problem (C1a) built from enksmpc's own BurgersDynamics."""
    from oracle import problems
    from paper_2410_09663_b200 import enks

    rm = _ref_mods()
    pr = problems.make_burgers_problem(rm, mode, horizon=3)
    st = rm.matvar.NoiseStreams(seed=2)
    ref, _ = rm.enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st)
    got, _ = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st)
    assert _rel(got, ref) < TOL
    n, l = pr.n, pr.l
    assert _rel(got[:, n:n + l], ref[:, n:n + l]) < TOL


def test_reference_test_enks_through_shim(tmp_path):
    """The reference's own pkg/tests/test_enks.py, unmodified except FP32_RELAX, against the
    B200 smoother through the INTEGRATION.md sys.modules shim."""
    _ref_mods()
    src = os.path.join(REF, "enksmpc_tests", "test_enks.py")
    if not os.path.exists(src):
        pytest.skip("reference tests not copied into baseline/_ref/enksmpc_tests")
    text = open(src).read()
    for a, b in FP32_RELAX:
        assert a in text, a
        text = text.replace(a, b)
    (tmp_path / "test_enks_fp32.py").write_text(text)
    (tmp_path / "conftest.py").write_text(
        "import sys\n"
        f"sys.path[:0] = [{REF!r}, {ROOT!r}]\n"
        "import paper_2410_09663_b200.enks as b200_enks\n"
        "import enksmpc\n"
        "sys.modules['enksmpc.enks'] = b200_enks   # INTEGRATION.md shim\n"
        "enksmpc.enks = b200_enks\n"
        "def pytest_sessionfinish(session, exitstatus):\n"
        "    import enksmpc.baselines as b\n"
        "    assert b.CH_W == b200_enks.CH_W\n"
        "    print('SHIM_ACTIVE', sys.modules['enksmpc.enks'].__name__)\n")
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-s", "-p", "no:cacheprovider",
                          str(tmp_path)], capture_output=True, text=True, cwd=str(tmp_path),
                         timeout=1200)
    out = res.stdout + res.stderr
    print(out[-3000:])
    assert res.returncode == 0, out[-3000:]
    assert "SHIM_ACTIVE paper_2410_09663_b200.enks" in out
    assert " passed" in out and "failed" not in out
