"""Reference arm / CPU baseline (bench.py only): time the UNMODIFIED reference smoother.

The reference (``enksmpc``, pure Python + NumPy/SciPy) is installed untouched into
baseline/_ref by __graft_entry__.install_reference().  Its smoother is driven through its own
public API -- ``enksmpc.enks.init_ensemble / predict / update`` (enks.py:105-253) with its own
``VirtualSystem``, ``MpcWeights``, ``AugmentedState`` and ``NoiseStreams`` -- on the benchmark
problem.  The reference ships no CNN, so its MatrixDynamics seam
(dynamics.py:40-50) gets the fp64 torch-CPU conv stack of oracle.models (the same surrogate the
device runs).  Nothing from the product package is on this path.

A full C3 horizon takes the reference about an hour, so a bench step times predict+update at a
given trajectory length T (slices before the predict); the horizon time is the sum over
T = 1..H of a + b T fitted to those samples.  The linear model is validated against a complete
measured C3 horizon (tools/reference_c3_full.py -> profiles/r02/reference_c3_full.json).
"""
from __future__ import annotations

import os
import subprocess
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def reference_modules():
    """The installed reference (None when baseline/_ref is missing)."""
    if not os.path.isdir(os.path.join(REF_INSTALL, "enksmpc")):
        return None
    from . import problems

    return problems.reference_modules(REF_INSTALL)


def cpu_topology() -> dict:
    """Sockets x physical cores of this host (lscpu), and the logical CPU count."""
    info = {"logical": os.cpu_count() or 1}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {k.strip(): v.strip() for k, _, v in (ln.partition(":") for ln in out.splitlines())}
        sockets = int(kv.get("Socket(s)", "1"))
        per = int(kv.get("Core(s) per socket", "0"))
        info.update(sockets=sockets, cores_per_socket=per, physical=sockets * per or info["logical"],
                    model=kv.get("Model name", ""))
    except (OSError, ValueError, subprocess.SubprocessError):
        info["physical"] = info["logical"]
    return info


def make_problem(rm, config: str, n_members=None, horizon=None):
    """The benchmark problem built from the reference's own types + the fp64 CNN surrogate."""
    from paper_2410_09663_b200.configs import CONFIGS, sine_field

    from .models import CnnSpec, OracleCNN

    n, N, H, widths = CONFIGS[config]
    N = n_members or N
    H = horizon or H
    m = l = n
    model = OracleCNN(CnnSpec(n, m, widths, alpha=0.1, seed=0), backend="torch")
    vsm = rm.virtualsys
    weights = vsm.MpcWeights(r=np.eye(n), q_u=np.eye(l), q_du=np.eye(l), x_ref=np.ones((n, m)),
                             u_ref=np.zeros((l, m)), scale=1.0)
    vs = vsm.build_virtual_system(model, weights)
    x0 = vsm.AugmentedState(sine_field(n, m, 0), np.zeros((l, m)), np.zeros((l, m)))
    from types import SimpleNamespace

    return SimpleNamespace(vs=vs, x0=x0, n=n, l=l, m=m, N=N, H=H, widths=tuple(widths),
                           y_ref=vs.reference_observation(), model=model)


class threads:
    """Context: BLAS (threadpoolctl) and torch intra-op threads limited to `n`."""

    def __init__(self, n: int):
        self.n = int(n)

    def __enter__(self):
        import torch
        from threadpoolctl import threadpool_limits

        self._torch = torch.get_num_threads()
        torch.set_num_threads(self.n)
        self._tp = threadpool_limits(limits=self.n)
        return self

    def __exit__(self, *exc):
        import torch

        self._tp.restore_original_limits()
        torch.set_num_threads(self._torch)


def time_step(rm, pr, T: int, seed: int = 0) -> float:
    """Seconds for one reference predict + update starting from a T-slice trajectory (t = T-1),
    i.e. step T of a horizon (enks.py:156-253).  Slices 1..T-1 are synthetic member spread."""
    ens = rm.enks.init_ensemble(pr.x0, pr.N, shared_col_cov=pr.vs.shared_col_cov)
    if T > 1:
        d = pr.x0.n + 2 * pr.x0.l
        rng = np.random.default_rng(seed)
        extra = pr.x0.packed[None, None] + 0.1 * rng.standard_normal((pr.N, T - 1, d, pr.m))
        ens.members = np.concatenate([ens.members, extra.reshape(pr.N, (T - 1) * d, pr.m)],
                                     axis=1)
        ens.t = T - 1
        ens.mean = ens.members.mean(axis=0)
    streams = rm.matvar.NoiseStreams(seed=seed)
    t0 = time.perf_counter()
    rm.enks.predict(ens, pr.vs, streams)
    rm.enks.update(ens, pr.y_ref, pr.vs, streams)
    dt = time.perf_counter() - t0
    del ens
    return dt


def fit_horizon(samples, H: int):
    """(horizon seconds, a, b) from [(T, seconds)] with the linear per-step model a + b T."""
    Ts = np.array([s[0] for s in samples], float)
    ys = np.array([s[1] for s in samples], float)
    if len(set(Ts.tolist())) >= 2:
        b, a = np.polyfit(Ts, ys, 1)
        b = max(float(b), 0.0)
        a = float(a)
    else:
        a, b = float(ys.mean()), 0.0
    return float(sum(a + b * T for T in range(1, H + 1))), a, b
