#!/usr/bin/env python
"""One complete C3 horizon (128x128, CNN 2-32-32-1, N=1024, H=50) of the UNMODIFIED reference
next to the B200 smoother on the same seeds, inputs and noise.

    python tools/reference_c3_full.py [--config C3] [--horizon 50] [--out gpurun_out/...json]

* reference: enksmpc (baseline/_ref) init_ensemble + H x (predict, update), fp64, all physical
  cores (BLAS + torch threads), the fp64 torch-CPU CNN as its MatrixDynamics; every step timed.
  This measures the reference's full horizon (no extrapolation) and validates the a + b T
  per-step model bench.py's reference arm fits on T <= 12 (oracle/refrun.py).
* device: enks.smooth_horizon eager and graph=True on cuda:0 with the reference's own
  NoiseStreams; relative errors (max |dev - ref| / max |ref|) over the mean trajectory and its
  X / U / dU blocks.
Runs on the GPU box (196 GB host RAM: the fp64 reference peaks near 65 GB at C3).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--horizon", type=int, default=None)
    ap.add_argument("--members", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "reference_c3_full.json"))
    args = ap.parse_args()

    from oracle import refrun

    rm = refrun.reference_modules()
    assert rm is not None, "baseline/_ref missing: run __graft_entry__.build() in the container"
    pr = refrun.make_problem(rm, args.config, args.members, args.horizon)
    topo = refrun.cpu_topology()
    cores = topo["physical"]
    res = {"config": args.config, "n": pr.n, "N": pr.N, "H": pr.H, "widths": list(pr.widths),
           "cores": cores, "topology": topo, "seed": args.seed}

    # ---- device first (fast), then the long reference run
    import torch

    from paper_2410_09663_b200 import build, enks

    build.build()
    pm_streams = rm.matvar.NoiseStreams(seed=args.seed)
    from paper_2410_09663_b200 import configs
    from types import SimpleNamespace

    import paper_2410_09663_b200 as pkg

    pm = SimpleNamespace(dynamics=pkg.dynamics, virtualsys=pkg.virtualsys, matvar=pkg.matvar)
    dpr = configs.make_cnn_problem(pm, args.config, n_members=pr.N, horizon=pr.H)
    assert np.array_equal(dpr.x0.packed, pr.x0.packed) and np.array_equal(dpr.y_ref, pr.y_ref)
    for w, v in zip(dpr.model.weights + dpr.model.biases, pr.model.weights + pr.model.biases):
        assert np.array_equal(w, v)
    t0 = time.perf_counter()
    got, _ = enks.smooth_horizon(dpr.x0, dpr.y_ref, dpr.vs, pr.H, pr.N, pm_streams)
    res["device_eager_s_incl_first_call"] = time.perf_counter() - t0
    got_g, _ = enks.smooth_horizon(dpr.x0, dpr.y_ref, dpr.vs, pr.H, pr.N, pm_streams, graph=True)
    res["graph_equals_eager"] = bool(np.array_equal(got, got_g))
    enks._GRAPHS.clear()
    torch.cuda.empty_cache()

    # ---- the reference, every step timed
    steps = []
    with refrun.threads(cores):
        t_start = time.perf_counter()
        ens = rm.enks.init_ensemble(pr.x0, pr.N, shared_col_cov=pr.vs.shared_col_cov)
        for k in range(pr.H):
            ts = time.perf_counter()
            rm.enks.predict(ens, pr.vs, pm_streams)
            tp = time.perf_counter()
            rm.enks.update(ens, pr.y_ref, pr.vs, pm_streams)
            te = time.perf_counter()
            steps.append({"T": k + 1, "predict_s": tp - ts, "update_s": te - tp, "step_s": te - ts})
            print(f"step {k + 1}/{pr.H}: {te - ts:.2f} s", flush=True)
        ref = ens.slices()
        res["horizon_s"] = time.perf_counter() - t_start
    del ens
    res["steps"] = steps
    Ts = np.array([s["T"] for s in steps], float)
    ys = np.array([s["step_s"] for s in steps], float)
    sel = Ts <= 12
    horizon_fit, a, b = refrun.fit_horizon(list(zip(Ts[sel], ys[sel])), pr.H)
    res.update(fit_T_le_12_horizon_s=horizon_fit, fit_a=a, fit_b=b,
               fit_error=horizon_fit / res["horizon_s"] - 1.0)
    b_all, a_all = np.polyfit(Ts, ys, 1)
    res.update(fit_all_a=float(a_all), fit_all_b=float(b_all))
    with refrun.threads(1):
        res["single_thread_step_T1_s"] = refrun.time_step(rm, pr, 1)

    def rel(x, y):
        return float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-30))

    n, l = pr.n, pr.l
    res["rel_err"] = {"all": rel(got, ref), "X": rel(got[:, :n], ref[:, :n]),
                      "U": rel(got[:, n:n + l], ref[:, n:n + l]),
                      "dU": rel(got[:, n + l:], ref[:, n + l:]),
                      "per_slice_all": [rel(got[t], ref[t]) for t in range(pr.H + 1)]}
    res["tolerance"] = 1e-4
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savez_compressed(args.out.replace(".json", "_means.npz"), reference=ref, device=got)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "steps"}))


if __name__ == "__main__":
    main()
