#!/usr/bin/env python
"""Horizons/s of smooth_horizon(track_cov=True) next to track_cov=False (both eager, host inputs
and host results, CUDA events) at C2 and C3 -- SURVEY §8 f3 "covariances at scale".  The tracked
run also materialises Sigma_traj ((T d)^2 fp64 on the host: 4032^2 at C2, 19584^2 = 3.1 GB at C3).

    python tools/trackcov_bench.py [--configs C2,C3] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from types import SimpleNamespace

    import paper_2410_09663_b200 as pkg
    from paper_2410_09663_b200 import build, configs, enks

    build.build()
    pm = SimpleNamespace(dynamics=pkg.dynamics, virtualsys=pkg.virtualsys, matvar=pkg.matvar)
    rows = []
    for cfg in args.configs.split(","):
        pr = configs.make_cnn_problem(pm, cfg)
        st = pm.matvar.NoiseStreams(seed=0)
        out = {"config": cfg, "n": pr.n, "N": pr.N, "H": pr.H, "traj_rows": (pr.H + 1) * (pr.n + 2 * pr.l)}
        for track in (False, True):
            def run():
                mean, cov = enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st,
                                                track_cov=track)
                if cov is not None:
                    _ = cov.sigma_traj, cov.sigma_cross, cov.sigma_pred  # host copies
                return mean
            run()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                run()
            torch.cuda.synchronize()
            sec = (time.perf_counter() - t0) / args.steps
            out["track_cov" if track else "plain"] = {"s_per_horizon": sec, "horizons_per_s": 1 / sec}
        rows.append(out)
        print(json.dumps(out), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "trackcov_bench.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
