#!/usr/bin/env python
"""The paper's Table 1 shapes on one B200: boundary-controlled
2-D Burgers (packed 2n x n state, l = 2), N = 100 members, H = 5, one OIC horizon solve through
enks.smooth_horizon (eager and graph=True), CUDA-event timed.  The paper's A100 column used a
trained PhyCRNet surrogate (not in the reference); here the reference's own Burgers FD model is the
forecast, so the rows are a context point, not a like-for-like comparison.

    python tools/table1.py [--sizes 64,80,128,200] [--steps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAPER_A100_S = {64: 0.42, 80: 0.51, 128: 0.954, 200: 2.097}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,80,128,200")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from types import SimpleNamespace

    import paper_2410_09663_b200 as pkg
    from paper_2410_09663_b200 import build, configs, enks

    build.build()
    pm = SimpleNamespace(dynamics=pkg.dynamics, virtualsys=pkg.virtualsys, matvar=pkg.matvar)
    rows = []
    for g in [int(s) for s in args.sizes.split(",")]:
        pr = configs.make_burgers_problem(pm, "boundary", grid_n=g, n_members=100, horizon=5)
        st = pm.matvar.NoiseStreams(seed=0)
        out = {"grid": f"2x{g}x{g}", "n": pr.n, "m": pr.m, "l": pr.l, "N": pr.N, "H": pr.H,
               "paper_a100_s": PAPER_A100_S.get(g)}
        for graph in (False, True):
            for _ in range(3):
                enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st, graph=graph)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.steps):
                enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, st, graph=graph)
            e.record()
            torch.cuda.synchronize()
            sec = s.elapsed_time(e) / 1e3 / args.steps
            out["graph_s" if graph else "eager_s"] = sec
        out["peak_mem_gb"] = torch.cuda.max_memory_allocated() / 1e9
        rows.append(out)
        print(json.dumps(out), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "table1.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
