#!/usr/bin/env python
"""Measured per-rank kernel time + modelled collectives for member sharding over R GPUs.

Only one B200 is available in this run, so the R-GPU horizon is modelled from MEASURED pieces:
rank 0 of an R-rank job is run for real on the one GPU (engine.SimComm: N/R members, exactly
the per-rank launches, every collective replaced by a local scale so the numbers stay sane and
its bytes logged), timed with CUDA events over whole horizons; the collectives are then costed
as alpha + bytes / bw per call (allreduce over NVLink 5 / NVSwitch; defaults alpha = 15 us,
bw = 275 GB/s algorithm bandwidth ~ 480 GB/s bus bandwidth at 8 ranks -- assumptions, stated
in the output).  Efficiency(R) = T(1) / (R * T_model(R)) with T the horizon time (strong scaling).

    python tools/shard_model.py [--config C3] [--ranks 1,2,4,8] [--steps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--members", type=int, default=None)
    ap.add_argument("--horizon", type=int, default=None)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--alpha-us", type=float, default=15.0)
    ap.add_argument("--bw-gbs", type=float, default=275.0)
    ap.add_argument("--graph", action="store_true", help="replay the per-rank horizon as a graph")
    args = ap.parse_args()
    import torch

    from paper_2410_09663_b200 import build, configs, enks
    from paper_2410_09663_b200.engine import SimComm
    import paper_2410_09663_b200 as pkg
    from types import SimpleNamespace

    build.build()
    pm = SimpleNamespace(dynamics=pkg.dynamics, virtualsys=pkg.virtualsys, matvar=pkg.matvar)
    pr = configs.make_cnn_problem(pm, args.config, n_members=args.members, horizon=args.horizon)
    ops = enks._ops()
    st = pm.matvar.NoiseStreams(seed=0)
    yref = ops.to_device(np.broadcast_to(pr.y_ref, (pr.H,) + pr.y_ref.shape).copy())
    rows = []
    base = None
    for R in [int(r) for r in args.ranks.split(",")]:
        comm = SimComm(R)
        if args.graph:
            g = enks.HorizonGraph(pr.x0, pr.vs, pr.H, pr.N, st, comm=comm)
            g.y_refs.copy_(yref)
            run = g.replay
        else:
            def run():
                return enks.smooth_horizon_device(pr.x0, yref, pr.vs, pr.H, pr.N, st, comm=comm)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        comm.log.clear()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            run()
        e.record()
        torch.cuda.synchronize()
        t_rank = s.elapsed_time(e) / 1e3 / args.steps
        per = len(comm.log) // args.steps
        nbytes = sum(b for _, b in comm.log) / args.steps
        t_coll = 0.0 if R == 1 else (per * args.alpha_us * 1e-6 + nbytes / (args.bw_gbs * 1e9))
        t_model = t_rank + t_coll
        if base is None:
            base = t_model if R == 1 else None
        row = {"ranks": R, "members_per_rank": -(-pr.N // R), "rank_horizon_ms": t_rank * 1e3,
               "collectives_per_horizon": per, "collective_bytes_per_horizon": nbytes,
               "collective_ms_model": t_coll * 1e3, "horizon_ms_model": t_model * 1e3,
               "horizons_per_s_model": 1.0 / t_model,
               "efficiency_vs_1": (base / (R * t_model)) if base else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
    out = {"config": args.config, "N": pr.N, "H": pr.H, "graph": args.graph,
           "assumptions": {"alpha_us": args.alpha_us, "bw_gbs": args.bw_gbs,
                           "note": "per-rank kernels measured on one B200 (SimComm); collectives "
                                   "modelled (NCCL over NVLink 5 / NVSwitch)"},
           "rows": rows}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"shard_model_{args.config.lower()}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
