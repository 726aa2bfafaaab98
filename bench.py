#!/usr/bin/env python
"""Benchmark: OIC horizon solves/sec (and member-CNN-steps/sec) of the B200 EnKS.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One bench "step" = one complete OIC horizon solve (reference enks.py:256-284
smooth_horizon: init + H x (predict, update)) of the configured problem
(default C3: 128x128 field, CNN 2-32-32-1, N=1024 members,
H=50), synthetic inputs, random-init CNN.

  value : horizons/s with inputs resident in HBM, CUDA-event timed (max over ranks); on one
          GPU the horizon is replayed as one CUDA graph (smooth_horizon(graph=True): the same
          kernels as the eager path, without per-launch host cost; --no-graph times eager)
  e2e   : the same metric through the public API enks.smooth_horizon (default eager call) with
          host (NumPy) inputs and the host result each step; e2e_graph: same with graph=True
  kernels : per-kernel-family CUDA-event brackets of one extra eager horizon (untimed)
  roofline : the dominant kernel (the cross-moment contraction P = [A; Yc] Yc^T)
          algorithmic FLOPs / its CUDA-event-measured launch time vs MEASURED_PEAKS.json
  cpu_baseline : the UNMODIFIED reference (enksmpc installed in baseline/_ref) timed on this
          host's physical cores on a bounded sample (rank 0, N=1 only), horizon time from the
          a + b T per-step model (oracle/refrun.py), plus one single-thread step

N > 1 (torchrun, or --gpus N re-executes itself under torchrun): members sharded over ranks,
NCCL allreduce of the covariance partials; strong scaling of one horizon.  --impl reference times
the unmodified reference on the host CPU (rank 0 prints; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--members", type=int, default=None)
    ap.add_argument("--horizon", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="(default on 1 GPU) time replays of a CUDA graph of the horizon -- "
                         "smooth_horizon(graph=True), the same kernels as the eager path")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time the eager path (one host launch per kernel)")
    return ap.parse_args()


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _tf32_peak():
    """Measured cuBLAS TF32 peak (tools/tf32_peak.py, committed under profiles/), or None."""
    for rnd in ("r02",):
        path = os.path.join(ROOT, "profiles", rnd, "tf32_peak.json")
        if os.path.exists(path):
            with open(path) as f:
                d = json.load(f)
            d["source"] = os.path.relpath(path, ROOT)
            return d
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _modules():
    from types import SimpleNamespace

    import paper_2410_09663_b200 as pkg

    return SimpleNamespace(dynamics=pkg.dynamics, virtualsys=pkg.virtualsys, matvar=pkg.matvar)


def _problem(config: str, members, horizon):
    from paper_2410_09663_b200 import configs  # synthetic inputs (shapes per SURVEY.md §8d)

    pm = _modules()
    return pm, configs.make_cnn_problem(pm, config, n_members=members, horizon=horizon)


def _algorithmic(pr):
    n, l, m, N, H = pr.n, pr.l, pr.m, pr.N, pr.H
    d, p, K = n + 2 * l, n + l, N * m
    cnn_flops = N * H * pr.model.flops_per_member_step()
    # P = [A_1..A_tau; Yc_1..Yc_tau] Yc_tau^T per step; A keeps the [X; dU] rows of each slice
    # under the derived-U chain (engine.py, U = prefix sums of dU), else all d rows
    ds = n + l if os.environ.get("ENKS_UCHAIN", "1") != "0" else d
    cross = sum(2 * tau * (ds + p) * p * K for tau in range(1, H + 1))
    enks_ref = sum(2 * p * p * K + 4 * (t + 1) * d * p * K + p ** 3 / 3 + 2 * p * p * (t + 1) * d
                   for t in range(1, H + 1))
    return dict(cnn_tflop=cnn_flops / 1e12, cross_tflop=cross / 1e12, enks_ref_tflop=enks_ref / 1e12)


# ---------------------------------------------------------------------- reference arm
def _ref_timer(config, members, horizon):
    """(modules, problem, kind) of the CPU path timed: the installed unmodified reference
    (baseline/_ref, kind "reference") or, if it is missing, the fp64 oracle port ("port")."""
    from oracle import refrun

    rm = refrun.reference_modules()
    if rm is not None:
        return rm, refrun.make_problem(rm, config, members, horizon), "reference"
    from types import SimpleNamespace

    from oracle import enks_oracle

    port = SimpleNamespace(enks=SimpleNamespace(
        init_ensemble=lambda x0, N, shared_col_cov=None: enks_oracle.oracle_init(
            x0.packed, x0.n, x0.l, N, shared_col_cov=shared_col_cov),
        predict=lambda e, vs, st: enks_oracle.oracle_predict(e, vs, st.seed, tuple(st.prefix),
                                                             backend="c"),
        update=lambda e, y, vs, st: enks_oracle.oracle_update(e, y, vs, st.seed, tuple(st.prefix),
                                                              backend="c")))
    pm = _modules()
    port.matvar = pm.matvar
    pr = refrun.make_problem(pm, config, members, horizon)
    return port, pr, "port"


def run_reference(args):
    """--impl reference: the UNMODIFIED reference smoother (enksmpc from baseline/_ref, fp64,
    NumPy/SciPy/OpenBLAS + the fp64 torch-CPU CNN) on all physical cores of this host, rank 0
    only.  Each step times one predict+update at trajectory length T (cycling T_SAMPLES); the
    horizon time is sum_{T=1..H} (a + b T) fitted over the timed steps (oracle/refrun.py)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import refrun

    rm, pr, kind = _ref_timer(args.config, args.members, args.horizon)
    topo = refrun.cpu_topology()
    cores = topo["physical"]
    ts = [t for t in T_SAMPLES if t <= pr.H] or [1]
    samples = []
    with refrun.threads(cores):
        for k in range(args.warmup + args.steps):
            T = ts[k % len(ts)]
            dt = refrun.time_step(rm, pr, T, seed=k)
            if k >= args.warmup:
                samples.append((T, dt))
    horizon, a, b = refrun.fit_horizon(samples, pr.H)
    value = 1.0 / horizon
    line = {
        "impl": "reference", "metric": "OIC horizon solves/sec", "value": value,
        "unit": "horizons/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": horizon * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(pr, args, world=1),
        "member_cnn_steps_per_s": pr.N * pr.H * value,
        "cpu_baseline": {"value": value, "unit": "horizons/s", "cores": cores, "kind": kind,
                         "topology": topo,
                         "sample": f"unmodified enksmpc.enks predict+update (baseline/_ref) with the "
                                   f"fp64 torch-CPU CNN, {cores} threads (BLAS + torch), at "
                                   f"T={[s[0] for s in samples]} "
                                   f"({[round(s[1], 2) for s in samples]} s) of {args.config} "
                                   f"(N={pr.N}); horizon = sum_(T=1..{pr.H}) (a + b T), "
                                   f"a={a:.3f} s, b={b:.3f} s"
                                   + ("" if kind == "reference" else " [reference not installed: "
                                      "fp64 oracle port]")},
        "fit_validation": _fit_validation(args.config),
        "e2e": {"value": value, "unit": "horizons/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


T_SAMPLES = (1, 4, 8, 12)


def _fit_validation(config):
    """The committed full-horizon reference measurement that validates the a + b T model."""
    path = os.path.join(ROOT, "profiles", "r02", f"reference_{config.lower()}_full.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return {"source": os.path.relpath(path, ROOT), "measured_horizon_s": d.get("horizon_s"),
            "fit_from_T_le_12_s": d.get("fit_T_le_12_horizon_s"), "cores": d.get("cores")}


def cpu_baseline(config, members, horizon):
    """Our arm's cpu_baseline: the unmodified reference at T = 1 and 8 on all physical cores
    (horizon by the a + b T model), plus one single-thread step at T = 1 (~30 s in all)."""
    from oracle import refrun

    rm, pr, kind = _ref_timer(config, members, horizon)
    topo = refrun.cpu_topology()
    cores = topo["physical"]
    with refrun.threads(cores):
        samples = [(T, refrun.time_step(rm, pr, T)) for T in (1, 8) if T <= pr.H] or \
            [(1, refrun.time_step(rm, pr, 1))]
    with refrun.threads(1):
        one = refrun.time_step(rm, pr, 1)
    horizon_s, a, b = refrun.fit_horizon(samples, pr.H)
    return {"value": 1.0 / horizon_s, "unit": "horizons/s", "cores": cores, "kind": kind,
            "topology": topo,
            "sample": f"unmodified enksmpc.enks predict+update at T={[s[0] for s in samples]} "
                      f"({[round(s[1], 2) for s in samples]} s, {cores} threads) of {config}; "
                      f"horizon = sum_T (a + b T), a={a:.3f} s, b={b:.3f} s",
            "single_thread_step_T1_s": one, "step_T1_s": samples[0][1]}


def _config(pr, args, world):
    return {"workload": f"{args.config}: OIC horizon solve, {pr.n}x{pr.m} field, "
                        f"CNN {'-'.join(map(str, pr.widths))}, N={pr.N} members, H={pr.H}",
            "n": pr.n, "m": pr.m, "l": pr.l, "members": pr.N, "horizon": pr.H,
            "cnn_widths": list(pr.widths),
            "parallelism": f"members sharded over {world} rank(s)" if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (append-only basis >> 126 MB at C2/C3)"}


# ---------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2410_09663_b200.engine import TorchComm

        comm = TorchComm()
    from paper_2410_09663_b200 import build, enks

    build.build()
    pm, pr = _problem(args.config, args.members, args.horizon)
    ops = enks._ops()
    if comm is not None:
        enks.set_default_comm(comm)
    streams = pm.matvar.NoiseStreams(seed=0)
    h = pr.H
    yref_dev = ops.to_device(np.broadcast_to(pr.y_ref, (h,) + pr.y_ref.shape).copy())

    # --graph (1 GPU): the horizon is one CUDA graph (all kernels of the eager path, replayed)
    graph = None
    # a captured horizon keeps its own engine; the extra profiled horizon and the e2e path need
    # room for another one, so very large problems (C4) run eager
    n, l, m = pr.n, pr.l, pr.m
    est = 4.4 * ((h + 1) * (n + l) + h * (n + l)) * pr.N * m  # fp16-pair basis + gains, bytes
    fits = est < 0.3 * torch.cuda.get_device_properties(local).total_memory
    if args.graph and fits:
        try:  # multi-rank: the NCCL collectives are captured inside the horizon graph
            graph = enks.HorizonGraph(pr.x0, pr.vs, h, pr.N, streams)
            graph.y_refs.copy_(yref_dev)
        except RuntimeError as exc:  # a backend that cannot be captured: time eager launches
            if world == 1:
                raise
            sys.stderr.write(f"bench.py: horizon graph capture failed ({exc}); eager\n")
            graph = None
            torch.cuda.synchronize()

    def one_step():
        if graph is not None:
            return graph.replay()
        return enks.smooth_horizon_device(pr.x0, yref_dev, pr.vs, h, pr.N, streams, comm=comm)

    for _ in range(args.warmup):
        eng = one_step()
        del eng
    torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ops.launches
    ops.profile = None  # no event brackets inside the timed region
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    for _ in range(args.steps):
        eng = one_step()
        del eng
    stop.record()
    torch.cuda.synchronize()
    prof, ops.profile = ops.profile, None
    clk = clocks.stop()
    launches = (ops.launches - launches0) // max(args.steps, 1)
    # one extra eager horizon, outside the timed region, for the per-kernel breakdown (CUDA-event
    # brackets on the launching streams)
    torch.cuda.empty_cache()
    l0 = ops.launches
    ops.profile = []
    enks.smooth_horizon_device(pr.x0, yref_dev, pr.vs, h, pr.N, streams, comm=comm)
    torch.cuda.synchronize()
    prof, ops.profile = ops.profile, None
    if graph is not None:
        launches = ops.launches - l0
    prof_steps = 1
    elapsed = start.elapsed_time(stop) / 1e3
    cross = [(s, e, f) for tag, s, e, f in prof if tag == "cross"]
    kern_s = sum(s.elapsed_time(e) for s, e, _ in cross) / 1e3
    kern_flops = sum(f for _, _, f in cross)
    n_kern = len(cross)
    if comm is not None:
        t = torch.tensor([elapsed, kern_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, kern_s = float(t[0]), float(t[1])
    value = args.steps / elapsed

    # e2e through the public API with host inputs and a host result each step: the default eager
    # smooth_horizon(...) (the call a reference user makes) is the headline, graph=True beside it
    e2e = e2e_graph = None
    if not args.no_e2e:
        e2e = _e2e(args, enks, ops, pr, streams, comm, graph=False)
        if graph is not None:
            e2e_graph = _e2e(args, enks, ops, pr, streams, comm, graph=True)

    peaks, peak_kind = _peaks()
    alg = _algorithmic(pr)
    achieved = (kern_flops / max(kern_s, 1e-12)) / 1e12
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    traffic, traffic_note = None, None
    tpath = next((q for q in (os.path.join(ROOT, "profiles", r, "roofline_traffic.json")
                              for r in ("r02", "r01")) if os.path.exists(q)), "")
    if tpath:
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes")
        traffic_note = {"launch": tj.get("launch"), "algorithmic_bytes": tj.get("algorithmic_bytes"),
                        "source": tj.get("source")}
    roofline = {
        "kernel": "cross-moment contraction P=[A;Yc]Yc^T (tcgen05 kind::f16 on fp16-pair "
                  "operands, CTA-pair f16p_gemm_pair_kernel)",
        "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak, "traffic": traffic, "traffic_capture": traffic_note,
        "peak_source": f"{peak_kind} bf16_tflops_sustained (MEASURED_PEAKS.json)",
        "launches_timed": n_kern, "kernel_share_of_step": kern_s / prof_steps / (elapsed / args.steps),
        "algorithmic_tflop_per_horizon": alg["cross_tflop"],
        "mma_work_frac": 3.0 * achieved / peak,
        "note": "achieved counts algorithmic flops (2 M N K); the kernel issues three kind::f16 "
                "MMAs (lo*hi, hi*lo, hi*hi) per algorithmic product for fp32-level accuracy, so "
                "the tensor pipe does mma_work_frac of the sustained peak",
    }
    # per-kernel-family breakdown (CUDA events around every tagged op of the timed region)
    hbm = float(peaks.get("hbm_gbs", 6536.0))
    fam = {}
    for tag, s_, e_, w in prof:
        t = s_.elapsed_time(e_) / 1e3
        f = fam.setdefault(tag, [0.0, 0.0, 0])
        f[0] += t
        f[1] += w
        f[2] += 1
    kinds = {"cross": ("tensor", "TFLOP/s"), "forecast": ("tensor", "TFLOP/s"),
             "correction": ("tensor", "TFLOP/s"), "gain": ("tensor", "TFLOP/s"),
             "mean": ("tensor", "TFLOP/s"),
             "shift": ("hbm", "GB/s"), "noise": ("issue", "Gnormal/s"), "stats": ("hbm", "GB/s"),
             "gain_solve": ("latency", "TFLOP/s")}
    # the newest-slice shift last = C0 + bias - G_tt Yc^T streams C0 (q x K fp32), the transposed
    # Yc pair planes (K x p, 2 x fp16) and writes last (q x K fp32): HBM-bound, reported in bytes
    q, K = pr.n + pr.l, pr.N * pr.m
    shift_bytes = (4 * q * K + 4 * K * (pr.n + pr.l) + 4 * q * K) * h
    tf32 = _tf32_peak()
    three_tf32 = {"correction", "gain", "mean"}  # 3xTF32 MMAs (gemm_tc.cu)
    kernels = {}
    for tag, (t, w, cnt) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        bound, unit = kinds.get(tag, ("?", "?"))
        if tag == "shift":
            w = shift_bytes * prof_steps
        rate = w / max(t, 1e-12) / (1e12 if unit == "TFLOP/s" else 1e9)
        pk = peak if bound == "tensor" else (hbm if bound == "hbm" else None)
        kernels[tag] = {"ms_per_horizon": t / prof_steps * 1e3,
                        "share": t / prof_steps / (elapsed / args.steps),
                        "launches": cnt // max(prof_steps, 1), "achieved": rate, "unit": unit,
                        "bound": bound, "peak": pk, "frac": (rate / pk) if pk else None}
        if tag in three_tf32 and tf32:
            # algorithmic flops against the 3xTF32 ceiling (three TF32 MMAs per product)
            kernels[tag]["peak_3xtf32"] = tf32["tf32_tflops_sustained"] / 3.0
            kernels[tag]["frac_3xtf32"] = rate / kernels[tag]["peak_3xtf32"]
            kernels[tag]["peak_3xtf32_source"] = tf32["source"]
    if "forecast" in kernels:
        kf = kernels["forecast"]
        kf["member_steps_per_s"] = pr.N * h * prof_steps / fam["forecast"][0]
        # fp16-pair kind::f16 MMAs, three per algorithmic product (cnn_tc.cu / cnn_deep.cu); the
        # bracket runs next to the concurrent noise launch, so this understates the kernel alone
        kf["peak_3xf16"] = peak / 3.0
        kf["frac_3xf16"] = kf["achieved"] / kf["peak_3xf16"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.members, args.horizon)

    if rank == 0:
        line = {
            "metric": "OIC horizon solves/sec", "value": value, "unit": "horizons/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (sine-field x0, random-init CNN, bit-exact numpy noise streams)",
            "config": _config(pr, args, world),
            "member_cnn_steps_per_s": pr.N * h * value,
            "e2e": e2e, "e2e_graph": e2e_graph,
            "gpu_launches": int(launches), "roofline": roofline, "kernels": kernels,
            "cuda_graph": graph is not None,
            "cpu_baseline": cpu, "clocks": clk,
            "algorithmic": alg,
        }
        print(json.dumps(line))
    if comm is not None:
        dist.barrier()
        dist.destroy_process_group()


def _e2e(args, enks, ops, pr, streams, comm, graph: bool):
    """horizons/s through enks.smooth_horizon with host NumPy inputs and the host fp64 result,
    all host<->device copies inside the timed region (bytes counted by DeviceOps)."""
    import torch
    import torch.distributed as dist

    h = pr.H
    enks.smooth_horizon(pr.x0, pr.y_ref, pr.vs, h, pr.N, streams, graph=graph)  # warm
    torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
    b_in, b_out = ops.h2d_bytes, ops.d2h_bytes
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        y_host = np.broadcast_to(pr.y_ref, (h,) + pr.y_ref.shape)
        out, _ = enks.smooth_horizon(pr.x0, y_host, pr.vs, h, pr.N, streams, graph=graph)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3
    if comm is not None:
        t = torch.tensor([sec], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t[0])
    return {"value": args.steps / sec, "unit": "horizons/s",
            "h2d_bytes_per_step": int((ops.h2d_bytes - b_in) // args.steps),
            "d2h_bytes_per_step": int((ops.d2h_bytes - b_out) // args.steps),
            "call": f"enks.smooth_horizon(x0, y_refs, vs, h, N, streams{', graph=True' if graph else ''})",
            "result": f"mean trajectory {tuple(out.shape)} fp64 on the host"}


def _relaunch_under_torchrun(args) -> None:
    """--gpus N > 1 without a torchrun environment: re-exec this command as N ranks (one process
    per GPU, NCCL), or fail loudly when this node has fewer GPUs -- never a 1-rank line."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has "
                         f"{have}\n")
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", "--master-port=29517",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = _args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch_under_torchrun(args)
    if args.impl == "ours" and int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE="
                         f"{os.environ.get('WORLD_SIZE')}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
