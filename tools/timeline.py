"""Per-op timeline of one eager C3 horizon (CUDA-event brackets relative to the horizon start).

    python tools/timeline.py [--config C3] [--steps 24,25]
Prints, for the chosen steps, every profiled op (tag, stream order) with start/end in ms.
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import problems  # noqa: E402  (synthetic inputs only)
from paper_2410_09663_b200 import enks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--members", type=int, default=None)
ap.add_argument("--horizon", type=int, default=None)
ap.add_argument("--steps", default="1,2,25,26")
ap.add_argument("--sim-ranks", type=int, default=1,
                help="rank 0 of a simulated R-rank job (engine.SimComm, N/R members)")
a = ap.parse_args()
pm = problems.product_modules()
pr = problems.make_cnn_problem(pm, a.config, n_members=a.members, horizon=a.horizon)
ops = enks._ops()
# bracket every C-ABI call that is not inside a tagged op as "misc:<entry point>"
from paper_2410_09663_b200 import _lib  # noqa: E402
import contextlib  # noqa: E402

_depth = [0]
_orig_prof, _orig_call = ops._prof, _lib.call


@contextlib.contextmanager
def _prof(tag, work):
    _depth[0] += 1
    try:
        with _orig_prof(tag, work):
            yield
    finally:
        _depth[0] -= 1


def _call(fn, *args):
    if ops.profile is None or _depth[0]:
        return _orig_call(fn, *args)
    with _prof("misc:" + fn.replace("enks_", ""), 0.0):
        return _orig_call(fn, *args)


ops._prof = _prof
_lib.call = _call
streams = pm.matvar.NoiseStreams(seed=0)
yref = ops.to_device(np.broadcast_to(pr.y_ref, (pr.H,) + pr.y_ref.shape).copy())
from paper_2410_09663_b200.engine import SimComm  # noqa: E402

comm = SimComm(a.sim_ranks) if a.sim_ranks > 1 else None
for _ in range(2):
    enks.smooth_horizon_device(pr.x0, yref, pr.vs, pr.H, pr.N, streams, comm=comm)
torch.cuda.synchronize()
ops.profile = []
base = torch.cuda.Event(enable_timing=True)
end = torch.cuda.Event(enable_timing=True)
base.record()
enks.smooth_horizon_device(pr.x0, yref, pr.vs, pr.H, pr.N, streams, comm=comm)
end.record()
torch.cuda.synchronize()
prof, ops.profile = ops.profile, None
total = base.elapsed_time(end)
rows = [(tag, base.elapsed_time(s), base.elapsed_time(e)) for tag, s, e, _ in prof]
# steps: a new step starts at each "forecast" op
starts = [i for i, r in enumerate(rows) if r[0] == "forecast"]
want = {int(x) for x in a.steps.split(",")}
print(f"horizon {total:.2f} ms, {len(rows)} profiled ops")
for k, i0 in enumerate(starts, start=1):
    if k not in want:
        continue
    i1 = starts[k] if k < len(starts) else len(rows)
    # include the noise op launched just before the forecast
    lo = i0 - 1 if i0 > 0 and rows[i0 - 1][0] == "noise" else i0
    t0 = rows[lo][1]
    print(f"--- step {k} (starts at {t0:.3f} ms)")
    for tag, s, e in rows[lo:i1 - (1 if i1 < len(rows) and rows[i1 - 1][0] == 'noise' else 0)]:
        print(f"  {tag:12s} {s - t0:8.3f} -> {e - t0:8.3f}  ({e - s:7.3f} ms)")
