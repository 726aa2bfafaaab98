"""Drop-in, B200-backed replacement for the reference smoother API.

Same names, signatures, return shapes and error behaviour as reference
pkg/src/enksmpc/enks.py:36-47:

    TrajectoryEnsemble, SmootherCovariances, CH_W, CH_VX, CH_VU, CH_EPS,
    init_ensemble (105-128), predict (156-186), update (212-253),
    smooth_horizon (256-284)

The ensemble lives on the GPU (engine.DeviceSmoother); ``members`` and
``mean`` are materialised as fp64 NumPy arrays on access (one device sync),
so code that inspects them keeps working.  Arithmetic is fp32 on device;
parity with the fp64 reference is <= 1e-4 relative (tests/test_parity_gpu.py).
Noise is bit-identical to the reference's NoiseStreams substreams.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from .covariance import SmootherCovariances, track_predict, track_update
from .engine import CH_EPS, CH_VU, CH_VX, CH_W, DeviceSmoother, LocalComm

__all__ = [
    "TrajectoryEnsemble",
    "SmootherCovariances",
    "CH_W",
    "CH_VX",
    "CH_VU",
    "CH_EPS",
    "init_ensemble",
    "predict",
    "update",
    "smooth_horizon",
    "set_default_comm",
    "HorizonGraph",
]

_OPS = None
_COMM = None


def _ops():
    global _OPS
    if _OPS is None:
        from .ops import DeviceOps

        _OPS = DeviceOps()
    return _OPS


def set_default_comm(comm) -> None:
    """Shard members over a torch.distributed group for subsequent ensembles
    (``engine.TorchComm()``); None restores single-process operation."""
    global _COMM
    _COMM = comm


def _comm():
    return _COMM or LocalComm()


class TrajectoryEnsemble:
    """N trajectory samples with their running mean (enks.py:56-93), device-resident.

    ``members`` has shape (N, (t+1)*slice_rows, m) and ``mean`` ((t+1)*slice_rows, m)
    when read.  Assigning ``members`` re-seeds the device state from explicit samples.
    """

    def __init__(self, members=None, mean=None, t: int = 0, lam: float | None = None,
                 n_x: int | None = None, n_u: int | None = None, jitter_events: int = 0, *,
                 _engine: DeviceSmoother | None = None):
        self._jitter0 = int(jitter_events)
        if _engine is not None:
            self._eng = _engine
            return
        if members is None or lam is None or n_x is None or n_u is None:
            raise TypeError("TrajectoryEnsemble needs members, mean, t, lam, n_x, n_u")
        members = np.asarray(members, dtype=float)
        d = n_x + 2 * n_u
        if members.ndim != 3 or members.shape[1] != (t + 1) * d:
            raise ValueError("members must be (N, (t+1)(n+2l), m)")
        comm = _comm()
        eng = DeviceSmoother(_ops(), members[0, :d], n_x, n_u, members.shape[0], lam,
                             capacity=max(t, 1), comm=comm)
        lo, cnt = eng.member0, eng.Nl
        eng.replace_members(members[lo:lo + cnt], t)
        self._eng = eng

    # -- reference dataclass fields ----------------------------------------
    @property
    def members(self) -> np.ndarray:
        eng = self._eng
        R = (eng.t + 1) * eng.d
        local = eng.ops.to_host(eng.members_device())
        local = local.reshape(R, eng.Nl, eng.m).transpose(1, 0, 2)
        if eng.slice0_zero and eng.x0_exact is not None:
            local[:, :eng.d] = eng.x0_exact  # identical copies of x0 (enks.py:108-110), exact
        if eng.comm.size > 1:
            import torch.distributed as dist

            parts = [None] * eng.comm.size
            dist.all_gather_object(parts, local, group=getattr(eng.comm, "group", None))
            local = np.concatenate(parts, axis=0)
        return np.ascontiguousarray(local)

    @members.setter
    def members(self, value) -> None:
        value = np.asarray(value, dtype=float)
        eng = self._eng
        if value.ndim != 3 or value.shape[1] % eng.d or value.shape[0] != eng.N:
            raise ValueError("members must be (N, (t+1)(n+2l), m) for this ensemble")
        eng.replace_members(value[eng.member0:eng.member0 + eng.Nl], value.shape[1] // eng.d - 1)

    @property
    def mean(self) -> np.ndarray:
        return self._eng.mean_host()

    @property
    def t(self) -> int:
        return self._eng.t

    @property
    def lam(self) -> float:
        return self._eng.lam

    @property
    def n_x(self) -> int:
        return self._eng.n

    @property
    def n_u(self) -> int:
        return self._eng.l

    @property
    def jitter_events(self) -> int:
        return self._jitter0 + self._eng.jitter_events()

    # -- reference helpers ------------------------------------------------------
    @property
    def n_members(self) -> int:
        return self._eng.N

    @property
    def slice_rows(self) -> int:
        return self._eng.d

    @property
    def n_cols(self) -> int:
        return self._eng.m

    def slices(self) -> np.ndarray:
        return self.mean.reshape(self.t + 1, self.slice_rows, self.n_cols)

    def last_slice_blocks(self):
        d, n, l = self.slice_rows, self.n_x, self.n_u
        tail = self.members[:, -d:, :]
        return tail[:, :n, :], tail[:, n:n + l, :], tail[:, n + l:, :]

    @property
    def engine(self) -> DeviceSmoother:
        return self._eng


def init_ensemble(x0, n_members: int, shared_col_cov: np.ndarray | None = None, *,
                  capacity: int = 8) -> TrajectoryEnsemble:
    """N identical copies of the current slice; lambda = 1/tr(shared_col_cov) (enks.py:105-128)."""
    if n_members < 2:
        raise ValueError("need at least 2 ensemble members")
    packed = np.asarray(x0.packed, dtype=float)
    lam = 1.0 / packed.shape[1] if shared_col_cov is None else \
        1.0 / float(np.trace(shared_col_cov))
    eng = DeviceSmoother(_ops(), packed, x0.n, x0.l, n_members, lam, capacity=capacity,
                         comm=_comm())
    return TrajectoryEnsemble(_engine=eng)


def predict(ens: TrajectoryEnsemble, vs, streams, cov: Optional[SmootherCovariances] = None
            ) -> TrajectoryEnsemble:
    """Advance every member one virtual step and append the new slice (enks.py:156-186)."""
    eng = ens._eng
    eng.predict(vs, streams)
    if cov is not None:
        track_predict(eng, cov)  # device-resident (covariance.py), read lazily as fp64
    return ens


def _device_yref(eng: DeviceSmoother, y_ref: np.ndarray):
    return eng.ops.to_device(np.asarray(y_ref, dtype=float))


def update(ens: TrajectoryEnsemble, y_ref: np.ndarray, vs, streams,
           cov: Optional[SmootherCovariances] = None) -> TrajectoryEnsemble:
    """Kalman-shift every member's whole trajectory toward the reference (enks.py:212-253)."""
    eng = ens._eng
    y_ref = np.asarray(y_ref, dtype=float)
    obs_shape = (vs.obs_rows, eng.m)
    if y_ref.shape != obs_shape:
        raise ValueError(f"y_ref shape {y_ref.shape} != observation {obs_shape}")
    eng.bind(vs)
    eng.update(_device_yref(eng, y_ref), streams)
    eng.check_status()
    if cov is not None:
        track_update(eng, cov)
    return ens


class HorizonGraph:
    """One whole horizon solve (reset + H x (predict, update)) captured as a CUDA graph.

    Static device inputs ``x0`` ((d x m)) and ``y_refs`` ((h, p, m)) are copied in before each
    ``replay``; the result is the engine's ``mean``.  The model and the virtual system are baked
    into the graph; the noise streams' entropy words live in device memory (ops.DeviceHead), so
    one capture serves every NoiseStreams / child(k) with the same number of entropy words
    (``set_streams``).  Every kernel of the eager path runs on replay (same launches, same order,
    side-stream gain solve included) -- the graph only removes the per-launch host cost, which
    dominates small problems."""

    def __init__(self, x0, vs, h: int, n_members: int, streams, comm=None):
        from .matvar import entropy_head
        from .ops import DeviceHead

        packed = np.asarray(x0.packed, dtype=float)
        lam = 1.0 / float(np.trace(vs.shared_col_cov))
        ops = _ops()
        self.h, self.vs, self.streams = int(h), vs, streams
        self.eng = DeviceSmoother(ops, packed, x0.n, x0.l, n_members, lam, capacity=h,
                                  comm=comm or _comm())
        self.eng.bind(vs)
        words = entropy_head(streams.seed, tuple(streams.prefix))
        self.head = DeviceHead(ops.zeros(max(32, len(words)), dtype=torch.int32), len(words))
        self.head.set(words)
        self.eng.dev_head = self.head
        self.x0 = ops.to_device(packed)
        self.y_refs = ops.zeros(h, vs.obs_rows, packed.shape[1])
        self._run()  # warm-up: kernel attributes, workspaces, tensor maps
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._run()

    def _run(self) -> None:
        eng = self.eng
        eng.reset(self.x0)
        for step in range(self.h):
            eng.predict(self.vs, self.streams)
            eng.update(self.y_refs[step], self.streams)

    def set_streams(self, streams) -> None:
        """Noise substreams for the next replays (same entropy word count as the capture)."""
        from .matvar import entropy_head

        self.head.set(entropy_head(streams.seed, tuple(streams.prefix)))
        self.streams = streams

    def replay(self) -> DeviceSmoother:
        eng = self.eng
        eng.clear_flags()  # per-solve failure flags, as a fresh eager engine would have
        self.graph.replay()
        eng.t = self.h
        eng.n_upd = self.h
        return eng


_GRAPHS: dict = {}


def _nccl(comm) -> bool:
    group = getattr(comm, "group", None)
    try:
        import torch.distributed as dist

        return getattr(comm, "dist", None) is not None and dist.get_backend(group) == "nccl"
    except (RuntimeError, ValueError):
        return False


GRAPH_CACHE_FRACTION = 0.25  # of device memory, summed over the cached horizon engines


def _graph_for(x0, vs, h, n_members, streams):
    """Cached HorizonGraph for this (virtual system, shapes, h, N, entropy word count), or None
    when its engine would not fit the cache budget (the caller then runs eager)."""
    from .matvar import entropy_head

    n_words = len(entropy_head(streams.seed, tuple(streams.prefix)))
    key = (id(vs), id(vs.model), tuple(np.shape(x0.packed)), x0.n, x0.l, int(h), int(n_members),
           n_words, id(_COMM))
    g = _GRAPHS.get(key)
    if g is not None and g.vs is vs:
        g.set_streams(streams)
        return g
    budget = GRAPH_CACHE_FRACTION * torch.cuda.get_device_properties(
        torch.cuda.current_device()).total_memory
    d, p, m = x0.n + 2 * x0.l, x0.n + x0.l, np.shape(x0.packed)[1]
    est = 4.4 * ((h + 1) * p + h * p) * n_members * m + 4 * (h + 1) * d * m  # basis + gains
    if est > budget:
        return None
    while _GRAPHS and sum(v.eng.memory_bytes() for v in _GRAPHS.values()) + est > budget:
        _GRAPHS.pop(next(iter(_GRAPHS)))
    g = _GRAPHS[key] = HorizonGraph(x0, vs, h, n_members, streams)
    return g


def smooth_horizon(x0, y_refs: np.ndarray, vs, h: int, n_members: int, streams,
                   track_cov: bool = False, *, graph: bool = False):
    """Forward predict/update sweep over an h-step horizon (enks.py:256-284).

    Returns the mean trajectory (h+1, n+2l, m) as fp64 and the covariances
    when ``track_cov``.  One host synchronisation at the end.  ``graph=True`` (keyword-only
    extension) replays a cached CUDA graph of the whole horizon for this (virtual system,
    shapes, h, N, noise streams): x0 and y_refs are copied into its static inputs, so the
    model / weights must not be mutated between calls (rebuild the VirtualSystem instead).
    """
    if h < 1:
        raise ValueError("horizon must be at least 1")
    y_refs = np.asarray(y_refs, dtype=float)
    if y_refs.ndim == 2:
        y_refs = np.broadcast_to(y_refs, (h, *y_refs.shape))
    elif y_refs.shape[0] != h:
        raise ValueError(f"need {h} reference observations, got {y_refs.shape[0]}")
    if y_refs.shape[1:] != (vs.obs_rows, x0.m):
        raise ValueError(f"y_ref shape {y_refs.shape[1:]} != observation {(vs.obs_rows, x0.m)}")
    if graph and not track_cov and n_members >= 2 and torch.cuda.is_available() and \
            (_comm().size == 1 or _nccl(_comm())):  # NCCL collectives are captured too
        g = _graph_for(x0, vs, h, n_members, streams)
    else:
        g = None
    if g is not None:
        ops = g.eng.ops
        ops.copy_from_host(g.x0, np.asarray(x0.packed, dtype=np.float32))
        g.eng.x0_exact = np.array(x0.packed, dtype=float)
        ops.copy_from_host(g.y_refs, np.ascontiguousarray(y_refs, dtype=np.float32))
        eng = g.replay()
        eng.check_status()
        return eng.mean_host().reshape(h + 1, eng.d, eng.m), None
    if n_members < 2:
        raise ValueError("need at least 2 ensemble members")
    ens = init_ensemble(x0, n_members, shared_col_cov=vs.shared_col_cov, capacity=h)
    eng = ens._eng
    eng.bind(vs)
    yref_dev = eng.ops.to_device(np.ascontiguousarray(y_refs))
    cov = SmootherCovariances(sigma_traj=np.zeros((eng.d, eng.d))) if track_cov else None
    for step in range(h):
        # tracking never feeds back into the smoother (test_enks.py:253-265), and every tracked
        # field is overwritten by the next predict / update (enks.py:173-185, 250-252), so only
        # the last step's values are observable: track there only
        last = cov is not None and step == h - 1
        eng.predict(vs, streams)
        if last:
            track_predict(eng, cov)
        eng.update(yref_dev[step], streams)
        if last:
            eng.check_status()
            track_update(eng, cov)
    eng.check_status()
    return ens.slices(), cov


def smooth_horizon_device(x0, yref_dev: torch.Tensor, vs, h: int, n_members: int, streams,
                          comm=None) -> DeviceSmoother:
    """Device-resident variant for benchmarks / closed loops: y refs already on
    device (h, p, m); returns the engine without any host synchronisation."""
    packed = np.asarray(x0.packed, dtype=float)
    lam = 1.0 / float(np.trace(vs.shared_col_cov))
    eng = DeviceSmoother(_ops(), packed, x0.n, x0.l, n_members, lam, capacity=h,
                         comm=comm or _comm())
    eng.bind(vs)
    for step in range(h):
        eng.predict(vs, streams)
        eng.update(yref_dev[step], streams)
    return eng
