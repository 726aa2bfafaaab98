"""Device-resident single-pass matrix-variate EnKS (the hot path).

Restructures reference pkg/src/enksmpc/enks.py:156-253 for the GPU without
changing the estimator.  The reference keeps every member's whole trajectory
and, at each update, (i) re-centres it, (ii) contracts it with the centred
observations (Sigma_xy, enks.py:233-236) and (iii) shifts it in place
(members += G (y_ref - obs), enks.py:247) -- three O(T d N m) passes over an
array that grows every step.

Here the trajectory is never rewritten.  For slice s and the update at step
tau the member deviations are

    M_s - mean_s = A_s - sum_{s <= tau' < tau} G_{tau', s} Yc_{tau'}

where A_s (d x Nm) are the centred predicted slices, Yc_tau (p x Nm) the
centred perturbed observations and G_{tau, s} (d x p) the gain rows of slice
s at step tau (the innovation's member-mean part only moves the mean).  So
with the append-only basis [A_0..A_tau ; Yc_1..Yc_tau] one tall-skinny
contraction per step,

    P = [A; Yc] Yc_tau^T            (the K = N m contraction, K6/K7)

gives Sigma_y (the Yc_tau block) and, after a small block-triangular
correction  S_s = P_{A_s} - sum_tau' G_{tau',s} P_{Yc_tau'},  Sigma_xy for
every slice.  G = (lam/N) S Sigma_y^{-1} (K8), the mean moves by
G (y_ref - y_bar) and only the newest slice's [x; u] blocks are materialised
for the next forecast.  Algebraically identical to the reference (checked to
5e-16 in fp64 by tests/test_engine_algebra.py); in fp32 it removes the
trajectory read-modify-write and one of the two O(T) contractions per step.

Anomalies are formed relative to global member 0 (stats.cu), so identical
members give exactly zero spread at any N (scale = 0 cases).

Multi-rank: members are sharded over ranks (global member ids name the noise
substreams, so draws do not depend on the rank count).  Per step the only
exchanges are the slice/observation member sums, the member-0 shift
(broadcast) and the allreduce of P; the gain, correction and mean update are
replicated.
"""
from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass

import numpy as np
import torch

from .matvar import entropy_head

CH_W, CH_VX, CH_VU, CH_EPS = 0, 1, 2, 3


def _nvtx(name: str):
    """NVTX range around an engine method on CUDA (nsys / ncu --nvtx see predict / update)."""
    def deco(fn):
        def wrapped(self, *args, **kw):
            if getattr(self.ops, "device", None) is None or self.ops.device.type != "cuda":
                return fn(self, *args, **kw)
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(self, *args, **kw)
            finally:
                torch.cuda.nvtx.range_pop()
        wrapped.__name__, wrapped.__doc__ = fn.__name__, fn.__doc__
        return wrapped
    return deco


class LocalComm:
    rank = 0
    size = 1

    def allreduce_(self, t):
        return t

    def allreduce_many(self, ts):
        return ts

    def reduce_scatter_rows(self, t):
        return t

    def all_gather_rows(self, t):
        return t

    def allreduce_max_(self, t):
        return t

    def broadcast_(self, t, src=0):
        return t


class SimComm:
    """Rank 0 of a SIMULATED `size`-rank job on one GPU (tools/shard_model.py): it owns N/size
    members and runs exactly the per-rank kernels; every collective is replaced by `t *= size`
    (as if each other rank held a copy of this rank's shard), which keeps the smoother numerically
    sane, and its bytes are logged for the collective-cost model.  Timing only."""

    rank = 0

    def __init__(self, size: int):
        self.size = int(size)
        self.log = []  # (kind, bytes)

    def allreduce_(self, t):
        self.log.append(("allreduce", t.numel() * t.element_size()))
        t.mul_(self.size)
        return t

    def allreduce_many(self, ts):
        self.log.append(("allreduce", sum(t.numel() * t.element_size() for t in ts)))
        for t in ts:
            t.mul_(self.size)
        return ts

    def allreduce_max_(self, t):
        self.log.append(("allreduce", t.numel() * t.element_size()))
        return t

    def broadcast_(self, t, src=0):
        self.log.append(("broadcast", t.numel() * t.element_size()))
        return t

    def reduce_scatter_rows(self, t):
        self.log.append(("reduce_scatter", t.numel() * t.element_size()))
        return t[:t.shape[0] // self.size].mul_(self.size)

    def all_gather_rows(self, t):
        self.log.append(("all_gather", t.numel() * t.element_size() * self.size))
        return t.repeat(self.size, 1)


class TorchComm:
    """torch.distributed process group (NCCL on B200, gloo on CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def allreduce_many(self, ts):
        """Sum-allreduce several tensors as ONE collective: one coalesced NCCL group launch
        (torch's coalescing manager); other backends issue them back to back."""
        ts = [t for t in ts if t.numel()]
        if len(ts) == 1:
            self.dist.all_reduce(ts[0], group=self.group)
        elif ts and self.dist.get_backend(self.group) == "nccl":
            from torch.distributed.distributed_c10d import _coalescing_manager

            with _coalescing_manager(group=self.group, device=ts[0].device):
                for t in ts:
                    self.dist.all_reduce(t, group=self.group)
        else:
            for t in ts:
                self.dist.all_reduce(t, group=self.group)
        return ts

    def reduce_scatter_rows(self, t):
        """Sum over ranks of t (R x C, R a multiple of the rank count); returns this rank's row
        block (R / size rows) -- row-sharded results (covariance tracking)."""
        rows = t.shape[0] // self.size
        if self.dist.get_backend(self.group) == "nccl":
            out = t.new_empty(rows, t.shape[1])
            self.dist.reduce_scatter_tensor(out, t, group=self.group)
            return out
        self.dist.all_reduce(t, group=self.group)  # gloo: no reduce_scatter
        return t[self.rank * rows:(self.rank + 1) * rows].clone()

    def all_gather_rows(self, t):
        """Concatenate every rank's row block (inverse of reduce_scatter_rows)."""
        if self.dist.get_backend(self.group) == "nccl":
            out = t.new_empty(t.shape[0] * self.size, t.shape[1])
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts)

    def allreduce_max_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def broadcast_(self, t, src=0):
        self.dist.broadcast(t, src=src, group=self.group)
        return t


def partition(n_members: int, size: int, rank: int) -> tuple[int, int]:
    """(first global member, count) of rank `rank` for an even split."""
    base, extra = divmod(n_members, size)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


@dataclass
class _Noise:
    kind: str           # "zero" | "diag" | "dense"
    diag: object = None  # device float64 (rows,)
    dense: object = None  # device float32 (rows, rows)


class Forecaster:
    """Device forecast for one dynamics model (dispatch on model type; no host fallback)."""

    def __init__(self, model, ops, n: int, l: int):
        self.model = model
        self.kind = None
        name = type(model).__name__
        if name == "CNNDynamics" and hasattr(model, "widths"):
            if l != n:
                raise ValueError("CNNDynamics needs input_rows == state_rows")
            if max(model.widths) > 32 or model.n_layers > 8:
                raise NotImplementedError("CNN widths > 32 or > 8 layers not supported on device")
            self.kind = "cnn"
            self.widths = tuple(model.widths)
            self.n_layers = len(self.widths) - 1
            self.alpha = float(model.alpha)
            self.cols = int(model.state_cols)
            self.w_dev = ops.to_device(np.concatenate([np.asarray(w, float).ravel()
                                                       for w in model.weights]))
            self.b_dev = ops.to_device(np.concatenate([np.asarray(b, float).ravel()
                                                       for b in model.biases]))
        elif name == "LinearDynamics" and hasattr(model, "a") and hasattr(model, "b"):
            self.kind = "linear"
            ab = np.concatenate([np.asarray(model.a, float), np.asarray(model.b, float)], axis=1)
            self.ab = ops.to_device(ab)  # n x (n + l)
        elif name == "BurgersDynamics" and hasattr(model, "cfg"):
            cfg = model.cfg
            g = int(cfg.grid_n)
            if n != 2 * g or l not in (2, 2 * g):
                raise ValueError("BurgersDynamics: state must be 2n x n and force 2 x n / 2n x n")
            self.kind = "burgers"
            self.grid_n, self.substeps = g, int(cfg.substeps)
            self.nu, self.dt, self.dx = float(cfg.nu), float(cfg.dt), float(cfg.dx)
            diff = self.nu * self.dt / self.dx ** 2
            if diff > 0.25:  # input-independent half of the CFL check (dynamics.py:172-177)
                from .dynamics import CflError
                raise CflError(f"CFL violated: nu*dt/dx^2 = {diff:.4g} (limit 0.25)")
            self.vmax = ops.zeros(1)                       # max |phi| over all substep inputs
            self.flags = ops.zeros(1, dtype=torch.int32)   # bit 0: non-finite entry
        else:
            raise TypeError(f"no device forecast for model type {name}; supported: "
                            "LinearDynamics, CNNDynamics, BurgersDynamics")

    def __call__(self, ops, last, out, n: int, n_members: int):
        """out (n x K) = f(x = last[:n], u = last[n:])."""
        if self.kind == "linear":
            ops.gemm(self.ab, last, out)
        elif self.kind == "burgers":
            ops.burgers_forward(self, last[:n], last[n:], out, n_members)
        else:
            ops.cnn_forward(self, last[:n], last[n:], out, n_members)


    def check_cfl(self, comm=None) -> None:
        """Raise CflError if any forecast so far saw max|phi| dt/dx > 1 or a non-finite
        entry (dynamics.py:168-180, checked lazily over the whole batch and all ranks)."""
        from .dynamics import CflError

        st = torch.stack([self.vmax[0], self.flags[0].float()])
        if comm is not None and comm.size > 1:
            comm.allreduce_max_(st)
        vmax, bad = float(st[0].item()), float(st[1].item())
        adv = vmax * self.dt / self.dx
        if bad or not np.isfinite(vmax):
            raise CflError("field contains non-finite entries")
        if adv > 1.0:
            raise CflError(f"CFL violated: max|phi|*dt/dx = {adv:.4g} (limit 1)")

    @property
    def advection_number(self) -> float:
        return float(self.vmax[0].item()) * self.dt / self.dx


@dataclass
class _Barrier:
    kind: int            # 0 linear functional, 1 max-abs over a row block
    coef: object         # device (d x m) fp32 for kind 0
    c0: float
    r0: int
    r1: int
    alpha: float
    beta: float
    sqrt_var: float


def _barrier_spec(con, ops, n: int, l: int, m: int) -> _Barrier:
    """Device form of ConstraintSpec.g: LinearConstraint / BoxConstraint only (no host g)."""
    from .virtualsys import BoxConstraint, LinearConstraint

    g = con.g
    common = dict(alpha=float(con.alpha), beta=float(con.beta),
                  sqrt_var=float(np.sqrt(con.noise_var)))
    if isinstance(g, LinearConstraint):
        coef = np.zeros((n + 2 * l, m))
        for r0, c in ((0, g.cx), (n, g.cu), (n + l, g.cdu)):
            if c is not None:
                c = np.asarray(c, float)
                coef[r0:r0 + c.shape[0]] = c
        return _Barrier(0, ops.to_device(coef), float(g.c0), 0, n + 2 * l, **common)
    if isinstance(g, BoxConstraint):
        r0, r1 = {"x": (0, n), "u": (n, n + l), "du": (n + l, n + 2 * l)}[g.block]
        return _Barrier(1, None, -float(g.bound), r0, r1, **common)
    raise TypeError("constraint g must be a LinearConstraint or BoxConstraint on the device "
                    f"path (got {type(g).__name__}); arbitrary host callables are not evaluated")


def _noise_params(params, ops, rows: int, cols: int) -> _Noise:
    if params is None:
        return _Noise("zero")
    L = np.asarray(params.row_chol, dtype=float)
    B = np.asarray(params.col_chol, dtype=float)
    if not np.array_equal(B, np.eye(cols)):
        raise NotImplementedError("device noise supports column Cholesky factor I_m only "
                                  "(the reference virtual system always uses I_m)")
    if np.any(np.asarray(params.mean) != 0):
        raise NotImplementedError("device noise supports zero-mean channels only")
    if L.shape != (rows, rows):
        raise ValueError("noise factor shape mismatch")
    if np.array_equal(L, np.diag(np.diag(L))):
        return _Noise("diag", diag=ops.to_device(np.diag(L).copy(), dtype=torch.float64))
    return _Noise("dense", dense=ops.to_device(L))


class DeviceSmoother:
    """Ensemble state + per-step orchestration for one horizon (see module docstring)."""

    def __init__(self, ops, x0_packed: np.ndarray, n: int, l: int, n_members: int, lam: float,
                 capacity: int = 8, comm=None, basis: str | None = None):
        self.ops = ops
        self.comm = comm or LocalComm()
        self.n, self.l = int(n), int(l)
        # d: slice rows [X; U; dU]; q: state rows [X; U] fed to the forecast; p: observation
        # rows [X; U] (+1 barrier row when a constraint is bound, enks.py:201-208)
        self.d, self.q = self.n + 2 * self.l, self.n + self.l
        self.p = self.q
        self.m = int(x0_packed.shape[1])
        self.N = int(n_members)
        if self.N < self.comm.size:
            raise ValueError("need at least one member per rank")
        self.member0, self.Nl = partition(self.N, self.comm.size, self.comm.rank)
        self.K = self.Nl * self.m
        self.lam = float(lam)
        self.t = 0
        self.n_upd = 0  # observation blocks Yc_1..Yc_n_upd in the basis (gains exist for these)
        self.cap = 0
        self.slice0_zero = True  # all members start as identical copies (enks.py:120)
        self._bound = None
        self.barrier = None
        self.dev_head = None  # ops.DeviceHead: noise entropy words read from device memory
        self.record = None    # dict: per-update Sigma_y / Sigma_xy / gain (tests, see _record_step)
        self._pending = None  # deferred centring of the newest predicted slice (_finish_slice)
        self._last_stale = False  # `last` lags the newest slice (a predict with no update yet)
        self._basis = basis
        self.sum2 = False  # set by bind()
        self._explicit = False  # explicit members (replace_members): no derived-U chain
        d, q, K = self.d, self.q, self.K
        self.slice_raw = ops.empty(d, K)      # [X; U; W] of the newest predicted slice
        self.last = ops.empty(q, K)           # materialised [x; u] of the newest updated slice
        self.status = ops.zeros(1, dtype=torch.int32)
        self.jitter = ops.zeros(1, dtype=torch.int32)
        self._alloc_obs()
        self._grow(max(1, int(capacity)))
        # slice 0 of identical copies is never moved (enks.py:108-110): read back exactly
        self.x0_exact = np.array(x0_packed, dtype=float)
        x0 = ops.to_device(self.x0_exact)
        self.mean[:d] = x0
        self.last.copy_(x0[:q].repeat(1, self.Nl))
        self._store_rows("A", 0, ops.zeros(self.ds, K))

    def _alloc_obs(self) -> None:
        """Buffers whose shape depends on the observation row count p."""
        ops, d, p, q, K, m = self.ops, self.d, self.p, self.q, self.K, self.m
        # every rank must take the same code path (the collectives follow it): decide on the
        # smallest local column count and on conditions every rank's K satisfies
        k_min = (self.N // self.comm.size) * m
        k_aligned = (m % 8 == 0) if self.comm.size > 1 else (K % 8 == 0)
        # tcgen05 cross moments (ENKS_TC=0 forces the SIMT engine for A/B checks)
        self.use_tc = (os.environ.get("ENKS_TC", "1") != "0" and hasattr(ops, "gemm_nt_tc")
                       and p <= 512 and k_min >= 128)
        # basis storage: fp16 pairs (tcgen05 kind::f16 contraction, gemm_f16p.cu) or fp32
        basis = self._basis or os.environ.get("ENKS_BASIS", "f16pair" if self.use_tc else "fp32")
        self.pair = basis == "f16pair" and k_aligned and hasattr(ops, "gemm_f16pair")
        # derived-U chain: slices are [X; U; dU] with U_s = U_{s-1} + dU_s member-wise
        # (enks.py:168, preserved by every linear update), so the basis, the cross moments and the
        # gains keep only the [X; dU] rows (ds = n + l per slice) and U follows by prefix sums
        # (enks_uchain_apply) -- l fewer rows per slice in the dominant contraction
        self.chain = (self.pair and self.l > 0 and not self._explicit and hasattr(ops, "uchain_apply")
                      and os.environ.get("ENKS_UCHAIN", "1") != "0")
        self.ds = self.n + self.l if self.chain else self.d
        self.gtt = ops.empty(self.q, p) if self.chain else None
        if self.use_tc and not self.pair:
            self.yc_hi = ops.empty(p, K)
            self.yc_lo = ops.empty(p, K)
        # newest-slice shift on the fp16-pair kernel: B = Yc_tau^T planes (K x p), re-split
        # from the basis rows; no fp32 copy of Yc_tau is kept
        self.shift_f16 = (self.pair and p <= 256 and p % 8 == 0 and m % 4 == 0
                          and hasattr(ops, "gemm_f16pair_ex"))
        # ... reading the Yc_tau basis rows themselves as an MN-major B operand (no transposed
        # planes: G_tt takes Yc_tau's per-row scale before its split); ENKS_SHIFT_MN=0: transposed
        self.shift_mn = (self.shift_f16 and hasattr(ops, "gemm_f16pair_ex_mn") and p % 32 == 0
                         and K % 8 == 0 and K > 128 and os.environ.get("ENKS_SHIFT_MN", "1") != "0")
        if self.pair:
            self.A_new = ops.empty(q, K)   # fp32 anomalies of the newest slice, [x; u] rows
            self.Yc_new = None if self.shift_f16 else ops.empty(p, K)  # fp32 centred obs
        if self.shift_f16:
            f16 = torch.float16
            self.ycT_h = self.ycT_l = self.ycT_inv = None
            if not self.shift_mn:
                self.ycT_h, self.ycT_l, self.ycT_inv = (ops.empty(K, p, dtype=f16),
                                                        ops.empty(K, p, dtype=f16), ops.empty(K))
            self.gtt_h, self.gtt_l, self.gtt_inv = (ops.empty(q, p, dtype=f16),
                                                    ops.empty(q, p, dtype=f16), ops.empty(q))
        # the gain-side products (correction, gain, newest-slice shift) on tcgen05 as well
        self.use_tc2 = self.use_tc and p % 4 == 0 and m % 4 == 0 and hasattr(ops, "gemm_tc")
        if self.use_tc2 and not self.shift_f16:
            self.ycT_hi = ops.empty(K, p)
            self.ycT_lo = ops.empty(K, p)
        if self.use_tc2:
            self.innT_hi, self.innT_lo = ops.empty(m, p), ops.empty(m, p)  # (y_ref - y_bar)^T
            self.sinvT_hi = ops.empty(p, p)
            self.sinvT_lo = ops.empty(p, p)
            self.pyT_hi = self.pyT_lo = None
        self.obs_raw = ops.empty(p, K)        # perturbed observations of the newest slice
        self.acc = ops.zeros(max(d, p), m, dtype=torch.float64)
        self.amax = ops.zeros(max(d, p), m)
        self.acc_obs = ops.zeros(p, m, dtype=torch.float64)  # observation sums (fused path)
        self.amax_obs = ops.zeros(p, m)
        self._obs_sums_t = -1
        self.ybar = ops.zeros(p, m)
        self.innov = ops.zeros(p, m)
        self.sinv = ops.zeros(p, p)
        self.eps = ops.empty(1, self.Nl) if p > q else None   # CH_EPS draws (barrier row)

    def _set_obs_rows(self, p: int) -> None:
        """Re-plan the observation-dependent storage (a constraint adds a barrier row);
        only before the first predict, when no observation history exists."""
        if p == self.p:
            return
        if self.t != 0:
            raise ValueError("the observation rows (constraint) cannot change mid-horizon")
        d, cap = self.d, self.cap
        x0 = self.mean[:d].clone()
        self.p = p
        self._alloc_obs()
        self.cap = 0
        self._grow(cap)
        self.reset(x0)

    def reset(self, x0) -> None:
        """Start a new horizon from N identical copies of x0 ((d x m), host or device),
        reusing every buffer (closed-loop driver: one smoother per MPC step, enks.py:105-128)."""
        d, q = self.d, self.q
        self.x0_exact = None if torch.is_tensor(x0) else np.array(x0, dtype=float)
        x0 = x0 if torch.is_tensor(x0) else self.ops.to_device(np.asarray(x0, float))
        self.t = 0
        self.n_upd = 0
        self.slice0_zero = True
        self._pending = None
        self._obs_t = -1
        self._obs_sums_t = -1
        self._last_stale = False
        self.mean[:d].copy_(x0)
        self.last.copy_(x0[:q].repeat(1, self.Nl))
        if self.pair:
            self.Ah[:self.ds].zero_()
            self.Al[:self.ds].zero_()
            self.a_inv[:self.ds].fill_(1.0)
        else:
            self.Abuf[:d].zero_()

    # ------------------------------------------------------------ storage
    def _grow(self, cap: int) -> None:
        """(Re)allocate the append-only basis for `cap` steps (slices 0..cap)."""
        if cap <= self.cap:
            return
        ops, d, ds, p, K, m = self.ops, self.d, self.ds, self.p, self.K, self.m
        ra, ry = (cap + 1) * ds, cap * p
        if self.pair:
            f16 = torch.float16
            new = dict(Ah=ops.empty(ra, K, dtype=f16), Al=ops.empty(ra, K, dtype=f16),
                       a_inv=ops.empty(ra), Yh=ops.empty(ry, K, dtype=f16),
                       Yl=ops.empty(ry, K, dtype=f16), y_inv=ops.empty(ry))
            a_keys, y_keys = ("Ah", "Al", "a_inv"), ("Yh", "Yl", "y_inv")
        else:
            new = dict(Abuf=ops.empty(ra, K), Ybuf=ops.empty(ry, K))
            a_keys, y_keys = ("Abuf",), ("Ybuf",)
        G = ops.zeros(ra, ry)
        mean = ops.zeros((cap + 1) * d, m)   # full [X; U; dU] slices
        PA = ops.empty(ra, p)
        PY = ops.empty(ry, p)
        if self.cap:
            rows_a, rows_y = (self.t + 1) * ds, self.t * p
            for k in a_keys:
                new[k][:rows_a] = getattr(self, k)[:rows_a]
            for k in y_keys:
                new[k][:rows_y] = getattr(self, k)[:rows_y]
            G[:rows_a, :rows_y] = self.G[:rows_a, :rows_y]
            mean[:(self.t + 1) * d] = self.mean[:(self.t + 1) * d]
        for k, v in new.items():
            setattr(self, k, v)
        self.G, self.mean, self.PA, self.PY = G, mean, PA, PY
        self.delta = ops.empty(ra, m) if self.chain else None
        if getattr(self, "use_tc2", False):
            self.pyT_hi = ops.empty(p * cap * p)
            self.pyT_lo = ops.empty(p * cap * p)
        self.cap = cap

    def memory_bytes(self) -> int:
        keys = ("Ah", "Al", "a_inv", "Yh", "Yl", "y_inv", "A_new") if self.pair \
            else ("Abuf", "Ybuf")
        return sum(t.numel() * t.element_size() for t in
                   [getattr(self, k) for k in keys] + [self.G, self.mean, self.PA, self.PY,
                                                       self.slice_raw, self.obs_raw, self.last])

    def _store_rows(self, which: str, r0: int, src) -> None:
        """Write fp32 rows (anomalies / centred observations) into the basis at row r0."""
        R = src.shape[0]
        if self.pair:
            h, l, inv = (self.Ah, self.Al, self.a_inv) if which == "A" else (self.Yh, self.Yl,
                                                                            self.y_inv)
            self.ops.f16pair_split(src, h[r0:r0 + R], l[r0:r0 + R], inv[r0:r0 + R])
        else:
            buf = self.Abuf if which == "A" else self.Ybuf
            if buf[r0:r0 + R].data_ptr() != src.data_ptr():
                buf[r0:r0 + R].copy_(src)

    def _rows_fp32(self, which: str, r0: int, r1: int):
        """fp32 view (fp32 basis) or reconstruction (fp16 pairs) of basis rows [r0, r1)."""
        if not self.pair:
            return (self.Abuf if which == "A" else self.Ybuf)[r0:r1]
        h, l, inv = (self.Ah, self.Al, self.a_inv) if which == "A" else (self.Yh, self.Yl,
                                                                        self.y_inv)
        out = self.ops.empty(r1 - r0, self.K)
        if r1 > r0:
            self.ops.f16pair_recon(h[r0:r1], l[r0:r1], inv[r0:r1], out)
        return out

    def newest_anomalies(self):
        """fp32 anomalies of the newest predicted slice (d x K)."""
        self._finish_slice()
        d, ds, t, q = self.d, self.ds, self.t, self.q
        if self.chain:  # [X; U] from the fp32 copy, dU from the basis
            out = self.ops.empty(d, self.K)
            out[:q] = self.A_new[:q]
            out[q:] = self._rows_fp32("A", t * ds + self.n, (t + 1) * ds)
            return out
        return self._rows_fp32("A", t * d, (t + 1) * d) if self.pair else self.Abuf[t * d:(t + 1) * d]

    # ------------------------------------------------------------ binding
    def bind(self, vs) -> None:
        if self._bound is vs:
            return
        ops = self.ops
        con = getattr(vs, "constraint", None)
        self.barrier = None if con is None else _barrier_spec(con, ops, self.n, self.l, self.m)
        self._set_obs_rows(self.q + (0 if con is None else 1))
        if (self.N - 1) * self.m < self.p:
            import warnings

            warnings.warn(
                f"rank-deficient Sigma_y: (N - 1) m = {(self.N - 1) * self.m} < p = {self.p}. The "
                "reference's 1e-9 relative jitter is below fp32 resolution; the device escalates "
                "it, and its fp32 gain is not a reliable match for the fp64 reference here "
                "(use N m > p).", RuntimeWarning, stacklevel=3)
        self.forecast = Forecaster(vs.model, ops, self.n, self.l)
        self.noise_w = _noise_params(vs.process_noise, ops, self.l, self.m)
        self.noise_vx = _noise_params(vs.obs_noise_x, ops, self.n, self.m)
        self.noise_vu = _noise_params(vs.obs_noise_u, ops, self.l, self.m)
        # all channels diagonal: draw W, V_X, V_U of a step in one launch during predict
        self.fused_noise = (all(c.kind == "diag" for c in (self.noise_w, self.noise_vx, self.noise_vu))
                            and hasattr(ops, "noise_fill_multi"))
        # the fused 2-32-32-1 forecast kernel can draw some of the step's noise jobs (W first) in
        # its three idle warps; ENKS_NOISE_IN_CNN = how many (0..3; default 0: measured slower --
        # three warps per SM cannot keep up with the stand-alone launch)
        fusable = (self.fused_noise and self.forecast.kind == "cnn"
                   and hasattr(ops, "cnn_forward_noise") and ops.cnn_noise_fusable(self.forecast, self.n))
        self.noise_in_forecast = (max(0, min(3, int(os.environ.get("ENKS_NOISE_IN_CNN", "0"))))
                                  if fusable else 0)
        # predict's slice and observation member sums in one pass (ENKS_SUM2=0: two passes)
        self.sum2 = hasattr(ops, "member_sum2") and os.environ.get("ENKS_SUM2", "1") != "0"
        # SMs the cross-moment grids leave to the concurrent side-stream gain solve (update())
        self.sm_reserve = (max(0, min(16, int(os.environ.get("ENKS_SM_RESERVE", "2"))))
                           if hasattr(ops, "set_sm_reserve") else 0)
        if self.fused_noise and getattr(self, "v_raw", None) is None:
            self.v_raw = ops.empty(self.q, self.K)  # raw [v_x; v_u] of the newest step
        # observation never materialised: its centring forms [x; u] + [v_x; v_u] on the fly (and,
        # without the MN-major shift, writes the transposed Yc_tau planes the shift reads)
        self.obs_fused = (self.fused_noise and self.shift_f16 and self.barrier is None
                          and self.p == self.q and hasattr(ops, "member_center_f16pair_t")
                          and os.environ.get("ENKS_OBS_FUSED", "1") != "0")
        self._obs_t = -1
        self._obs_key = None
        self._bound = vs

    # ------------------------------------------------------------ helpers
    def _head(self, streams):
        """Entropy words of the streams' (seed, prefix), or the device-resident words."""
        if self.dev_head is not None:
            return self.dev_head
        return entropy_head(streams.seed, tuple(streams.prefix))

    def _noise_stream(self):
        """Stream for the noise draws that overlap the forecast (None off-GPU, or when
        ENKS_NOISE_CONCURRENT=0: drawn on the main stream before the forecast)."""
        if getattr(self.ops, "device", None) is None or self.ops.device.type != "cuda":
            return None
        if os.environ.get("ENKS_NOISE_CONCURRENT", "1") == "0":
            return None
        if getattr(self, "_nstream", None) is None:
            self._nstream = torch.cuda.Stream(device=self.ops.device)
        return self._nstream

    def _side_stream(self):
        """Second CUDA stream for the gain solve (None off-GPU)."""
        if getattr(self.ops, "device", None) is None or self.ops.device.type != "cuda":
            return None
        if getattr(self, "_side", None) is None:
            # high priority: the one-CTA gain solve is dispatched ahead of the cross-moment CTAs
            # queued behind it on the main stream, instead of waiting for an SM to drain
            prio = int(os.environ.get("ENKS_SIDE_PRIORITY", "-1"))
            self._side = torch.cuda.Stream(device=self.ops.device, priority=prio)
        return self._side

    @_nvtx("enks.gain_solve")
    def _spd_async(self, side, S, scale) -> None:
        """Sigma_y^{-1} with the reference's jitter fallback (enks.py:234-244), on `side`
        after everything queued so far on the main stream."""
        if side is None:
            self.ops.spd_inverse(S, scale, self.sinv, self.status, self.jitter)
            return
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.ops.spd_inverse(S, scale, self.sinv, self.status, self.jitter)

    def _join_side(self, side) -> None:
        if side is not None:
            torch.cuda.current_stream().wait_stream(side)

    def _barrier_row(self, head, t) -> None:
        """Observation row q: softplus(g(slice_i)) + sqrt(var) eps_i, eps_i the first draw of
        substream (i, t, CH_EPS)  (enks.py:201-208, virtualsys.py:289-302)."""
        if self.barrier is None:
            return
        ops = self.ops
        ops.noise_fill(head, t, CH_EPS, self.member0, self.Nl, 1, 1, out=self.eps)
        ops.barrier_row(self.barrier, self.slice_raw, self.n, self.l, self.m, self.Nl, self.eps,
                        self.obs_raw[self.q:self.q + 1])

    def _noise(self, spec: _Noise, head, t, ch, rows, out=None, base=None, out_plus=None):
        """out = L z ; out_plus = base + L z for this rank's members."""
        ops = self.ops
        if spec.kind == "zero":
            if out is not None:
                out.zero_()
            if out_plus is not None:
                out_plus.copy_(base)
            return
        if spec.kind == "diag":
            ops.noise_fill(head, t, ch, self.member0, self.Nl, rows, self.m, diag=spec.diag,
                           out=out, base=base, out_plus=out_plus)
            return
        z = ops.empty(rows, self.K)
        ops.noise_fill(head, t, ch, self.member0, self.Nl, rows, self.m, out=z)
        if out is not None:
            ops.gemm(spec.dense, z, out)
        if out_plus is not None:
            ops.gemm(spec.dense, z, out_plus, beta=1.0, C0=base)

    def _local_sums(self, src, acc, amax=None, src2=None) -> None:
        """This rank's member sums of src (+ src2) relative to its own first member; under
        sharding converted to absolute sums (+ n_local * s) ready for the allreduce."""
        self.ops.member_sum(src, self.Nl, self.m, None, acc, amax, src2=src2)
        if self.comm.size > 1:
            self.ops.member_sum_rebase(src, self.m, acc, float(self.Nl), src2=src2)

    def _global_sums(self, items) -> None:
        """ONE collective for every (src, acc, src2) of `items`, then each acc back to sums
        relative to this rank's first member (-N * s) -- what the centring kernels expect with
        z0 = NULL.  No broadcast of global member 0 (enks_member_sum_rebase)."""
        if self.comm.size <= 1:
            return
        self.comm.allreduce_many([acc for _, acc, _ in items])
        for src, acc, src2 in items:
            self.ops.member_sum_rebase(src, self.m, acc, -float(self.N), src2=src2)

    def _center(self, src, mean_out, anom_out, pair_rows=None, f32_rows=0, skip=(0, 0),
                obs_sums=False, defer=False):
        """Member mean (rows x m) and anomalies of `src` (rows x K) relative to each rank's first
        member (identical members give exactly zero anomalies at any N and any rank count).

        pair_rows=(which, r0): write the anomalies straight into the fp16-pair basis at row r0
        (plus an fp32 copy of the first f32_rows rows into anom_out).  obs_sums: also form this
        step's observation sums (slice [x; u] + [v_x; v_u], enks.py:194-200, 231) in the same
        collective, for the fused observation centring of update()."""
        ops, rows = self.ops, src.shape[0]
        if rows > self.acc.shape[0]:
            self.acc = ops.zeros(rows, self.m, dtype=torch.float64)
            self.amax = ops.zeros(rows, self.m)
        acc = self.acc[:rows]
        amax = None if pair_rows is None else self.amax[:rows]
        p = self.p
        if (obs_sums and self.sum2 and src.data_ptr() == self.slice_raw.data_ptr()
                and amax is not None and self.m % 4 == 0):
            # slice and observation sums in one pass over the slice (its [x; u] rows read once)
            self.ops.member_sum2(src, p, self.v_raw, self.Nl, self.m, acc, amax, self.acc_obs,
                                 self.amax_obs)
            if self.comm.size > 1:
                self.ops.member_sum_rebase(src, self.m, acc, float(self.Nl))
                self.ops.member_sum_rebase(self.slice_raw[:p], self.m, self.acc_obs,
                                           float(self.Nl), src2=self.v_raw)
        else:
            self._local_sums(src, acc, amax)
            if obs_sums:
                self._local_sums(self.slice_raw[:p], self.acc_obs, self.amax_obs, src2=self.v_raw)
        items = [(src, acc, None)]
        if obs_sums:
            items.append((self.slice_raw[:p], self.acc_obs, self.v_raw))
            self._obs_sums_t = self.t + 1
        self._global_sums(items)

        def centre():
            if pair_rows is None:
                ops.member_center(src, self.Nl, self.m, None, acc, self.N, mean=mean_out,
                                  anom=anom_out)
                return
            which, r0 = pair_rows
            h, l, inv = (self.Ah, self.Al, self.a_inv) if which == "A" else (self.Yh, self.Yl,
                                                                            self.y_inv)
            hr = rows - (skip[1] - skip[0])  # basis rows written
            ops.member_center_f16pair(src, self.Nl, self.m, None, acc, amax, self.N, mean_out,
                                      h[r0:r0 + hr], l[r0:r0 + hr], inv[r0:r0 + hr],
                                      f32=anom_out, rows_f32=f32_rows, skip=skip)

        if defer:  # the new slice's centring waits for update(), behind the gain-solve launch
            self._pending = centre
        else:
            centre()

    def _finish_slice(self) -> None:
        """Run the deferred centring of the newest predicted slice (predict's last stage), if any:
        update() issues it after launching the side-stream gain solve, so at small ensembles the
        two overlap; every reader of the slice's basis rows / mean calls this first."""
        f, self._pending = self._pending, None
        if f is not None:
            f()

    def _center_obs_fused(self, tau) -> None:
        """Centre y = [x; u] + [v_x; v_u] (never materialised) into the basis rows of Yc_tau and
        (without the MN-major shift) the transposed planes of the newest-slice shift; y_bar = member
        mean (enks.py:231-232).
        The member sums normally come from predict's collective (obs_sums)."""
        ops, p, m = self.ops, self.p, self.m
        src, src2 = self.slice_raw[:p], self.v_raw
        acc, amax = self.acc_obs, self.amax_obs
        if self._obs_sums_t != tau:
            self._local_sums(src, acc, amax, src2=src2)
            self._global_sums([(src, acc, src2)])
        r0 = (tau - 1) * p
        ops.member_center_f16pair_t(src, src2, self.Nl, m, None, acc, amax, self.N, self.ybar,
                                    self.Yh[r0:r0 + p], self.Yl[r0:r0 + p], self.y_inv[r0:r0 + p],
                                    self.ycT_h, self.ycT_l, self.ycT_inv)

    # ------------------------------------------------------------ predict
    @_nvtx("enks.predict")
    def predict(self, vs, streams) -> None:
        """enks.py:156-171: W draw, new slice [f(x,u); u+w; w], append, mean."""
        self.bind(vs)
        tau = self.t + 1
        if tau > self.cap:
            self._grow(max(2 * self.cap, tau))
        ops, n, l, d = self.ops, self.n, self.l, self.d
        head = self._head(streams)
        sr, ob = self.slice_raw, self.obs_raw
        self._finish_slice()  # (a predict with no update in between)
        if self.t >= 1 and self.n_upd < self.t:
            # the previous step had no update (predict twice in a row, as the reference allows):
            # its observation block and gain column hold no information -- zero them so the
            # later cross moments / corrections read exact zeros, not stale or uninitialised rows
            self._zero_obs_block(self.t)
        if self._last_stale:  # newest members are the un-updated predicted slice [f; u + w]
            self.last.copy_(sr[:self.q])
        self._last_stale = True
        if self.fused_noise:
            # W (enks.py:165-168) and this step's observation noise V_X, V_U (enks.py:194-200,
            # drawn at t = tau with the same substream ids update() would use) in one launch on a
            # second stream, concurrently with the forecast (both are SIMT-issue / latency bound
            # and share SMs): dU = w, U = u + w, raw v_x, raw v_u; the two sums that need the
            # forecast (x' + v_x, U + v_u) follow on the main stream.
            jobs = [dict(t=tau, ch=CH_W, rows=l, diag=self.noise_w.diag, out=sr[n + l:],
                         base=self.last[n:], out_plus=sr[n:n + l]),
                    dict(t=tau, ch=CH_VX, rows=n, diag=self.noise_vx.diag, out=self.v_raw[:n]),
                    dict(t=tau, ch=CH_VU, rows=l, diag=self.noise_vu.diag,
                         out=self.v_raw[n:n + l])]
            # the first `noise_in_forecast` jobs are drawn by the fused CNN's idle warps (cnn_tc.cu),
            # the rest by the noise kernel on a second stream
            k = self.noise_in_forecast
            ns = self._noise_stream()
            if k < len(jobs):
                if ns is not None:
                    ns.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(ns) if ns is not None else contextlib.nullcontext():
                    ops.noise_fill_multi(head, self.member0, self.Nl, self.m, jobs[k:])
            if k:
                ops.cnn_forward_noise(self.forecast, self.last[:n], self.last[n:], sr[:n], self.Nl,
                                      head, self.member0, jobs[:k])
            else:
                self.forecast(ops, self.last, sr[:n], n, self.Nl)
            if ns is not None and k < len(jobs):
                torch.cuda.current_stream().wait_stream(ns)
            if not self.obs_fused:
                ops.add(sr[:n + l], self.v_raw, ob[:n + l])
            self._barrier_row(head, tau)
            self._obs_t = tau
            self._obs_key = (streams.seed, tuple(streams.prefix))
        else:
            self.forecast(ops, self.last, sr[:n], n, self.Nl)
            # ΔU slot = w, U slot = u + w  (one draw fills both, enks.py:168)
            self._noise(self.noise_w, head, tau, CH_W, l, out=sr[n + l:], base=self.last[n:],
                        out_plus=sr[n:n + l])
        if self.pair:
            # fp32 copy of the [x; u] rows only (the newest-slice shift's C0)
            # (derived-U chain: the U rows stay out of the basis; A_new keeps them in fp32)
            self._center(sr, self.mean[tau * d:(tau + 1) * d], self.A_new,
                         pair_rows=("A", tau * self.ds), f32_rows=self.q,
                         skip=(n, n + l) if self.chain else (0, 0),
                         obs_sums=self.obs_fused and self.fused_noise, defer=True)
        else:
            self._center(sr, self.mean[tau * d:(tau + 1) * d], self.Abuf[tau * d:(tau + 1) * d],
                         defer=True)
        self.t = tau

    # ------------------------------------------------------------ update
    @_nvtx("enks.update")
    def update(self, y_ref_dev, streams) -> None:
        """enks.py:212-248 restated on the append-only basis (module docstring)."""
        ops, comm = self.ops, self.comm
        if self.t < 1:
            self._update_t0(y_ref_dev, streams)
            return
        if self.n_upd >= self.t:
            # a second update at the same t (the reference allows it: enks.py:212-253 shifts the
            # members again): the append-only basis holds one observation block per slice, so
            # re-seed from the explicit members first (slow path, exact)
            self._reseed_from_members()
        n, l, d, p, tau = self.n, self.l, self.d, self.p, self.t
        head = self._head(streams)
        sr, ob = self.slice_raw, self.obs_raw
        # perturbed observations [x + v_x; u + v_u]  (enks.py:194-200)
        redraw = self._obs_t != tau or self._obs_key != (streams.seed, tuple(streams.prefix))
        if redraw:
            self._noise(self.noise_vx, head, tau, CH_VX, n, base=sr[:n], out_plus=ob[:n])
            self._noise(self.noise_vu, head, tau, CH_VU, l, base=sr[n:n + l],
                        out_plus=ob[n:n + l])
            self._barrier_row(head, tau)
        yc = self.Yc_new if self.pair else self.Ybuf[(tau - 1) * p:tau * p]
        fused_obs = self.obs_fused and not redraw
        if not (fused_obs and self.pair):
            self._finish_slice()  # the observation centring below reuses the sum buffers
        if fused_obs:
            self._center_obs_fused(tau)
        elif self.pair:
            self._center(ob, self.ybar, yc, pair_rows=("Y", (tau - 1) * p),
                         f32_rows=0 if yc is None else p)
        else:
            self._center(ob, self.ybar, yc)

        # P = [A_s0..A_tau ; Yc_1..Yc_tau] Yc_tau^T  (local K-partial, then allreduce)
        ds = self.ds  # basis rows per slice (n + l under the derived-U chain, else d)
        a0 = ds if self.slice0_zero else 0
        rows_a = (tau + 1) * ds
        PA, PY = self.PA[a0:rows_a], self.PY[:tau * p]
        scale = self.lam / self.N
        side = self._side_stream()
        if self.pair:
            yb = slice((tau - 1) * p, tau * p)
            yh, yl, yi = self.Yh[yb], self.Yl[yb], self.y_inv[yb]
            # Sigma_y block first, so the gain solve (one SM, latency-bound) overlaps the big
            # contraction on a second stream (enks.py:234-246)
            ops.gemm_f16pair(yh, yl, yi, yh, yl, yi, PY[(tau - 1) * p:], tag="cross")
            comm.allreduce_(PY[(tau - 1) * p:])
            self._spd_async(side, PY[(tau - 1) * p:], scale)
            self._finish_slice()  # the new slice's centring, next to the gain solve
            # the cross-moment grids leave SMs to the side-stream gain solve (one CTA that
            # otherwise waits for the first cross CTA to drain: exposed at small ensembles)
            reserve = self.sm_reserve if side is not None else 0
            if reserve:
                ops.set_sm_reserve(reserve)
            ops.gemm_f16pair(self.Ah[a0:rows_a], self.Al[a0:rows_a], self.a_inv[a0:rows_a],
                             yh, yl, yi, PA, tag="cross")
            if tau > 1:
                ops.gemm_f16pair(self.Yh[:(tau - 1) * p], self.Yl[:(tau - 1) * p],
                                 self.y_inv[:(tau - 1) * p], yh, yl, yi, PY[:(tau - 1) * p],
                                 tag="cross")
            if reserve:
                ops.set_sm_reserve(0)
            comm.allreduce_many([PY[:(tau - 1) * p], PA])  # one collective for the rest of P
        else:
            if self.use_tc:
                ops.tf32_split(yc, self.yc_hi, self.yc_lo)
                ops.gemm_nt_tc(self.Abuf[a0:rows_a], self.yc_hi, self.yc_lo, PA, tag="cross")
                ops.gemm_nt_tc(self.Ybuf[:tau * p], self.yc_hi, self.yc_lo, PY, tag="cross")
            else:
                ops.gemm(self.Abuf[a0:rows_a], yc, PA, trans_b=True, tag="cross")
                ops.gemm(self.Ybuf[:tau * p], yc, PY, trans_b=True, tag="cross")
            comm.allreduce_many([PA, PY])
            # Sigma_y^{-1} with the reference's jitter fallback (enks.py:234-244)
            self._spd_async(None, PY[(tau - 1) * p:], scale)

        # S_s = P_{A_s} - sum_{tau' < tau} G_{tau',s} P_{Yc_tau'}  (block upper-triangular G)
        tri = (ds, p) if a0 == ds else (0, 0)
        gcol = self.G[a0:rows_a, (tau - 1) * p:tau * p]
        r0 = tau * d
        # under sharding the correction and gain GEMMs are row-sharded: this rank owns a
        # contiguous run of slices [s_lo, s_lo + s_cnt) (rows lo..hi of S), and the gain rows are
        # allgathered afterwards so G stays replicated (mean / shift / readback read all of it)
        nsl = (rows_a - a0) // ds
        s_lo, s_cnt = partition(nsl, comm.size, comm.rank) if comm.size > 1 else (0, nsl)
        lo, hi = s_lo * ds, (s_lo + s_cnt) * ds
        kk = (tau - 1) * p
        k0 = min(s_lo * p, kk) if tri[0] else 0  # block-triangular: owned slices skip early K
        PAo, Go = PA[lo:hi], self.G[a0 + lo:a0 + hi]
        if self.use_tc2:
            if tau > 1:
                pth = self.pyT_hi[:p * kk].view(p, kk)
                ptl = self.pyT_lo[:p * kk].view(p, kk)
                ops.tf32_split(self.PY[:kk], pth, ptl, transpose=True)
                if hi > lo and kk > k0:
                    ops.gemm_tc(Go[:, k0:kk], pth[:, k0:], ptl[:, k0:], PAo, alpha=-1.0, beta=1.0,
                                C0=PAo, tri=tri, tag="correction")
            # G_{tau,s} = (lam/N) S_s Sigma_y^{-1}
            self._join_side(side)
            ops.tf32_split(self.sinv, self.sinvT_hi, self.sinvT_lo, transpose=True)
            if hi > lo:
                ops.gemm_tc(PAo, self.sinvT_hi, self.sinvT_lo, gcol[lo:hi], alpha=scale,
                            tag="gain")
        else:
            if tau > 1 and hi > lo and kk > k0:
                ops.gemm(Go[:, k0:kk], self.PY[k0:kk], PAo, alpha=-1.0, beta=1.0, C0=PAo, tri=tri)
            self._join_side(side)
            if hi > lo:
                ops.gemm(PAo, self.sinv, gcol[lo:hi], alpha=scale)
        if comm.size > 1:
            self._allgather_gain_rows(gcol, nsl, ds)
        if self.record is not None:
            self._record_step(tau, a0, rows_a, scale)
        # mean_s += G_{tau,s} (y_ref - y_bar)   (enks.py:247-248 on the mean)
        self.n_upd = tau
        ops.sub(y_ref_dev, self.ybar, self.innov)
        q = self.q
        if self.chain:
            # compact increments, then U rows by prefix sums; newest-slice [X; U] gain rows
            dl = self.delta[:rows_a - a0]
            if self.use_tc2 and ops.tc_applicable(gcol, self.innT_hi):
                ops.tf32_split(self.innov, self.innT_hi, self.innT_lo, transpose=True)
                ops.gemm_tc(gcol, self.innT_hi, self.innT_lo, dl, tag="mean")
            else:
                ops.gemm(gcol, self.innov, dl)
            ops.uchain_apply(dl, self.mean[d:], gcol, self.gtt, tau, n, l, self.m, p)
            g_tt = self.gtt
        else:
            mv = self.mean[a0 // ds * d:(tau + 1) * d]
            ops.gemm(gcol, self.innov, mv, beta=1.0, C0=mv)
            g_tt = self.G[tau * ds:tau * ds + q, (tau - 1) * p:tau * p]
        # newest slice [x; u] for the next forecast: mean + A_tau - G_{tau,tau} Yc_tau
        a_new = self.A_new if self.pair else self.Abuf[r0:r0 + d]  # (fp32 basis: ds == d)
        if self.shift_mn:
            yb = slice((tau - 1) * p, tau * p)
            ops.f16pair_split_cs(g_tt, self.y_inv[yb], self.gtt_h, self.gtt_l, self.gtt_inv)
            ops.gemm_f16pair_ex_mn(self.gtt_h, self.gtt_l, self.gtt_inv, self.Yh[yb], self.Yl[yb],
                                   self.last, alpha=-1.0, beta=1.0, C0=a_new[:q],
                                   bias=self.mean[r0:r0 + q], bias_cols=self.m, tag="shift")
        elif self.shift_f16:
            yb = slice((tau - 1) * p, tau * p)
            ops.f16pair_split(g_tt, self.gtt_h, self.gtt_l, self.gtt_inv)
            if not fused_obs:  # (the fused centring wrote the transposed planes)
                ops.f16pair_transpose(self.Yh[yb], self.Yl[yb], self.y_inv[yb], self.ycT_h,
                                      self.ycT_l, self.ycT_inv)
            ops.gemm_f16pair_ex(self.gtt_h, self.gtt_l, self.gtt_inv, self.ycT_h, self.ycT_l,
                                self.ycT_inv, self.last, alpha=-1.0, beta=1.0, C0=a_new[:q],
                                bias=self.mean[r0:r0 + q], bias_cols=self.m, tag="shift")
        elif self.use_tc2:
            ops.tf32_split(yc, self.ycT_hi, self.ycT_lo, transpose=True)
            ops.gemm_tc(g_tt, self.ycT_hi, self.ycT_lo, self.last, alpha=-1.0, beta=1.0,
                        C0=a_new[:q], bias=self.mean[r0:r0 + q], bias_cols=self.m, tag="shift")
        else:
            ops.gemm(g_tt, yc, self.last, alpha=-1.0, beta=1.0, C0=a_new[:q],
                     bias=self.mean[r0:r0 + q], bias_cols=self.m)
        self._last_stale = False

    def _allgather_gain_rows(self, gcol, nsl: int, ds: int) -> None:
        """Every rank's gain rows (slice-aligned, uneven) into every rank's G column block: one
        all-gather of equal padded row blocks through a staging buffer."""
        comm, p = self.comm, self.p
        per = -(-nsl // comm.size) * ds
        if getattr(self, "_gstage", None) is None or self._gstage.shape[0] < per:
            self._gstage = self.ops.empty(max(per, ds), p)
        st = self._gstage[:per]
        s_lo, s_cnt = partition(nsl, comm.size, comm.rank)
        if s_cnt:
            st[:s_cnt * ds].copy_(gcol[s_lo * ds:(s_lo + s_cnt) * ds])
        full = comm.all_gather_rows(st)
        for r in range(comm.size):
            r_lo, r_cnt = partition(nsl, comm.size, r)
            if r_cnt and r != comm.rank:
                gcol[r_lo * ds:(r_lo + r_cnt) * ds].copy_(full[r * per:r * per + r_cnt * ds])

    def _zero_obs_block(self, tau: int) -> None:
        """Zero the basis rows of Yc_tau and the gain column block of step tau."""
        p = self.p
        r0, r1 = (tau - 1) * p, tau * p
        if self.pair:
            self.Yh[r0:r1].zero_()
            self.Yl[r0:r1].zero_()
            self.y_inv[r0:r1].fill_(1.0)
        else:
            self.Ybuf[r0:r1].zero_()
        self.G[:, r0:r1].zero_()

    @_nvtx("enks.update_t0")
    def _update_t0(self, y_ref_dev, streams) -> None:
        """update() before the first predict (enks.py:212-253 at t = 0): the trajectory is slice 0
        alone.  Observation noise is drawn with t = 0 (enks.py:224); Sigma_y goes through the
        jittered Cholesky (jitter_events / LinAlgError as the reference); the gain is
        Sigma_xy Sigma_y^-1 with Sigma_xy = (lam/N) A_0 Yc^T, which is exactly zero for the
        identical copies of init_ensemble (enks.py:108-110), so only explicit members move.
        Rare, small path: fp32 SIMT GEMMs, members re-seeded afterwards."""
        ops, comm = self.ops, self.comm
        n, l, d, p, q, K = self.n, self.l, self.d, self.p, self.q, self.K
        head = self._head(streams)
        self.slice_raw.copy_(self.members_device()[:d])  # slice 0 [x; u; dU] of every member
        sr, ob = self.slice_raw, self.obs_raw
        self._noise(self.noise_vx, head, 0, CH_VX, n, base=sr[:n], out_plus=ob[:n])
        self._noise(self.noise_vu, head, 0, CH_VU, l, base=sr[n:q], out_plus=ob[n:q])
        self._barrier_row(head, 0)
        self._obs_t = -1
        yc = ops.empty(p, K)
        self._center(ob, self.ybar, yc)
        scale = self.lam / self.N
        sy = ops.empty(p, p)
        ops.gemm(yc, yc, sy, trans_b=True)
        comm.allreduce_(sy)
        ops.spd_inverse(sy, scale, self.sinv, self.status, self.jitter)
        if self.slice0_zero:
            return
        a0 = self.deviations()[:d]
        sxy = ops.empty(d, p)
        ops.gemm(a0, yc, sxy, trans_b=True)
        comm.allreduce_(sxy)
        g = ops.empty(d, p)
        ops.gemm(sxy, self.sinv, g, alpha=scale)
        ops.sub(y_ref_dev, self.ybar, self.innov)
        mean0 = self.mean[:d].clone()
        ops.gemm(g, self.innov, mean0, beta=1.0, C0=mean0)
        # members = mean' + A_0 - G Yc
        new = ops.empty(d, K)
        ops.gemm(g, yc, new, alpha=-1.0, beta=1.0, C0=a0, bias=mean0, bias_cols=self.m)
        self._replace_members_dev(new, 0)

    def _reseed_from_members(self) -> None:
        """Re-seed the representation from the current explicit members (device, exact)."""
        self._replace_members_dev(self.members_device(), self.t)

    # ------------------------------------------------------------ per-step record (tests)
    def _expand_rows(self, compact: np.ndarray, a0: int) -> np.ndarray:
        """Rows of slices a0/ds..t in the basis layout -> full (T d, cols) rows of slices 0..t
        (zero rows for a skipped slice 0; U rows = prefix sums of dU under the derived-U chain)."""
        ds, d, n, l, t = self.ds, self.d, self.n, self.l, self.t
        cols = compact.shape[1]
        full_c = np.zeros(((t + 1) * ds, cols))
        full_c[a0:] = compact
        if not self.chain:
            return full_c
        cv = full_c.reshape(t + 1, ds, cols)
        out = np.zeros((t + 1, d, cols))
        out[:, :n] = cv[:, :n]
        out[:, n + l:] = cv[:, n:]
        out[:, n:n + l] = np.cumsum(cv[:, n:], axis=0)
        return out.reshape((t + 1) * d, cols)

    def _record_step(self, tau: int, a0: int, rows_a: int, scale: float) -> None:
        """Append this update's Sigma_y (p x p, symmetrised as enks.py:234), Sigma_xy
        (T d x p, enks.py:235-236) and gain (T d x p, enks.py:246) as fp64 host arrays to
        ``self.record`` -- the same keys as the oracle's ``record=`` hook.  Test-only: syncs;
        single rank (under sharding each rank corrects only its own rows of P)."""
        if self.comm.size > 1:
            raise RuntimeError("record= is single-rank only")
        if self.ops.device.type == "cuda":
            torch.cuda.synchronize(self.ops.device)
        p = self.p
        sy = scale * self.PY[(tau - 1) * p:tau * p].double().cpu().numpy()
        S = scale * self.PA[a0:rows_a].double().cpu().numpy()
        G = self.G[a0:rows_a, (tau - 1) * p:tau * p].double().cpu().numpy()
        rec = self.record
        rec.setdefault("sigma_y", []).append(0.5 * (sy + sy.T))
        rec.setdefault("sigma_xy", []).append(self._expand_rows(S, a0))
        rec.setdefault("gain", []).append(self._expand_rows(G, a0))

    # ------------------------------------------------------------ readback
    def deviations(self, rows: int | None = None):
        """Member deviations M - mean for slices 0..t, (T d x K) on device."""
        self._finish_slice()
        ops, d, ds, p, t = self.ops, self.d, self.ds, self.p, self.t
        R, Rc = (t + 1) * d, (t + 1) * ds
        out = ops.empty(Rc, self.K)
        a0 = ds if self.slice0_zero else 0
        A = self._rows_fp32("A", 0, Rc)
        out[:a0] = A[:a0]
        ku = min(self.n_upd, t) * p  # only observation blocks that have been drawn
        if ku:
            ops.gemm(self.G[a0:Rc, :ku], self._rows_fp32("Y", 0, ku), out[a0:], alpha=-1.0,
                     beta=1.0, C0=A[a0:Rc], tri=(ds, p) if a0 else (0, 0))
        else:
            out[a0:] = A[a0:Rc]
        if not self.chain:
            return out
        # expand [X; dU] slices to [X; U; dU] with U_s = sum_{s' <= s} dU_s' (slice 0 is zero)
        n, l, K = self.n, self.l, self.K
        full = ops.zeros(R, K)
        fv, cv = full.view(t + 1, d, K), out.view(t + 1, ds, K)
        fv[:, :n] = cv[:, :n]
        fv[:, n + l:] = cv[:, n:]
        fv[:, n:n + l] = torch.cumsum(cv[:, n:], dim=0)
        return full

    def members_device(self):
        dev = self.deviations()
        R = dev.shape[0]
        mean = self.mean[:R]
        return dev + mean.repeat(1, self.Nl)

    def mean_host(self) -> np.ndarray:
        self._finish_slice()
        R = (self.t + 1) * self.d
        out = self.ops.to_host(self.mean[:R])
        if self.slice0_zero and self.x0_exact is not None:
            out[:self.d] = self.x0_exact  # identical copies: slice 0 is x0 itself, in fp64
        return out

    def clear_flags(self) -> None:
        """Per-solve device flags back to a fresh engine's: failure status, jitter count and the
        Burgers CFL maxima (a reused engine must not inherit an earlier solve's failure)."""
        self.status.zero_()
        self.jitter.zero_()
        fc = getattr(self, "forecast", None)
        if fc is not None and fc.kind == "burgers":
            fc.vmax.zero_()
            fc.flags.zero_()

    def jitter_events(self) -> int:
        return int(self.ops.read_scalar(self.jitter))

    def check_status(self) -> None:
        fc = getattr(self, "forecast", None)
        if fc is not None and fc.kind == "burgers":
            fc.check_cfl(self.comm)
        if int(self.ops.read_scalar(self.status)) != 0:
            raise np.linalg.LinAlgError("observation covariance not positive definite even "
                                        "after jitter")

    def replace_members(self, members_local: np.ndarray, t: int) -> None:
        """Reset the representation to explicit members (local shard, (Nl, (t+1)d, m))."""
        ops, d = self.ops, self.d
        R = (int(t) + 1) * d
        members_local = np.asarray(members_local, dtype=float)
        M = members_local.transpose(1, 0, 2).reshape(R, self.K)
        self.slice0_zero = True  # re-derived from the data below
        self.x0_exact = members_local[0, :d].copy() if len(members_local) else None
        self._replace_members_dev(ops.to_device(M), t)

    def _replace_members_dev(self, Mdev, t: int) -> None:
        """replace_members for a device tensor in the member-column layout ((t+1) d x K)."""
        ops, d = self.ops, self.d
        self._pending = None  # the explicit members replace any deferred centring
        self._obs_t = -1
        self.t = 0
        if self.chain:  # explicit members need not obey U_s = U_{s-1} + dU_s: full rows
            self._explicit = True
            self._alloc_obs()
            self.cap = 0
        self._grow(max(t, 1))
        self.t = int(t)
        R = (self.t + 1) * d
        self.G.zero_()
        anom = ops.empty(R, self.K)
        self._center(Mdev, self.mean[:R], anom)
        self._store_rows("A", 0, anom)
        self.n_upd = 0  # no observation history: the explicit members carry it
        if self.t:  # zero observation rows: the cross moments read them (their gains are zero)
            self._store_rows("Y", 0, ops.zeros(self.t * self.p, self.K))
        if self.pair:
            self.A_new[:self.q].copy_(anom[self.t * d:self.t * d + self.q])
        spread = torch.any(anom[:d] != 0).to(torch.float32).reshape(1)
        if self.comm.size > 1:  # every rank must take the same path (slice0_zero picks rows)
            self.comm.allreduce_max_(spread)
        x0_spread = bool(spread.item())
        if x0_spread or not self.slice0_zero:
            self.x0_exact = None
        self.slice0_zero = not x0_spread
        last = Mdev[self.t * d:self.t * d + self.q]
        self.last.copy_(last)
        self._last_stale = False
