"""Covariance tracking on the device (reference enks.py:96-102, 173-185, 250-252).

The reference keeps three lambda-scaled covariances as fp64 host arrays and rebuilds them on
every call: after predict the cross covariance of the whole trajectory with the new slice
(sigma_cross, (T d) x d), the new slice's covariance (sigma_pred, d x d) and the block-grown
trajectory covariance; after update the full trajectory covariance
sigma_traj = (lam/N) D D^T, D = members - mean ((T d) x (N m)) -- (T d)^2 N m flops per update.

Here they stay on the device between calls:

* D is formed once per tracked call (engine.deviations()), split into fp16-pair planes and
  contracted on the tcgen05 kind::f16 kernel (3 products, fp32-level accuracy);
* sigma_traj after an update is a SYRK: only the 256-wide block columns on and below the
  diagonal are computed (half the flops), the upper triangle is mirrored when the host reads it;
* sigma_pred is the last d rows of sigma_cross (the same contraction, reference enks.py:176-177);
* after predict the grown sigma_traj is an unevaluated block assembly [old, cross; cross^T,
  pred] -- evaluated only if read before the next update replaces it;
* under member sharding each rank contracts its own members and the SYRK partials are
  reduce-scattered by row blocks (each rank keeps its rows: row-sharded storage); sigma_cross
  is allreduced.

Host fp64 copies are made only when a field is read (the SmootherCovariances properties), so a
tracked horizon does no per-step host assembly.
"""
from __future__ import annotations

import numpy as np
import torch

BLOCK = 256  # SYRK block columns (one fp16-pair tcgen05 launch each)


class _Dense:
    """A device matrix, identical on every rank."""

    def __init__(self, t, ops):
        self.t, self.ops = t, ops

    def host(self):
        return self.ops.to_host(self.t)


class _SymRows:
    """Row-sharded lower-block SYRK result: this rank holds padded rows [r0, r0 + rows) of the
    R x R matrix whose 256-column blocks on and below the diagonal are valid."""

    def __init__(self, local, R, comm, ops):
        self.local, self.R, self.comm, self.ops = local, R, comm, ops

    def host(self):
        full = self.comm.all_gather_rows(self.local)[:self.R, :self.R]
        a = self.ops.to_host(full)
        # lower triangle as computed, upper mirrored (the diagonal blocks' upper halves were
        # computed too, in a different summation order -- mirroring keeps sigma_traj exactly
        # symmetric like the reference's D @ D.T)
        i = np.arange(self.R)
        return np.where(i[:, None] >= i[None, :], a, a.T)


class _Assembled:
    """sigma_traj grown by predict (enks.py:179-185): [old, cross[:old]; cross[:old]^T, pred]."""

    def __init__(self, old, cross, d):
        self.old, self.cross, self.d = old, cross, d

    def host(self):
        old = self.old.host() if hasattr(self.old, "host") else np.asarray(self.old, float)
        cross = self.cross.host()
        o = old.shape[0]
        block = np.zeros((o + self.d, o + self.d))
        block[:o, :o] = old
        block[:o, o:] = cross[:o]
        block[o:, :o] = cross[:o].T
        block[o:, o:] = cross[o:]
        return block


class SmootherCovariances:
    """lambda-scaled covariance tracking (enks.py:96-102).  The fields read as fp64 host arrays
    (materialised from device state on first read after each predict / update, then cached) and
    may be assigned like the reference dataclass's fields."""

    _FIELDS = ("sigma_traj", "sigma_pred", "sigma_cross")

    def __init__(self, sigma_traj, sigma_pred=None, sigma_cross=None):
        self._host = {"sigma_traj": sigma_traj, "sigma_pred": sigma_pred,
                      "sigma_cross": sigma_cross}
        self._dev = {}

    def _get(self, name):
        src = self._dev.get(name)
        if src is not None and self._host.get(name) is None:
            self._host[name] = src.host()
        return self._host.get(name)

    def _set(self, name, value):
        self._host[name] = value
        self._dev.pop(name, None)

    def _set_dev(self, name, src):
        self._dev[name] = src
        self._host[name] = None

    def _source(self, name):
        """Device source of a field, or its host array."""
        return self._dev.get(name) or self._host.get(name)

    sigma_traj = property(lambda s: s._get("sigma_traj"), lambda s, v: s._set("sigma_traj", v))
    sigma_pred = property(lambda s: s._get("sigma_pred"), lambda s, v: s._set("sigma_pred", v))
    sigma_cross = property(lambda s: s._get("sigma_cross"), lambda s, v: s._set("sigma_cross", v))

    def __repr__(self):
        shapes = {k: (None if self._source(k) is None else "device" if k in self._dev
                      else np.shape(self._host[k])) for k in self._FIELDS}
        return f"SmootherCovariances({shapes})"


def _planes(ops, D):
    f16 = torch.float16
    R, K = D.shape
    h, l, s = ops.empty(R, K, dtype=f16), ops.empty(R, K, dtype=f16), ops.empty(R)
    ops.f16pair_split(D, h, l, s)
    return h, l, s


def _tc_ok(ops, K):
    return hasattr(ops, "gemm_f16pair") and K >= 128 and K % 8 == 0


def track_predict(eng, cov: SmootherCovariances) -> None:
    """After predict: sigma_cross = (lam/N) D dev_new^T, sigma_pred = its last d rows
    (enks.py:173-178), sigma_traj = the block assembly (enks.py:179-185), left unevaluated."""
    ops, d = eng.ops, eng.d
    D = eng.deviations()                      # (T d) x K, the new slice last
    R, K = D.shape
    scale = eng.lam / eng.N
    cross = ops.empty(R, d)
    if _tc_ok(ops, K):
        h, l, s = _planes(ops, D)
        ops.gemm_f16pair(h, l, s, h[R - d:], l[R - d:], s[R - d:], cross, alpha=scale,
                         tag="cov")
    else:
        ops.gemm(D, D[R - d:], cross, trans_b=True, alpha=scale)
    eng.comm.allreduce_(cross)
    cross_src = _Dense(cross, ops)
    cov._set_dev("sigma_traj", _Assembled(cov._source("sigma_traj"), cross_src, d))
    cov._set_dev("sigma_cross", cross_src)
    cov._set_dev("sigma_pred", _Dense(cross[R - d:], ops))


def track_update(eng, cov: SmootherCovariances) -> None:
    """After update: sigma_traj = (lam/N) D D^T (enks.py:250-252) as a lower-block SYRK, partial
    over this rank's members, reduce-scattered by row blocks."""
    ops, comm = eng.ops, eng.comm
    D = eng.deviations()
    R, K = D.shape
    scale = eng.lam / eng.N
    Rp = -(-R // comm.size) * comm.size
    full = ops.zeros(Rp, R)
    if _tc_ok(ops, K):
        h, l, s = _planes(ops, D)
        del D
        for j0 in range(0, R, BLOCK):
            j1 = min(R, j0 + BLOCK)
            ops.gemm_f16pair(h[j0:], l[j0:], s[j0:], h[j0:j1], l[j0:j1], s[j0:j1],
                             full[j0:R, j0:j1], alpha=scale, tag="cov")
    else:
        ops.gemm(D, D, full[:R], trans_b=True, alpha=scale)
    cov._set_dev("sigma_traj", _SymRows(comm.reduce_scatter_rows(full), R, comm, ops))
