"""Host-side mirror of the reference's matrix-normal parameters and noise streams.

Mirrors reference pkg/src/enksmpc/matvar.py: ``MatrixNormalParams``
(matvar.py:59-93; cached Cholesky factors), ``NoiseStreams`` (matvar.py:136-154;
substreams keyed by (seed, prefix + ids)) and ``transform_standard_normal``
(matvar.py:183-188).  These are configuration objects: the smoother never
draws through them on the hot path -- the device noise kernel regenerates the
identical bitstream from (seed, prefix, member, t, channel) alone
(csrc/noise.cu).  The host ``substream`` stays available for users and tests.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["MatrixNormalParams", "NoiseStreams", "transform_standard_normal", "entropy_head"]

_SYM_TOL = 1e-12


def _lower_cholesky(mat: np.ndarray, what: str) -> np.ndarray:
    mat = np.asarray(mat, dtype=float)
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1]:
        raise ValueError(f"{what} must be square, got {mat.shape}")
    if mat.size:
        scale = max(1.0, float(np.abs(mat).max()))
        if float(np.abs(mat - mat.T).max()) > _SYM_TOL * scale:
            raise ValueError(f"{what} is not symmetric")
    try:
        return np.linalg.cholesky(0.5 * (mat + mat.T))
    except np.linalg.LinAlgError as exc:
        raise np.linalg.LinAlgError(f"{what} is not positive definite: {exc}") from exc


@dataclass
class MatrixNormalParams:
    """MN(mean; row_cov, col_cov) with lower Cholesky factors computed once."""

    mean: np.ndarray
    row_cov: np.ndarray
    col_cov: np.ndarray
    row_chol: np.ndarray = field(init=False, repr=False)
    col_chol: np.ndarray = field(init=False, repr=False)

    def __post_init__(self) -> None:
        self.mean = np.asarray(self.mean, dtype=float)
        if self.mean.ndim != 2:
            raise ValueError("mean must be a matrix")
        self.row_cov = np.asarray(self.row_cov, dtype=float)
        self.col_cov = np.asarray(self.col_cov, dtype=float)
        self.row_chol = _lower_cholesky(self.row_cov, "row_cov")
        self.col_chol = _lower_cholesky(self.col_cov, "col_cov")
        rows, cols = self.mean.shape
        if self.row_cov.shape != (rows, rows) or self.col_cov.shape != (cols, cols):
            raise ValueError("covariance shapes do not match the mean")

    @property
    def n(self) -> int:
        return self.mean.shape[0]

    @property
    def m(self) -> int:
        return self.mean.shape[1]


def _uint32_words(v: int) -> list[int]:
    v = int(v)
    if v < 0:
        raise ValueError("seed and stream ids must be non-negative")
    words = [v & 0xFFFFFFFF] if v == 0 else []
    while v > 0:
        words.append(v & 0xFFFFFFFF)
        v >>= 32
    return words


def entropy_head(seed: int, prefix: tuple) -> list[int]:
    """SeedSequence entropy words shared by every (member, t, channel) substream.

    numpy assembles [seed words zero-padded to the pool size 4] + [spawn-key
    words]; the spawn key is prefix + (member, t, channel), so everything up to
    the prefix is common and the device appends the last three ids.
    """
    head = _uint32_words(seed)
    if len(head) < 4:
        head = head + [0] * (4 - len(head))
    for k in prefix:
        head.extend(_uint32_words(k))
    return head


@dataclass(frozen=True)
class NoiseStreams:
    """Reproducible substreams named by (seed, prefix + ids)."""

    seed: int
    prefix: tuple = ()

    def substream(self, *ids: int) -> np.random.Generator:
        seq = np.random.SeedSequence(entropy=self.seed, spawn_key=tuple(self.prefix) + ids)
        return np.random.Generator(np.random.Philox(seq))

    def child(self, *ids: int) -> "NoiseStreams":
        return NoiseStreams(self.seed, tuple(self.prefix) + ids)


def transform_standard_normal(params: MatrixNormalParams, z: np.ndarray) -> np.ndarray:
    """mean + row_chol z col_chol^T, batched over leading axes."""
    return params.mean + params.row_chol @ z @ params.col_chol.T
