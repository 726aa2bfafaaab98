"""ORACLE (test infrastructure only) — noise substreams of the reference.

Restates reference pkg/src/enksmpc/matvar.py:136-154 (NoiseStreams) and the
per-member draw loop of enks.py:131-145 (_member_noise).  Two interchangeable
back ends:

* ``numpy`` — the third-party implementation the reference itself calls
  (numpy.random SeedSequence/Philox/Generator.standard_normal).
* ``c``     — oracle/npy_noise.c, a plain-C restatement of the same bitstream,
  pinned bit-for-bit against numpy by tests/test_oracle_noise.py.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

MASK32 = 0xFFFFFFFF
POOL_SIZE = 4  # numpy SeedSequence DEFAULT_POOL_SIZE


def int_to_words(v: int) -> list[int]:
    """numpy bit_generator._int_to_uint32_array: little-endian uint32 words; 0 -> [0]."""
    v = int(v)
    if v < 0:
        raise ValueError("expected non-negative integer")
    if v == 0:
        return [0]
    out = []
    while v > 0:
        out.append(v & MASK32)
        v >>= 32
    return out


def assemble_entropy(seed: int, spawn_key: Sequence[int]) -> list[int]:
    """SeedSequence.get_assembled_entropy: seed words (zero-padded to the pool
    size when a spawn key is present) followed by each spawn id's words."""
    run = int_to_words(seed)
    spawn: list[int] = []
    for k in spawn_key:
        spawn.extend(int_to_words(k))
    if spawn and len(run) < POOL_SIZE:
        run = run + [0] * (POOL_SIZE - len(run))
    return run + spawn


def head_words(seed: int, prefix: Sequence[int]) -> list[int]:
    """Entropy words common to every (member, t, channel) substream: the seed
    words zero-padded to the pool size (a spawn key is always present) and the
    prefix ids.  The per-stream ids (i, t, ch) follow, one word each (< 2**32)."""
    return assemble_entropy(seed, tuple(prefix) + (0,))[:-1]


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "lib", "libnpy_noise.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.npyo_seedseq_key.argtypes = [u32p, ctypes.c_int, u64p]
        lib.npyo_standard_normal.argtypes = [u64p, ctypes.c_int64, dp]
        lib.npyo_standard_normal_words.argtypes = [u64p, ctypes.c_int64, dp]
        lib.npyo_standard_normal_words.restype = ctypes.c_int64
        lib.npyo_member_noise.argtypes = [u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_int64, ctypes.c_int64, dp]
        lib.npyo_member_noise_range.argtypes = [u32p, ctypes.c_int, ctypes.c_uint32,
                                                ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_int64, dp]
        lib.npyo_philox_block.argtypes = [u64p, u64p, u64p]
        _LIB = lib
    return _LIB


def c_key(seed: int, spawn_key: Sequence[int]) -> np.ndarray:
    ent = np.asarray(assemble_entropy(seed, spawn_key), dtype=np.uint32)
    key = np.zeros(2, dtype=np.uint64)
    _lib().npyo_seedseq_key(ent.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), len(ent),
                            key.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return key


def c_standard_normal(seed: int, spawn_key: Sequence[int], count: int, return_words=False):
    key = c_key(seed, spawn_key)
    out = np.empty(count, dtype=np.float64)
    lib = _lib()
    fn = lib.npyo_standard_normal_words if return_words else lib.npyo_standard_normal
    words = fn(key.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), count,
               out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return (out, words) if return_words else out


def substream(seed: int, prefix: Sequence[int], *ids: int) -> np.random.Generator:
    """matvar.py:149-151 NoiseStreams.substream via numpy (the reference's own dependency)."""
    seq = np.random.SeedSequence(entropy=seed, spawn_key=tuple(prefix) + tuple(ids))
    return np.random.Generator(np.random.Philox(seq))


def member_normals(seed: int, prefix: Sequence[int], t: int, channel: int, n_members: int,
                   shape: tuple[int, int], backend: str = "numpy") -> np.ndarray:
    """Raw standard normals z[i] for members 0..N-1, enks.py:142-144. Returns (N, rows, cols)."""
    rows, cols = shape
    if backend == "numpy":
        z = np.empty((n_members, rows, cols))
        for i in range(n_members):
            z[i] = substream(seed, prefix, i, t, channel).standard_normal((rows, cols))
        return z
    if backend != "c":
        raise ValueError(backend)
    head = np.asarray(head_words(seed, prefix), dtype=np.uint32)
    out = np.empty((n_members, rows * cols), dtype=np.float64)
    hp = head.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    lib = _lib()

    def run(i0, i1):  # ctypes releases the GIL: member ranges draw in parallel
        lib.npyo_member_noise_range(hp, len(head), t, channel, i0, i1 - i0, rows * cols,
                                    out[i0:].ctypes.data_as(ctypes.POINTER(ctypes.c_double)))

    workers = min(os.cpu_count() or 1, 32) if n_members * rows * cols >= (1 << 22) else 1
    if workers == 1:
        run(0, n_members)
    else:
        from concurrent.futures import ThreadPoolExecutor

        cuts = np.linspace(0, n_members, workers + 1).astype(int)
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(lambda k: run(cuts[k], cuts[k + 1]), range(workers)))
    return out.reshape(n_members, rows, cols)
