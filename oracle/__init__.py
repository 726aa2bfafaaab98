"""ORACLE — CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import anything from this package, and only as
the checker (or the timed CPU baseline).  The product package
``paper_2410_09663_b200`` never imports it; its GPU path fails loudly when the
CUDA library is missing instead of falling back here.

Contents (each function cites the reference file:line it restates):
  noise.py        numpy-RNG bitstream restated in C (npy_noise.c) + entropy assembly
  enks_oracle.py  fp64 NumPy restatement of pkg/src/enksmpc/enks.py (init/predict/update/smooth_horizon)
  models.py       fp64 dynamics used with the oracle: linear (dynamics.py:53-85),
                  the CNN surrogate (not in the reference) and Burgers FD (dynamics.py:156-270)
  problems.py     synthetic problem builders for configs C1..C5

Parity pinning: the restatement is checked against the reference itself
(imported read-only from /root/reference in this container) by
tests/golden/make_golden.py, which commits the golden vectors under
tests/golden/; tests/test_oracle_*.py re-check the oracle against those
fixtures on any box.
"""
