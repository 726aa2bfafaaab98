"""Vector-EnKS comparator (reference baselines.py:95-197).

Golden fixtures are the UNMODIFIED reference vector_enks_smooth (tests/golden/
make_golden.py).  CPU: the product's orchestration on the fp64 CPU operator set
equals them to rounding; GPU: the device run within the fp32 tolerance; the
memory-budget projection rejects C3-sized vector problems that the matrix smoother
holds in a fraction of one B200.
"""
import os

import numpy as np
import pytest

from cpu_ops import CpuOps
from oracle import problems

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _case(pm, name):
    from golden.make_golden import VECTOR_CASES

    _, kw, seed, N, h, sseed = next(c for c in VECTOR_CASES if c[0] == name)
    _, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(seed), **kw)
    return vs, x0, N, h, sseed, np.load(os.path.join(GOLD, name + ".npz"))


@pytest.mark.parametrize("name", ["vec_m1", "vec_m2", "vec_m4"])
def test_vector_smoother_cpu_ops_equals_reference(pm, name):
    from paper_2410_09663_b200.baselines import vector_enks_smooth

    vs, x0, N, h, sseed, gold = _case(pm, name)
    assert np.array_equal(x0.packed, gold["x0"])
    mean, rep = vector_enks_smooth(x0, vs.reference_observation(), vs, h, N,
                                   pm.matvar.NoiseStreams(seed=sseed), ops=CpuOps())
    np.testing.assert_allclose(mean, gold["mean"], rtol=1e-9, atol=1e-9)
    assert rep.obs_cov_entries == int(gold["obs_cov_entries"])
    assert rep.cross_cov_entries == int(gold["cross_cov_entries"])
    assert rep.jitter_events == int(gold["jitter_events"])


def test_entry_counts_and_budget_error(pm):
    from paper_2410_09663_b200.baselines import (MemoryBudgetError, covariance_entry_counts,
                                                 vector_enks_smooth)

    assert covariance_entry_counts(256, 128) == {"vector": (256 * 128) ** 2, "matrix": 256 ** 2}
    vs, x0, N, h, sseed, _ = _case(pm, "vec_m2")
    with pytest.raises(MemoryBudgetError, match="budget"):
        vector_enks_smooth(x0, vs.reference_observation(), vs, h, N,
                           pm.matvar.NoiseStreams(seed=sseed), memory_budget_bytes=10_000,
                           ops=CpuOps())
    with pytest.raises(ValueError):
        vector_enks_smooth(x0, vs.reference_observation(), vs, h, 1,
                           pm.matvar.NoiseStreams(seed=sseed), ops=CpuOps())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["vec_m1", "vec_m2", "vec_m4"])
def test_vector_smoother_gpu_matches_reference(pm, name):
    from paper_2410_09663_b200.baselines import vector_enks_smooth

    vs, x0, N, h, sseed, gold = _case(pm, name)
    mean, rep = vector_enks_smooth(x0, vs.reference_observation(), vs, h, N,
                                   pm.matvar.NoiseStreams(seed=sseed))
    assert np.abs(mean - gold["mean"]).max() < 1e-4 * np.abs(gold["mean"]).max()
    assert rep.jitter_events == int(gold["jitter_events"])


@pytest.mark.gpu
def test_memory_outage_contrast_c3(pm):
    """Table 1's point on B200: at C3 (128 x 128, N = 1024, H = 50) the vector smoother's
    projected covariance storage exceeds the device memory, the matrix smoother's whole
    state needs a small fraction of it."""
    import torch

    from paper_2410_09663_b200 import enks
    from paper_2410_09663_b200.baselines import MemoryBudgetError, vector_enks_smooth

    pr = problems.make_cnn_problem(pm, "C3")
    with pytest.raises(MemoryBudgetError):
        vector_enks_smooth(pr.x0, pr.y_ref, pr.vs, pr.H, pr.N, pm.matvar.NoiseStreams(seed=0))
    free, total = torch.cuda.mem_get_info()
    eng = enks.init_ensemble(pr.x0, pr.N, capacity=pr.H).engine
    assert eng.memory_bytes() < 0.25 * total
