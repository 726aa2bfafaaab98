"""Member sharding on the DEVICE path: 2 ranks with DeviceOps on the one B200, gloo collectives.

The product's multi-rank path (engine.py: members sharded by global id, collectives through
engine.TorchComm) runs with the real sm_100a kernels in both ranks -- the member-0-offset noise
launches (member0 > 0), the sharded statistics and contractions -- and must reproduce the
single-rank result.  NCCL refuses two ranks on one GPU, so the collectives go through gloo on
CUDA tensors (host-staged: the ranks' kernels never wait on one another, this is a correctness
test, not a timing).  On a multi-GPU node bench.py runs the same code with NCCL.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
# fp32 rounding only: the ranks' member sums and K-partial cross moments are summed in another
# order than one rank's (and each rank picks its own fp16-pair row scales); noise is bit-identical
TOL = 5e-6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(kind):
    from oracle import problems

    pm = problems.product_modules()
    if kind == "cnn_tc":  # fused tcgen05 CNN, fp16-pair basis, derived-U chain, odd split
        pr = problems.make_cnn_problem(pm, "C1", size=32, n_members=45, horizon=4,
                                       widths=(2, 32, 32, 1))
        return pm, pr.vs, pr.x0, pr.y_ref, pr.N, pr.H
    if kind == "burgers":
        pr = problems.make_burgers_problem(pm, "pointwise", grid_n=16, n_members=21, horizon=3)
        return pm, pr.vs, pr.x0, pr.y_ref, pr.N, pr.H
    model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(2), n=24, l=8, m=8)
    if kind == "constraint":
        con = problems.make_constraint(pm, "linear", x0.n, x0.l, x0.m)
        vs = pm.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
    return pm, vs, x0, vs.reference_observation(), 33, 4


def _smooth(kind):
    from paper_2410_09663_b200 import enks

    pm, vs, x0, y, N, h = _problem(kind)
    ens = enks.init_ensemble(x0, N, shared_col_cov=vs.shared_col_cov, capacity=h)
    st = pm.matvar.NoiseStreams(seed=5)
    for _ in range(h):
        enks.predict(ens, vs, st)
        enks.update(ens, y, vs, st)
    return ens.slices(), ens.members, ens.jitter_events


def _worker(rank, world, port, kind, out):
    sys.path[:0] = [os.path.dirname(HERE), HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_09663_b200 import enks
    from paper_2410_09663_b200.engine import TorchComm

    enks.set_default_comm(TorchComm())
    mean, members, jit = _smooth(kind)
    if rank == 0:
        np.savez(out, mean=mean, members=members, jitter=jit)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["cnn_tc", "linear", "burgers", "constraint"])
def test_two_device_ranks_equal_one(kind, tmp_path):
    from paper_2410_09663_b200 import enks

    enks.set_default_comm(None)
    ref_mean, ref_members, ref_jit = _smooth(kind)
    out = str(tmp_path / "r0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), kind, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    scale = np.abs(ref_mean).max()
    assert np.abs(got["mean"] - ref_mean).max() < TOL * scale
    assert got["members"].shape == ref_members.shape
    assert np.abs(got["members"] - ref_members).max() < 10 * TOL * np.abs(ref_members).max()
    assert int(got["jitter"]) == ref_jit
