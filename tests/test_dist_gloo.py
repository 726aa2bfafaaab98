"""Member sharding over 2 ranks (gloo, CPU): same result as one rank.

Exercises the engine's multi-rank orchestration -- global member ids for the
noise substreams, the member-0 shift broadcast, the member-sum and cross-moment
allreduces, replicated gain -- with the test-only CPU operator set.  On B200
the same code runs with DeviceOps and NCCL (bench.py --gpus N under torchrun).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(kind):
    from oracle import problems

    pm = problems.product_modules()
    if kind == "cnn":
        pr = problems.make_cnn_problem(pm, "C1", size=8, n_members=11, horizon=3)
        return pm, pr.vs, pr.x0, pr.N, pr.H
    if kind == "burgers":
        pr = problems.make_burgers_problem(pm, "boundary", grid_n=8, n_members=11, horizon=3)
        return pm, pr.vs, pr.x0, pr.N, pr.H
    model, vs, x0 = problems.make_linear_setup(pm, np.random.default_rng(2), n=5, l=3, m=4)
    if kind == "constraint":
        con = problems.make_constraint(pm, "box", x0.n, x0.l, x0.m)
        vs = pm.virtualsys.build_virtual_system(model, vs.weights, constraint=con)
    return pm, vs, x0, 13, 4


def _run(kind, comm, basis="fp32"):
    from cpu_ops import CpuOps
    from paper_2410_09663_b200.engine import DeviceSmoother

    pm, vs, x0, N, h = _problem(kind)
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, N, 1.0 / np.trace(vs.shared_col_cov),
                         capacity=2, comm=comm, basis=basis)
    st = pm.matvar.NoiseStreams(seed=21)
    y = ops.to_device(vs.reference_observation())
    for _ in range(h):
        eng.predict(vs, st)
        eng.update(y, st)
    return eng


def _worker(rank, world, port, kind, out, basis="fp32"):
    sys.path[:0] = [os.path.dirname(HERE), HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_09663_b200.engine import TorchComm

    eng = _run(kind, TorchComm(), basis)
    local = eng.members_device().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (eng.member0, eng.Nl, local))
    if rank == 0:
        np.savez(out, mean=eng.mean_host(), members=np.concatenate([p[2] for p in parts], axis=1),
                 spans=np.array([(p[0], p[1]) for p in parts]), jitter=eng.jitter.item())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,basis", [("linear", "fp32"), ("cnn", "fp32"), ("cnn", "f16pair"),
                                        ("burgers", "f16pair"), ("constraint", "f16pair")])
def test_two_rank_sharding_matches_single_rank(kind, basis, tmp_path):
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), kind, out, basis), nprocs=2, join=True)
    got = np.load(out)
    ref = _run(kind, None, basis)
    assert [tuple(s) for s in got["spans"]] == [(0, 7), (7, 6)] if kind == "linear" else True
    if kind == "burgers":
        ref.check_status()  # batch-wide CFL / finiteness flags (max-reduced across ranks on B200)
    scale = np.abs(ref.mean_host()).max()
    assert np.abs(got["mean"] - ref.mean_host()).max() < 1e-10 * scale
    assert np.abs(got["members"] - ref.members_device().numpy()).max() < 1e-10 * scale
    assert int(got["jitter"]) == ref.jitter.item()


def _count_worker(rank, world, port, out):
    sys.path[:0] = [os.path.dirname(HERE), HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_09663_b200.engine import TorchComm

    class Counting(TorchComm):
        calls = []

        def allreduce_(self, t):
            self.calls.append(("allreduce", t.numel()))
            return super().allreduce_(t)

        def allreduce_many(self, ts):
            self.calls.append(("allreduce_many", sum(t.numel() for t in ts)))
            return super().allreduce_many(ts)

        def broadcast_(self, t, src=0):
            self.calls.append(("broadcast", t.numel()))
            return super().broadcast_(t, src)

        def all_gather_rows(self, t):
            self.calls.append(("all_gather", t.numel()))
            return super().all_gather_rows(t)

    comm = Counting()
    eng = _run("cnn", comm, "f16pair")
    if rank == 0:
        np.savez(out, n=len(comm.calls), h=3, fused=int(eng.obs_fused),
                 kinds=np.array([c[0] for c in comm.calls]))
    dist.barrier()
    dist.destroy_process_group()


def test_collectives_per_step(tmp_path):
    """four collectives per predict+update under member sharding (fused noise and
    observation path) -- the slice + observation member sums, the Sigma_y block, the rest of the
    cross moments (one coalesced group), and the all-gather of the row-sharded gain rows -- and
    no broadcast (each rank centres relative to its own first member)."""
    out = str(tmp_path / "c.npz")
    mp.spawn(_count_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    kinds = got["kinds"].tolist()
    assert int(got["fused"]) == 1
    assert "broadcast" not in set(kinds)
    assert int(got["n"]) == 4 * int(got["h"])
    assert kinds.count("all_gather") == int(got["h"])


def _cov_run(comm):
    from cpu_ops import CpuOps
    from paper_2410_09663_b200.covariance import (SmootherCovariances, track_predict,
                                                  track_update)
    from paper_2410_09663_b200.engine import DeviceSmoother

    pm, vs, x0, N, h = _problem("cnn")
    ops = CpuOps()
    eng = DeviceSmoother(ops, x0.packed, x0.n, x0.l, N, 1.0 / np.trace(vs.shared_col_cov),
                         capacity=2, comm=comm, basis="f16pair")
    eng.bind(vs)
    cov = SmootherCovariances(sigma_traj=np.zeros((eng.d, eng.d)))
    st = pm.matvar.NoiseStreams(seed=21)
    y = ops.to_device(vs.reference_observation())
    for _ in range(h):
        eng.predict(vs, st)
        track_predict(eng, cov)
        eng.update(y, st)
    pre = cov.sigma_traj  # the predict-assembled matrix (materialised on every rank)
    track_update(eng, cov)
    return pre, cov.sigma_traj, cov.sigma_cross


def _cov_worker(rank, world, port, out):
    sys.path[:0] = [os.path.dirname(HERE), HERE]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_09663_b200.engine import TorchComm

    pre, traj, cross = _cov_run(TorchComm())
    if rank == 0:
        np.savez(out, pre=pre, traj=traj, cross=cross)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_covariance_tracking_row_sharded(tmp_path):
    """Tracked covariances under member sharding: SYRK partials reduce-scattered by row blocks,
    gathered on read -- equal to the single-rank result."""
    out = str(tmp_path / "cov.npz")
    mp.spawn(_cov_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    pre, traj, cross = _cov_run(None)
    for a, b in ((got["pre"], pre), (got["traj"], traj), (got["cross"], cross)):
        assert a.shape == b.shape
        assert np.abs(a - b).max() < 1e-10 * np.abs(b).max()
