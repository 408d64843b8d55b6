"""The phase entry points (plq_sweep_segments ... plq_finalize) driven by the
horizon-sharding orchestration on a real GPU: a world-size-1 NCCL group must
reproduce the one-call solve bitwise."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cfg_id,T,J", [(2, 512, 16), (1, 64, 8), (4, 64, 4)])
def test_phases_equal_one_call_solve(cfg_id, T, J):
    import torch
    import torch.distributed as dist

    from paper_1809_06360_b200 import solve_parallel_batch, synth
    from paper_1809_06360_b200.sharded import sharded_solve_device
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=5, count=2)
    ref = solve_parallel_batch(batch, J=J)
    dev = torch.device("cuda", 0)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    try:
        solver, res = sharded_solve_device(inputs, J=J, dist=dist)
        torch.cuda.synchronize()
        for k in ("K", "k", "x", "u", "lam", "links", "objective", "kkt_inf", "link_mismatch", "link_residual"):
            a = solver.out[k].cpu().numpy()
            b = ref.out[k].cpu().numpy()
            assert np.array_equal(a, b), k
    finally:
        dist.destroy_process_group()


class HostStagedDist:
    """torch.distributed over gloo for CUDA tensors: every collective is
    staged through host memory.  Lets two processes sharing ONE GPU run the
    horizon-sharded phases as two ranks -- the exchange happens on the host
    between kernel launches, so no kernel of one rank ever waits on another
    rank (the NCCL path on N GPUs uses the same orchestration)."""

    def __init__(self, dist):
        self.d = dist

    def get_world_size(self, group=None):
        return self.d.get_world_size(group)

    def get_rank(self, group=None):
        return self.d.get_rank(group)

    def all_gather_into_tensor(self, out, inp, group=None):
        import torch
        host = torch.empty(out.shape, dtype=out.dtype)
        self.d.all_gather_into_tensor(host, inp.cpu(), group=group)
        out.copy_(host)


def _rank_worker(rank, world, port, cfg_id, T, J, outdir):
    import os

    import torch
    import torch.distributed as dist

    from paper_1809_06360_b200 import BatchSolver, synth
    from paper_1809_06360_b200.sharded import DeviceBackend, shard_range, solve_sharded, stage_window
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
        batch = synth.generate_batch(cfg, seed=5, count=1)
        solver = BatchSolver(1, T, cfg.n, cfg.m, J=J, device=dev, degenerate=False)
        j0, j1 = shard_range(J, world, rank)
        win, t0 = stage_window(batch, solver.partition.split_times, j0, j1)
        inputs = {k: torch.from_numpy(v.copy()).to(dev) for k, v in win.items()}
        be = DeviceBackend(solver, inputs, t0=t0)
        res = solve_sharded(be, HostStagedDist(dist))
        torch.cuda.synchronize()
        lo, hi = solver.partition.split_times[j0], solver.partition.split_times[j1]
        o = solver.out
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), lo=lo, hi=hi, t0=t0,
                 K=o["K"][0, lo:hi].cpu().numpy(), k=o["k"][0, lo:hi].cpu().numpy(),
                 x=o["x"][0, lo:hi].cpu().numpy(), u=o["u"][0, lo:hi].cpu().numpy(),
                 lam=o["lam"][0, lo:hi].cpu().numpy(),
                 **{k: v.cpu().numpy() for k, v in res.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_id,T,J", [(2, 2, 512, 16), (2, 3, 64, 8), (3, 0, 96, 6)])
def test_two_ranks_windowed_inputs_equal_one_call_solve(world, cfg_id, T, J):
    """The CUDA phases across `world` ranks (processes on one GPU, host-staged
    gloo exchange), each rank holding only its segments' stages: every
    rank's slice of K, k, x, u, lambda and the replicated links / scalars
    equal the single-call solve bit for bit."""
    import os
    import tempfile

    import torch.multiprocessing as mp

    from paper_1809_06360_b200 import solve_parallel_batch, synth
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=5, count=1)
    ref = {k: v.cpu().numpy() for k, v in solve_parallel_batch(batch, J=J).out.items() if v is not None}
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_worker, args=(world, _free_port(), cfg_id, T, J, d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    for o in outs:
        lo, hi = int(o["lo"]), int(o["hi"])
        for k in ("K", "k", "x", "u", "lam"):
            assert np.array_equal(o[k], ref[k][0, lo:hi]), k
        for k in ("objective", "kkt_inf", "link_mismatch", "link_residual"):
            assert np.array_equal(o[k], ref[k]), k
        assert np.array_equal(o["links"], ref["links"])
