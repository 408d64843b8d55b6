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


@pytest.mark.parametrize("cfg_id,T,J,count", [(2, 512, 16, 1), (1, 64, 8, 3), (4, 64, 4, 2), (0, 96, 6, 1)])
def test_native_sharded_entry_equals_one_call_solve(cfg_id, T, J, count):
    """plq_solve_parallel_sharded over a real (one-rank) NCCL communicator:
    the in-place all-gather (B = 1, equal shards) and grouped-broadcast
    (B > 1) exchanges run, and every output equals the one-call solve bit
    for bit.  NULL communicator with nranks = 1 takes the same phases."""
    import torch

    from paper_1809_06360_b200 import BatchSolver, solve_parallel_batch, synth
    from paper_1809_06360_b200.sharded import NcclComm, solve_sharded_native
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=5, count=count)
    ref = solve_parallel_batch(batch, J=J)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    comm = NcclComm()
    try:
        for c in (comm, None):
            solver = BatchSolver(count, T, cfg.n, cfg.m, J=J, device=dev)
            solve_sharded_native(solver, inputs, c)
            torch.cuda.synchronize()
            assert solver.launches == ref.launches
            for k in ("K", "k", "x", "u", "lam", "links", "objective", "kkt_inf", "link_mismatch",
                      "link_residual", "status"):
                assert np.array_equal(solver.out[k].cpu().numpy(), ref.out[k].cpu().numpy()), k
    finally:
        comm.close()


def test_native_sharded_entry_degenerate_partition():
    """A partition with segments too short to reach arbitrary endpoints
    (feasibility rows, parallel.py:320-384) through the sharded entry: the rows
    travel with the value blocks and the constrained link solve is replicated."""
    import torch

    from paper_1809_06360_b200 import BatchSolver, Partition, solve_parallel_batch, synth
    from paper_1809_06360_b200.sharded import NcclComm, solve_sharded_native
    cfg = synth.CONFIGS[0].scaled(T=24, J=4)
    batch = synth.generate_batch(cfg, seed=2, count=2)
    part = Partition(4, (0, 2, 12, 14, 24))          # L = 2 stages of m = 4 controls < n = 12
    ref = solve_parallel_batch(batch, partition=part)
    assert int(ref.out["feas_rows"].sum()) > 0
    dev = torch.device("cuda", 0)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    comm = NcclComm()
    try:
        solver = BatchSolver(2, 24, cfg.n, cfg.m, partition=part, device=dev)
        solve_sharded_native(solver, inputs, comm)
        torch.cuda.synchronize()
        for k in ("K", "k", "x", "u", "lam", "links", "objective", "kkt_inf", "feas_rows", "feas_residual"):
            assert np.array_equal(solver.out[k].cpu().numpy(), ref.out[k].cpu().numpy()), k
    finally:
        comm.close()


# ---------------------------------------------------------------------------
# plq_solve_parallel_sharded across several ranks on ONE GPU: the library's
# NCCL binding is pointed (PLQ_NCCL_LIB) at tests/nccl_host_shim.c, which
# stages every collective through host shared memory between kernel launches.

SHIM_CAP = 64 << 20


def _build_shim(workdir):
    import os
    import subprocess
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "nccl_host_shim.c")
    so = os.path.join(workdir, "libnccl_host_shim.so")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-shared", "-fPIC", "-O1", f"-I{cuda}/include", src, "-o", so, f"-L{cuda}/lib64",
                    f"-Wl,-rpath,{cuda}/lib64", "-lcudart", "-lpthread", "-lrt"], check=True)
    return so


class _ShimComm:
    def __init__(self, so, name, rank, world):
        import ctypes
        self.lib = ctypes.CDLL(so)
        self.lib.shim_attach.restype = ctypes.c_void_p
        self.lib.shim_attach.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_size_t]
        self.lib.shim_calls.restype = ctypes.c_ulonglong
        self.lib.shim_calls.argtypes = [ctypes.c_void_p]
        self.comm = ctypes.c_void_p(self.lib.shim_attach(name.encode(), rank, world, SHIM_CAP))
        assert self.comm.value, "shim attach failed"
        self.rank, self.world = rank, world

    def calls(self):
        return int(self.lib.shim_calls(self.comm))


def _native_rank_worker(rank, world, so, name, case, outdir):
    import os
    os.environ["PLQ_NCCL_LIB"] = so          # read once, at the library's first sharded call
    import torch

    from paper_1809_06360_b200 import BatchSolver, Partition, synth
    from paper_1809_06360_b200.sharded import shard_range, solve_sharded_native, stage_window
    cfg_id, T, J, count, splits, windowed = case
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=5, count=count)
    part = None if splits is None else Partition(J, tuple(splits))
    solver = BatchSolver(count, T, cfg.n, cfg.m, J=J, partition=part, device=dev)
    j0, j1 = shard_range(J, world, rank)
    t0 = 0
    if windowed:
        batch, t0 = stage_window(batch, solver.partition.split_times, j0, j1)
    inputs = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in batch.items()}
    comm = _ShimComm(so, name, rank, world)
    res = solve_sharded_native(solver, inputs, comm, t0=t0)
    torch.cuda.synchronize()
    st = solver.partition.split_times
    lo, hi = int(st[j0]), int(st[j1])
    o = solver.out
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), lo=lo, hi=hi, calls=comm.calls(),
             status=o["status"].cpu().numpy(), feas_rows=o["feas_rows"].cpu().numpy(),
             **{k: o[k][:, lo:hi].cpu().numpy() for k in ("K", "k", "x", "u", "lam")},
             **{k: v.cpu().numpy() for k, v in res.items()})


@pytest.mark.parametrize("world,case", [
    (2, (2, 512, 16, 1, None, True)),                      # equal shards, B = 1: in-place all-gathers, stage windows
    (4, (0, 96, 6, 1, None, True)),                        # unequal shards (2,2,1,1): grouped broadcasts
    (2, (1, 64, 8, 3, None, False)),                       # B > 1: one broadcast per owner and problem
    (3, (3, 64, 8, 1, None, True)),                        # n = 128 generic kernels, shards (3,3,2)
    (2, (0, 24, 4, 2, (0, 2, 12, 14, 24), False)),         # degenerate partition: feasibility rows exchanged
])
def test_native_sharded_entry_multi_rank(world, case):
    """Every rank's slice of K, k, x, u, lambda and the replicated links /
    scalars / status equal the one-call solve bit for bit, for any rank count."""
    import ctypes
    import os
    import tempfile

    import torch.multiprocessing as mp

    from paper_1809_06360_b200 import Partition, solve_parallel_batch, synth
    cfg_id, T, J, count, splits, _ = case
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=5, count=count)
    part = None if splits is None else Partition(J, tuple(splits))
    ref = {k: v.cpu().numpy() for k, v in solve_parallel_batch(batch, J=J, partition=part).out.items()
           if v is not None}
    if splits is not None:
        assert int(ref["feas_rows"].sum()) > 0
    name = f"/plq_shim_{os.getpid()}_{world}_{cfg_id}"
    with tempfile.TemporaryDirectory() as d:
        so = _build_shim(d)
        parent = ctypes.CDLL(so)
        parent.shim_create.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_size_t]
        assert parent.shim_create(name.encode(), world, SHIM_CAP) == 0
        try:
            ctx = mp.get_context("spawn")
            procs = [ctx.Process(target=_native_rank_worker, args=(r, world, so, name, case, d)) for r in range(world)]
            for p in procs:
                p.start()
            for p in procs:
                p.join(240)
            hung = [p for p in procs if p.is_alive()]
            for p in hung:                       # a rank that died leaves its peers in the barrier
                p.kill()
            assert not hung and all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
            outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        finally:
            parent.shim_destroy(name.encode())
    for o in outs:
        lo, hi = int(o["lo"]), int(o["hi"])
        assert int(o["calls"]) > 0
        for k in ("K", "k", "x", "u", "lam"):
            assert np.array_equal(o[k], ref[k][:, lo:hi]), k
        for k in ("objective", "kkt_inf", "link_mismatch", "link_residual", "links", "status", "feas_rows"):
            assert np.array_equal(o[k], ref[k]), k
