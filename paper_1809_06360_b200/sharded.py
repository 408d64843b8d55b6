"""Horizon sharding of one (batch of) partitioned solve(s) across ranks.

One process per GPU (``torch.distributed``, NCCL over NVLink for the GPU
backend).  Rank r owns a contiguous range of segments; the phases of the C ABI
(``include/parlqr_b200.h``) run on it with three exchanges:

1. sweeps of the local segments (``plq_sweep_segments``), then ONE all-gather
   of the segment-start value blocks ``vf0`` (the only data the coupling needs
   -- the reference ships the same blocks back from its worker pool,
   ``parallel.py:230-240``) and of the per-segment status;
2. the link solve, replicated: every rank factors the same system from the
   same bytes, so the links are bitwise identical on all ranks;
3. local reconstruction, an all-gather of the ``mu_left / lambda_right`` rows
   (the link-stage KKT rows need the right neighbour's multiplier), the
   link-stage rows, and an all-gather of the per-segment partials followed by
   a fixed-order reduction -- objective / KKT / mismatch are identical for any
   rank count.

The orchestration is backend-agnostic: :class:`DeviceBackend` drives the CUDA
library; the tests drive the same code with a CPU (oracle) backend over gloo.
"""

from __future__ import annotations

import ctypes

from . import _native
from .parallel import BatchSolver, raise_for_status


def shard_range(J, world, rank):
    """Balanced contiguous segment range of ``rank`` (remainder to early ranks)."""
    base, extra = divmod(J, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def batch_shard(B, world, rank):
    """Problems ``[first, first + count)`` of a batch of ``B`` owned by ``rank``:
    independent problems shard with no data-path collective (cfg1, cfg4;
    SURVEY.md 8e).  Equal shares; ``B`` must divide over the ranks."""
    if B % world:
        raise ValueError(f"batch {B} does not shard over {world} ranks")
    count = B // world
    return rank * count, count


def _gather_rows(dist, group, local, J, world, torch):
    """All-gather per-segment rows.

    ``local``: tensor (B, S_r, X) holding this rank's segments' rows.  Returns
    a (B, J, X) tensor with every rank's rows in segment order.  Ranks own
    unequal counts, so rows are padded to the largest shard for the
    equal-size collective.
    """
    B, _, X = local.shape
    smax = -(-J // world)
    send = torch.zeros((B, smax, X), dtype=local.dtype, device=local.device)
    send[:, :local.shape[1]] = local
    flat = torch.empty((world * B, smax, X), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(flat, send.contiguous(), group=group)   # concatenation form (NCCL and gloo)
    recv = flat.view(world, B, smax, X)
    out = torch.empty((B, J, X), dtype=local.dtype, device=local.device)
    for r in range(world):
        lo, hi = shard_range(J, world, r)
        out[:, lo:hi] = recv[r, :, :hi - lo]
    return out


def solve_sharded(backend, dist, group=None, check=True):
    """Run one sharded solve; every rank returns the same scalar results.

    The per-segment status rows are exchanged with the value blocks and kept
    on the device: with ``check=False`` the solve makes no host
    synchronization (stream-ordered launches and collectives only) and the
    caller raises the reference's exceptions afterwards with
    :func:`raise_sharded_status`.  ``check=True`` does that at the end.
    """
    torch = backend.torch
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    J = backend.J
    j0, j1 = shard_range(J, world, rank)
    backend.launches = 0
    # 1. local sweeps, exchange of segment-start value blocks and status
    if j1 > j0:
        backend.sweep(j0, j1)
    vf0 = _gather_rows(dist, group, backend.vf0_rows(j0, j1), J, world, torch)
    backend.seg_status = _gather_rows(dist, group, backend.status_rows(j0, j1), J, world, torch)
    backend.set_vf0(vf0)
    # 2. replicated coupling solve
    backend.link()
    # 3. local reconstruction, multiplier rows, link-stage KKT rows, partials
    if j1 > j0:
        backend.recon(j0, j1)
    ml = _gather_rows(dist, group, backend.multiplier_rows(j0, j1), J, world, torch)
    backend.set_multiplier_rows(ml)
    if j1 > j0:
        backend.boundary(j0, j1)
    parts = _gather_rows(dist, group, backend.partial_rows(j0, j1), J, world, torch)
    backend.set_partials(parts)
    backend.finalize()
    if check:
        raise_sharded_status(backend)
    return backend.results()


def raise_sharded_status(backend):
    """The reference's exceptions for a finished sharded solve, in the
    reference's order: segment sweeps first (gathered rows), then the link
    solve (this rank's replicated flags)."""
    raise_for_status(backend.seg_status[:, :, 0].cpu().numpy())
    raise_for_status(backend.status_all())


class DeviceBackend:
    """GPU backend: a :class:`BatchSolver`'s buffers driven phase by phase."""

    def __init__(self, solver: BatchSolver, inputs, t0=0):
        """``inputs``: the full stacked device arrays, or (``t0`` > 0, B = 1)
        only this rank's window of stages starting at stage ``t0``
        (:func:`stage_window`) -- each rank then uploads and holds only its
        segments' stage data."""
        self.solver = solver
        self.torch = solver.torch
        self.lib = solver.lib
        self.J = solver.J
        self.n = solver.n
        solver.check_inputs(inputs, T_held=inputs["qx1"].shape[1])
        self.prob = solver._problem_struct(inputs, t0=t0)
        self.inputs = inputs          # keep the (windowed) buffers alive
        self.t0 = t0
        self.seg_status = None
        self.launches = 0
        torch = self.torch
        self.partials = torch.zeros((solver.B, solver.J, 3), dtype=torch.float64, device=solver.device)
        self.stream = torch.cuda.current_stream(solver.device)

    def _call(self, name, *args):
        fn = getattr(self.lib, name)
        s = self.solver
        head = (ctypes.byref(self.prob), ctypes.byref(s._outs))
        rc = fn(*head, *args)
        _native.check(rc, name)
        self.launches += int(self.lib.plq_last_launch_count())

    def _ws(self):
        s = self.solver
        return ctypes.c_void_p(s.workspace.data_ptr()), s.ws_bytes, ctypes.c_void_p(self.stream.cuda_stream)

    def sweep(self, j0, j1):
        self._call("plq_sweep_segments", j0, j1, *self._ws())

    def vf0_rows(self, j0, j1):
        return self.solver.out["vf0"][:, j0:j1]

    def status_rows(self, j0, j1):
        return self.solver.out["status"][:, j0:j1, None].to(self.torch.float64)

    def set_vf0(self, vf0):
        self.solver.out["vf0"].copy_(vf0)
        # status rows gathered separately; keep the local copy in sync for link flags
        self.solver.out["status"].zero_()

    def status_all(self):
        return self.solver.out["status"].cpu().numpy()

    def link(self):
        self._call("plq_link_solve", *self._ws())

    def recon(self, j0, j1):
        ws = self._ws()
        self._call("plq_reconstruct_segments", j0, j1, ctypes.c_void_p(self.partials.data_ptr()), *ws)

    def multiplier_rows(self, j0, j1):
        # row j: [mu_left[j] (j < J-1) | lambda_right[j-1] (j > 0)]
        torch = self.torch
        s = self.solver
        B, n, J = s.B, s.n, s.J
        rows = torch.zeros((B, j1 - j0, 2 * n), dtype=torch.float64, device=s.device)
        a, b = j0, min(j1, J - 1)
        if b > a:
            rows[:, a - j0:b - j0, :n] = s.out["mu_left"][:, a:b]
        a, b = max(j0, 1), j1
        if b > a:
            rows[:, a - j0:b - j0, n:] = s.out["lambda_right"][:, a - 1:b - 1]
        return rows

    def set_multiplier_rows(self, rows):
        s = self.solver
        n, J = s.n, s.J
        if J > 1:
            s.out["mu_left"][:, :J - 1] = rows[:, :J - 1, :n]
            s.out["lambda_right"][:, :J - 1] = rows[:, 1:, n:]

    def boundary(self, j0, j1):
        self._call("plq_boundary_segments", j0, j1, ctypes.c_void_p(self.partials.data_ptr()), *self._ws())

    def partial_rows(self, j0, j1):
        return self.partials[:, j0:j1]

    def set_partials(self, parts):
        self.partials.copy_(parts)

    def finalize(self):
        self._call("plq_finalize", ctypes.c_void_p(self.partials.data_ptr()), *self._ws())

    def results(self):
        o = self.solver.out
        return {k: o[k] for k in ("objective", "kkt_inf", "link_mismatch", "link_residual", "links")}


class NcclComm:
    """An ``ncclComm_t`` of this process's own, for ``plq_solve_parallel_sharded``
    (torch does not expose its communicators).  The 128-byte unique id is made
    on rank 0 and broadcast through the given ``torch.distributed`` group (any
    backend); every rank then calls ``ncclCommInitRank`` on its current CUDA
    device.  The library is the one torch already loaded (``libnccl.so.2``)."""

    def __init__(self, dist=None, group=None, rank=0, world=1):
        import torch
        name = None
        for cand in ("libnccl.so.2", "libnccl.so"):
            try:
                self.nccl = ctypes.CDLL(cand)
                name = cand
                break
            except OSError:
                continue
        if name is None:
            raise RuntimeError("libnccl.so.2 not found (import torch with CUDA support first)")
        if dist is not None:
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.rank, self.world = int(rank), int(world)

        class UniqueId(ctypes.Structure):
            _fields_ = [("internal", ctypes.c_char * 128)]

        uid = UniqueId()
        self.nccl.ncclGetErrorString.restype = ctypes.c_char_p
        if self.rank == 0:
            self._ok(self.nccl.ncclGetUniqueId(ctypes.byref(uid)), "ncclGetUniqueId")
        if self.world > 1:
            box = [bytes(uid.internal) if self.rank == 0 else None]
            src = 0 if group is None else dist.get_global_rank(group, 0)
            dist.broadcast_object_list(box, src=src, group=group)
            ctypes.memmove(ctypes.byref(uid), box[0], 128)
        self.comm = ctypes.c_void_p()
        self.nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
        torch.cuda.current_stream().synchronize()
        self._ok(self.nccl.ncclCommInitRank(ctypes.byref(self.comm), self.world, uid, self.rank), "ncclCommInitRank")

    def _ok(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: NCCL error {rc} ({self.nccl.ncclGetErrorString(rc).decode()})")

    def close(self):
        if getattr(self, "comm", None):
            self.nccl.ncclCommDestroy.argtypes = [ctypes.c_void_p]
            self.nccl.ncclCommDestroy(self.comm)
            self.comm = None


def solve_sharded_native(solver: BatchSolver, inputs, comm: NcclComm = None, t0=0, stream=None, check=True):
    """One horizon-sharded solve through ``plq_solve_parallel_sharded``: the
    library runs the phases and issues the NCCL exchanges itself on one stream
    (no host synchronization, no temporaries).  ``inputs``: full stacked device
    arrays, or this rank's stage window (``t0`` = its first stage, B = 1).
    Degenerate partitions are supported (the feasibility rows travel with the
    value blocks).  Returns the replicated scalar results; ``solver.out`` holds
    this rank's segments of ``K, k, x, u, lam``."""
    torch = solver.torch
    solver.check_inputs(inputs, T_held=inputs["qx1"].shape[1])
    prob = solver._problem_struct(inputs, t0=t0)
    stream = torch.cuda.current_stream(solver.device) if stream is None else stream
    rank, world = (comm.rank, comm.world) if comm is not None else (0, 1)
    rc = solver.lib.plq_solve_parallel_sharded(
        ctypes.byref(prob), ctypes.byref(solver._outs), ctypes.c_void_p(solver.workspace.data_ptr()),
        solver.ws_bytes, comm.comm if comm is not None else None, rank, world,
        ctypes.c_void_p(stream.cuda_stream))
    _native.check(rc, "plq_solve_parallel_sharded")
    solver.launches = int(solver.lib.plq_last_launch_count())
    if check:
        solver.raise_for_status()
    o = solver.out
    return {k: o[k] for k in ("objective", "kkt_inf", "link_mismatch", "link_residual", "links")}


def stage_window(arrays, splits, j0, j1):
    """Host arrays of one problem (B = 1) cut to the stages of segments
    [j0, j1) -- what a rank of a horizon-sharded solve needs (its sweeps,
    reconstruction and link-stage KKT rows read nothing else; terminal cost
    and x_init are replicated).  Returns (window arrays, first stage)."""
    t0, t1 = int(splits[j0]), int(splits[j1])
    out = {}
    for k, v in arrays.items():
        out[k] = v[:, t0:t1] if v.ndim >= 2 and k not in ("QxxT", "qx1T", "x_init") else v
    return out, t0


def sharded_solve_device(inputs, J=None, partition=None, dist=None, group=None, device=None, tolerances=None):
    """Convenience wrapper: a horizon-sharded solve of device ``inputs`` (each
    rank holds the full stacked inputs; it only reads its segments')."""
    from .problem import DEFAULT_TOLERANCES
    B, T, n = (int(s) for s in inputs["qx1"].shape)
    m = int(inputs["qu1"].shape[2])
    solver = BatchSolver(B, T, n, m, J=J, partition=partition, device=device,
                         tolerances=tolerances or DEFAULT_TOLERANCES, degenerate=False)
    backend = DeviceBackend(solver, inputs)
    res = solve_sharded(backend, dist, group)
    return solver, res


__all__ = ["batch_shard", "shard_range", "solve_sharded", "raise_sharded_status", "DeviceBackend", "stage_window",
           "sharded_solve_device", "NcclComm", "solve_sharded_native"]
