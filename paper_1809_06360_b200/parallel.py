"""Horizon-partitioned Riccati solve on B200: the drop-in for
``parlqr.solve_parallel`` (/root/reference/pkg/src/parlqr/parallel.py:422-553).

Same signature, partition rules, error contract and result types; the
compute runs in ``libparlqr_b200.so`` (hand-written sm_100a CUDA) through its
C ABI.  torch supplies device memory and streams only.  There is no CPU
fallback: without the library or a CUDA device the call raises.

Batched problems (the reference has no batch API) go through
:class:`BatchSolver` / :func:`solve_parallel_batch` with stacked
``(B, T, ...)`` arrays -- the reference's own transport layout
(``_stacked_stages``, parallel.py:108,141-149) with a leading batch axis.
"""

from __future__ import annotations

import collections.abc
import ctypes
import dataclasses
import os

import numpy as np

from . import _native, compat
from .errors import CholeskyFailure, Infeasible, LinkSingular, UnsupportedPartition
from .problem import DEFAULT_TOLERANCES, AffinePolicy, LqrSolution

__all__ = [
    "Partition", "ParallelDetails", "make_partition", "default_workers", "solve_parallel",
    "solve_parallel_batch", "solve_parallel_host", "BatchSolver", "stack_problem",
]

STAGE_FIELDS = ("Qxx", "Qux", "Quu", "qx1", "qu1", "Fx", "Fu", "f1")
TERMINAL_FIELDS = ("QxxT", "qx1T", "x_init")
INPUT_FIELDS = STAGE_FIELDS + TERMINAL_FIELDS
WORKERS_ENV_VAR = "PAR_RICCATI_WORKERS"


@dataclasses.dataclass(frozen=True)
class _Partition:
    """Split of the horizon into ``J`` contiguous segments (parallel.py:67-79)."""

    J: int
    split_times: tuple

    def segment(self, j):
        return self.split_times[j], self.split_times[j + 1]

    @property
    def interior(self):
        return self.split_times[1:-1]


_ref_parallel = compat.reference_module("parallel")
# the reference's own Partition when parlqr is importable (see compat.py)
Partition = _ref_parallel.Partition if _ref_parallel is not None else _Partition


def make_partition(T, J):
    """Balanced partition, remainder to the earliest segments (parallel.py:82-94)."""
    if not 1 <= J <= T:
        raise ValueError(f"J must be in [1, {T}], got {J}")
    base, extra = divmod(T, J)
    splits = [0]
    for j in range(J):
        splits.append(splits[-1] + base + (1 if j < extra else 0))
    return Partition(J, tuple(splits))


def default_workers(J):
    """parallel.py:97-102; accepted for signature parity, the GPU ignores it."""
    env = os.environ.get(WORKERS_ENV_VAR)
    if env:
        return max(1, int(env))
    return max(1, min(J, os.cpu_count() or 1))


@dataclasses.dataclass(eq=False, repr=False)
class _ParallelDetails:
    """Diagnostics of a partitioned solve (parallel.py:390-405)."""

    partition: Partition
    link_points: np.ndarray
    link_residual: float
    mu_left: np.ndarray
    lambda_right: np.ndarray
    link_mismatch: float
    segment_values0: tuple
    segment_feasibility: tuple
    feasibility_residuals: tuple
    degenerate: bool
    segment_diagnostics: tuple = None
    smooth_deviation: float = None


ParallelDetails = _ref_parallel.ParallelDetails if _ref_parallel is not None else _ParallelDetails


class PolicySequence(collections.abc.Sequence):
    """Lazy ``AffinePolicy.state_feedback(K_t, k_t)`` views (``policies``).

    The reference builds T policy objects eagerly (parallel.py:503-504); a
    lazy sequence keeps ``T = 65536`` solves from spending their time in
    Python object construction.
    """

    def __init__(self, K, k):
        self._K, self._k = K, k

    def __len__(self):
        return self._K.shape[0]

    def __getitem__(self, t):
        if isinstance(t, slice):
            return tuple(self[i] for i in range(*t.indices(len(self))))
        return AffinePolicy.state_feedback(self._K[t], self._k[t])


def _check_partition(partition, T):
    splits = tuple(int(s) for s in partition.split_times)
    if splits[0] != 0 or splits[-1] != T:
        raise ValueError("partition does not cover the horizon")
    if len(splits) != partition.J + 1 or np.diff(splits).min() < 1:
        raise ValueError("split times must be strictly increasing")
    return Partition(partition.J, splits)


def stack_problem(problem):
    """Stacked float64 arrays of one problem, memoized on the instance like
    the reference's ``_stacked_stages`` (parallel.py:141-149)."""
    cached = getattr(problem, "_plq_b200_stacked", None)
    if cached is not None:
        return cached
    ref = getattr(problem, "_stacked_stages", None)
    out = {}
    for f in STAGE_FIELDS:
        if ref is not None and f in ref:
            out[f] = np.ascontiguousarray(ref[f], dtype=np.float64)
        else:
            out[f] = np.ascontiguousarray(np.stack(
                [getattr(c if f[0] in "Qq" else d, f) for c, d in problem.stages]), dtype=np.float64)
    out["QxxT"] = np.ascontiguousarray(problem.terminal.Qxx, dtype=np.float64)
    out["qx1T"] = np.ascontiguousarray(problem.terminal.qx1, dtype=np.float64)
    out["x_init"] = np.ascontiguousarray(problem.x_init, dtype=np.float64)
    try:
        object.__setattr__(problem, "_plq_b200_stacked", out)
    except (AttributeError, TypeError):
        pass
    return out


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1809_06360_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


class BatchSolver:
    """Pre-allocated device solver for a batch of ``B`` problems sharing
    ``(T, n, m)`` and one partition.  ``run`` only launches (stream-ordered,
    capturable in a CUDA graph); ``raise_for_status`` synchronizes and maps
    the per-segment status to the reference's exceptions."""

    def __init__(self, B, T, n, m, J=None, partition=None, tolerances=DEFAULT_TOLERANCES,
                 device=None, keep_unfolded=False, degenerate=True, diagnostics=False):
        torch = _torch()
        self.torch = torch
        self.lib = _native.lib()
        if partition is None:
            partition = make_partition(T, J)
        else:
            partition = _check_partition(partition, T)
        self.partition = partition
        self.B, self.T, self.n, self.m, self.J = int(B), int(T), int(n), int(m), partition.J
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.tolerances = tolerances
        dev = dict(device=self.device, dtype=torch.float64)
        B, T, n, m, J = self.B, self.T, self.n, self.m, self.J
        with torch.cuda.device(self.device):
            self.split_times = torch.tensor(partition.split_times, dtype=torch.int32, device=self.device)
            self.out = {
                "K": torch.empty((B, T, m, n), **dev),
                "k": torch.empty((B, T, m), **dev),
                "x": torch.empty((B, T + 1, n), **dev),
                "u": torch.empty((B, T, m), **dev),
                "lam": torch.empty((B, T + 1, n), **dev),
                "links": torch.empty((B, max(J - 1, 1), n), **dev),
                "mu_left": torch.empty((B, max(J - 1, 1), n), **dev),
                "lambda_right": torch.empty((B, max(J - 1, 1), n), **dev),
                "vf0": torch.empty((B, J, 3 * n * n + 2 * n), **dev),
                "Kz": torch.empty((B, T, m, n), **dev) if keep_unfolded else None,
                "k1": torch.empty((B, T, m), **dev) if keep_unfolded else None,
                "objective": torch.empty((B,), **dev),
                "kkt_inf": torch.empty((B,), **dev),
                "link_mismatch": torch.zeros((B,), **dev),
                "link_residual": torch.zeros((B,), **dev),
                "status": torch.zeros((B, J), dtype=torch.int32, device=self.device),
                # degenerate partitions (parallel.py:320-384): rows, counts, residuals
                "feas": torch.empty((B, J, n, 2 * n + 1), **dev) if degenerate else None,
                "feas_rows": torch.zeros((B, J), dtype=torch.int32, device=self.device) if degenerate else None,
                "feas_residual": torch.zeros((B, J), **dev) if degenerate else None,
                # collect_diagnostics (StageDiagnostics, endpoint.py:108-115): defects, max rows
                "diag": torch.zeros((B, J, 2), **dev) if diagnostics else None,
                "diag_rows": torch.zeros((B, J), dtype=torch.int32, device=self.device) if diagnostics else None,
            }
        self._outs = _native.PlqOutputs(**{f: _ptr(self.out[f]) for f in _native.OUTPUT_FIELDS})
        self._prob = self._problem_struct(None)
        with torch.cuda.device(self.device):
            self.ws_bytes = int(self.lib.plq_workspace_bytes(ctypes.byref(self._prob)))
            if self.ws_bytes == 0:
                _native.check(-1, "plq_workspace_bytes")
            self.workspace = torch.empty((self.ws_bytes,), dtype=torch.uint8, device=self.device)
        self.launches = 0

    def _problem_struct(self, inputs, t0=0):
        """C-ABI problem struct over device ``inputs``.  ``t0 > 0`` (B = 1,
        horizon sharding): the stage arrays hold only a window of stages
        starting at ``t0``; their pointers are shifted back by ``t0`` stages
        so the kernels' global stage index lands in the window (the phase
        entry points read only the stages of their segment range,
        include/parlqr_b200.h)."""
        splits = np.asarray(self.partition.split_times)
        P = _native.PlqProblem()
        P.B, P.T, P.n, P.m, P.J = self.B, self.T, self.n, self.m, self.J
        P.max_seg_len = int(np.diff(splits).max())
        P.split_times = _ptr(self.split_times)
        dummy = self.split_times   # non-null placeholder for sizing queries
        if t0 and self.B != 1:
            raise ValueError("stage windows are for single-problem horizon sharding (B = 1)")
        for f in INPUT_FIELDS:
            if inputs is None:
                setattr(P, f, _ptr(dummy))
            elif t0 and f in STAGE_FIELDS:
                t = inputs[f]
                stride = t[0, 0].numel() * t.element_size()
                setattr(P, f, ctypes.c_void_p(t.data_ptr() - t0 * stride))
            else:
                setattr(P, f, _ptr(inputs[f]))
        P.rank_tol = float(self.tolerances.rank_tol)
        P.feas_tol = float(self.tolerances.feas_tol)
        return P

    def check_inputs(self, inputs, T_held=None):
        torch = self.torch
        B, n, m = self.B, self.n, self.m
        T = self.T if T_held is None else int(T_held)
        shapes = {"Qxx": (B, T, n, n), "Qux": (B, T, m, n), "Quu": (B, T, m, m), "qx1": (B, T, n),
                  "qu1": (B, T, m), "Fx": (B, T, n, n), "Fu": (B, T, n, m), "f1": (B, T, n),
                  "QxxT": (B, n, n), "qx1T": (B, n), "x_init": (B, n)}
        for f, shp in shapes.items():
            t = inputs[f]
            if tuple(t.shape) != shp or t.dtype != torch.float64 or t.device != self.device \
                    or not t.is_contiguous():
                raise ValueError(f"{f}: expected contiguous float64 {shp} on {self.device}, "
                                 f"got {tuple(t.shape)} {t.dtype} {t.device}")

    def run(self, inputs, stream=None):
        """Launch the solve of device-resident ``inputs`` (no host sync)."""
        torch = self.torch
        prob = self._problem_struct(inputs)
        stream = torch.cuda.current_stream(self.device) if stream is None else stream
        rc = self.lib.plq_solve_parallel(ctypes.byref(prob), ctypes.byref(self._outs),
                                         _ptr(self.workspace), self.ws_bytes,
                                         ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, "plq_solve_parallel")
        self.launches = int(self.lib.plq_last_launch_count())

    def capture(self, inputs, stream=None):
        """Capture ``run(inputs)`` into a CUDA graph (the launches are
        stream-ordered and allocation-free, so the whole solve replays as one
        graph launch).  Returns the ``torch.cuda.CUDAGraph``; ``replay()``
        re-solves whatever the captured input tensors hold."""
        torch = self.torch
        with torch.cuda.device(self.device):
            self.run(inputs)                     # warm: one-time kernel attributes
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(self.device) if stream is None else stream
            with torch.cuda.graph(g, stream=s):
                self.run(inputs, stream=s)
            self._graph_inputs = inputs          # keep the captured buffers alive
        return g

    def raise_for_status(self):
        status = self.out["status"].cpu().numpy()
        fr = self.out.get("feas_residual")
        raise_for_status(status, None if fr is None else fr.cpu().numpy())

    def smooth(self, inputs, stream=None):
        """Launch the smoothing pass (``plq_smooth``) over this solver's last
        solve of the same ``inputs`` (no host sync).  Returns the device dict
        of smoothed ``K, k, x, u, objective, kkt_inf, deviation, status``."""
        torch = self.torch
        if getattr(self, "smooth_out", None) is None:
            B, T, n, m, J = self.B, self.T, self.n, self.m, self.J
            dev = dict(device=self.device, dtype=torch.float64)
            with torch.cuda.device(self.device):
                self.smooth_out = {
                    "K": torch.empty((B, T, m, n), **dev), "k": torch.empty((B, T, m), **dev),
                    "x": torch.empty((B, T + 1, n), **dev), "u": torch.empty((B, T, m), **dev),
                    "objective": torch.empty((B,), **dev), "kkt_inf": torch.empty((B,), **dev),
                    "deviation": torch.empty((B,), **dev),
                    "status": torch.zeros((B, J), dtype=torch.int32, device=self.device),
                }
            self._smooth_outs = _native.PlqSmoothOutputs(
                **{f: _ptr(self.smooth_out[f]) for f in _native.SMOOTH_FIELDS})
        prob = self._problem_struct(inputs)
        stream = torch.cuda.current_stream(self.device) if stream is None else stream
        rc = self.lib.plq_smooth(ctypes.byref(prob), ctypes.byref(self._outs), ctypes.byref(self._smooth_outs),
                                 _ptr(self.workspace), self.ws_bytes, ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, "plq_smooth")
        self.launches = int(self.lib.plq_last_launch_count())
        return self.smooth_out


def raise_for_status(status, feas_residual=None):
    """Map per-(problem, segment) status codes to the reference exceptions,
    in the order the reference raises them: segment sweeps first, in segment
    order (pool.map, parallel.py:207), then the link solve, then the
    feasibility check at the solved links (parallel.py:462-475)."""
    status = np.atleast_2d(status)
    if np.any(status == _native.PLQ_STATUS_BAD_PARTITION):
        j = int(np.argwhere(status == _native.PLQ_STATUS_BAD_PARTITION)[0][1])
        raise ValueError(f"malformed partition at segment {j}: split times must increase from 0 to T "
                         "with no segment longer than max_seg_len")
    bad = np.argwhere((status > 0) | (status == _native.PLQ_STATUS_DEGENERATE))
    if bad.size:
        b, j = (int(v) for v in bad[np.lexsort((bad[:, 1], bad[:, 0]))][0])
        s = int(status[b, j])
        if s > 0:
            raise CholeskyFailure(s - 1, segment=j)
        raise UnsupportedPartition(j)
    if np.any(status == _native.PLQ_STATUS_LINK_SINGULAR):
        raise LinkSingular("singular pivot block in the link system")
    inf = np.argwhere(status == _native.PLQ_STATUS_INFEASIBLE)
    if inf.size:
        b, j = (int(v) for v in inf[np.lexsort((inf[:, 1], inf[:, 0]))][0])
        res = float(np.atleast_2d(feas_residual)[b, j]) if feas_residual is not None else float("nan")
        raise Infeasible(res, segment=j)


def _to_device(arrays, device, torch):
    out = {}
    for f in INPUT_FIELDS:
        a = arrays[f]
        if isinstance(a, torch.Tensor):
            t = a.to(device=device, dtype=torch.float64)
        else:
            t = torch.from_numpy(np.require(a, dtype=np.float64, requirements=["C", "W"])).to(device)
        out[f] = t.contiguous()
    return out


def _symmetrize_blocks(inputs, torch, chunk=1 << 24):
    """The reference symmetrizes ``Qxx`` / ``Quu`` when a problem is built
    (problem.py:106-116, 129-133); raw stacked arrays skip those constructors,
    and the kernels read only one triangle of the symmetric blocks on some
    paths.  Blocks that are already symmetric (the usual case) are left
    untouched and unallocated; others are replaced by ``0.5 (Q + Q')``."""
    for f in ("Qxx", "Quu", "QxxT"):
        t = inputs[f]
        d = t.shape[-1]
        flat = t.reshape(-1, d, d)
        step = max(1, chunk // (d * d))
        fixed = None
        for i in range(0, flat.shape[0], step):
            blk = flat[i:i + step]
            if not torch.equal(blk, blk.transpose(1, 2)):
                if fixed is None:
                    fixed = flat.clone()
                fixed[i:i + step] = 0.5 * (blk + blk.transpose(1, 2))
        if fixed is not None:
            inputs[f] = fixed.reshape(t.shape)
    return inputs


def solve_parallel_batch(arrays, J=None, partition=None, tolerances=DEFAULT_TOLERANCES, device=None,
                         keep_unfolded=False, check=True, symmetrize=True, diagnostics=False):
    """Solve ``B`` stacked problems (dict of ``(B, T, ...)`` arrays or
    tensors).  Returns the :class:`BatchSolver` whose ``out`` dict holds the
    device results.  ``symmetrize`` applies the reference constructors'
    ``0.5 (Q + Q')`` to unsymmetric quadratic blocks (a C-ABI caller must
    pass symmetric blocks, include/parlqr_b200.h)."""
    torch = _torch()
    B, T, n = (int(s) for s in arrays["qx1"].shape)
    m = int(arrays["qu1"].shape[2])
    solver = BatchSolver(B, T, n, m, J=J, partition=partition, tolerances=tolerances, device=device,
                         keep_unfolded=keep_unfolded, diagnostics=diagnostics)
    inputs = _to_device(arrays, solver.device, torch)
    solver.check_inputs(inputs)
    if symmetrize:
        inputs = _symmetrize_blocks(inputs, torch)
    with torch.cuda.device(solver.device):
        solver.run(inputs)
    if check:
        solver.raise_for_status()
    return solver


def solve_parallel(problem, J, workers=None, tolerances=DEFAULT_TOLERANCES, collect_diagnostics=False,
                   partition=None, *, device=None):
    """Drop-in for ``parlqr.solve_parallel`` (parallel.py:422-553).

    ``workers`` is accepted for signature parity and ignored (the segments
    run concurrently on the GPU).  ``J = 1`` runs the single (serial)
    segment on the GPU; its multipliers follow the stationarity recursion,
    which equals the reference's value-gradient form ``-(Vxx x + vx1)``
    (serial.py:86-88) up to rounding.
    """
    T = len(problem.stages)
    if partition is not None:
        partition = _check_partition(partition, T)
        J = partition.J
    else:
        partition = make_partition(T, J)
    a = stack_problem(problem)
    batch = {f: a[f][None] for f in INPUT_FIELDS}
    solver = solve_parallel_batch(batch, partition=partition, tolerances=tolerances, device=device,
                                  diagnostics=bool(collect_diagnostics))
    o = {k: (v.cpu().numpy()[0] if v is not None else None) for k, v in solver.out.items()}
    return solution_from_outputs(o, partition)


@dataclasses.dataclass(eq=False, repr=False)
class _StageDiagnostics:
    """endpoint.py:108-115 (stand-in when ``parlqr`` is not importable)."""

    basis_defect: float = 0.0
    projector_defect: float = 0.0
    max_rows: int = 0


def _segment_diagnostics(o, Jp):
    """``details.segment_diagnostics``: one ``StageDiagnostics`` per endpoint
    segment (``None`` for the last, serial one, and for every segment without
    ``collect_diagnostics``; parallel.py:239, 549).  The defects come from the
    rank-revealing kernel's singular vectors (include/parlqr_b200.h)."""
    if o.get("diag") is None:
        return tuple(None for _ in range(Jp))
    ref = compat.reference_module("endpoint")
    cls = ref.StageDiagnostics if ref is not None else _StageDiagnostics
    return tuple(cls(basis_defect=float(o["diag"][j][0]), projector_defect=float(o["diag"][j][1]),
                     max_rows=int(o["diag_rows"][j])) if j < Jp - 1 else None for j in range(Jp))


def solution_from_outputs(o, partition):
    """``LqrSolution`` + ``ParallelDetails`` (the reference's classes when
    ``parlqr`` is importable) from one problem's host outputs ``o`` (the
    ``BatchSolver.out`` fields of one batch row, parallel.py:529-553)."""
    n = o["x"].shape[1]
    Jp = partition.J
    nn = n * n
    vf = o["vf0"]
    values = []
    for j in range(Jp):
        row = vf[j]
        Vxx = row[:nn].reshape(n, n)
        vx1 = row[3 * nn:3 * nn + n]
        if j == Jp - 1:
            values.append((Vxx, vx1))
        else:
            values.append((Vxx, row[nn:2 * nn].reshape(n, n), row[2 * nn:3 * nn].reshape(n, n),
                           vx1, row[3 * nn + n:3 * nn + 2 * n]))
    links = o["links"][:Jp - 1]
    # feasibility triples of the endpoint segments (rows in the GPU's
    # orthonormal basis; parallel.py:398-401) and their residuals (:462-475)
    rows = o["feas_rows"] if o.get("feas_rows") is not None else np.zeros(Jp, dtype=np.int32)
    feas = []
    for j in range(Jp):
        if j == Jp - 1:
            feas.append(None)
            continue
        r = int(rows[j])
        F = o["feas"][j][:r] if r else np.zeros((0, 2 * n + 1))
        feas.append((F[:, :n].copy(), F[:, n:2 * n].copy(), F[:, 2 * n].copy()))
    fres = o.get("feas_residual")
    details = ParallelDetails(
        partition=Partition(partition.J, tuple(partition.split_times)),
        link_points=links,
        link_residual=float(o["link_residual"]),
        mu_left=o["mu_left"][:Jp - 1],
        lambda_right=o["lambda_right"][:Jp - 1],
        link_mismatch=float(o["link_mismatch"]) if Jp > 1 else 0.0,
        segment_values0=tuple(values),
        segment_feasibility=tuple(feas),
        feasibility_residuals=tuple(float(fres[j]) if fres is not None and int(rows[j]) else 0.0
                                    for j in range(Jp)),
        degenerate=bool(np.any(rows[:Jp - 1] > 0)),
        segment_diagnostics=_segment_diagnostics(o, Jp),
    )
    return LqrSolution(
        states=o["x"], controls=o["u"], lambdas=o["lam"],
        policies=PolicySequence(o["K"], o["k"]),
        objective=float(o["objective"]), kkt_residual_inf=float(o["kkt_inf"]),
        details=details,
    )


def _policy_arrays(policies):
    if isinstance(policies, PolicySequence):
        return policies._K, policies._k
    return (np.stack([np.asarray(p.Kx, dtype=np.float64) for p in policies]),
            np.stack([np.asarray(p.k1, dtype=np.float64) for p in policies]))


def _vf0_rows(values, n):
    rows = np.zeros((len(values), 3 * n * n + 2 * n))
    nn = n * n
    for j, v in enumerate(values):
        if len(v) == 2:
            rows[j, :nn] = np.ravel(v[0])
            rows[j, 3 * nn:3 * nn + n] = v[1]
        else:
            Vxx, Vzx, Vzz, vx1, vz1 = v
            rows[j] = np.concatenate([np.ravel(Vxx), np.ravel(Vzx), np.ravel(Vzz), vx1, vz1])
    return rows


def smooth(problem, result, workers=None, tolerances=DEFAULT_TOLERANCES, *, device=None):
    """Drop-in for ``parlqr.parallel.smooth`` (parallel.py:567-633).

    The sweeps of segments ``0..J-2`` with conditioned terminal costs and the
    rollout of the resulting policies run on the GPU (``plq_smooth``).
    ``workers`` is accepted for signature parity and ignored.  A ``J = 1``
    (or non-partitioned) result is returned unchanged, and a partition whose
    conditioning segment cannot reach arbitrary endpoints raises
    ``ValueError`` -- the reference's contract.
    """
    details = result.details
    if details is None or not hasattr(details, "segment_values0"):
        return result
    partition = details.partition
    J = partition.J
    if J == 1:
        return result
    for j in range(1, J - 1):
        feas = details.segment_feasibility[j]
        if feas is not None and feas[0].shape[0]:
            raise ValueError(
                f"segment {j} cannot reach arbitrary endpoints "
                f"({feas[0].shape[0]} feasibility rows); smoothing undefined "
                "for this partition")
    torch = _torch()
    a = stack_problem(problem)
    T, n = a["qx1"].shape
    m = a["qu1"].shape[1]
    batch = {f: a[f][None] for f in INPUT_FIELDS}
    solver = BatchSolver(1, T, n, m, partition=_check_partition(partition, T), tolerances=tolerances,
                         device=device)
    inputs = _to_device(batch, solver.device, torch)
    K, k = _policy_arrays(result.policies)
    parent = {"K": K, "k": k, "x": result.states, "u": result.controls, "lam": result.lambdas,
              "links": np.asarray(details.link_points).reshape(J - 1, n),
              "vf0": _vf0_rows(details.segment_values0, n)}
    for f, v in parent.items():
        solver.out[f][0].copy_(torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)))
    with torch.cuda.device(solver.device):
        so = solver.smooth(inputs)
    o = {f: v.cpu().numpy()[0] for f, v in so.items()}
    raise_for_status(o["status"])
    deviation = float(o["deviation"])
    return LqrSolution(
        states=o["x"], controls=o["u"], lambdas=result.lambdas,
        policies=PolicySequence(o["K"], o["k"]),
        objective=float(o["objective"]), kkt_residual_inf=float(o["kkt_inf"]),
        details=dataclasses.replace(details, smooth_deviation=deviation),
    )


HOST_OUTPUTS = ("K", "k", "x", "u", "lam", "links", "mu_left", "lambda_right", "vf0",
                "objective", "kkt_inf", "link_mismatch", "link_residual", "status")


class HostSolver:
    """End-to-end entry through ``plq_solve_parallel_host``: host input
    buffers in, host results out, H2D/D2H inside the call (the path a
    ctypes/cgo binding of the reference would take)."""

    def __init__(self, B, T, n, m, J=None, partition=None, tolerances=DEFAULT_TOLERANCES, device=None,
                 pin=True, keep_feas=False):
        torch = _torch()
        self.torch = torch
        self.lib = _native.lib()
        self.partition = make_partition(T, J) if partition is None else _check_partition(partition, T)
        self.B, self.T, self.n, self.m, self.J = int(B), int(T), int(n), int(m), self.partition.J
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.tolerances = tolerances
        self.splits = np.ascontiguousarray(self.partition.split_times, dtype=np.int32)
        B, T, n, m, J = self.B, self.T, self.n, self.m, self.J
        shapes = {"K": (B, T, m, n), "k": (B, T, m), "x": (B, T + 1, n), "u": (B, T, m),
                  "lam": (B, T + 1, n), "links": (B, max(J - 1, 1), n), "mu_left": (B, max(J - 1, 1), n),
                  "lambda_right": (B, max(J - 1, 1), n), "vf0": (B, J, 3 * n * n + 2 * n),
                  "objective": (B,), "kkt_inf": (B,), "link_mismatch": (B,), "link_residual": (B,)}
        if keep_feas:   # degenerate partitions' feasibility rows (details.segment_feasibility)
            shapes["feas"] = (B, J, n, 2 * n + 1)
        shapes["feas_residual"] = (B, J)
        self.out = {k: torch.empty(s, dtype=torch.float64, pin_memory=pin) for k, s in shapes.items()}
        self.out["status"] = torch.zeros((B, J), dtype=torch.int32, pin_memory=pin)
        self.out["feas_rows"] = torch.zeros((B, J), dtype=torch.int32, pin_memory=pin)
        P = self._problem_struct(None)
        with torch.cuda.device(self.device):
            self.arena_bytes = int(self.lib.plq_host_arena_bytes(ctypes.byref(P)))
            if self.arena_bytes == 0:
                _native.check(-1, "plq_host_arena_bytes")
            self.arena = torch.empty((self.arena_bytes,), dtype=torch.uint8, device=self.device)
        self.h2d_bytes = 0
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in self.out.values())

    def _problem_struct(self, inputs):
        P = _native.PlqProblem()
        P.B, P.T, P.n, P.m, P.J = self.B, self.T, self.n, self.m, self.J
        P.max_seg_len = int(np.diff(self.splits).max())
        P.split_times = ctypes.c_void_p(self.splits.ctypes.data)
        for f in INPUT_FIELDS:
            setattr(P, f, _ptr(inputs[f]) if inputs is not None else ctypes.c_void_p(self.splits.ctypes.data))
        P.rank_tol = float(self.tolerances.rank_tol)
        P.feas_tol = float(self.tolerances.feas_tol)
        return P

    def run(self, host_inputs, stream=None):
        """``host_inputs``: dict of contiguous float64 CPU tensors (pinned for speed)."""
        torch = self.torch
        self.h2d_bytes = sum(host_inputs[f].numel() * 8 for f in INPUT_FIELDS) + self.splits.nbytes
        P = self._problem_struct(host_inputs)
        outs = _native.PlqOutputs(**{f: (_ptr(self.out[f]) if f in self.out else ctypes.c_void_p(0))
                                     for f in _native.OUTPUT_FIELDS})
        stream = torch.cuda.current_stream(self.device) if stream is None else stream
        rc = self.lib.plq_solve_parallel_host(ctypes.byref(P), ctypes.byref(outs), _ptr(self.arena),
                                              self.arena_bytes, ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, "plq_solve_parallel_host")
        raise_for_status(self.out["status"].numpy(), self.out["feas_residual"].numpy())
        return self.out


def solve_parallel_host(arrays, J=None, partition=None, tolerances=DEFAULT_TOLERANCES, device=None):
    """One end-to-end batch solve from host arrays; returns host numpy results."""
    torch = _torch()
    B, T, n = (int(s) for s in arrays["qx1"].shape)
    m = int(arrays["qu1"].shape[2])
    hs = HostSolver(B, T, n, m, J=J, partition=partition, tolerances=tolerances, device=device, pin=False,
                    keep_feas=True)
    host = {f: torch.from_numpy(np.require(arrays[f], dtype=np.float64, requirements=["C", "W"]))
            for f in INPUT_FIELDS}
    out = hs.run(host)
    return {k: v.numpy().copy() for k, v in out.items()}
