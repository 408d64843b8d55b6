"""Two-point-boundary solve on the GPU: drop-ins for
``parlqr.endpoint.solve_endpoint_affine`` / ``solve_endpoint``
(``endpoint.py:603-653``) and their result types, over the C ABI entries
``plq_endpoint_affine`` / ``plq_endpoint_evaluate``.

The backward pass, the forward affine maps, the multiplier normal equations
and the evaluation at concrete endpoints all run on the device
(``csrc/plq_endpoint.cu``).  Differences a caller can observe:

* ``values`` / ``constraints`` hold the t = 0 entries only (the ones
  ``evaluate`` needs); ``values[0].const`` is taken lazily from one device
  evaluation at a feasible endpoint pair;
* problems whose endpoint cannot be reached in every direction (feasibility
  rows, e.g. ``T m < n``) are solved like the reference does: no multiplier
  maps, ``evaluate`` checks the rows (``Infeasible``) and takes the
  multipliers from the value-function gradient and the stationarity recursion
  (``gradient_duals``, ``endpoint.py:566-587``) on the device; the rows in
  ``constraints[0]`` are an orthonormal rotation of the reference's;
* ``collect_diagnostics=True`` routes the backward pass through the
  rank-revealing kernel and returns its singular-vector defects as the
  reference's ``StageDiagnostics`` (include/parlqr_b200.h).
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _native
from .errors import CholeskyFailure, FactorizationFailure, Infeasible, UnsupportedPartition
from .parallel import INPUT_FIELDS, _ptr, _to_device, _torch, stack_problem
from .problem import DEFAULT_TOLERANCES, AffinePolicy, LqrSolution


class ValueFunction:
    """endpoint.py:61-83: ``value(x, z) = 1/2 x'Vxx x + z'Vzx x + 1/2 z'Vzz z
    + vx1'x + vz1'z + const``.  The sweep kernels do not carry ``const``;
    it is taken on first use from one device evaluation at a feasible endpoint
    pair (``const`` may be given as a callable returning it)."""

    def __init__(self, Vxx, Vzx, Vzz, vx1, vz1, const=0.0):
        self.Vxx, self.Vzx, self.Vzz, self.vx1, self.vz1 = Vxx, Vzx, Vzz, vx1, vz1
        self._const = const

    @property
    def const(self):
        if callable(self._const):
            self._const = float(self._const())
        return self._const

    def gradient_x(self, x, z):
        return self.Vxx @ x + self.Vzx.T @ z + self.vx1

    def gradient_z(self, x, z):
        return self.Vzx @ x + self.Vzz @ z + self.vz1

    def _quadratic(self, x, z):
        return float(0.5 * x @ (self.Vxx @ x) + z @ (self.Vzx @ x) + 0.5 * z @ (self.Vzz @ z)
                     + self.vx1 @ x + self.vz1 @ z)

    def value(self, x, z):
        return self._quadratic(x, z) + self.const


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class ConstraintToGo:
    """endpoint.py:86-105."""

    Hx: np.ndarray
    Hz: np.ndarray
    h1: np.ndarray

    @property
    def rows(self):
        return self.Hx.shape[0]

    def residual(self, x, z):
        if self.rows == 0:
            return np.zeros(0)
        return self.Hx @ x + self.Hz @ z + self.h1

    def residual(self, x, z):
        return np.zeros(0) if self.rows == 0 else self.Hx @ x + self.Hz @ z + self.h1


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class TrajectoryMaps:
    """endpoint.py:303-323: x_t = Ra x_init + Rz x_term + r1, u_t = Sa ... ."""

    Ra: np.ndarray
    Rz: np.ndarray
    r1: np.ndarray
    Sa: np.ndarray
    Sz: np.ndarray
    s1: np.ndarray

    def states(self, x_init, x_term):
        return self.Ra @ x_init + self.Rz @ x_term + self.r1

    def controls(self, x_init, x_term):
        return self.Sa @ x_init + self.Sz @ x_term + self.s1


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class MultiplierMaps:
    """endpoint.py:441-456: lam_t = La x_init + Lz x_term + l1, mu = Ea ... ."""

    La: np.ndarray
    Lz: np.ndarray
    l1: np.ndarray
    Ea: np.ndarray
    Ez: np.ndarray
    e1: np.ndarray

    def lambdas(self, x_init, x_term):
        return self.La @ x_init + self.Lz @ x_term + self.l1

    def mu(self, x_init, x_term):
        return self.Ea @ x_init + self.Ez @ x_term + self.e1


class EndpointBatch:
    """Device two-point-boundary solver for ``B`` problems sharing
    ``(T, n, m)``.  ``affine(inputs)`` launches the backward pass, the maps
    and the multiplier system; ``evaluate(x_term[, x_init])`` the trajectories,
    objective and KKT residual at concrete endpoints (stream-ordered; call
    ``raise_for_status`` to synchronize and map failures)."""

    def __init__(self, B, T, n, m, tolerances=DEFAULT_TOLERANCES, device=None, diagnostics=False):
        torch = _torch()
        self.torch = torch
        self.lib = _native.lib()
        self.B, self.T, self.n, self.m = int(B), int(T), int(n), int(m)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.tolerances = tolerances
        B, T, n, m = self.B, self.T, self.n, self.m
        W = 2 * n + 1
        f64 = dict(device=self.device, dtype=torch.float64)
        with torch.cuda.device(self.device):
            self.split_times = torch.tensor([0, T], dtype=torch.int32, device=self.device)
            self.out = {
                "Kx": torch.empty((B, T, m, n), **f64), "Kz": torch.empty((B, T, m, n), **f64),
                "k1": torch.empty((B, T, m), **f64), "value0": torch.empty((B, 3 * n * n + 2 * n), **f64),
                "X": torch.empty((B, T + 1, n, W), **f64), "S": torch.empty((B, T, m, W), **f64),
                "Lam": torch.empty((B, T + 1, n, W), **f64), "E": torch.empty((B, n, W), **f64),
                "status": torch.zeros((B,), dtype=torch.int32, device=self.device),
                "gram_status": torch.zeros((B,), dtype=torch.int32, device=self.device),
                "feas": torch.zeros((B, n, W), **f64),
                "feas_rows": torch.zeros((B,), dtype=torch.int32, device=self.device),
            }
            if diagnostics:
                self.out["diag"] = torch.zeros((B, 2), **f64)
                self.out["diag_rows"] = torch.zeros((B,), dtype=torch.int32, device=self.device)
            self.point = {
                "x": torch.empty((B, T + 1, n), **f64), "u": torch.empty((B, T, m), **f64),
                "lam": torch.empty((B, T + 1, n), **f64), "mu": torch.empty((B, n), **f64),
                "objective": torch.empty((B,), **f64), "kkt_inf": torch.empty((B,), **f64),
                "feas_residual": torch.zeros((B,), **f64),
            }
        self._outs = _native.PlqEndpointOutputs(**{f: _ptr(self.out.get(f)) for f in _native.ENDPOINT_FIELDS})
        P = self._problem_struct(None)
        with torch.cuda.device(self.device):
            self.ws_bytes = int(self.lib.plq_endpoint_workspace_bytes(ctypes.byref(P)))
            if self.ws_bytes == 0:
                _native.check(-1, "plq_endpoint_workspace_bytes")
            self.workspace = torch.empty((self.ws_bytes,), dtype=torch.uint8, device=self.device)
        self.launches = 0
        self._inputs = None

    def _problem_struct(self, inputs):
        P = _native.PlqProblem()
        P.B, P.T, P.n, P.m, P.J = self.B, self.T, self.n, self.m, 1
        P.max_seg_len = self.T
        P.split_times = _ptr(self.split_times)
        for f in INPUT_FIELDS:
            setattr(P, f, _ptr(inputs[f]) if inputs is not None else _ptr(self.split_times))
        P.rank_tol = float(self.tolerances.rank_tol)
        P.feas_tol = float(self.tolerances.feas_tol)
        return P

    def affine(self, inputs, stream=None):
        torch = self.torch
        self._inputs = inputs
        P = self._problem_struct(inputs)
        stream = torch.cuda.current_stream(self.device) if stream is None else stream
        rc = self.lib.plq_endpoint_affine(ctypes.byref(P), ctypes.byref(self._outs), _ptr(self.workspace),
                                          self.ws_bytes, ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, "plq_endpoint_affine")
        self.launches = int(self.lib.plq_last_launch_count())

    def evaluate(self, x_term, x_init=None, stream=None):
        torch = self.torch
        P = self._problem_struct(self._inputs)
        pt = _native.PlqEndpointPoint(x_init=_ptr(x_init), x_term=_ptr(x_term),
                                      **{f: _ptr(self.point[f]) for f in _native.POINT_FIELDS[2:]})
        stream = torch.cuda.current_stream(self.device) if stream is None else stream
        rc = self.lib.plq_endpoint_evaluate(ctypes.byref(P), ctypes.byref(self._outs), ctypes.byref(pt),
                                            _ptr(self.workspace), self.ws_bytes, ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, "plq_endpoint_evaluate")
        self.launches = int(self.lib.plq_last_launch_count())
        xi = x_init if x_init is not None else self._inputs["x_init"]
        self._last_endpoints = (xi.cpu().numpy(), x_term.cpu().numpy())
        return self.point

    def raise_for_status(self, require_multipliers=True, check_feasibility=False):
        """Map the device status to the reference's exceptions.  ``require_multipliers``:
        ``"strict"`` = ``solve_endpoint_affine(require_multipliers=True)`` (rows raise
        ``FactorizationFailure``, endpoint.py:614-617); truthy = a failed Gram factorization
        raises.  ``check_feasibility``: after ``evaluate``, rows violated by the endpoint pair
        raise ``Infeasible`` (endpoint.py:516-523)."""
        st = self.out["status"].cpu().numpy()
        gs = self.out["gram_status"].cpu().numpy()
        rows = self.out["feas_rows"].cpu().numpy()
        for b in range(self.B):
            if st[b] > 0:
                raise CholeskyFailure(int(st[b]) - 1)
            if st[b] < 0:
                raise UnsupportedPartition(0, "feasibility rows left but no buffer to return them")
            if rows[b] > 0 and require_multipliers == "strict":
                raise FactorizationFailure(None, "boundary constraints are linearly dependent "
                                                 f"({int(rows[b])} unreachable endpoint rows)")
            if gs[b] > 0 and require_multipliers:
                raise FactorizationFailure(int(gs[b]) - 1)
        if check_feasibility and rows.any():
            res = self.point["feas_residual"].cpu().numpy()
            xi, xt = self._last_endpoints
            for b in range(self.B):
                scale = 1.0 + float(np.abs(xi[b]).max(initial=0.0)) + float(np.abs(xt[b]).max(initial=0.0))
                if rows[b] > 0 and res[b] > self.tolerances.feas_tol * scale:
                    raise Infeasible(float(res[b]))


class EndpointAffineSolution:
    """endpoint.py:479-575: the solution as affine maps of (x_init, x_term);
    ``evaluate`` runs on the GPU."""

    def __init__(self, problem, batch, index=0):
        o = {k: v[index].cpu().numpy() for k, v in batch.out.items()}
        n, m, T = batch.n, batch.m, batch.T
        nn = n * n
        self.stages = problem.stages
        self.terminal = problem.terminal
        self.policies = tuple(AffinePolicy(o["Kx"][t], o["Kz"][t], o["k1"][t]) for t in range(T))
        v = o["value0"]
        self.values = (ValueFunction(v[:nn].reshape(n, n), v[nn:2 * nn].reshape(n, n),
                                     v[2 * nn:3 * nn].reshape(n, n), v[3 * nn:3 * nn + n], v[3 * nn + n:],
                                     const=self._const0),)
        r = int(o["feas_rows"])
        Hf = o["feas"][:r]
        self.constraints = (ConstraintToGo(Hf[:, :n].copy(), Hf[:, n:2 * n].copy(), Hf[:, 2 * n].copy()),)
        X, S, L, E = o["X"], o["S"], o["Lam"], o["E"]
        self.maps = TrajectoryMaps(X[:, :, :n], X[:, :, n:2 * n], X[:, :, 2 * n],
                                   S[:, :, :n], S[:, :, n:2 * n], S[:, :, 2 * n])
        self.multipliers = None if (int(o["gram_status"]) or r) else MultiplierMaps(
            L[:, :, :n], L[:, :, n:2 * n], L[:, :, 2 * n], E[:, :n], E[:, n:2 * n], E[:, 2 * n])
        self.diagnostics = None
        if "diag" in o:
            from .parallel import _segment_diagnostics
            self.diagnostics = _segment_diagnostics({"diag": o["diag"][None], "diag_rows": o["diag_rows"][None]}, 2)[0]
        self._batch, self._index, self._problem = batch, index, problem

    @property
    def feasibility(self):
        return self.constraints[0]

    def _const0(self):
        """``values[0].const`` (endpoint.py:283-284, 296): the objective of one device
        evaluation at a feasible endpoint pair minus the value function's other terms
        there -- (0, 0) when every endpoint is reachable, else the least-norm pair on
        the feasibility rows."""
        c = self.feasibility
        n = self._batch.n
        xz = np.zeros(2 * n)
        if c.rows:
            xz = np.linalg.lstsq(np.concatenate([c.Hx, c.Hz], axis=1), -c.h1, rcond=None)[0]
        x, z = xz[:n], xz[n:]
        return self._objective_at(x, z) - self.values[0]._quadratic(x, z)

    def _objective_at(self, x_init, x_term):
        torch = self._batch.torch
        B, n, dev = self._batch.B, self._batch.n, self._batch.device
        xi = torch.zeros((B, n), dtype=torch.float64, device=dev)
        xt = torch.zeros((B, n), dtype=torch.float64, device=dev)
        xi[self._index] = torch.from_numpy(np.asarray(x_init, dtype=np.float64))
        xt[self._index] = torch.from_numpy(np.asarray(x_term, dtype=np.float64))
        with torch.cuda.device(dev):
            pt = self._batch.evaluate(xt, xi)
        return float(pt["objective"][self._index].cpu())

    def feasibility_residual(self, x_init, x_term):
        res = self.feasibility.residual(np.asarray(x_init, float), np.asarray(x_term, float))
        return float(np.abs(res).max()) if res.size else 0.0

    def evaluate(self, x_init, x_term, tolerances=DEFAULT_TOLERANCES):
        """Numeric solution at concrete endpoints (endpoint.py:507-546).  With
        feasibility rows: ``Infeasible`` when the pair violates them, else the
        multipliers come from ``gradient_duals`` (computed on the device)."""
        x_init = np.asarray(x_init, dtype=np.float64)
        x_term = np.asarray(x_term, dtype=np.float64)
        if self.feasibility.rows:
            residual = self.feasibility_residual(x_init, x_term)
            scale = 1.0 + float(np.abs(x_init).max(initial=0.0)) + float(np.abs(x_term).max(initial=0.0))
            if residual > tolerances.feas_tol * scale:
                raise Infeasible(residual)
        elif self.multipliers is None:
            raise FactorizationFailure(int(self._batch.out["gram_status"][self._index]) - 1)
        torch = self._batch.torch
        B, n = self._batch.B, self._batch.n
        dev = self._batch.device
        xi = torch.zeros((B, n), dtype=torch.float64, device=dev)
        xt = torch.zeros((B, n), dtype=torch.float64, device=dev)
        xi[self._index] = torch.from_numpy(np.asarray(x_init, dtype=np.float64))
        xt[self._index] = torch.from_numpy(np.asarray(x_term, dtype=np.float64))
        with torch.cuda.device(dev):
            pt = self._batch.evaluate(xt, xi)
        o = {k: v[self._index].cpu().numpy() for k, v in pt.items()}
        return LqrSolution(states=o["x"], controls=o["u"], lambdas=o["lam"], policies=self.policies,
                           objective=float(o["objective"]), kkt_residual_inf=float(o["kkt_inf"]),
                           mu=o["mu"], x_term=np.asarray(x_term, dtype=np.float64))


def _batch_for(problem, tolerances, device, diagnostics=False):
    torch = _torch()
    a = stack_problem(problem)
    T, n = a["qx1"].shape
    m = a["qu1"].shape[1]
    batch = EndpointBatch(1, T, n, m, tolerances=tolerances, device=device, diagnostics=diagnostics)
    inputs = _to_device({f: a[f][None] for f in INPUT_FIELDS}, batch.device, torch)
    with torch.cuda.device(batch.device):
        batch.affine(inputs)
    return batch


def solve_endpoint_affine(problem, tolerances=DEFAULT_TOLERANCES, collect_diagnostics=False,
                          require_multipliers=False, *, device=None):
    """Drop-in for ``parlqr.endpoint.solve_endpoint_affine`` (endpoint.py:603-636)."""
    batch = _batch_for(problem, tolerances, device, diagnostics=bool(collect_diagnostics))
    batch.raise_for_status(require_multipliers="strict" if require_multipliers else False)
    return EndpointAffineSolution(problem, batch)


def solve_endpoint(problem, x_init, x_term, tolerances=DEFAULT_TOLERANCES, *, device=None):
    """Drop-in for ``parlqr.endpoint.solve_endpoint`` (endpoint.py:639-653):
    ``problem.x_init`` is ignored in favour of ``x_init``."""
    batch = _batch_for(problem, tolerances, device)
    batch.raise_for_status(require_multipliers=True)
    return EndpointAffineSolution(problem, batch).evaluate(x_init, x_term, tolerances)   # Infeasible inside


def solve_endpoint_batch(arrays, x_term, x_init=None, tolerances=DEFAULT_TOLERANCES, device=None):
    """Batched two-point-boundary solve of stacked ``(B, T, ...)`` arrays at
    endpoints ``x_term (B, n)`` (and ``x_init``, default the problems').
    Returns the :class:`EndpointBatch` (device results in ``out`` / ``point``)."""
    torch = _torch()
    B, T, n = (int(s) for s in arrays["qx1"].shape)
    m = int(arrays["qu1"].shape[2])
    batch = EndpointBatch(B, T, n, m, tolerances=tolerances, device=device)
    inputs = _to_device(arrays, batch.device, torch)
    dev = batch.device
    xt = torch.as_tensor(np.asarray(x_term, dtype=np.float64) if not isinstance(x_term, torch.Tensor) else x_term,
                         dtype=torch.float64).to(dev).contiguous()
    xi = None if x_init is None else torch.as_tensor(x_init, dtype=torch.float64).to(dev).contiguous()
    with torch.cuda.device(dev):
        batch.affine(inputs)
        batch.evaluate(xt, xi)
    batch.raise_for_status(check_feasibility=True)
    batch._keep = (inputs, xt, xi)
    return batch


__all__ = ["ConstraintToGo", "EndpointAffineSolution", "EndpointBatch", "MultiplierMaps", "TrajectoryMaps",
           "ValueFunction", "solve_endpoint", "solve_endpoint_affine", "solve_endpoint_batch"]
