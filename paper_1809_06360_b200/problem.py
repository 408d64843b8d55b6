"""Problem / solution containers of the drop-in.

When the reference package ``parlqr`` is importable, this module re-exports
ITS classes (``parlqr.problem``: ``StageCost``, ``StageDynamics``,
``TerminalCost``, ``LqrProblem``, ``AffinePolicy``, ``LqrSolution``,
``ToleranceSet``), so a caller of the drop-in receives exactly the reference's
types (``isinstance(sol, parlqr.LqrSolution)`` holds).  Without ``parlqr``
(e.g. on a GPU box that only has this package) small stand-ins with the same
field names and conventions are used (problem.py:44-280): the solver itself
only reads ``stages[t] = (cost, dynamics)``, ``terminal`` and ``x_init``.

Stage cost ``1/2 x'Qxx x + 1/2 u'Quu u + u'Qux x + qx1'x + qu1'u``, dynamics
``x' = Fx x + Fu u + f1``, terminal ``1/2 x'Qxx_T x + qx1_T'x``; multipliers
satisfy ``lam_t = -dV_t/dx`` (problem.py:1-17).
"""

from __future__ import annotations

import dataclasses

import numpy as np

from . import compat

__all__ = [
    "ToleranceSet", "DEFAULT_TOLERANCES", "StageCost", "TerminalCost",
    "StageDynamics", "LqrProblem", "AffinePolicy", "LqrSolution", "problem_from_arrays",
    "USING_REFERENCE_TYPES",
]


def _frozen(value, shape=None, what="array"):
    """float64 copy, shape-checked, read-only (the reference's arrays are)."""
    out = np.array(value, dtype=np.float64)
    if shape is not None and out.shape != tuple(shape):
        raise ValueError(f"{what} must have shape {tuple(shape)}, got {out.shape}")
    out.setflags(write=False)
    return out


def _symmetric_part(value, what):
    """(0.5 (A + A'), relative asymmetry of A) -- problem.py:81-88."""
    a = np.array(value, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"{what} must be square, got shape {a.shape}")
    scale = float(np.abs(a).max()) if a.size else 0.0
    asym = float(np.abs(a - a.T).max()) / scale if scale else 0.0
    return _frozen(0.5 * (a + a.T)), asym


def _set(obj, **fields):
    for k, v in fields.items():
        object.__setattr__(obj, k, v)


@dataclasses.dataclass(frozen=True)
class _ToleranceSet:
    """Numerical thresholds (problem.py:44-58)."""

    rank_tol: float = 1e-10
    feas_tol: float = 1e-8
    kkt_tol: float = 1e-8


@dataclasses.dataclass(frozen=True, eq=False, repr=False, init=False)
class _StageCost:
    """Quadratic stage cost; ``Qxx``/``Quu`` symmetrized on construction."""

    Qxx: np.ndarray
    Qux: np.ndarray
    Quu: np.ndarray
    qx1: np.ndarray
    qu1: np.ndarray
    asymmetry: float

    def __init__(self, Qxx, Qux, Quu, qx1, qu1):
        sxx, ax = _symmetric_part(Qxx, "Qxx")
        suu, au = _symmetric_part(Quu, "Quu")
        n, m = len(sxx), len(suu)
        _set(self, Qxx=sxx, Quu=suu, Qux=_frozen(Qux, (m, n), "Qux"), qx1=_frozen(qx1, (n,), "qx1"),
             qu1=_frozen(qu1, (m,), "qu1"), asymmetry=max(ax, au))

    n = property(lambda self: self.Qxx.shape[0])
    m = property(lambda self: self.Quu.shape[0])


@dataclasses.dataclass(frozen=True, eq=False, repr=False, init=False)
class _TerminalCost:
    Qxx: np.ndarray
    qx1: np.ndarray
    asymmetry: float

    def __init__(self, Qxx, qx1):
        sxx, ax = _symmetric_part(Qxx, "terminal Qxx")
        _set(self, Qxx=sxx, qx1=_frozen(qx1, (len(sxx),), "terminal qx1"), asymmetry=ax)

    n = property(lambda self: self.Qxx.shape[0])

    @classmethod
    def zero(cls, n):
        return cls(np.zeros((n, n)), np.zeros(n))


@dataclasses.dataclass(frozen=True, eq=False, repr=False, init=False)
class _StageDynamics:
    Fx: np.ndarray
    Fu: np.ndarray
    f1: np.ndarray

    def __init__(self, Fx, Fu, f1):
        fx, fu = _frozen(Fx), _frozen(Fu)
        if fx.ndim != 2 or fx.shape[0] != fx.shape[1]:
            raise ValueError(f"Fx must be square, got shape {fx.shape}")
        if fu.ndim != 2 or fu.shape[0] != fx.shape[0]:
            raise ValueError(f"Fu must have {fx.shape[0]} rows, got shape {fu.shape}")
        _set(self, Fx=fx, Fu=fu, f1=_frozen(f1, (fx.shape[0],), "f1"))

    n = property(lambda self: self.Fx.shape[0])
    m = property(lambda self: self.Fu.shape[1])


@dataclasses.dataclass(frozen=True, eq=False, repr=False, init=False)
class _LqrProblem:
    stages: tuple
    terminal: object
    x_init: np.ndarray

    def __init__(self, stages, terminal, x_init):
        stages = tuple((c, d) for c, d in stages)
        if not stages:
            raise ValueError("horizon must contain at least one stage")
        n, m = stages[0][0].n, stages[0][0].m
        bad = [t for t, (c, d) in enumerate(stages) if (c.n, c.m, d.n, d.m) != (n, m, n, m)]
        if bad:
            raise ValueError(f"inconsistent dimensions at stage {bad[0]}")
        if terminal.n != n:
            raise ValueError("terminal cost dimension mismatch")
        _set(self, stages=stages, terminal=terminal, x_init=_frozen(x_init, (n,), "x_init"))

    n = property(lambda self: self.stages[0][0].n)
    m = property(lambda self: self.stages[0][0].m)
    T = property(lambda self: len(self.stages))

    def __repr__(self):
        return f"LqrProblem(n={self.n}, m={self.m}, T={self.T})"


@dataclasses.dataclass(frozen=True, eq=False, repr=False, init=False)
class _AffinePolicy:
    """``u = Kx x + Kz x_term + k1`` (problem.py:224-259)."""

    Kx: np.ndarray
    Kz: np.ndarray
    k1: np.ndarray

    def __init__(self, Kx, Kz, k1):
        kx = _frozen(Kx)
        if kx.ndim != 2:
            raise ValueError("Kx must be a matrix")
        kz = _frozen(Kz, kx.shape, "Kz")
        _set(self, Kx=kx, Kz=kz, k1=_frozen(k1, kx.shape[:1], "k1"), _uses_terminal=bool(kz.any()))

    @classmethod
    def state_feedback(cls, Kx, k1):
        return cls(Kx, np.zeros(np.shape(Kx)), k1)

    def __call__(self, x, x_term=None):
        u = self.Kx @ x + self.k1
        if not self._uses_terminal:
            return u
        if x_term is None:
            raise ValueError("policy depends on x_term but none was given")
        return u + self.Kz @ x_term


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class _LqrSolution:
    """Numeric solution (problem.py:262-280)."""

    states: np.ndarray
    controls: np.ndarray
    lambdas: np.ndarray
    policies: tuple
    objective: float
    kkt_residual_inf: float
    mu: np.ndarray = None
    x_term: np.ndarray = None
    details: object = None


_ref = compat.reference_module("problem")
USING_REFERENCE_TYPES = _ref is not None
if _ref is not None:
    ToleranceSet = _ref.ToleranceSet
    DEFAULT_TOLERANCES = _ref.DEFAULT_TOLERANCES
    StageCost = _ref.StageCost
    TerminalCost = _ref.TerminalCost
    StageDynamics = _ref.StageDynamics
    LqrProblem = _ref.LqrProblem
    AffinePolicy = _ref.AffinePolicy
    LqrSolution = _ref.LqrSolution
else:
    ToleranceSet = _ToleranceSet
    DEFAULT_TOLERANCES = _ToleranceSet()
    StageCost = _StageCost
    TerminalCost = _TerminalCost
    StageDynamics = _StageDynamics
    LqrProblem = _LqrProblem
    AffinePolicy = _AffinePolicy
    LqrSolution = _LqrSolution


def problem_from_arrays(a):
    """An ``LqrProblem`` (the active class) from one problem's stacked arrays
    (``synth`` layout: ``Qxx (T,n,n) ... f1 (T,n)``, ``QxxT``, ``qx1T``,
    ``x_init``)."""
    T = a["qx1"].shape[0]
    stages = [(StageCost(a["Qxx"][t], a["Qux"][t], a["Quu"][t], a["qx1"][t], a["qu1"][t]),
               StageDynamics(a["Fx"][t], a["Fu"][t], a["f1"][t])) for t in range(T)]
    return LqrProblem(stages, TerminalCost(a["QxxT"], a["qx1T"]), a["x_init"])
