"""Problem / solution containers with the reference's field names and
conventions (parlqr/problem.py:44-280), so code written against ``parlqr``
runs unchanged.  Objects of the reference package itself are accepted too:
the solver only reads ``stages[t] = (cost, dynamics)``, ``terminal`` and
``x_init`` attributes.

Stage cost ``1/2 x'Qxx x + 1/2 u'Quu u + u'Qux x + qx1'x + qu1'u``, dynamics
``x' = Fx x + Fu u + f1``, terminal ``1/2 x'Qxx_T x + qx1_T'x``; multipliers
satisfy ``lam_t = -dV_t/dx`` (problem.py:1-17).
"""

from __future__ import annotations

import dataclasses

import numpy as np

__all__ = [
    "ToleranceSet", "DEFAULT_TOLERANCES", "StageCost", "TerminalCost",
    "StageDynamics", "LqrProblem", "AffinePolicy", "LqrSolution",
]


@dataclasses.dataclass(frozen=True)
class ToleranceSet:
    """Numerical thresholds (problem.py:44-58)."""

    rank_tol: float = 1e-10
    feas_tol: float = 1e-8
    kkt_tol: float = 1e-8


DEFAULT_TOLERANCES = ToleranceSet()


def _ro(a, shape=None, name="array"):
    arr = np.array(a, dtype=np.float64)
    if shape is not None and arr.shape != shape:
        raise ValueError(f"{name} must have shape {shape}, got {arr.shape}")
    arr.setflags(write=False)
    return arr


def _sym(a, name):
    arr = np.array(a, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise ValueError(f"{name} must be square, got shape {arr.shape}")
    amax = float(np.abs(arr).max()) if arr.size else 0.0
    defect = float(np.abs(arr - arr.T).max()) / amax if amax else 0.0
    out = 0.5 * (arr + arr.T)
    out.setflags(write=False)
    return out, defect


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class StageCost:
    """Quadratic stage cost; ``Qxx``/``Quu`` symmetrized on construction."""

    Qxx: np.ndarray
    Qux: np.ndarray
    Quu: np.ndarray
    qx1: np.ndarray
    qu1: np.ndarray
    asymmetry: float = 0.0

    def __init__(self, Qxx, Qux, Quu, qx1, qu1):
        Qxx, dx = _sym(Qxx, "Qxx")
        Quu, du = _sym(Quu, "Quu")
        n, m = Qxx.shape[0], Quu.shape[0]
        object.__setattr__(self, "Qxx", Qxx)
        object.__setattr__(self, "Quu", Quu)
        object.__setattr__(self, "Qux", _ro(Qux, (m, n), "Qux"))
        object.__setattr__(self, "qx1", _ro(qx1, (n,), "qx1"))
        object.__setattr__(self, "qu1", _ro(qu1, (m,), "qu1"))
        object.__setattr__(self, "asymmetry", max(dx, du))

    @property
    def n(self):
        return self.Qxx.shape[0]

    @property
    def m(self):
        return self.Quu.shape[0]


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class TerminalCost:
    Qxx: np.ndarray
    qx1: np.ndarray
    asymmetry: float = 0.0

    def __init__(self, Qxx, qx1):
        Qxx, d = _sym(Qxx, "terminal Qxx")
        object.__setattr__(self, "Qxx", Qxx)
        object.__setattr__(self, "qx1", _ro(qx1, (Qxx.shape[0],), "terminal qx1"))
        object.__setattr__(self, "asymmetry", d)

    @property
    def n(self):
        return self.Qxx.shape[0]

    @classmethod
    def zero(cls, n):
        return cls(np.zeros((n, n)), np.zeros(n))


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class StageDynamics:
    Fx: np.ndarray
    Fu: np.ndarray
    f1: np.ndarray

    def __init__(self, Fx, Fu, f1):
        Fx = np.array(Fx, dtype=np.float64)
        if Fx.ndim != 2 or Fx.shape[0] != Fx.shape[1]:
            raise ValueError(f"Fx must be square, got shape {Fx.shape}")
        n = Fx.shape[0]
        Fu = np.array(Fu, dtype=np.float64)
        if Fu.ndim != 2 or Fu.shape[0] != n:
            raise ValueError(f"Fu must have {n} rows, got shape {Fu.shape}")
        Fx.setflags(write=False)
        Fu.setflags(write=False)
        object.__setattr__(self, "Fx", Fx)
        object.__setattr__(self, "Fu", Fu)
        object.__setattr__(self, "f1", _ro(f1, (n,), "f1"))

    @property
    def n(self):
        return self.Fx.shape[0]

    @property
    def m(self):
        return self.Fu.shape[1]


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class LqrProblem:
    stages: tuple
    terminal: TerminalCost
    x_init: np.ndarray

    def __init__(self, stages, terminal, x_init):
        stages = tuple((c, d) for c, d in stages)
        if not stages:
            raise ValueError("horizon must contain at least one stage")
        n, m = stages[0][0].n, stages[0][0].m
        for t, (c, d) in enumerate(stages):
            if c.n != n or c.m != m or d.n != n or d.m != m:
                raise ValueError(f"inconsistent dimensions at stage {t}")
        if terminal.n != n:
            raise ValueError("terminal cost dimension mismatch")
        object.__setattr__(self, "stages", stages)
        object.__setattr__(self, "terminal", terminal)
        object.__setattr__(self, "x_init", _ro(x_init, (n,), "x_init"))

    @classmethod
    def from_arrays(cls, a):
        """Build from one problem's stacked arrays (``synth`` layout)."""
        T = a["qx1"].shape[0]
        stages = [(StageCost(a["Qxx"][t], a["Qux"][t], a["Quu"][t], a["qx1"][t], a["qu1"][t]),
                   StageDynamics(a["Fx"][t], a["Fu"][t], a["f1"][t])) for t in range(T)]
        return cls(stages, TerminalCost(a["QxxT"], a["qx1T"]), a["x_init"])

    @property
    def n(self):
        return self.stages[0][0].n

    @property
    def m(self):
        return self.stages[0][0].m

    @property
    def T(self):
        return len(self.stages)

    def __repr__(self):
        return f"LqrProblem(n={self.n}, m={self.m}, T={self.T})"


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class AffinePolicy:
    """``u = Kx x + Kz x_term + k1`` (problem.py:224-259)."""

    Kx: np.ndarray
    Kz: np.ndarray
    k1: np.ndarray

    def __init__(self, Kx, Kz, k1):
        Kx = np.array(Kx, dtype=np.float64)
        if Kx.ndim != 2:
            raise ValueError("Kx must be a matrix")
        m, n = Kx.shape
        Kx.setflags(write=False)
        object.__setattr__(self, "Kx", Kx)
        object.__setattr__(self, "Kz", _ro(Kz, (m, n), "Kz"))
        object.__setattr__(self, "k1", _ro(k1, (m,), "k1"))
        object.__setattr__(self, "_uses_terminal", bool(np.any(self.Kz)))

    @classmethod
    def state_feedback(cls, Kx, k1):
        Kx = np.asarray(Kx, dtype=np.float64)
        return cls(Kx, np.zeros_like(Kx), k1)

    def __call__(self, x, x_term=None):
        u = self.Kx @ x + self.k1
        if self._uses_terminal:
            if x_term is None:
                raise ValueError("policy depends on x_term but none was given")
            u = u + self.Kz @ x_term
        return u


@dataclasses.dataclass(frozen=True, eq=False, repr=False)
class LqrSolution:
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
