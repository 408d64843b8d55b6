"""Seeded synthetic LQR instances following BASELINE.json's five configs.

This is input generation only (host, numpy); it is not on the solve path.
The recipe is BASELINE.json ``configs`` as interpreted in SURVEY.md
Appendix B:

* ``Fx = I + a*G`` with ``G ~ N(0, 1/n)``; ``Fu ~ N(0, 0.01/n)``;
  ``f1 ~ N(0, 0.01)`` (``N(0, v)`` has variance ``v``);
* ``Qxx = W W'/n + q_eps*I``; ``Quu = V V'/m + r_eps*I``; ``Qux = 0``;
* ``qx1, qu1 ~ N(0, 1)``; terminal ``Qxx_T`` from the ``Qxx`` recipe and
  ``qx1_T ~ N(0, 1)``; ``x_init ~ N(0, 1)``.

One ``numpy.random.default_rng(seed + i)`` per problem ``i``.  Draw order
(fixed, documented in DESIGN.md): ``G (T,n,n), Bu (T,n,m), c (T,n),
W (T,n,n), V (T,m,m), q (T,n), r (T,m), W_T (n,n), qT (n), x0 (n)``.
Quadratic blocks are symmetrized exactly once here, so the reference's
``StageCost`` symmetrization (``parlqr/problem.py:81-88``) is a no-op and
both solvers see byte-identical data.
"""

from __future__ import annotations

import dataclasses

import numpy as np

STAGE_FIELDS = ("Qxx", "Qux", "Quu", "qx1", "qu1", "Fx", "Fu", "f1")


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    B: int
    n: int
    m: int
    T: int
    J: int
    a_scale: float = 0.1
    q_eps: float = 1e-2
    r_eps: float = 1e-1

    @property
    def knots(self):
        return self.B * self.T

    def scaled(self, **kw):
        return dataclasses.replace(self, **kw)


CONFIGS = {
    0: Config("cfg0_n12_m4_T256_J4", 1, 12, 4, 256, 4),
    1: Config("cfg1_batch4096_n12_m4_T64_J8", 4096, 12, 4, 64, 8),
    2: Config("cfg2_n32_m8_T65536_J1024", 1, 32, 8, 65536, 1024),
    3: Config("cfg3_n128_m64_T4096_J256", 1, 128, 64, 4096, 256,
              q_eps=1e-3, r_eps=1e-3),
    4: Config("cfg4_batch256_n64_m32_T1024_J32", 256, 64, 32, 1024, 32,
              a_scale=0.5, r_eps=1e-4),
}


def _sym(a):
    return 0.5 * (a + np.swapaxes(a, -1, -2))


def generate_one(n, m, T, seed, a_scale=0.1, q_eps=1e-2, r_eps=1e-1):
    """One problem as a dict of stacked arrays (``(T, ...)`` per field)."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((T, n, n))
    Bu = rng.standard_normal((T, n, m))
    c = rng.standard_normal((T, n))
    W = rng.standard_normal((T, n, n))
    V = rng.standard_normal((T, m, m))
    q = rng.standard_normal((T, n))
    r = rng.standard_normal((T, m))
    WT = rng.standard_normal((n, n))
    qT = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    eye_n = np.eye(n)
    eye_m = np.eye(m)
    out = {
        "Fx": eye_n + a_scale * G / np.sqrt(n),
        "Fu": 0.1 * Bu / np.sqrt(n),
        "f1": 0.1 * c,
        "Qxx": _sym(W @ np.swapaxes(W, 1, 2) / n + q_eps * eye_n),
        "Qux": np.zeros((T, m, n)),
        "Quu": _sym(V @ np.swapaxes(V, 1, 2) / m + r_eps * eye_m),
        "qx1": q,
        "qu1": r,
        "QxxT": _sym(WT @ WT.T / n + q_eps * eye_n),
        "qx1T": qT,
        "x_init": x0,
    }
    return {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in out.items()}


def generate_batch(cfg, seed=0, count=None, first=0):
    """Problems ``first .. first+count-1`` of ``cfg`` stacked as ``(B, T, ...)``."""
    count = cfg.B if count is None else count
    probs = [generate_one(cfg.n, cfg.m, cfg.T, seed + first + i, cfg.a_scale,
                          cfg.q_eps, cfg.r_eps) for i in range(count)]
    return {k: np.ascontiguousarray(np.stack([p[k] for p in probs]))
            for k in probs[0]}


def batch_nbytes(cfg, B=None):
    B = cfg.B if B is None else B
    n, m, T = cfg.n, cfg.m, cfg.T
    per_stage = 8 * (2 * n * n + 2 * n * m + m * m + 2 * n + m)
    return B * (T * per_stage + 8 * (n * n + 2 * n))
