"""Seeded synthetic LQR instances following BASELINE.json's five configs.

This is input generation only (host, numpy); it is not on the solve path.
The recipe is BASELINE.json ``configs`` as interpreted in SURVEY.md
Appendix B:

* ``Fx = I + a*G`` with ``G ~ N(0, 1/n)``; ``Fu ~ N(0, 0.01/n)``;
  ``f1 ~ N(0, 0.01)`` (``N(0, v)`` has variance ``v``);
* ``Qxx = W W'/n + q_eps*I``; ``Quu = V V'/m + r_eps*I``; ``Qux = 0``;
* ``qx1, qu1 ~ N(0, 1)``; terminal ``Qxx_T`` from the ``Qxx`` recipe and
  ``qx1_T ~ N(0, 1)``; ``x_init ~ N(0, 1)``.

``cross > 0`` (not a BASELINE config: test data for the ``Qux`` paths of
the kernels) adds ``Qux = cross * N(0, 1)``, drawn after everything else and
halved until the control-eliminated state cost ``Qxx - Qux' Quu^-1 Qux`` is
PSD -- the shrink rule of the reference's generator (generate.py:27-32).

:func:`generate_reference_recipe` restates the reference's own generator
(``parlqr.generate``, generate.py:14-47) for the fuzz / cross-term tests.

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
    cross: float = 0.0

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


def _shrink_cross(Qxx, Quu, Qux):
    """Halve each stage's ``Qux`` until ``Qxx - Qux' Quu^-1 Qux`` is PSD
    (the acceptance loop of generate.py:29-32, applied stage-wise)."""
    for t in range(Qux.shape[0]):
        while np.linalg.eigvalsh(Qxx[t] - Qux[t].T @ np.linalg.solve(Quu[t], Qux[t])).min() < 0.0:
            Qux[t] *= 0.5
    return Qux


def generate_one(n, m, T, seed, a_scale=0.1, q_eps=1e-2, r_eps=1e-1, cross=0.0):
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
    if cross:
        Qux = cross * rng.standard_normal((T, m, n))
        out["Qux"] = _shrink_cross(out["Qxx"], out["Quu"], Qux)
    return {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in out.items()}


def generate_reference_recipe(n, m, T, seed):
    """The reference's random problem (``parlqr.generate``, generate.py:14-47)
    restated on stacked arrays: per stage ``Quu = B B' + I``, ``Qxx = C C'``,
    ``Qux = 0.3 N(0,1)`` halved until ``Qxx - Qux' Quu^-1 Qux`` is PSD,
    ``qx1, qu1 ~ N(0,1)``, ``Fx ~ N(0,1)`` rescaled to spectral radius
    <= 1.05, ``Fu, f1 ~ N(0,1)``; then terminal ``D D'``, ``qx1_T`` and
    ``x_init``.  Same draw order as the reference, so a given seed yields the
    reference's problem (up to the symmetrization of its constructors, which
    is applied here as well)."""
    if min(n, m, T) < 1:
        raise ValueError("n, m and T must all be at least 1")
    rng = np.random.default_rng(seed)
    f = {k: [] for k in STAGE_FIELDS}
    for _ in range(T):
        Bm = rng.standard_normal((m, m))
        Quu = Bm @ Bm.T + np.eye(m)
        C = rng.standard_normal((n, n))
        Qxx = C @ C.T
        Qux = 0.3 * rng.standard_normal((m, n))
        while np.linalg.eigvalsh(Qxx - Qux.T @ np.linalg.solve(Quu, Qux)).min() < 0.0:
            Qux = Qux * 0.5
        f["qx1"].append(rng.standard_normal(n))
        f["qu1"].append(rng.standard_normal(m))
        Fx = rng.standard_normal((n, n))
        rho = float(np.abs(np.linalg.eigvals(Fx)).max())
        if rho > 1.05:
            Fx = Fx * (1.05 / rho)
        f["Fx"].append(Fx)
        f["Fu"].append(rng.standard_normal((n, m)))
        f["f1"].append(rng.standard_normal(n))
        f["Qxx"].append(_sym(Qxx))
        f["Quu"].append(_sym(Quu))
        f["Qux"].append(Qux)
    D = rng.standard_normal((n, n))
    out = {k: np.stack(v) for k, v in f.items()}
    out["QxxT"] = _sym(D @ D.T)
    out["qx1T"] = rng.standard_normal(n)
    out["x_init"] = rng.standard_normal(n)
    return {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in out.items()}


def generate_batch(cfg, seed=0, count=None, first=0):
    """Problems ``first .. first+count-1`` of ``cfg`` stacked as ``(B, T, ...)``."""
    count = cfg.B if count is None else count
    probs = [generate_one(cfg.n, cfg.m, cfg.T, seed + first + i, cfg.a_scale,
                          cfg.q_eps, cfg.r_eps, cfg.cross) for i in range(count)]
    return {k: np.ascontiguousarray(np.stack([p[k] for p in probs]))
            for k in probs[0]}


def _fill_rows(args):
    cfg, seed, first, lo, hi = args
    for i in range(lo, hi):
        one = generate_one(cfg.n, cfg.m, cfg.T, seed + first + i, cfg.a_scale, cfg.q_eps, cfg.r_eps, cfg.cross)
        for k, v in one.items():
            _SHARED[k][i] = v
    return hi - lo


_SHARED = {}


def generate_batch_parallel(cfg, seed=0, count=None, first=0, workers=None):
    """:func:`generate_batch` with the problems drawn by a fork pool into one
    shared anonymous mapping (same bytes; cfg4's 28 GB batch takes seconds
    instead of minutes).  Returns numpy arrays backed by that mapping."""
    import mmap
    import multiprocessing
    import os
    count = cfg.B if count is None else count
    workers = workers or min(count, os.cpu_count() or 1)
    if workers <= 1 or count < 4:
        return generate_batch(cfg, seed, count, first)
    one = generate_one(cfg.n, cfg.m, 1, 0)
    shapes = {k: (count, cfg.T, *v.shape[1:]) if k in STAGE_FIELDS else (count, *v.shape)
              for k, v in one.items()}
    sizes = {k: 8 * int(np.prod(s)) for k, s in shapes.items()}
    buf = mmap.mmap(-1, sum(sizes.values()))
    off = 0
    out = {}
    for k, shp in shapes.items():
        out[k] = np.frombuffer(buf, dtype=np.float64, count=sizes[k] // 8, offset=off).reshape(shp)
        off += sizes[k]
    _SHARED.clear()
    _SHARED.update(out)
    step = -(-count // (4 * workers))
    chunks = [(cfg, seed, first, lo, min(count, lo + step)) for lo in range(0, count, step)]
    try:
        with multiprocessing.get_context("fork").Pool(workers) as pool:
            done = sum(pool.map(_fill_rows, chunks))
    finally:
        _SHARED.clear()
    assert done == count
    return out


def batch_nbytes(cfg, B=None):
    B = cfg.B if B is None else B
    n, m, T = cfg.n, cfg.m, cfg.T
    per_stage = 8 * (2 * n * n + 2 * n * m + m * m + 2 * n + m)
    return B * (T * per_stage + 8 * (n * n + 2 * n))


# ---------------------------------------------------------------------------
# device-side generator (plq_generate_batch) and the host restatement of its
# random stream

_FIELD_IDS = {"G": 0, "Bu": 1, "c": 2, "W": 3, "V": 4, "q": 5, "r": 6, "WT": 7, "qT": 8, "x0": 9}


def generate_batch_device(cfg, seed=0, count=None, first=0, device=None, out=None):
    """Problems ``first .. first+count-1`` of ``cfg``'s seeded family generated
    ON THE DEVICE (``plq_generate_batch``, csrc/plq_generate.cu): a dict of
    ``(B, T, ...)`` float64 CUDA tensors in the solver's input layout.  The
    family has the distributions of :func:`generate_one` (BASELINE.json recipe,
    ``Qux = 0``) but its own counter-based stream (Philox-4x32-10 + Box-Muller,
    restated in :func:`device_stream_reference`), so the values differ from the
    numpy generator's for the same seed.  ``out``: tensors to fill in place."""
    import ctypes

    import torch

    from . import _native
    if cfg.cross:
        raise ValueError("the device generator has no cross term (BASELINE recipe: Qux = 0)")
    count = cfg.B if count is None else count
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    n, m, T = cfg.n, cfg.m, cfg.T
    shapes = {"Qxx": (count, T, n, n), "Qux": (count, T, m, n), "Quu": (count, T, m, m), "qx1": (count, T, n),
              "qu1": (count, T, m), "Fx": (count, T, n, n), "Fu": (count, T, n, m), "f1": (count, T, n),
              "QxxT": (count, n, n), "qx1T": (count, n), "x_init": (count, n)}
    if out is None:
        out = {k: torch.empty(s, dtype=torch.float64, device=dev) for k, s in shapes.items()}
    P = _native.PlqProblem()
    P.B, P.T, P.n, P.m, P.J, P.max_seg_len = count, T, n, m, 1, T
    for k, s in shapes.items():
        t = out[k]
        if tuple(t.shape) != s or t.dtype != torch.float64 or not t.is_contiguous() or not t.is_cuda:
            raise ValueError(f"{k}: expected a contiguous float64 CUDA tensor of shape {s}")
        setattr(P, k, ctypes.c_void_p(t.data_ptr()))
    R = _native.PlqRecipe(cfg.a_scale, cfg.q_eps, cfg.r_eps, int(seed) & (2 ** 64 - 1), int(first))
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        rc = _native.lib().plq_generate_batch(ctypes.byref(P), ctypes.byref(R), ctypes.c_void_p(stream.cuda_stream))
    _native.check(rc, "plq_generate_batch")
    return out


def _philox4x32_10(c0, c1, c2, c3, k0, k1):
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    mask = np.uint64(0xFFFFFFFF)
    c = [np.asarray(x, dtype=np.uint64) & mask for x in (c0, c1, c2, c3)]
    k0, k1 = np.uint64(k0), np.uint64(k1)
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        hi0, lo0, hi1, lo1 = p0 >> np.uint64(32), p0 & mask, p1 >> np.uint64(32), p1 & mask
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + np.uint64(0x9E3779B9)) & mask
        k1 = (k1 + np.uint64(0xBB67AE85)) & mask
    return c


def _device_normals(seed, problem, field, count):
    """The first ``count`` standard normals of (seed, problem, field) in the
    device generator's stream (csrc/plq_generate.cu: normal_at)."""
    e = np.arange(count, dtype=np.uint64)
    k = e >> np.uint64(1)
    seed = int(seed) & (2 ** 64 - 1)
    w = _philox4x32_10(k & np.uint64(0xFFFFFFFF), k >> np.uint64(32), np.full(count, _FIELD_IDS[field], np.uint64),
                       np.full(count, problem, np.uint64), seed & 0xFFFFFFFF, seed >> 32)
    u0 = (w[0] >> np.uint64(5)).astype(np.float64) / 134217728.0 + (w[1] >> np.uint64(6)).astype(np.float64) / 9007199254740992.0
    u1 = (w[2] >> np.uint64(5)).astype(np.float64) / 134217728.0 + (w[3] >> np.uint64(6)).astype(np.float64) / 9007199254740992.0
    r = np.sqrt(-2.0 * np.log(1.0 - u0))
    return np.where(e & np.uint64(1), r * np.sin(2.0 * np.pi * u1), r * np.cos(2.0 * np.pi * u1))


def device_stream_reference(cfg, seed=0, problem=0):
    """Host (numpy) restatement of ONE problem of the device generator's
    family: same Philox counters, Box-Muller pairing and recipe, so the
    device output can be checked to rounding (libm vs CUDA ``log`` /
    ``sincospi`` differ in the last bits).  Test infrastructure."""
    n, m, T = cfg.n, cfg.m, cfg.T
    nrm = lambda f, shape: _device_normals(seed, problem, f, int(np.prod(shape))).reshape(shape)  # noqa: E731
    G, Bu, c = nrm("G", (T, n, n)), nrm("Bu", (T, n, m)), nrm("c", (T, n))
    W, V = nrm("W", (T, n, n)), nrm("V", (T, m, m))
    WT = nrm("WT", (n, n))
    return {
        "Fx": np.eye(n) + (cfg.a_scale / np.sqrt(n)) * G,
        "Fu": (0.1 / np.sqrt(n)) * Bu,
        "f1": 0.1 * c,
        "Qxx": W @ np.swapaxes(W, 1, 2) / n + cfg.q_eps * np.eye(n),
        "Qux": np.zeros((T, m, n)),
        "Quu": V @ np.swapaxes(V, 1, 2) / m + cfg.r_eps * np.eye(m),
        "qx1": nrm("q", (T, n)),
        "qu1": nrm("r", (T, m)),
        "QxxT": WT @ WT.T / n + cfg.q_eps * np.eye(n),
        "qx1T": nrm("qT", (n,)),
        "x_init": nrm("x0", (n,)),
    }
