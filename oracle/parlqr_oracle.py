"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's horizon-partitioned Riccati
solve (``parlqr.solve_parallel``, ``/root/reference/pkg/src/parlqr``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path (``paper_1809_06360_b200``) never
imports it and has no CPU fallback.

Parity of this restatement is pinned against outputs of the reference itself
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src`` in the
build container and writes ``tests/golden/*.npz``; ``tests/test_oracle.py``
checks this module against them).

Layout: one problem is a dict of stacked float64 arrays, the reference's own
transport layout (``parallel.py:108,141-149``): ``Qxx (T,n,n) Qux (T,m,n)
Quu (T,m,m) qx1 (T,n) qu1 (T,m) Fx (T,n,n) Fu (T,n,m) f1 (T,n)`` plus
``QxxT (n,n) qx1T (n) x_init (n)``.
"""

from __future__ import annotations

import concurrent.futures
import multiprocessing
import os

import numpy as np
import scipy.linalg

STAGE_FIELDS = ("Qxx", "Qux", "Quu", "qx1", "qu1", "Fx", "Fu", "f1")
RANK_TOL = 1e-10      # problem.py:53 ToleranceSet.rank_tol
FEAS_TOL = 1e-8       # problem.py:54 ToleranceSet.feas_tol


class OracleCholeskyFailure(Exception):
    """errors.py:8-13 -- stage index is segment-local (endpoint.py:243-245)."""

    def __init__(self, stage):
        self.stage = stage
        super().__init__(f"Cholesky failed at stage {stage}")


class OracleLinkSingular(Exception):
    """errors.py:29-30 (raised from parallel.py:267-271)."""


class OracleDegenerate(Exception):
    """Segment left feasibility rows (parallel.py:452-456); the GPU path
    raises for these partitions, so the oracle does too."""


def make_partition(T, J):
    """Balanced split, remainder to early segments (parallel.py:82-94)."""
    if not 1 <= J <= T:
        raise ValueError(f"J must be in [1, {T}], got {J}")
    base, extra = divmod(T, J)
    splits = [0]
    for j in range(J):
        splits.append(splits[-1] + base + (1 if j < extra else 0))
    return tuple(splits)


def _compress(Hx, Hz, h1, rank_tol, scale, cert_scale):
    """Row compression + infeasibility certificate (endpoint.py:130-165)."""
    r = Hx.shape[0]
    if r == 0:
        return Hx, Hz, h1
    U, s, _ = np.linalg.svd(np.concatenate([Hx, Hz], axis=1),
                            full_matrices=False)
    thr = rank_tol * max(scale, s[0] if s.size else 0.0)
    q = int(np.sum(s > thr))
    if q == r:
        return Hx, Hz, h1
    n = Hx.shape[1]
    if q:
        Uq = U[:, :q]
        body = Uq.T @ np.concatenate([Hx, Hz, h1[:, None]], axis=1)
        nHx, nHz, nh1 = body[:, :n], body[:, n:2 * n], body[:, 2 * n]
        rest = h1 - Uq @ (Uq.T @ h1)
    else:
        nHx, nHz, nh1 = np.zeros((0, n)), np.zeros((0, n)), np.zeros(0)
        rest = h1
    res = float(np.linalg.norm(rest))
    if res > rank_tol * cert_scale:
        nHx = np.concatenate([nHx, np.zeros((1, n))], axis=0)
        nHz = np.concatenate([nHz, np.zeros((1, n))], axis=0)
        nh1 = np.concatenate([nh1, [res]])
    return nHx, nHz, nh1


def endpoint_sweep(st, rank_tol=RANK_TOL, QxxT=None, qx1T=None):
    """Endpoint-explicit backward sweep of one segment with terminal rows
    ``Hx=I, Hz=-I`` and zero terminal cost (endpoint.py:168-301 as called by
    parallel.py:228-229) -- or the terminal cost ``(QxxT, qx1T)`` when given
    (backward_pass(stages, terminal), endpoint.py:178-184, as called by
    solve_endpoint[_affine], :618-619, :640).  Returns per-stage ``Kx, Kz,
    k1`` and the start blocks ``vf0 = (Vxx, Vzx, Vzz, vx1, vz1)`` and
    feasibility rows.
    """
    L, n = st["qx1"].shape
    m = st["qu1"].shape[1]
    Vxx = np.zeros((n, n)) if QxxT is None else 0.5 * (QxxT + QxxT.T)
    vx1 = np.zeros(n) if qx1T is None else np.array(qx1T, dtype=float)
    Vzx = np.zeros((n, n))
    Vzz = np.zeros((n, n))
    vz1 = np.zeros(n)
    Hx, Hz, h1 = np.eye(n), -np.eye(n), np.zeros(n)
    Kx_all = np.empty((L, m, n))
    Kz_all = np.empty((L, m, n))
    k1_all = np.empty((L, m))
    eye_m = np.eye(m)
    # StageDiagnostics (endpoint.py:108-115, 200): worst defects, largest row count
    diag = {"basis_defect": 0.0, "projector_defect": 0.0, "max_rows": int(Hx.shape[0])}
    for t in range(L - 1, -1, -1):
        Fx, Fu, f1 = st["Fx"][t], st["Fu"][t], st["f1"][t]
        # M-terms (endpoint.py:206-217)
        VFx = Vxx @ Fx
        VFu = Vxx @ Fu
        w = vx1 + Vxx @ f1
        Mxx = st["Qxx"][t] + Fx.T @ VFx
        Muu = st["Quu"][t] + Fu.T @ VFu
        Mux = st["Qux"][t] + Fu.T @ VFx
        Mzx = Vzx @ Fx
        Mzu = Vzx @ Fu
        mx1 = st["qx1"][t] + Fx.T @ w
        mu1 = st["qu1"][t] + Fu.T @ w
        mz1 = vz1 + Vzx @ f1
        # constraint-to-go and its rank (endpoint.py:219-231)
        r = Hx.shape[0]
        p = 0
        if r:
            Nx = Hx @ Fx
            Nu = Hx @ Fu
            Nz = Hz
            n1 = Hx @ f1 + h1
            U, s, Vt = np.linalg.svd(Nu)
            nu_scale = float(np.linalg.norm(Hx)) * float(np.linalg.norm(Fu))
            if s.size:
                p = int(np.sum(s > rank_tol * max(nu_scale, s[0])))
        # gains [Kx|Kz|k1]: range-space move + null-space Cholesky
        # (endpoint.py:233-256)
        if p:
            stack = np.concatenate([Nx, Nz, n1[:, None]], axis=1)
            base = ((Vt[:p].T / s[:p]) @ U[:, :p].T) @ stack
        else:
            base = np.zeros((m, 2 * n + 1))
        if p < m:
            Zw = Vt[p:].T if p else eye_m
            Wn = Zw.T @ Muu @ Zw
            try:
                Lw = np.linalg.cholesky(Wn)
            except np.linalg.LinAlgError:
                raise OracleCholeskyFailure(t) from None
            C = np.concatenate([Mux, Mzu.T, mu1[:, None]], axis=1)
            if p:
                C = C - Muu @ base
            G = -(base + Zw @ scipy.linalg.cho_solve((Lw, True), Zw.T @ C,
                                                     check_finite=False))
        else:
            G = -base
        Kx, Kz, k1 = G[:, :n], G[:, n:2 * n], G[:, 2 * n]
        Kx_all[t], Kz_all[t], k1_all[t] = Kx, Kz, k1
        if p:   # endpoint.py:258-265, 275-277
            Zfull = Vt[p:].T if p < m else np.zeros((m, 0))
            comp = Vt[:p].T @ Vt[:p] + Zfull @ Zfull.T - eye_m
            diag["basis_defect"] = max(diag["basis_defect"], float(np.abs(comp).max()))
            Pr = np.eye(r) - U[:, :p] @ U[:, :p].T
            diag["projector_defect"] = max(diag["projector_defect"], float(np.abs(Pr @ Pr - Pr).max()))
        # constraint projection + compression (endpoint.py:267-281)
        if r:
            pre = float(np.linalg.norm(np.concatenate([Nx, Nz], axis=1)))
            cert = max(1.0, float(np.abs(n1).max(initial=0.0)))
            if p:
                Up = U[:, :p]
                stk = np.concatenate([Nx, Nz, n1[:, None]], axis=1)
                stk = stk - Up @ (Up.T @ stk)
                Hx, Hz, h1 = stk[:, :n], stk[:, n:2 * n], stk[:, 2 * n]
            else:
                Hx, Hz, h1 = Nx, Nz, n1
            Hx, Hz, h1 = _compress(Hx, Hz, h1, rank_tol, pre, cert)
        # value update (endpoint.py:285-294)
        MuuKx = Muu @ Kx
        MuuKz = Muu @ Kz
        MuxTKx = Mux.T @ Kx
        Vxx = Mxx + MuxTKx + MuxTKx.T + Kx.T @ MuuKx
        Vxx = 0.5 * (Vxx + Vxx.T)
        Vzx_new = Mzx + Mzu @ Kx + Kz.T @ Mux + Kz.T @ MuuKx
        Vzz = Vzz + Mzu @ Kz + (Mzu @ Kz).T + Kz.T @ MuuKz
        Vzz = 0.5 * (Vzz + Vzz.T)
        vx1 = mx1 + Kx.T @ mu1 + (Mux.T + Kx.T @ Muu) @ k1
        vz1 = mz1 + Mzu @ k1 + Kz.T @ mu1 + Kz.T @ (Muu @ k1)
        Vzx = Vzx_new
        diag["max_rows"] = max(diag["max_rows"], int(Hx.shape[0]))   # endpoint.py:298-299
    return {"Kx": Kx_all, "Kz": Kz_all, "k1": k1_all,
            "vf0": (Vxx, Vzx, Vzz, vx1, vz1), "feas": (Hx, Hz, h1), "diagnostics": diag}


def serial_sweep(st, QxxT, qx1T):
    """Plain Riccati sweep of the last segment (serial.py:37-79)."""
    L, n = st["qx1"].shape
    m = st["qu1"].shape[1]
    Vxx, vx1 = QxxT, qx1T
    Kx_all = np.empty((L, m, n))
    k1_all = np.empty((L, m))
    for t in range(L - 1, -1, -1):
        Fx, Fu, f1 = st["Fx"][t], st["Fu"][t], st["f1"][t]
        VFx = Vxx @ Fx
        VFu = Vxx @ Fu
        w = vx1 + Vxx @ f1
        Mxx = st["Qxx"][t] + Fx.T @ VFx
        Muu = st["Quu"][t] + Fu.T @ VFu
        Mux = st["Qux"][t] + Fu.T @ VFx
        mx1 = st["qx1"][t] + Fx.T @ w
        mu1 = st["qu1"][t] + Fu.T @ w
        try:
            Lc = np.linalg.cholesky(Muu)
        except np.linalg.LinAlgError:
            raise OracleCholeskyFailure(t) from None
        G = -scipy.linalg.cho_solve((Lc, True), np.column_stack([Mux, mu1]),
                                    check_finite=False)
        Kx, k1 = G[:, :-1], G[:, -1]
        Kx_all[t], k1_all[t] = Kx, k1
        Vxx = Mxx + Mux.T @ Kx + Kx.T @ Mux + Kx.T @ (Muu @ Kx)
        Vxx = 0.5 * (Vxx + Vxx.T)
        vx1 = mx1 + Kx.T @ mu1 + (Mux.T + Kx.T @ Muu) @ k1
    return {"Kx": Kx_all, "k1": k1_all, "vf0": (Vxx, vx1)}


def block_tridiagonal_solve(D, S, b):
    """SPD block-tridiagonal solve by block Cholesky without inter-block
    pivoting (endpoint.py:410-438).  ``S[i]`` couples row ``i+1`` to ``i``."""
    K = len(D)
    X = [None] * K
    d = [None] * K
    P = D[0]
    for i in range(K):
        if i:
            P = D[i] - S[i - 1] @ X[i - 1]
        try:
            Lc = np.linalg.cholesky(P)
        except np.linalg.LinAlgError:
            raise OracleLinkSingular(f"singular pivot block {i}") from None
        g = b[i] if not i else b[i] - S[i - 1] @ d[i - 1]
        d[i] = scipy.linalg.cho_solve((Lc, True), g, check_finite=False)
        if i < K - 1:
            X[i] = scipy.linalg.cho_solve((Lc, True), S[i].T,
                                          check_finite=False)
    out = [None] * K
    out[K - 1] = d[K - 1]
    for i in range(K - 2, -1, -1):
        out[i] = d[i] - X[i] @ out[i + 1]
    return np.array(out)


# ---------------------------------------------------------------------------
# two-point-boundary solve (endpoint.py:303-653)

class OracleFactorizationFailure(Exception):
    """errors.py FactorizationFailure(block) from the multiplier Gram system."""

    def __init__(self, block):
        super().__init__(f"factorization failed at block {block}")
        self.block = block


def forward_maps(st, Kx, Kz, k1):
    """forward_pass (endpoint.py:326-349): states / controls as affine maps
    of (x_init, x_term), packed ``X[t] = [Ra | Rz | r1]`` (T+1, n, 2n+1) and
    ``S[t] = [Sa | Sz | s1]`` (T, m, 2n+1)."""
    T, n = st["qx1"].shape
    m = st["qu1"].shape[1]
    W = 2 * n + 1
    X = np.empty((T + 1, n, W))
    S = np.empty((T, m, W))
    X[0] = 0.0
    X[0, :, :n] = np.eye(n)
    for t in range(T):
        S[t, :, :n] = Kx[t] @ X[t, :, :n]
        S[t, :, n:2 * n] = Kx[t] @ X[t, :, n:2 * n] + Kz[t]
        S[t, :, 2 * n] = Kx[t] @ X[t, :, 2 * n] + k1[t]
        Fx, Fu = st["Fx"][t], st["Fu"][t]
        X[t + 1, :, :n] = Fx @ X[t, :, :n] + Fu @ S[t, :, :n]
        X[t + 1, :, n:2 * n] = Fx @ X[t, :, n:2 * n] + Fu @ S[t, :, n:2 * n]
        X[t + 1, :, 2 * n] = Fx @ X[t, :, 2 * n] + Fu @ S[t, :, 2 * n] + st["f1"][t]
    return X, S


def multiplier_maps(st, QxxT, qx1T, X, S):
    """assemble_normal_equations + multiplier_pass (endpoint.py:370-476):
    the (T+2)-block Gram system over ``lam_0..lam_T, mu`` with a (2n+1)-wide
    affine right-hand side, solved by block Cholesky.  Returns ``Lam`` (T+1,
    n, 2n+1) and ``E`` (n, 2n+1)."""
    T, n = st["qx1"].shape
    m = st["qu1"].shape[1]
    W = 2 * n + 1
    bx = np.empty((T + 1, n, W))
    bu = np.empty((T, m, W))
    for t in range(T):
        bx[t] = -(st["Qxx"][t] @ X[t] + st["Qux"][t].T @ S[t])
        bx[t, :, -1] -= st["qx1"][t]
        bu[t] = -(st["Qux"][t] @ X[t] + st["Quu"][t] @ S[t])
        bu[t, :, -1] -= st["qu1"][t]
    QT = 0.5 * (QxxT + QxxT.T)
    bx[T] = -(QT @ X[T])
    bx[T, :, -1] -= qx1T
    eye = np.eye(n)
    D = np.empty((T + 2, n, n))
    Sb = np.empty((T + 1, n, n))
    rhs = np.empty((T + 2, n, W))
    D[0] = eye
    D[T + 1] = eye
    rhs[0] = bx[0]
    for t in range(T):
        Fx, Fu = st["Fx"][t], st["Fu"][t]
        D[t + 1] = eye + Fx @ Fx.T + Fu @ Fu.T
        Sb[t] = -Fx
        rhs[t + 1] = -Fx @ bx[t] - Fu @ bu[t] + bx[t + 1]
    Sb[T] = eye
    rhs[T + 1] = bx[T]
    try:
        sol = block_tridiagonal_solve(D, Sb, rhs)
    except OracleLinkSingular as exc:
        raise OracleFactorizationFailure(int(str(exc).split()[-1])) from None
    return sol[:-1], sol[-1]


def full_kkt_residual(prob, states, controls, lambdas, mu, x_term):
    """kkt_residual with an endpoint constraint (problem.py:385-420): every
    stationarity, dynamics, terminal (+mu), initial and endpoint row."""
    worst = 0.0
    for t in range(controls.shape[0]):
        x, u = states[t], controls[t]
        Fx, Fu = prob["Fx"][t], prob["Fu"][t]
        r1 = prob["Qxx"][t] @ x + prob["Qux"][t].T @ u + prob["qx1"][t] + lambdas[t] - Fx.T @ lambdas[t + 1]
        r2 = prob["Qux"][t] @ x + prob["Quu"][t] @ u + prob["qu1"][t] - Fu.T @ lambdas[t + 1]
        r3 = states[t + 1] - (Fx @ x + Fu @ u + prob["f1"][t])
        worst = max(worst, float(np.abs(r1).max()), float(np.abs(r2).max()), float(np.abs(r3).max()))
    term = prob["QxxT"] @ states[-1] + prob["qx1T"] + lambdas[-1] + mu
    return max(worst, float(np.abs(term).max()), float(np.abs(states[0] - prob["x_init"]).max()),
               float(np.abs(states[-1] - x_term).max()))


def solve_endpoint_affine(prob, rank_tol=RANK_TOL):
    """solve_endpoint_affine (endpoint.py:589-620).  With feasibility rows
    left at t = 0 (unreachable endpoint directions) the boundary constraints
    are linearly dependent and no multiplier maps are computed (``Lam``/``E``
    absent); ``feas`` holds the rows."""
    st = {f: np.asarray(prob[f]) for f in STAGE_FIELDS}
    sw = endpoint_sweep(st, rank_tol, prob["QxxT"], prob["qx1T"])
    X, S = forward_maps(st, sw["Kx"], sw["Kz"], sw["k1"])
    out = {"Kx": sw["Kx"], "Kz": sw["Kz"], "k1": sw["k1"], "vf0": sw["vf0"], "X": X, "S": S,
           "feas": sw["feas"]}
    if sw["feas"][0].shape[0] == 0:
        out["Lam"], out["E"] = multiplier_maps(st, prob["QxxT"], prob["qx1T"], X, S)
    return out


def gradient_duals(prob, vf0, states, controls, x_init, x_term):
    """Multipliers from the value-function gradient and the backward
    stationarity recursion (endpoint.py:566-587)."""
    Vxx, Vzx, Vzz, vx1, vz1 = vf0
    mu = -(Vzx @ x_init + Vzz @ x_term + vz1)
    T, n = controls.shape[0], states.shape[1]
    lambdas = np.empty((T + 1, n))
    lambdas[T] = -(prob["QxxT"] @ states[T] + prob["qx1T"]) - mu
    for t in range(T - 1, -1, -1):
        lambdas[t] = prob["Fx"][t].T @ lambdas[t + 1] - (
            prob["Qxx"][t] @ states[t] + prob["Qux"][t].T @ controls[t] + prob["qx1"][t])
    return lambdas, mu


def evaluate_endpoint(prob, aff, x_init, x_term):
    """EndpointAffineSolution.evaluate (endpoint.py:507-546): states,
    controls, lambdas, mu, objective, full KKT residual, and the residual of
    the feasibility rows at the endpoint pair; multipliers from the maps, or
    from :func:`gradient_duals` when there are none."""
    x_init = np.asarray(x_init, dtype=float)
    x_term = np.asarray(x_term, dtype=float)
    v = np.concatenate([x_init, x_term, [1.0]])
    states = aff["X"] @ v
    controls = aff["S"] @ v
    Hx, Hz, h1 = aff["feas"]
    res = Hx @ x_init + Hz @ x_term + h1
    if "Lam" in aff:
        lambdas = aff["Lam"] @ v
        mu = aff["E"] @ v
    else:
        lambdas, mu = gradient_duals(prob, aff["vf0"], states, controls, x_init, x_term)
    p = dict(prob)
    p["x_init"] = x_init
    return {"states": states, "controls": controls, "lambdas": lambdas, "mu": mu,
            "objective": objective(p, states, controls),
            "kkt": full_kkt_residual(p, states, controls, lambdas, mu, x_term),
            "feas_residual": float(np.abs(res).max()) if res.size else 0.0}


def link_system(vf0, x_init):
    """Multiplier-matching system over the J-1 links (parallel.py:286-319),
    returned in the reference's sign convention ``diag, sub, rhs`` with
    ``sub[k-1] l_{k-1} + diag[k] l_k + sub[k]' l_{k+1} + rhs[k] = 0``."""
    J = len(vf0)
    n = x_init.shape[0]
    diag = np.empty((J - 1, n, n))
    sub = np.empty((J - 2, n, n)) if J > 2 else np.zeros((0, n, n))
    rhs = np.empty((J - 1, n))
    for k in range(1, J):
        right = vf0[k]
        if len(right) == 2:            # serial (last) segment: (Vxx, vx1)
            La_r, l1_r = -right[0], -right[1]
        else:
            La_r, l1_r = -right[0], -right[3]
        _, Vzx_l, Vzz_l, _, vz1_l = vf0[k - 1]
        diag[k - 1] = -Vzz_l + La_r
        rhs[k - 1] = -vz1_l + l1_r
        if k == 1:
            rhs[k - 1] += -Vzx_l @ x_init
        else:
            sub[k - 2] = -Vzx_l
    return diag, sub, rhs


def solve_links(diag, sub, rhs):
    """LinkSystem.solve (parallel.py:264-283): links and max residual."""
    links = block_tridiagonal_solve(-diag, -sub, rhs[:, :, None])[:, :, 0]
    K = len(diag)
    worst = 0.0
    for k in range(K):
        r = diag[k] @ links[k] + rhs[k]
        if k:
            r = r + sub[k - 1] @ links[k - 1]
        if k < K - 1:
            r = r + sub[k].T @ links[k + 1]
        worst = max(worst, float(np.abs(r).max()))
    return links, worst


def objective(prob, states, controls):
    """evaluate_objective (problem.py:366-382)."""
    total = 0.0
    for t in range(controls.shape[0]):
        x, u = states[t], controls[t]
        total += 0.5 * (x @ (prob["Qxx"][t] @ x)) + 0.5 * (u @ (prob["Quu"][t] @ u))
        total += u @ (prob["Qux"][t] @ x) + prob["qx1"][t] @ x + prob["qu1"][t] @ u
    xT = states[-1]
    total += 0.5 * (xT @ (prob["QxxT"] @ xT)) + prob["qx1T"] @ xT
    return float(total)


def kkt_residual(prob, states, controls, lambdas):
    """Infinity norm of stationarity + dynamics + initial residuals
    (problem.py:385-420 with mu=None, x_term=None)."""
    worst = 0.0
    for t in range(controls.shape[0]):
        x, u = states[t], controls[t]
        lam, lam_next = lambdas[t], lambdas[t + 1]
        Fx, Fu = prob["Fx"][t], prob["Fu"][t]
        r1 = prob["Qxx"][t] @ x + prob["Qux"][t].T @ u + prob["qx1"][t] + lam - Fx.T @ lam_next
        r2 = prob["Qux"][t] @ x + prob["Quu"][t] @ u + prob["qu1"][t] - Fu.T @ lam_next
        r3 = states[t + 1] - (Fx @ x + Fu @ u + prob["f1"][t])
        worst = max(worst, float(np.abs(r1).max()), float(np.abs(r2).max()),
                    float(np.abs(r3).max()))
    term = prob["QxxT"] @ states[-1] + prob["qx1T"] + lambdas[-1]
    worst = max(worst, float(np.abs(term).max()),
                float(np.abs(states[0] - prob["x_init"]).max()))
    return worst


def _segment_task(args):
    kind, st, QxxT, qx1T, rank_tol = args
    if kind == "serial":
        return serial_sweep(st, QxxT, qx1T)
    return endpoint_sweep(st, rank_tol)


_POOLS = {}


def _pool(workers):
    pool = _POOLS.get(workers)
    if pool is None:
        pool = concurrent.futures.ProcessPoolExecutor(
            max_workers=workers, mp_context=multiprocessing.get_context("fork"))
        _POOLS[workers] = pool
    return pool


def sweep_segments(prob, splits, rank_tol=RANK_TOL, workers=1):
    """Per-segment sweeps (parallel.py:408-419, 197-240): endpoint kind for
    every segment but the last, which keeps the terminal cost."""
    J = len(splits) - 1
    tasks = []
    for j in range(J):
        lo, hi = splits[j], splits[j + 1]
        st = {f: np.array(prob[f][lo:hi]) for f in STAGE_FIELDS}
        kind = "serial" if j == J - 1 else "endpoint"
        tasks.append((kind, st, prob["QxxT"], prob["qx1T"], rank_tol))
    if workers > 1 and J > 1:
        return list(_pool(workers).map(_segment_task, tasks))
    return [_segment_task(t) for t in tasks]


def solve(prob, J=None, splits=None, rank_tol=RANK_TOL, workers=1):
    """Restatement of ``solve_parallel`` (parallel.py:422-553) for J >= 2.

    Returns a dict with the reference's outputs plus the unfolded per-stage
    segment gains (``Kz``, ``k1``) for kernel-level parity checks.
    """
    T, n = prob["qx1"].shape
    m = prob["qu1"].shape[1]
    if splits is None:
        splits = make_partition(T, J)
    J = len(splits) - 1
    if J < 2:
        raise ValueError("the oracle restates the J >= 2 partitioned path")
    segs = sweep_segments(prob, splits, rank_tol, workers)
    for j, seg in enumerate(segs[:-1]):
        if seg["feas"][0].shape[0]:
            raise OracleDegenerate(f"segment {j} keeps {seg['feas'][0].shape[0]} rows")
    vf0 = [s["vf0"] for s in segs]
    x_init = prob["x_init"]
    diag, sub, rhs = link_system(vf0, x_init)
    links, link_res = solve_links(diag, sub, rhs)

    states = np.empty((T + 1, n))
    controls = np.empty((T, m))
    lambdas = np.empty((T + 1, n))
    K = np.empty((T, m, n))
    k = np.empty((T, m))
    Kz = np.zeros((T, m, n))
    k1u = np.empty((T, m))
    mu_left = np.empty((J - 1, n))
    lambda_right = np.empty((J - 1, n))
    # reconstruction (parallel.py:485-525), segment by segment
    for j, seg in enumerate(segs):
        lo, hi = splits[j], splits[j + 1]
        r = reconstruct_segment(prob, splits, j, seg, links)
        K[lo:hi] = seg["Kx"]
        k[lo:hi] = r["fold"]
        k1u[lo:hi] = seg["k1"]
        if "Kz" in seg:
            Kz[lo:hi] = seg["Kz"]
        controls[lo:hi] = r["us"]
        states[lo:hi] = r["xs"][:-1]
        lambdas[lo:hi] = r["lam"]
        if j == J - 1:
            states[T] = r["xs"][-1]
            lambdas[T] = r["lam_T"]
        else:
            mu_left[j] = r["mu"]
        if j:
            lambda_right[j - 1] = r["lam"][0]
    mismatch = float(np.abs(mu_left + lambda_right).max())
    return {
        "states": states, "controls": controls, "lambdas": lambdas,
        "K": K, "k": k, "Kz": Kz, "k1": k1u,
        "links": links, "link_residual": link_res,
        "mu_left": mu_left, "lambda_right": lambda_right,
        "link_mismatch": mismatch, "vf0": vf0,
        "objective": objective(prob, states, controls),
        "kkt": kkt_residual(prob, states, controls, lambdas),
        "splits": tuple(splits),
    }


def reconstruct_segment(prob, splits, j, seg, links):
    """The reconstruction of one segment (parallel.py:485-525): fold
    ``k = Kz z + k1`` (:495), rollout (:498-502), multiplier seed (:505-515)
    and backward multiplier recursion (:518-523).  Returns the segment's
    rollout ``xs`` (L+1 states, the last one the rollout end), ``us``,
    ``fold``, multipliers ``lam`` at stages lo..hi-1 and the seed values."""
    J = len(splits) - 1
    lo, hi = splits[j], splits[j + 1]
    n = prob["x_init"].shape[0]
    m = prob["qu1"].shape[1]
    a = prob["x_init"] if j == 0 else links[j - 1]
    last = j == J - 1
    if last:
        fold = seg["k1"]
    else:
        z = links[j]
        fold = seg["Kz"] @ z + seg["k1"]
    xs = np.empty((hi - lo + 1, n))
    us = np.empty((hi - lo, m))
    xs[0] = a
    for s in range(hi - lo):
        us[s] = seg["Kx"][s] @ xs[s] + fold[s]
        xs[s + 1] = prob["Fx"][lo + s] @ xs[s] + prob["Fu"][lo + s] @ us[s] + prob["f1"][lo + s]
    out = {"xs": xs, "us": us, "fold": fold}
    if last:
        lam = -(prob["QxxT"] @ xs[-1] + prob["qx1T"])
        out["lam_T"] = lam
    else:
        Vxx0, Vzx0, Vzz0, vx10, vz10 = seg["vf0"]
        mu = -(Vzx0 @ a + Vzz0 @ z + vz10)
        out["mu"] = mu
        lam = -mu
    lams = np.empty((hi - lo, n))
    for s in range(hi - lo - 1, -1, -1):
        t = lo + s
        lam = prob["Fx"][t].T @ lam - (prob["Qxx"][t] @ xs[s] + prob["Qux"][t].T @ us[s] + prob["qx1"][t])
        lams[s] = lam
    out["lam"] = lams
    return out


def smooth(prob, sol, workers=1):
    """Second pass trading endpoint constraints for conditioned value costs
    (parallel.py:567-633): for each segment ahead of the last, a plain
    Riccati sweep whose terminal cost is the next segment's start value
    conditioned on its link point, then a full rollout of all T policies.
    ``sol`` is a dict returned by :func:`solve`."""
    splits = sol["splits"]
    J = len(splits) - 1
    if J == 1:
        return sol
    links = sol["links"]
    vf0 = sol["vf0"]
    T, n = prob["qx1"].shape
    m = prob["qu1"].shape[1]
    tasks = []
    for j in range(J - 1):
        lo, hi = splits[j], splits[j + 1]
        vf = vf0[j + 1]
        if j + 1 == J - 1:
            QT, qT = vf[0], vf[1]
        else:
            QT, qT = vf[0], vf[3] + vf[1].T @ links[j + 1]
        QT = 0.5 * (QT + QT.T)          # TerminalCost symmetrizes (problem.py:135-139)
        st = {f: np.array(prob[f][lo:hi]) for f in STAGE_FIELDS}
        tasks.append(("serial", st, QT, qT, RANK_TOL))
    if workers > 1 and len(tasks) > 1:
        rep = list(_pool(workers).map(_segment_task, tasks))
    else:
        rep = [_segment_task(t) for t in tasks]
    K = sol["K"].copy()
    k = sol["k"].copy()
    for j in range(J - 1):
        lo, hi = splits[j], splits[j + 1]
        K[lo:hi] = rep[j]["Kx"]
        k[lo:hi] = rep[j]["k1"]
    # _rollout_policies (parallel.py:556-564)
    xs = np.empty((T + 1, n))
    us = np.empty((T, m))
    xs[0] = prob["x_init"]
    for t in range(T):
        us[t] = K[t] @ xs[t] + k[t]
        xs[t + 1] = prob["Fx"][t] @ xs[t] + prob["Fu"][t] @ us[t] + prob["f1"][t]
    dev = max(float(np.abs(xs - sol["states"]).max()), float(np.abs(us - sol["controls"]).max()))
    out = dict(sol)
    out.update({"K": K, "k": k, "states": xs, "controls": us, "smooth_deviation": dev,
                "objective": objective(prob, xs, us),
                "kkt": kkt_residual(prob, xs, us, sol["lambdas"])})
    return out


def _solve_one(args):
    prob, J, splits, rank_tol = args
    return solve(prob, J=J, splits=splits, rank_tol=rank_tol)


def problem_slice(batch, i):
    return {k: v[i] for k, v in batch.items()}


def solve_batch(batch, J=None, splits=None, rank_tol=RANK_TOL, workers=1):
    """Loop (or problem-level fork pool, a harness around the reference API
    -- the reference has no batch entry) over the leading batch axis."""
    B = batch["x_init"].shape[0]
    tasks = [(problem_slice(batch, i), J, splits, rank_tol) for i in range(B)]
    if workers > 1 and B > 1:
        return list(_pool(workers).map(_solve_one, tasks,
                                       chunksize=max(1, B // (4 * workers))))
    return [_solve_one(t) for t in tasks]


def perturbed(prob, eps, seed):
    """Inputs multiplied by ``1 + eps*N(0,1)`` elementwise;
    symmetric blocks stay symmetric."""
    rng = np.random.default_rng(seed)
    out = {}
    for k, v in prob.items():
        p = v * (1.0 + eps * rng.standard_normal(v.shape))
        if k in ("Qxx", "Quu", "QxxT"):
            p = 0.5 * (p + np.swapaxes(p, -1, -2))
        out[k] = p
    return out


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
