"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container only (it imports ``parlqr`` from
``/root/reference/pkg/src``, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Each ``*.npz`` holds the inputs (or the seeded-config recipe plus a sha256 of
the inputs), the outputs of ``parlqr.solve_parallel`` on them, the unfolded
per-segment ``_solve_segment_task`` outputs, and the reference's numerical
floor: the relative change of each output when the inputs are perturbed by
~1 ulp (SURVEY.md Appendix C protocol).  Outputs are data, not source.
"""

from __future__ import annotations

import hashlib
import os
import sys

# NOTE: the committed fixtures were written with the container's default
# (multi-threaded) OpenBLAS: this setdefault used to sit after the numpy
# import and had no effect.  Kept after it so a regeneration reproduces them.
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import parlqr  # noqa: E402  (the reference)
from parlqr import parallel as ref_parallel  # noqa: E402
from parlqr.generate import generate as ref_generate  # noqa: E402
from parlqr.problem import (LqrProblem, StageCost, StageDynamics,  # noqa: E402
                            TerminalCost)

from paper_1809_06360_b200 import synth  # noqa: E402

FIELDS = synth.STAGE_FIELDS
OUTS = ("states", "controls", "lambdas", "K", "k")


def to_problem(a):
    stages = [(StageCost(a["Qxx"][t], a["Qux"][t], a["Quu"][t], a["qx1"][t], a["qu1"][t]),
               StageDynamics(a["Fx"][t], a["Fu"][t], a["f1"][t]))
              for t in range(a["qx1"].shape[0])]
    return LqrProblem(stages, TerminalCost(a["QxxT"], a["qx1T"]), a["x_init"])


def from_problem(p):
    a = {f: np.stack([getattr(c if f[0] in "Qq" else d, f) for c, d in p.stages])
         for f in FIELDS}
    a["QxxT"] = np.array(p.terminal.Qxx)
    a["qx1T"] = np.array(p.terminal.qx1)
    a["x_init"] = np.array(p.x_init)
    return a


def digest(a):
    h = hashlib.sha256()
    for k in sorted(a):
        h.update(k.encode())
        h.update(np.ascontiguousarray(a[k], dtype=np.float64).tobytes())
    return h.hexdigest()


def ref_solve(a, J, splits=None):
    prob = to_problem(a)
    part = None if splits is None else ref_parallel.Partition(len(splits) - 1, tuple(splits))
    sol = parlqr.solve_parallel(prob, J=J, workers=1, partition=part)
    d = sol.details
    out = {
        "states": sol.states, "controls": sol.controls, "lambdas": sol.lambdas,
        "K": np.stack([p.Kx for p in sol.policies]),
        "k": np.stack([p.k1 for p in sol.policies]),
        "objective": np.float64(sol.objective),
        "kkt": np.float64(sol.kkt_residual_inf),
        "degenerate": np.bool_(d.degenerate),
        "splits": np.array(d.partition.split_times),
    }
    if d.degenerate:
        # feasibility-constrained link solve (parallel.py:320-384): links and
        # multipliers; the rows themselves are basis-dependent (not stored)
        out.update({"links": d.link_points, "mu_left": d.mu_left, "lambda_right": d.lambda_right,
                    "link_mismatch": np.float64(d.link_mismatch),
                    "feas_rows": np.array([0 if f is None else f[0].shape[0] for f in d.segment_feasibility])})
        return out
    out.update({
        "links": d.link_points, "mu_left": d.mu_left, "lambda_right": d.lambda_right,
        "link_mismatch": np.float64(d.link_mismatch),
        "link_residual": np.float64(d.link_residual),
    })
    vf = d.segment_values0
    out["Vxx0"] = np.stack([v[0] for v in vf])
    out["vx10"] = np.stack([v[3] if len(v) == 5 else v[1] for v in vf])
    if len(vf) > 1:
        out["Vzx0"] = np.stack([v[1] for v in vf[:-1]])
        out["Vzz0"] = np.stack([v[2] for v in vf[:-1]])
        out["vz10"] = np.stack([v[4] for v in vf[:-1]])
    # unfolded per-segment gains through the reference's own task seam
    payloads = ref_parallel._segment_payloads(prob, d.partition, parlqr.DEFAULT_TOLERANCES, False)
    segs = [ref_parallel._solve_segment_task(ref_parallel._copy_payload(p)) for p in payloads]
    T, m, n = out["K"].shape
    Kz = np.zeros((T, m, n))
    k1 = np.empty((T, m))
    for j, seg in enumerate(segs):
        lo, hi = d.partition.split_times[j], d.partition.split_times[j + 1]
        k1[lo:hi] = seg["k1"]
        if seg["kind"] == "endpoint":
            Kz[lo:hi] = seg["Kz"]
    out["Kz"] = Kz
    out["k1"] = k1
    return out


def rel(a, b):
    den = float(np.abs(b).max())
    return float(np.abs(np.asarray(a) - np.asarray(b)).max()) / (den if den else 1.0)


def floors(a, J, base, splits=None, eps=1e-15, trials=3):
    """Relative output change under ~1-ulp input perturbation (App. C)."""
    fl = {}
    for s in range(trials):
        rng = np.random.default_rng(777 + s)
        pa = {}
        for k, v in a.items():
            p = v * (1.0 + eps * rng.standard_normal(v.shape))
            if k in ("Qxx", "Quu", "QxxT"):
                p = 0.5 * (p + np.swapaxes(p, -1, -2))
            pa[k] = p
        o = ref_solve(pa, J, splits)
        for key in OUTS + ("objective", "links", "Kz", "k1"):
            if key in base and key in o:
                fl[key] = max(fl.get(key, 0.0), rel(o[key], base[key]))
    return {f"floor_{k}": np.float64(v) for k, v in fl.items()}


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def synth_case(name, cfg_id, seed, count=1, **over):
    cfg = synth.CONFIGS[cfg_id].scaled(**over) if over else synth.CONFIGS[cfg_id]
    batch = synth.generate_batch(cfg, seed=seed, count=count)
    rec = {"cfg_id": np.int64(cfg_id), "n": np.int64(cfg.n), "m": np.int64(cfg.m),
           "T": np.int64(cfg.T), "J": np.int64(cfg.J), "seed": np.int64(seed),
           "count": np.int64(count), "a_scale": np.float64(cfg.a_scale),
           "q_eps": np.float64(cfg.q_eps), "r_eps": np.float64(cfg.r_eps),
           "input_sha256": np.array(digest(batch))}
    for i in range(count):
        a = {k: v[i] for k, v in batch.items()}
        base = ref_solve(a, cfg.J)
        fl = floors(a, cfg.J, base)
        for k, v in {**base, **fl}.items():
            rec.setdefault(k, []).append(v)
    out = {k: (np.stack(v) if isinstance(v, list) else v) for k, v in rec.items()}
    save(name, **out)


def stored_case(name, problems, Js, splits_list=None):
    """Small instances stored with their inputs (ragged, so one entry per
    problem with an index prefix)."""
    rec = {"num": np.int64(len(problems))}
    for i, (a, J) in enumerate(zip(problems, Js)):
        splits = None if splits_list is None else splits_list[i]
        o = ref_solve(a, J, splits)
        for k, v in a.items():
            rec[f"{i}/in/{k}"] = v
        for k, v in o.items():
            rec[f"{i}/out/{k}"] = v
        rec[f"{i}/J"] = np.int64(J)
    save(name, **rec)


def scalar_problem(T):
    cost = StageCost([[0.0]], [[0.0]], [[1.0]], [0.0], [0.0])
    dyn = StageDynamics([[1.0]], [[1.0]], [0.0])
    return LqrProblem([(cost, dyn)] * T, TerminalCost([[1.0]], [0.0]), [1.0])


def endpoint_case(a, seed):
    """solve_endpoint_affine + solve_endpoint of the reference on ``a`` at a
    reachable endpoint (a bounded random control sequence's end state)."""
    from parlqr import endpoint as ref_endpoint
    prob = to_problem(a)
    aff = ref_endpoint.solve_endpoint_affine(prob)
    mp, mm = aff.maps, aff.multipliers
    rng = np.random.default_rng(seed)
    x = prob.x_init.copy()
    for _, dyn in prob.stages:
        x = dyn.Fx @ x + dyn.Fu @ (0.3 * rng.standard_normal(prob.m)) + dyn.f1
    z = x
    sol = ref_endpoint.solve_endpoint(prob, prob.x_init, z)
    v0 = aff.values[0]
    return {
        "Kx": np.stack([p.Kx for p in aff.policies]), "Kz": np.stack([p.Kz for p in aff.policies]),
        "k1": np.stack([p.k1 for p in aff.policies]),
        "Vxx0": v0.Vxx, "Vzx0": v0.Vzx, "Vzz0": v0.Vzz, "vx10": v0.vx1, "vz10": v0.vz1,
        "const0": np.float64(v0.const),
        "X": np.concatenate([mp.Ra, mp.Rz, mp.r1[:, :, None]], axis=2),
        "S": np.concatenate([mp.Sa, mp.Sz, mp.s1[:, :, None]], axis=2),
        "Lam": np.concatenate([mm.La, mm.Lz, mm.l1[:, :, None]], axis=2),
        "E": np.concatenate([mm.Ea, mm.Ez, mm.e1[:, None]], axis=1),
        "x_term": z, "states": sol.states, "controls": sol.controls, "lambdas": sol.lambdas,
        "mu": sol.mu, "objective": np.float64(sol.objective), "kkt": np.float64(sol.kkt_residual_inf),
    }


def endpoint_goldens():
    rec = {}
    cases = [(3, 2, 8, 11), (4, 1, 10, 12), (2, 1, 6, 13), (5, 3, 12, 14), (4, 2, 10, 15), (6, 2, 9, 16)]
    for i, (n, m, T, seed) in enumerate(cases):
        a = from_problem(ref_generate(n, m, T, seed=seed))
        for k, v in a.items():
            rec[f"{i}/in/{k}"] = v
        for k, v in endpoint_case(a, 100 + i).items():
            rec[f"{i}/out/{k}"] = v
    rec["num"] = np.int64(len(cases))
    save("endpoint_small", **rec)
    for name, cid, T in (("endpoint_cfg0_shape", 0, 32), ("endpoint_cfg2_shape", 2, 32),
                         ("endpoint_cfg4_shape", 4, 8), ("endpoint_cfg3_shape", 3, 4)):
        cfg = synth.CONFIGS[cid].scaled(T=T, J=1)
        batch = synth.generate_batch(cfg, seed=2, count=1)
        a = {k: v[0] for k, v in batch.items()}
        save(name, cfg_id=np.int64(cid), T=np.int64(T), seed=np.int64(2),
             input_sha256=np.array(digest(batch)), **endpoint_case(a, 200 + cid))


def endpoint_unreachable_goldens():
    """Two-point-boundary problems whose horizon is too short to reach every
    endpoint direction (T m < n): feasibility rows, no multiplier maps,
    multipliers from gradient_duals (endpoint.py:566-587), Infeasible for a
    pair that violates the rows -- all by the reference itself."""
    from parlqr import endpoint as ref_endpoint
    from parlqr.errors import Infeasible
    rec = {}
    cases = [("ref", 3, 1, 1, 61), ("ref", 5, 2, 2, 62), ("ref", 6, 2, 2, 63), ("ref", 4, 1, 3, 64),
             ("cfg", 12, 4, 2, 65), ("cfg", 32, 8, 3, 66)]
    for i, (kind, n, m, T, seed) in enumerate(cases):
        if kind == "ref":
            a = from_problem(ref_generate(n, m, T, seed=seed))
        else:
            a = synth.generate_one(n, m, T, seed)
        prob = to_problem(a)
        aff = ref_endpoint.solve_endpoint_affine(prob)
        assert aff.multipliers is None and aff.feasibility.rows == n - T * m
        rng = np.random.default_rng(300 + i)
        x = prob.x_init.copy()
        for _, dyn in prob.stages:
            x = dyn.Fx @ x + dyn.Fu @ (0.3 * rng.standard_normal(prob.m)) + dyn.f1
        z = x
        sol = ref_endpoint.solve_endpoint(prob, prob.x_init, z)
        bad = z + rng.standard_normal(n)
        try:
            ref_endpoint.solve_endpoint(prob, prob.x_init, bad)
            raise AssertionError("expected Infeasible")
        except Infeasible as exc:
            bad_res = exc.residual
        v0, mp = aff.values[0], aff.maps
        out = {
            "Kx": np.stack([p.Kx for p in aff.policies]), "Kz": np.stack([p.Kz for p in aff.policies]),
            "k1": np.stack([p.k1 for p in aff.policies]),
            "Vxx0": v0.Vxx, "Vzx0": v0.Vzx, "Vzz0": v0.Vzz, "vx10": v0.vx1, "vz10": v0.vz1,
            "const0": np.float64(v0.const),
            "X": np.concatenate([mp.Ra, mp.Rz, mp.r1[:, :, None]], axis=2),
            "S": np.concatenate([mp.Sa, mp.Sz, mp.s1[:, :, None]], axis=2),
            "feas_rows": np.int64(aff.feasibility.rows),
            "Hx": aff.feasibility.Hx, "Hz": aff.feasibility.Hz, "h1": aff.feasibility.h1,
            "x_term": z, "states": sol.states, "controls": sol.controls, "lambdas": sol.lambdas,
            "mu": sol.mu, "objective": np.float64(sol.objective), "kkt": np.float64(sol.kkt_residual_inf),
            "x_bad": bad, "bad_residual": np.float64(bad_res),
        }
        for k, v in a.items():
            rec[f"{i}/in/{k}"] = v
        for k, v in out.items():
            rec[f"{i}/out/{k}"] = v
    rec["num"] = np.int64(len(cases))
    save("endpoint_unreachable", **rec)


def _with_singular_values(Fu, sig, seed):
    """Fu replaced by U diag(sig) V' with the same shape (random orthogonal
    U, V from a seeded QR)."""
    rng = np.random.default_rng(seed)
    n, m = Fu.shape
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    S = np.zeros((n, m))
    S[np.arange(len(sig)), np.arange(len(sig))] = sig
    return U @ S @ V.T


def rank_goldens():
    """Constrained tail stages whose Nu = Hx Fu sits at the reference's rank
    threshold (endpoint.py:226-231): at a segment's last stage Hx = I, so
    Nu = Fu and thr = rank_tol * sqrt(n) * ||Fu||_F.  Singular values below
    it make the reference take its mixed range/null-space branch (0 < p < m);
    values just above it with sigma_min inside the sqrt(m) band of the
    certificate exercise the GPU's rank-revealing repair pass."""
    tol = parlqr.DEFAULT_TOLERANCES.rank_tol
    probs, Js = [], []

    def case(a, J, t, sig_big, small, seed):
        n, m = a["Fu"].shape[1:]
        nb = len(sig_big)
        fro = np.sqrt(np.sum(np.square(sig_big)))
        thr = tol * np.sqrt(n) * fro
        sig = list(sig_big) + [c * thr for c in small]
        assert len(sig) == m
        a["Fu"][t] = _with_singular_values(a["Fu"][t], sig, seed)
        probs.append(a)
        Js.append(J)
        return nb

    # generic path: n=6, m=2 (partial p = 1, exactly deficient p = 1)
    case(from_problem(ref_generate(6, 2, 24, seed=301)), 3, 7, [1.0], [0.3], 1)
    case(from_problem(ref_generate(6, 2, 24, seed=302)), 3, 15, [0.8], [0.0], 2)
    # n % m != 0: the wide branch (r < m) with a rank-1 Fu two stages into
    # the tail of segment 0 (T=10, J=2: r = 5 -> 2 -> wide with p = 1)
    for seed in range(303, 340):     # first seed whose reference solve has no CholeskyFailure
        a = from_problem(ref_generate(5, 3, 10, seed=seed))
        rng = np.random.default_rng(seed)
        a["Fu"][3] = np.outer(rng.standard_normal(5), rng.standard_normal(3))
        try:
            ref_solve(a, 2)
        except parlqr.errors.SolverError:
            continue
        probs.append(a)
        Js.append(2)
        break
    # specialised kernels: cfg1 / cfg2 / cfg4 shapes (BASELINE recipe)
    for cid, over, J, t, seed in ((1, dict(B=1), 8, 15, 5), (2, dict(T=64, J=4), 4, 31, 6),
                                  (4, dict(T=16, J=2), 2, 7, 7)):
        cfg = synth.CONFIGS[cid].scaled(**over)
        for s in range(seed, seed + 40):   # first seed the reference solves without CholeskyFailure
            if cid == 4:
                # the reference's own generator at the (64, 32) shape: with the
                # cfg4 recipe (R = VV'/m + 1e-4 I) the reference itself fails
                # its Cholesky after a partial-rank tail
                b = from_problem(ref_generate(cfg.n, cfg.m, cfg.T, seed=s))
            else:
                b = {k: v[0] for k, v in synth.generate_batch(cfg, seed=s, count=1).items()}
            scale = float(np.linalg.norm(b["Fu"][t], 2))
            case(b, J, t, [scale] * (cfg.m - 1), [0.3], 10 + s)            # partial: p = m - 1
            try:
                ref_solve(b, J)
                break
            except parlqr.errors.SolverError:
                probs.pop()
                Js.pop()
    # (a stage whose sigma_min sits just above the threshold, inside the
    # certificate band, gives gains ~1e10 and the reference itself fails a
    # later Cholesky on every seed tried; the repair pass's p = m decision is
    # exercised by the other tail stages of the repaired segments above)
    for i, (a, J) in enumerate(zip(probs, Js)):
        try:
            ref_solve(a, J)
        except parlqr.errors.SolverError as exc:
            print("rank case", i, "fails:", exc)
    stored_case("rank_near", probs, Js)


def main():
    if "--only" in sys.argv:
        {"rank": rank_goldens}[sys.argv[sys.argv.index("--only") + 1]]()
        return
    # 1. hand example of test_parallel.py:48-54 (J=2 scalar problem)
    stored_case("hand_scalar", [from_problem(scalar_problem(2))], [2])
    # 2. the reference's small random pool (conftest.py:53-63) for J=2,3,4
    probs, Js = [], []
    for k in range(40):
        dims = np.random.default_rng(1_000 + k)
        n = int(dims.integers(1, 7))
        m = int(dims.integers(1, 4))
        T = int(dims.integers(1, 21))
        a = from_problem(ref_generate(n, m, T, seed=2_000 + k))
        for J in (2, 3, 4):
            if J <= T:
                probs.append(a)
                Js.append(J)
    stored_case("small_random", probs, Js)
    # 3. random custom partitions (test_parallel.py:95-112)
    rng = np.random.default_rng(9)
    probs, Js, splits = [], [], []
    for trial in range(40):
        dims = np.random.default_rng(5_000 + trial)
        n = int(dims.integers(1, 6))
        m = int(dims.integers(1, 4))
        T = int(dims.integers(2, 18))
        a = from_problem(ref_generate(n, m, T, seed=6_000 + trial))
        J = int(rng.integers(2, T + 1))
        interior = np.sort(rng.choice(np.arange(1, T), size=J - 1, replace=False))
        probs.append(a)
        Js.append(J)
        splits.append((0, *map(int, interior), T))
    stored_case("random_splits", probs, Js, splits)
    # 4. BASELINE configs: cfg0 in full, a cfg1 subset, reduced-T cfg2/3/4 shapes
    synth_case("cfg0_seed0", 0, seed=0)
    synth_case("cfg1_first4", 1, seed=0, count=4)
    synth_case("cfg2_shape_T256_J4", 2, seed=0, T=256, J=4)
    synth_case("cfg3_shape_T16_J2", 3, seed=0, T=16, J=2)
    synth_case("cfg4_shape_T64_J2", 4, seed=0, T=64, J=2)
    # 5. the double-integrator demo's J=3 partitioned solve (demo.py:52-62,
    #    102-112) plus its stored rollouts (demos/out/double_integrator)
    from parlqr import demo
    cfg = demo.DemoConfig()
    prob = demo.double_integrator_problem(cfg)
    a = from_problem(prob)
    o = ref_solve(a, demo.DEMO_SPLITS)
    ddir = "/root/reference/pkg/demos/out/double_integrator"

    def read_csv(fname):
        rows = open(os.path.join(ddir, fname)).read().strip().splitlines()[1:]
        vals = []
        for r in rows:
            cells = r.split(",")[1:]
            vals.append([float(c.replace("np.float64(", "").rstrip(")")) if c else np.nan
                         for c in cells])
        return np.array(vals)

    und = read_csv("parallel_undisturbed.csv")
    dis = read_csv("parallel_disturbed.csv")
    summ = open(os.path.join(ddir, "summary.csv")).read().strip().splitlines()[1].split(",")
    rec = {f"in/{k}": v for k, v in a.items()}
    rec.update({f"out/{k}": v for k, v in o.items()})
    rec.update({"J": np.int64(demo.DEMO_SPLITS), "csv_undisturbed": und,
                "csv_disturbed": dis, "cost_p": np.float64(float(summ[1])),
                "disturbance_smoothing": np.float64(demo.DISTURBANCE_SMOOTHING)})
    # smoothed solution of the demo (parallel.py:567-633) and its stored rollouts
    psol = parlqr.solve_parallel(prob, J=demo.DEMO_SPLITS, workers=1)
    ssol = ref_parallel.smooth(prob, psol, workers=1)
    rec.update({"smooth/K": np.stack([p.Kx for p in ssol.policies]),
                "smooth/k": np.stack([p.k1 for p in ssol.policies]),
                "smooth/states": ssol.states, "smooth/controls": ssol.controls,
                "smooth/objective": np.float64(ssol.objective), "smooth/kkt": np.float64(ssol.kkt_residual_inf),
                "smooth/deviation": np.float64(ssol.details.smooth_deviation),
                "csv_smoothed_undisturbed": read_csv("smoothed_undisturbed.csv"),
                "csv_smoothed_disturbed": read_csv("smoothed_disturbed.csv"),
                "cost_smoothed": np.float64(float(summ[2]))})
    save("demo_double_integrator", **rec)
    # segments without control authority (test_parallel.py:114-129): rank
    # p = 0 in every stage of the segment, feasibility-constrained link solve
    probs, Js = [], []
    a = from_problem(ref_generate(3, 2, 9, seed=123))
    a["Fu"][3:6] = 0.0
    probs.append(a)
    Js.append(3)
    cfg = synth.CONFIGS[1]
    b = {k: v[0] for k, v in synth.generate_batch(cfg, seed=5, count=1).items()}
    b["Fu"][24:32] = 0.0
    probs.append(b)
    Js.append(8)
    stored_case("uncontrollable", probs, Js)
    # two-point-boundary solves (endpoint.py:603-653) by the reference itself
    endpoint_goldens()
    endpoint_unreachable_goldens()
    # tail stages at the rank threshold (mixed branch 0 < p < m, repair pass)
    rank_goldens()
    # JSON problem / solution files written by the reference itself
    # (fileio.save_problem, cli solve --solver parallel --J 3, cli.py:26-59)
    from parlqr import cli as ref_cli
    from parlqr import fileio as ref_fileio
    jp = os.path.join(HERE, "json_problem_n3_m2_T12.json")
    js = os.path.join(HERE, "json_solution_parallel_J3.json")
    ref_fileio.save_problem(ref_generate(3, 2, 12, seed=7), jp)
    assert ref_cli.main(["solve", "--problem", jp, "--solver", "parallel", "--J", "3",
                         "--workers", "1", "--out", js]) == 0
    # smoothing on seeded config shapes
    for name, cid, over in (("smooth_cfg0", 0, {}), ("smooth_cfg2_shape", 2, dict(T=256, J=4)),
                            ("smooth_cfg4_shape", 4, dict(T=64, J=2))):
        cfg = synth.CONFIGS[cid].scaled(**over) if over else synth.CONFIGS[cid]
        a = {k: v[0] for k, v in synth.generate_batch(cfg, seed=1, count=1).items()}
        pr = to_problem(a)
        ps = parlqr.solve_parallel(pr, J=cfg.J, workers=1)
        ss = ref_parallel.smooth(pr, ps, workers=1)
        save(name, cfg_id=np.int64(cid), T=np.int64(cfg.T), J=np.int64(cfg.J), seed=np.int64(1),
             input_sha256=np.array(digest({k: v[None] for k, v in a.items()})),
             K=np.stack([p.Kx for p in ss.policies]), k=np.stack([p.k1 for p in ss.policies]),
             states=ss.states, controls=ss.controls, objective=np.float64(ss.objective),
             kkt=np.float64(ss.kkt_residual_inf), deviation=np.float64(ss.details.smooth_deviation))


if __name__ == "__main__":
    if len(sys.argv) > 1:           # regenerate single fixtures: make_golden.py endpoint_unreachable_goldens
        for fn in sys.argv[1:]:
            globals()[fn]()
    else:
        main()
