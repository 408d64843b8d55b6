"""GPU parity of the two-point-boundary solve (``plq_endpoint_affine`` /
``plq_endpoint_evaluate``; parlqr.endpoint.solve_endpoint_affine /
solve_endpoint, endpoint.py:603-653) against the reference's own outputs
(tests/golden/endpoint_*.npz) and the oracle, plus the reference's
test_endpoint.py properties restated.

Gate: err = |y_gpu - y_ref|_inf / |y_ref|_inf <= max(1e-9, 10 * floor) for
gains, maps, multiplier maps, trajectories and the objective; floor = the
reference's own output change under ~1-ulp input perturbation (oracle).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from oracle import parlqr_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9
KEYS = ("Kx", "Kz", "k1", "X", "S", "Lam", "E")
PT = (("x", "states"), ("u", "controls"), ("lam", "lambdas"), ("mu", "mu"))


@pytest.fixture(params=["specialized", "generic"])
def kernel_path(request, monkeypatch):
    if request.param == "generic":
        monkeypatch.setenv("PLQ_FORCE_GENERIC", "1")
    else:
        monkeypatch.delenv("PLQ_FORCE_GENERIC", raising=False)
    return request.param


def _scale(a):
    return 1.0 + max(float(np.abs(v).max()) for v in a.values() if np.size(v))


def _floor(a, z, ref_aff, ref_ev):
    fl = {}
    for s in range(2):
        pa = O.perturbed(a, 1e-15, 900 + s)
        aff = O.solve_endpoint_affine(pa)
        ev = O.evaluate_endpoint(pa, aff, pa["x_init"], z)
        for k in KEYS:
            fl[k] = max(fl.get(k, 0.0), rel_err(aff[k], ref_aff[k]))
        for k in ("states", "controls", "lambdas", "mu", "objective"):
            fl[k] = max(fl.get(k, 0.0), rel_err(ev[k], ref_ev[k]))
    return fl


def _run(batch_arrays, z):
    from paper_1809_06360_b200 import solve_endpoint_batch
    eb = solve_endpoint_batch(batch_arrays, z)
    out = {k: v.cpu().numpy() for k, v in eb.out.items()}
    pt = {k: v.cpu().numpy() for k, v in eb.point.items()}
    return out, pt, eb


def _check(out, pt, i, ref, a, floors):
    for k in KEYS:
        gate = max(TOL, 10 * floors.get(k, 0.0))
        assert rel_err(out[k][i], ref[k]) <= gate, (k, rel_err(out[k][i], ref[k]), gate)
    for k, rk in PT + (("objective", "objective"),):
        gate = max(TOL, 10 * floors.get(rk, 0.0))
        assert rel_err(pt[k][i], ref[rk]) <= gate, (k, rel_err(pt[k][i], ref[rk]), gate)
    assert pt["kkt_inf"][i] <= max(10 * float(ref["kkt"]), 1e-8 * _scale(a))


def test_endpoint_reference_goldens_small():
    z = np.load(os.path.join(GOLDEN, "endpoint_small.npz"))
    for i in range(int(z["num"])):
        a = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/in/")}
        o = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/out/")}
        out, pt, eb = _run({k: v[None] for k, v in a.items()}, o["x_term"][None])
        aff = O.solve_endpoint_affine(a)
        fl = _floor(a, o["x_term"], aff, O.evaluate_endpoint(a, aff, a["x_init"], o["x_term"]))
        _check(out, pt, 0, o, a, fl)


@pytest.mark.parametrize("name", ["endpoint_cfg0_shape", "endpoint_cfg2_shape", "endpoint_cfg4_shape",
                                  "endpoint_cfg3_shape"])
def test_endpoint_reference_goldens_configs(name, kernel_path):
    from paper_1809_06360_b200 import synth
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = synth.CONFIGS[int(z["cfg_id"])].scaled(T=int(z["T"]), J=1)
    batch = synth.generate_batch(cfg, seed=int(z["seed"]), count=1)
    a = O.problem_slice(batch, 0)
    out, pt, eb = _run(batch, z["x_term"][None])
    assert eb.launches == 4                      # point, duals (no-op without rows), evaluation, reduction
    ref = {k: z[k] for k in z.files}
    aff = O.solve_endpoint_affine(a)
    _check(out, pt, 0, ref, a, _floor(a, z["x_term"], aff, O.evaluate_endpoint(a, aff, a["x_init"], z["x_term"])))


def test_endpoint_batch_vs_oracle_fresh_seeds(kernel_path):
    from paper_1809_06360_b200 import synth
    cfg = synth.CONFIGS[1].scaled(T=16, J=1)
    batch = synth.generate_batch(cfg, seed=77, count=6)
    rng = np.random.default_rng(3)
    zs = rng.standard_normal((6, cfg.n))
    out, pt, _ = _run(batch, zs)
    for i in range(6):
        a = O.problem_slice(batch, i)
        aff = O.solve_endpoint_affine(a)
        ev = O.evaluate_endpoint(a, aff, a["x_init"], zs[i])
        ref = {**aff, **ev}
        _check(out, pt, i, ref, a, _floor(a, zs[i], aff, ev))


def _interp(T=2):
    import paper_1809_06360_b200 as plq
    cost = plq.StageCost([[0.0]], [[0.0]], [[1.0]], [0.0], [0.0])
    dyn = plq.StageDynamics([[1.0]], [[1.0]], [0.0])
    return plq.LqrProblem([(cost, dyn)] * T, plq.TerminalCost.zero(1), [0.0])


def test_interpolation_full_stack_and_split():
    # test_endpoint.py:125-130, 191-194
    import paper_1809_06360_b200 as plq
    sol = plq.solve_endpoint(_interp(), [0.0], [1.0])
    assert sol.kkt_residual_inf <= 1e-10
    np.testing.assert_allclose(sol.lambdas.ravel(), [0.5, 0.5, 0.5], atol=1e-12)
    np.testing.assert_allclose(sol.mu, [-0.5], atol=1e-12)
    np.testing.assert_allclose(sol.controls.ravel(), [0.5, 0.5], atol=1e-12)
    assert sol.objective == pytest.approx(0.25)


def test_zero_data_means_zero_multipliers():
    # test_endpoint.py:132-140
    import paper_1809_06360_b200 as plq
    cost = plq.StageCost(np.zeros((2, 2)), np.zeros((2, 2)), np.eye(2), np.zeros(2), np.zeros(2))
    dyn = plq.StageDynamics(np.eye(2), np.eye(2), np.zeros(2))
    prob = plq.LqrProblem([(cost, dyn)] * 4, plq.TerminalCost.zero(2), np.zeros(2))
    sol = plq.solve_endpoint(prob, np.zeros(2), np.zeros(2))
    assert np.abs(sol.lambdas).max() <= 1e-12 and np.abs(sol.mu).max() <= 1e-12


def test_dependent_constraints():
    # test_endpoint.py:171-175: one step cannot pin three states with one control
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    prob = plq.problem_from_arrays(synth.generate_one(3, 1, 1, seed=61))
    with pytest.raises(plq.FactorizationFailure):
        plq.solve_endpoint_affine(prob, require_multipliers=True)
    with pytest.raises(plq.Infeasible):
        plq.solve_endpoint(prob, np.zeros(3), np.ones(3))
    aff = plq.solve_endpoint_affine(prob)
    assert aff.multipliers is None and aff.feasibility.rows == 2


def test_endpoint_unreachable_directions_reference_goldens(kernel_path):
    """Horizons too short to reach every endpoint direction (T m < n): the
    rows are returned, no multiplier maps are computed, and evaluate takes the
    multipliers from gradient_duals (endpoint.py:566-587) on the device --
    against the reference's own outputs, batched and through the drop-in."""
    import paper_1809_06360_b200 as plq
    z = np.load(os.path.join(GOLDEN, "endpoint_unreachable.npz"))
    for i in range(int(z["num"])):
        a = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/in/")}
        o = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/out/")}
        out, pt, eb = _run({k: v[None] for k, v in a.items()}, o["x_term"][None])
        assert eb.launches == 4                      # point, duals, evaluation, reduction
        r = int(o["feas_rows"])
        assert int(out["feas_rows"][0]) == r and int(out["gram_status"][0]) == -1
        sc = _scale(a)
        for k in ("Kx", "Kz", "k1", "X", "S"):
            assert rel_err(out[k][0], o[k]) <= 1e-9 * sc, (k, rel_err(out[k][0], o[k]))
        # the rows span the reference's row space (an orthonormal rotation of them)
        mine = out["feas"][0][:r]
        ref_rows = np.concatenate([o["Hx"], o["Hz"], o["h1"][:, None]], axis=1)
        coef = np.linalg.lstsq(ref_rows.T, mine.T, rcond=None)[0]
        assert np.abs(ref_rows.T @ coef - mine.T).max() <= 1e-9 * sc
        assert np.abs(coef @ coef.T - np.eye(r)).max() <= 1e-8 * sc
        for k, rk in PT + (("objective", "objective"),):
            assert rel_err(pt[k][0], o[rk]) <= 1e-8 * sc, (k, rel_err(pt[k][0], o[rk]))
        assert pt["kkt_inf"][0] <= max(10 * float(o["kkt"]), 1e-8 * sc)
        assert pt["feas_residual"][0] <= 1e-9 * sc
        # drop-in: same solution, Infeasible for a pair off the rows, strict mode raises
        prob = plq.problem_from_arrays(a)
        sol = plq.solve_endpoint(prob, a["x_init"], o["x_term"])
        assert rel_err(sol.lambdas, o["lambdas"]) <= 1e-8 * sc and rel_err(sol.mu, o["mu"]) <= 1e-8 * sc
        with pytest.raises(plq.Infeasible) as ei:
            plq.solve_endpoint(prob, a["x_init"], o["x_bad"])
        assert 0.2 * float(o["bad_residual"]) <= ei.value.residual <= 5 * float(o["bad_residual"])
        with pytest.raises(plq.FactorizationFailure):
            plq.solve_endpoint_affine(prob, require_multipliers=True)
    # a batch mixing reachable and unreachable problems is not possible (one T per batch);
    # mixed ROW COUNTS are: an uncontrollable direction in one problem of a reachable batch
    from paper_1809_06360_b200 import solve_endpoint_batch, synth
    cfg = synth.CONFIGS[1].scaled(T=8, J=1)
    batch = synth.generate_batch(cfg, seed=31, count=3)
    batch["Fu"][1][:, 0, :] = 0.0                  # state 0 of problem 1 gets no direct control ...
    batch["Fx"][1][:, 0, :] = 0.0                  # ... and no coupling: x0' = f1 only
    batch["Fx"][1][:, 0, 0] = 1.0
    zt = np.zeros((3, cfg.n))
    for i in range(3):
        a = O.problem_slice(batch, i)
        x = a["x_init"].copy()
        for t in range(cfg.T):
            x = a["Fx"][t] @ x + a["f1"][t]
        zt[i] = x                                     # reachable with u = 0
    eb = solve_endpoint_batch(batch, zt)
    rows = eb.out["feas_rows"].cpu().numpy()
    assert rows[0] == 0 and rows[2] == 0 and rows[1] >= 1
    for i in range(3):
        a = O.problem_slice(batch, i)
        aff = O.solve_endpoint_affine(a)
        ev = O.evaluate_endpoint(a, aff, a["x_init"], zt[i])
        assert aff["feas"][0].shape[0] == rows[i]
        for k, rk in PT:
            assert rel_err(eb.point[k][i].cpu().numpy(), ev[rk]) <= 1e-7, (i, k)


def test_map_boundary_blocks_equal_value_gradients():
    # test_endpoint.py:177-189 -- ties the backward pass to the multiplier pass
    import paper_1809_06360_b200 as plq
    from conftest import load_stored
    a, _, _ = load_stored("small_random")[5]
    prob = plq.problem_from_arrays(a)
    aff = plq.solve_endpoint_affine(prob)
    v0, mm = aff.values[0], aff.multipliers
    tol = 1e-7 * _scale(a)
    for got, want in ((mm.La[0], -v0.Vxx), (mm.Lz[0], -v0.Vzx.T), (mm.l1[0], -v0.vx1), (mm.Ea, -v0.Vzx),
                      (mm.Ez, -v0.Vzz), (mm.e1, -v0.vz1)):
        assert np.abs(got - want).max() <= tol


def test_endpoint_exactness_over_many_targets():
    # test_endpoint.py:213-221 through the GPU evaluation
    import paper_1809_06360_b200 as plq
    from conftest import load_stored
    a, _, _ = load_stored("small_random")[9]
    prob = plq.problem_from_arrays(a)
    aff = plq.solve_endpoint_affine(prob)
    rng = np.random.default_rng(5)
    n = a["x_init"].shape[0]
    for _ in range(10):
        x0, z = rng.standard_normal(n), rng.standard_normal(n)
        sol = aff.evaluate(x0, z)
        assert np.abs(sol.states[-1] - z).max() <= 1e-8 * (1 + np.abs(z).max())
        assert np.abs(sol.states[0] - x0).max() <= 1e-12 * (1 + np.abs(x0).max())
        assert sol.kkt_residual_inf <= 1e-8 * _scale(a) * (1 + np.abs(z).max() + np.abs(x0).max())


def test_endpoint_collect_diagnostics():
    """solve_endpoint_affine(collect_diagnostics=True): StageDiagnostics from the
    rank-revealing kernel (bounds of test_endpoint.py:73-78), same solution."""
    import paper_1809_06360_b200 as plq
    from conftest import load_stored
    a, _, _ = load_stored("small_random")[5]
    prob = plq.problem_from_arrays(a)
    base = plq.solve_endpoint_affine(prob)
    aff = plq.solve_endpoint_affine(prob, collect_diagnostics=True)
    assert base.diagnostics is None
    d = aff.diagnostics
    assert d.max_rows == a["x_init"].shape[0]
    assert 0.0 <= d.basis_defect <= 1e-10 and 0.0 <= d.projector_defect <= 1e-12
    for t in (0, len(aff.policies) - 1):
        assert rel_err(aff.policies[t].Kx, base.policies[t].Kx) <= 1e-8
    assert rel_err(aff.maps.Ra, base.maps.Ra) <= 1e-8


def test_initial_value_constant_and_objective_identity():
    """``values[0].const`` (endpoint.py:283-284, 296) against the reference's own
    goldens -- reachable problems (taken at the pair (0, 0)) and problems with
    feasibility rows (least-norm pair on the rows) -- and test_endpoint.py:223-231
    restated: the objective at a reachable endpoint equals ``values[0].value``."""
    import paper_1809_06360_b200 as plq
    for name in ("endpoint_small", "endpoint_unreachable"):
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        for i in range(int(z["num"])):
            a = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/in/")}
            o = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/out/")}
            prob = plq.problem_from_arrays(a)
            aff = plq.solve_endpoint_affine(prob)
            v0 = aff.values[0]
            sc = _scale(a)
            for k, mine in (("Vxx0", v0.Vxx), ("Vzx0", v0.Vzx), ("Vzz0", v0.Vzz), ("vx10", v0.vx1), ("vz10", v0.vz1)):
                assert rel_err(mine, o[k]) <= 1e-8 * sc, (name, i, k, rel_err(mine, o[k]))
            quad = abs(float(o["objective"])) + abs(float(o["const0"])) + 1.0
            assert abs(v0.const - float(o["const0"])) <= 1e-8 * sc * quad, (name, i, v0.const, float(o["const0"]))
            sol = aff.evaluate(a["x_init"], o["x_term"])
            val = v0.value(a["x_init"], o["x_term"])
            assert sol.objective == pytest.approx(val, rel=1e-8 * sc, abs=1e-8 * sc * (1 + abs(val)))
            assert val == pytest.approx(float(o["objective"]), rel=1e-8 * sc, abs=1e-8 * sc * (1 + abs(val)))
