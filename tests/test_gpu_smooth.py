"""GPU parity of the smoothing pass (``plq_smooth``; parlqr.parallel.smooth,
parallel.py:567-633) against the reference's smoothed solutions
(tests/golden) and against the oracle's restatement on fresh seeds, plus the
reference's own smoothing tests (test_parallel.py:184-231) restated.

Gates: smoothed K, k, states, controls and the objective within
max(1e-9, 10 * floor) relative, floor = the reference's own output change
under ~1-ulp input perturbation; smooth_deviation and the smoothed KKT
residual (taken with the parent multipliers) within the reference test's
scale 1e-8 * (1 + data magnitude) (test_parallel.py:211) or, on
ill-conditioned problems, the reference's own value plus that floor.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from oracle import parlqr_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _scale(a):
    return 1.0 + max(float(np.abs(v).max()) for v in a.values() if np.size(v))


@pytest.fixture(params=["specialized", "generic"])
def kernel_path(request, monkeypatch):
    if request.param == "generic":
        monkeypatch.setenv("PLQ_FORCE_GENERIC", "1")
    else:
        monkeypatch.delenv("PLQ_FORCE_GENERIC", raising=False)
    return request.param


def _smooth_batch(batch, J):
    from paper_1809_06360_b200 import solve_parallel_batch
    from paper_1809_06360_b200.parallel import raise_for_status
    s = solve_parallel_batch(batch, J=J)
    so = s.smooth({f: s.torch.from_numpy(np.ascontiguousarray(batch[f])).to(s.device) for f in batch})
    out = {k: v.cpu().numpy() for k, v in so.items()}
    raise_for_status(out["status"])
    assert s.launches in (2, 5)   # walk kernel, or maps + segment rollouts + evaluation
    return out, {k: (v.cpu().numpy() if v is not None else None) for k, v in s.out.items()}


def _floor(a, J, ref):
    """The reference's own smoothed-output change under ~1-ulp input
    perturbation, measured with the oracle."""
    fl = {}
    for s in range(2):
        pa = O.perturbed(a, 1e-15, 300 + s)
        r = O.smooth(pa, O.solve(pa, J=J))
        for k in ("K", "k", "states", "controls", "objective"):
            fl[k] = max(fl.get(k, 0.0), rel_err(r[k], ref[k]))
    return fl


def _check(o, i, ref, a, floors=None):
    floors = floors or {}
    for key, rk in (("K", "K"), ("k", "k"), ("x", "states"), ("u", "controls"), ("objective", "objective")):
        gate = max(TOL, 10.0 * floors.get(rk, 0.0))
        err = rel_err(o[key][i], ref[rk])
        assert err <= gate, (key, err, gate)
    # smooth_deviation compares two trajectories that agree to the problem's
    # conditioning: the GPU's must be within the reference test's bound or
    # the reference's own deviation plus its perturbation floor
    sc = _scale(a)
    slack = 10.0 * max(floors.get("states", 0.0) * float(np.abs(ref["states"]).max()),
                       floors.get("controls", 0.0) * float(np.abs(ref["controls"]).max()))
    assert o["deviation"][i] <= max(1e-8 * sc, 10 * float(ref["deviation"]) + slack)
    assert o["kkt_inf"][i] <= max(10 * float(ref["kkt"]), 1e-8 * sc) + slack


@pytest.mark.parametrize("name", ["smooth_cfg0", "smooth_cfg2_shape", "smooth_cfg4_shape"])
def test_smooth_reference_goldens(name, kernel_path):
    from paper_1809_06360_b200 import synth
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = synth.CONFIGS[int(z["cfg_id"])].scaled(T=int(z["T"]), J=int(z["J"]))
    batch = synth.generate_batch(cfg, seed=int(z["seed"]), count=1)
    o, _ = _smooth_batch(batch, cfg.J)
    _check(o, 0, {k: z[k] for k in z.files}, O.problem_slice(batch, 0))


@pytest.mark.parametrize("cfg_id,T,J,count", [(1, 64, 8, 16), (2, 512, 8, 1), (2, 4096, 64, 1),
                                              (3, 32, 4, 1), (4, 128, 4, 2), (0, 96, 5, 2)])
def test_smooth_vs_oracle_fresh_seeds(cfg_id, T, J, count, kernel_path):
    from paper_1809_06360_b200 import synth
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=515, count=count)
    o, _ = _smooth_batch(batch, J)
    for i in range(count):
        a = O.problem_slice(batch, i)
        ref = O.smooth(a, O.solve(a, J=J))
        ref["deviation"] = ref["smooth_deviation"]
        _check(o, i, ref, a, _floor(a, J, ref))


def test_smooth_drop_in_api_on_demo():
    """Drop-in smooth() on the reference demo (demo.py:102-130): policies,
    objective and the stored smoothed rollouts, nominal and disturbed."""
    import paper_1809_06360_b200 as plq
    z = np.load(os.path.join(GOLDEN, "demo_double_integrator.npz"))
    a = {k[3:]: z[k] for k in z.files if k.startswith("in/")}
    prob = plq.problem_from_arrays(a)
    psol = plq.solve_parallel(prob, J=int(z["J"]))
    sm = plq.smooth(prob, psol, workers=1)
    K = np.stack([p.Kx for p in sm.policies])
    k = np.stack([p.k1 for p in sm.policies])
    assert rel_err(K, z["smooth/K"]) <= TOL and rel_err(k, z["smooth/k"]) <= TOL
    assert rel_err(sm.states, z["smooth/states"]) <= TOL
    assert rel_err(sm.objective, z["smooth/objective"]) <= TOL
    assert sm.lambdas is psol.lambdas
    assert sm.details.smooth_deviation <= 1e-8 * _scale(a)
    assert psol.details.smooth_deviation is None
    for disturbed, key in ((False, "csv_smoothed_undisturbed"), (True, "csv_smoothed_disturbed")):
        x = a["x_init"].copy()
        xs = [x]
        for t in range(a["qx1"].shape[0]):
            u = sm.policies[t](x)
            xn = a["Fx"][t] @ x + a["Fu"][t] @ u + a["f1"][t]
            if disturbed:
                xn = xn + np.array([0.0, x[0] / (x[0] * x[0] + float(z["disturbance_smoothing"]))])
            x = xn
            xs.append(x)
        assert rel_err(np.array(xs), z[key][:, :2]) <= TOL, key


def _problem(a):
    import paper_1809_06360_b200 as plq
    return plq.problem_from_arrays(a)


def test_two_way_smoothing_recovers_global_gain():
    # test_parallel.py:185-191: J=2 scalar problem, smoothed first gain equals
    # the serial (global) Riccati gain
    import paper_1809_06360_b200 as plq
    from conftest import load_stored
    (a, _, _), = load_stored("hand_scalar")
    prob = _problem(a)
    sm = plq.smooth(prob, plq.solve_parallel(prob, J=2, workers=1), workers=1)
    ser = O.serial_sweep({f: a[f] for f in O.STAGE_FIELDS}, a["QxxT"], a["qx1T"])
    np.testing.assert_allclose(sm.policies[0].Kx, ser["Kx"][0], atol=1e-12)


def test_single_segment_noop():
    # test_parallel.py:193-196
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    prob = _problem(synth.generate_one(3, 1, 6, seed=18))
    psol = plq.solve_parallel(prob, J=1, workers=1)
    assert plq.smooth(prob, psol) is psol


def test_smoothed_rollout_reproduces_parallel_trajectory():
    # test_parallel.py:198-211 over the reference's small random pool
    import paper_1809_06360_b200 as plq
    from conftest import load_stored
    checked = 0
    seen = set()
    for a, o, _ in load_stored("small_random"):
        key = a["x_init"].tobytes() + a["qx1"].tobytes()
        if key in seen:
            continue
        seen.add(key)
        T = a["qx1"].shape[0]
        J = min(3, T)
        if J < 2:
            continue
        prob = _problem(a)
        psol = plq.solve_parallel(prob, J=J, workers=1)
        try:
            sm = plq.smooth(prob, psol, workers=1)
        except ValueError:
            # reachability-deficient conditioning segment: undefined
            assert psol.details.degenerate
            continue
        assert sm.details.smooth_deviation <= 1e-8 * _scale(a)
        if psol.details.degenerate:
            checked += 1
            continue    # rows only in segment 0: the oracle does not restate the dense link path
        ref = O.smooth(a, O.solve(a, J=J))
        assert rel_err(sm.states, ref["states"]) <= TOL
        assert rel_err(np.stack([p.Kx for p in sm.policies]), ref["K"]) <= TOL
        checked += 1
    assert checked >= 10


def test_smoothing_rejects_deficient_partitions():
    # test_parallel.py:213-218: length-3 segments with one control reach rank
    # 3 < 4, the solve takes the feasibility-constrained link path and
    # smoothing is undefined
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    a = synth.generate_one(4, 1, 12, seed=19)
    prob = _problem(a)
    psol = plq.solve_parallel(prob, J=4, workers=1)
    assert psol.details.degenerate
    with pytest.raises(ValueError):
        plq.smooth(prob, psol, workers=1)


def test_smoothed_policies_differ_from_both_parents():
    # test_parallel.py:220-231
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    a = synth.generate_one(2, 1, 30, seed=20)
    prob = _problem(a)
    psol = plq.solve_parallel(prob, J=3, workers=1)
    sm = plq.smooth(prob, psol, workers=1)
    ser = O.serial_sweep({f: a[f] for f in O.STAGE_FIELDS}, a["QxxT"], a["qx1T"])
    Ks = np.stack([p.Kx for p in sm.policies])
    Kp = np.stack([p.Kx for p in psol.policies])
    assert np.abs(Ks - Kp).max() > 1e-6
    assert np.abs(Ks - ser["Kx"]).max() > 1e-6


def test_smooth_full_size_cfg1_properties():
    """BASELINE config 1 at full size: every smoothed trajectory reproduces
    its parent's; samples equal the oracle's smoothing."""
    from paper_1809_06360_b200 import synth
    cfg = synth.CONFIGS[1]
    batch = synth.generate_batch(cfg, seed=0)
    o, parent = _smooth_batch(batch, cfg.J)
    assert np.all(np.isfinite(o["x"])) and np.all(np.isfinite(o["K"]))
    scale = np.abs(parent["x"]).reshape(cfg.B, -1).max(axis=1) + 1.0
    assert np.median(o["deviation"] / scale) <= 1e-10
    for i in (0, 1, 777, 4095):
        a = O.problem_slice(batch, i)
        ref = O.smooth(a, O.solve(a, J=cfg.J))
        assert rel_err(o["K"][i], ref["K"]) <= TOL
        assert rel_err(o["x"][i], ref["states"]) <= TOL
        assert rel_err(o["objective"][i], ref["objective"]) <= TOL
