"""The reference's own property / acceptance tests for the hot path, restated
against the GPU drop-in on the reference's problem family
(``synth.generate_reference_recipe`` = ``parlqr.generate``, same draw order):

* test_parallel.py:74-112, 131-162 -- x / u equal the serial optimum, links
  equal the serial states at the split times, global KKT residual, multiplier
  matching at the links, link-system residual, for J in {1, 2, 3, 4, T};
* test_acceptance.py criteria 1, 3 (oracle equivalence, link condition) and 4
  (infeasibility detection with the free-evolution gap as the residual);
* test_endpoint.py:42-50, 196-201 -- the feasibility triple of an
  uncontrollable system is the free-evolution gap.

Tolerances are the reference's (1e-8 x (1 + data magnitude), 1e-9 absolute for
the gap).  The serial truth comes from the oracle's J = 1 solve."""

import numpy as np
import pytest

from oracle import parlqr_oracle as O

pytestmark = pytest.mark.gpu

ORACLE_TOL = 1e-8


def _scale(a):
    return 1.0 + max(float(np.abs(v).max()) for v in a.values() if np.size(v))


def _instance(k):
    from paper_1809_06360_b200 import synth
    dims = np.random.default_rng(10_000 + k)          # test_acceptance.py:28-33
    n, m, T = int(dims.integers(1, 7)), int(dims.integers(1, 4)), int(dims.integers(1, 21))
    return synth.generate_reference_recipe(n, m, T, 20_000 + k)


def _serial(a):
    """serial.solve (serial.py:37-98): Riccati sweep, rollout, objective -- the unique optimum."""
    sw = O.serial_sweep({f: a[f] for f in O.STAGE_FIELDS}, a["QxxT"], a["qx1T"])
    T, n = a["qx1"].shape
    xs, us = np.empty((T + 1, n)), np.empty((T, a["qu1"].shape[1]))
    xs[0] = a["x_init"]
    for t in range(T):
        us[t] = sw["Kx"][t] @ xs[t] + sw["k1"][t]
        xs[t + 1] = a["Fx"][t] @ xs[t] + a["Fu"][t] @ us[t] + a["f1"][t]
    return {"states": xs, "controls": us, "objective": O.objective(a, xs, us)}


def _free_evolution(a):
    x = a["x_init"].copy()
    for t in range(a["qx1"].shape[0]):
        x = a["Fx"][t] @ x + a["f1"][t]
    return x


def _drop_controls(a):
    b = {k: v.copy() for k, v in a.items()}
    b["Fu"][:] = 0.0
    return b


@pytest.mark.parametrize("block", range(3))
def test_acceptance_oracle_equivalence_and_link_condition(block):
    import paper_1809_06360_b200 as plq
    checked_links = 0
    for k in range(8 * block, 8 * block + 8):
        a = _instance(k)
        T = a["qx1"].shape[0]
        prob = plq.problem_from_arrays(a)
        ser = _serial(a)
        tol = ORACLE_TOL * _scale(a)
        for J in sorted({1, 2, 3, 4, T}):
            if J > T:
                continue
            sol = plq.solve_parallel(prob, J)
            assert np.abs(sol.states - ser["states"]).max() <= tol, (k, J)           # criterion 1
            assert np.abs(sol.controls - ser["controls"]).max() <= tol, (k, J)
            assert abs(sol.objective - ser["objective"]) <= tol * (1 + abs(ser["objective"])), (k, J)
            assert sol.kkt_residual_inf <= tol, (k, J, sol.kkt_residual_inf)          # test_parallel.py:131-135
            if J > 1:
                assert sol.details.link_mismatch <= tol, (k, J)                       # criterion 3
                for i, tau in enumerate(sol.details.partition.split_times[1:-1]):     # test_parallel.py:64-71
                    assert np.abs(sol.details.link_points[i] - ser["states"][tau]).max() <= tol, (k, J, i)
                checked_links += J - 1
    assert checked_links > 20


def test_link_residual_small():
    # test_parallel.py:147-162
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    a = synth.generate_reference_recipe(4, 2, 16, 14)
    sol = plq.solve_parallel(plq.problem_from_arrays(a), 4)
    vf = sol.details.segment_values0
    rhs = max(float(np.abs(vf[j][4] + vf[j + 1][3 if j + 1 < 3 else 1]).max()) for j in range(3))
    assert sol.details.link_residual <= 1e-9 * (1.0 + rhs) * _scale(a)
    ser = _serial(a)
    for i, tau in enumerate(sol.details.partition.split_times[1:-1]):
        assert np.abs(sol.details.link_points[i] - ser["states"][tau]).max() <= 1e-8 * _scale(a)


def test_uncontrollable_feasibility_triple_is_free_evolution_gap():
    # test_endpoint.py:42-50: with Fu = 0 no row is ever eliminated or rotated,
    # so the rows keep their meaning -- x_free(x_init) - x_term per state
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    a = _drop_controls(synth.generate_reference_recipe(3, 2, 6, 11))
    aff = plq.solve_endpoint_affine(plq.problem_from_arrays(a))
    assert aff.feasibility.rows == 3 and aff.multipliers is None
    x_free = _free_evolution(a)
    x_term = x_free + np.array([0.7, -0.2, 0.1])
    res = aff.feasibility.residual(a["x_init"], x_term)
    assert np.abs(res).max() == pytest.approx(np.abs(x_free - x_term).max(), abs=1e-9)


def test_unreachable_endpoint_is_infeasible():
    # test_endpoint.py:196-201
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import synth
    a = _drop_controls(synth.generate_reference_recipe(2, 1, 1, 70))
    x_term = _free_evolution(a) + np.array([1.0, 0.0])
    with pytest.raises(plq.Infeasible) as info:
        plq.solve_endpoint(plq.problem_from_arrays(a), a["x_init"], x_term)
    assert info.value.residual == pytest.approx(1.0, abs=1e-9)


def test_acceptance_infeasibility_detection():
    # test_acceptance.py:123-139 (criterion 4), first 10 instances
    import paper_1809_06360_b200 as plq
    for k in range(10):
        a = _drop_controls(_instance(k))
        prob = plq.problem_from_arrays(a)
        rng = np.random.default_rng(30_000 + k)
        x_free = _free_evolution(a)
        x_term = x_free + rng.standard_normal(x_free.shape[0])
        gap = float(np.abs(x_free - x_term).max())
        with pytest.raises(plq.Infeasible) as info:
            plq.solve_endpoint(prob, a["x_init"], x_term)
        assert info.value.residual == pytest.approx(gap, abs=1e-9), k
        sol = plq.solve_endpoint(prob, a["x_init"], x_free)       # the uncontrolled evolution itself stays feasible
        assert np.abs(sol.states[-1] - x_free).max() <= 1e-9 * _scale(a)
