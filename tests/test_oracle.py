"""The CPU oracle (oracle/parlqr_oracle.py) pinned against outputs of the
reference implementation itself (tests/golden/*.npz, written by
tests/golden/make_golden.py from /root/reference/pkg/src)."""

import hashlib

import numpy as np
import pytest

from conftest import SYNTH_FIXTURES, load_stored, load_synth, rel_err
from oracle import parlqr_oracle as O

KEYS = ("states", "controls", "lambdas", "K", "k", "links", "Kz", "k1")


def _digest(a):
    h = hashlib.sha256()
    for k in sorted(a):
        h.update(k.encode())
        h.update(np.ascontiguousarray(a[k], dtype=np.float64).tobytes())
    return h.hexdigest()


def test_hand_example_two_way_split():
    # test_parallel.py:48-54: link 2/3, u = (-1/3, -1/3), objective 1/6
    (a, o, J), = load_stored("hand_scalar")
    r = O.solve(a, J=J)
    np.testing.assert_allclose(r["links"], [[2 / 3]], atol=1e-12)
    np.testing.assert_allclose(r["controls"].ravel(), [-1 / 3, -1 / 3], atol=1e-12)
    assert r["objective"] == pytest.approx(1 / 6)
    for k in KEYS:
        assert np.array_equal(r[k], o[k]), k


def test_interpolation_sweep_by_hand():
    # test_endpoint.py:28-40: last stage Kx=-1, Kz=1, k1=0; value 0.25 at z=1
    st = {"Qxx": np.zeros((2, 1, 1)), "Qux": np.zeros((2, 1, 1)), "Quu": np.ones((2, 1, 1)),
          "qx1": np.zeros((2, 1)), "qu1": np.zeros((2, 1)), "Fx": np.ones((2, 1, 1)),
          "Fu": np.ones((2, 1, 1)), "f1": np.zeros((2, 1))}
    r = O.endpoint_sweep(st)
    np.testing.assert_allclose(r["Kx"][1], [[-1.0]])
    np.testing.assert_allclose(r["Kz"][1], [[1.0]])
    np.testing.assert_allclose(r["k1"][1], [0.0])
    assert r["feas"][0].shape[0] == 0
    Vxx, Vzx, Vzz, vx1, vz1 = r["vf0"]
    z = np.ones(1)
    assert float(0.5 * z @ Vzz @ z + vz1 @ z) == pytest.approx(0.25)


@pytest.mark.parametrize("name", ["small_random", "random_splits"])
def test_oracle_matches_reference_small(name):
    checked = 0
    for a, o, J in load_stored(name):
        if bool(o["degenerate"]):
            with pytest.raises(O.OracleDegenerate):
                O.solve(a, splits=tuple(int(s) for s in o["splits"]))
            continue
        r = O.solve(a, splits=tuple(int(s) for s in o["splits"]))
        scale = 1.0 + max(float(np.abs(v).max()) for v in a.values())
        for k in KEYS:
            assert np.abs(r[k] - o[k]).max() <= 1e-12 * scale, k
        assert abs(r["objective"] - float(o["objective"])) <= 1e-12 * scale * (1 + abs(float(o["objective"])))
        checked += 1
    assert checked >= 20


@pytest.mark.parametrize("name", SYNTH_FIXTURES)
def test_oracle_matches_reference_configs(name):
    cfg, batch, z = load_synth(name)
    assert _digest(batch) == str(z["input_sha256"]), "generator drifted from the golden inputs"
    for i in range(int(z["count"])):
        r = O.solve(O.problem_slice(batch, i), J=cfg.J)
        for k in ("states", "controls", "lambdas", "K", "k", "Kz", "k1"):
            # same numpy call sequence; allow BLAS summation-order noise (the
            # fixtures were written with multi-threaded OpenBLAS, the tests
            # run it single-threaded, conftest.py)
            assert rel_err(r[k], z[k][i]) <= 1e-12, (k, rel_err(r[k], z[k][i]))
        assert rel_err(r["objective"], z["objective"][i]) <= 1e-14


def test_demo_policies_reproduce_stored_rollouts():
    # demos/out/double_integrator/parallel_undisturbed.csv came from rolling
    # the J=3 partitioned policies out on the nominal dynamics (demo.py:69-82)
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "demo_double_integrator.npz"))
    a = {k[3:]: z[k] for k in z.files if k.startswith("in/")}
    r = O.solve(a, J=int(z["J"]))
    T = a["qx1"].shape[0]
    x = a["x_init"].copy()
    xs, us = [x], []
    for t in range(T):
        u = r["K"][t] @ x + r["k"][t]
        x = a["Fx"][t] @ x + a["Fu"][t] @ u + a["f1"][t]
        xs.append(x)
        us.append(u)
    und = z["csv_undisturbed"]
    np.testing.assert_allclose(np.array(xs), und[:, :2], rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.array(us)[:, 0], und[:-1, 2], rtol=0, atol=1e-9)


SMOOTH_FIXTURES = ("smooth_cfg0", "smooth_cfg2_shape", "smooth_cfg4_shape")


def test_oracle_smooth_matches_reference():
    """oracle.smooth restates parallel.py:567-633; pinned against the
    reference's own smoothed solutions (tests/golden/make_golden.py)."""
    import os
    from conftest import GOLDEN
    from paper_1809_06360_b200 import synth
    z = np.load(os.path.join(GOLDEN, "demo_double_integrator.npz"))
    a = {k[3:]: z[k] for k in z.files if k.startswith("in/")}
    sm = O.smooth(a, O.solve(a, J=int(z["J"])))
    for k in ("K", "k", "states", "controls"):
        assert rel_err(sm[k], z["smooth/" + k]) <= 1e-13, k
    assert abs(sm["objective"] - float(z["smooth/objective"])) <= 1e-13 * abs(float(z["smooth/objective"]))
    # the demo's stored smoothed rollouts (demo.py: smoothed_undisturbed.csv)
    np.testing.assert_allclose(sm["states"], z["csv_smoothed_undisturbed"][:, :2], rtol=0, atol=1e-12)
    for name in SMOOTH_FIXTURES:
        zz = np.load(os.path.join(GOLDEN, name + ".npz"))
        cfg = synth.CONFIGS[int(zz["cfg_id"])].scaled(T=int(zz["T"]), J=int(zz["J"]))
        batch = synth.generate_batch(cfg, seed=int(zz["seed"]), count=1)
        a = O.problem_slice(batch, 0)
        sm = O.smooth(a, O.solve(a, J=cfg.J))
        for k in ("K", "k", "states", "controls"):
            assert rel_err(sm[k], zz[k]) <= 1e-12, (name, k)
        assert abs(sm["objective"] - float(zz["objective"])) <= 1e-12 * abs(float(zz["objective"]))
        assert sm["smooth_deviation"] <= 1e-8 and float(zz["deviation"]) <= 1e-8


def test_oracle_endpoint_unreachable_matches_reference():
    """Two-point-boundary problems with unreachable endpoint directions
    (T m < n): the reference's own gains, maps, gradient-dual multipliers
    (endpoint.py:566-587) and trajectories (tests/golden/endpoint_unreachable.npz)."""
    import os

    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "endpoint_unreachable.npz"))
    for i in range(int(z["num"])):
        a = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/in/")}
        o = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/out/")}
        aff = O.solve_endpoint_affine(a)
        assert "Lam" not in aff and aff["feas"][0].shape[0] == int(o["feas_rows"])
        scale = 1.0 + max(float(np.abs(v).max()) for v in a.values())
        for k in ("Kx", "Kz", "k1", "X", "S"):
            assert np.abs(aff[k] - o[k]).max() <= 1e-12 * scale * (1 + np.abs(o[k]).max()), k
        for k, v in zip(("Hx", "Hz", "h1"), aff["feas"]):
            assert np.abs(v - o[k]).max() <= 1e-11 * scale, k
        ev = O.evaluate_endpoint(a, aff, a["x_init"], o["x_term"])
        for k in ("states", "controls", "lambdas", "mu"):
            assert np.abs(ev[k] - o[k]).max() <= 1e-11 * scale * (1 + np.abs(o[k]).max()), k
        assert abs(ev["objective"] - float(o["objective"])) <= 1e-11 * scale * (1 + abs(float(o["objective"])))
        assert ev["feas_residual"] <= 1e-9 * scale
        bad = O.evaluate_endpoint(a, aff, a["x_init"], o["x_bad"])
        assert bad["feas_residual"] == pytest.approx(float(o["bad_residual"]), rel=1e-9)
