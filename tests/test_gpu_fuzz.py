"""Randomised GPU parity over odd shapes: n = 1..9, m = 1..5 (m > n, n % m != 0
mixed branch), J up to T (one-stage segments), random unbalanced partitions,
generated alternately by the reference's own generator restated
(``synth.generate_reference_recipe``, generate.py:14-47: cross term
``Qux = 0.3 N(0,1)``, spectral radius 1.05) and by the BASELINE recipe with a
cross term (``synth.generate_one(..., cross=0.3)``).  Non-degenerate partitions are compared with the
oracle (max(1e-9, 10 * floor) on x/u/lambda, 1e-9 on K and the objective);
degenerate ones (feasibility-constrained link path) must reach the method's
own KKT accuracy and link mismatch (test_parallel.py:131-135, 105-119)."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import parlqr_oracle as O

pytestmark = pytest.mark.gpu


def _cases(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(count):
        n = int(rng.integers(1, 10))
        m = int(rng.integers(1, 6))
        T = int(rng.integers(2, 41))
        J = int(rng.integers(2, min(T, 12) + 1))    # J = 1: test_single_segment_matches_serial_riccati
        if rng.random() < 0.4 and J > 1:
            cuts = np.sort(rng.choice(np.arange(1, T), size=J - 1, replace=False))
            splits = (0, *(int(c) for c in cuts), T)
        else:
            splits = None
        out.append((n, m, T, J, splits, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("block", range(4))
def test_random_shapes_and_partitions(block):
    from paper_1809_06360_b200 import Partition, solve_parallel_batch, synth
    checked = degenerate = 0
    for c, (n, m, T, J, splits, seed) in enumerate(_cases(40, 1000 + block)):
        if c % 2 == 0:
            a = synth.generate_reference_recipe(n, m, T, seed=seed)
        else:
            a = synth.generate_one(n, m, T, seed=seed, cross=0.3)
        sp = splits if splits is not None else tuple(O.make_partition(T, J))
        part = Partition(len(sp) - 1, tuple(sp))
        s = solve_parallel_batch({k: v[None] for k, v in a.items()}, partition=part)
        g = {k: (v.cpu().numpy()[0] if v is not None else None) for k, v in s.out.items()}
        sc = 1.0 + max(float(np.abs(v).max()) for v in a.values())
        rows = g["feas_rows"]
        if len(sp) > 2 and np.any(rows[:len(sp) - 2] > 0):
            degenerate += 1
            assert g["kkt_inf"] <= 1e-7 * sc, (n, m, T, sp, g["kkt_inf"])
            assert g["link_mismatch"] <= 1e-7 * sc
            continue
        ref = O.solve(a, splits=sp)
        fl = {}
        for t in range(2):
            r = O.solve(O.perturbed(a, 1e-15, 50 + t), splits=sp)
            for key in ("states", "controls", "lambdas", "k"):
                fl[key] = max(fl.get(key, 0.0), rel_err(r[key], ref[key]))
        for key, rk in (("x", "states"), ("u", "controls"), ("lam", "lambdas"), ("k", "k")):
            gate = max(1e-9, 10 * fl[rk])
            assert rel_err(g[key], ref[rk]) <= gate, (key, n, m, T, sp, rel_err(g[key], ref[rk]), gate)
        assert rel_err(g["K"], ref["K"]) <= 1e-9, (n, m, T, sp)
        assert abs(g["objective"] - ref["objective"]) <= 1e-9 * max(1.0, abs(ref["objective"]))
        checked += 1
    assert checked >= 20
