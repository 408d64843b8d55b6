"""The drop-in speaks the reference's types and exceptions when ``parlqr`` is
importable: a caller that switched
``parlqr.solve_parallel`` to the GPU path keeps catching
``parlqr.SolverError`` and the reference CLI keeps its exit codes
(cli.py:20-23, 47-52).  No GPU needed: the GPU's per-segment status codes
are fed through the same mapping the solver uses (``raise_for_status``).

Runs in a subprocess with the reference on ``PYTHONPATH`` (this container
only; the reference is not on the GPU box).
"""

import os
import subprocess
import sys
import textwrap

import pytest

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r'''
    import json, os, sys, tempfile
    import numpy as np
    import parlqr, parlqr.cli, parlqr.fileio, parlqr.parallel
    import paper_1809_06360_b200 as plq
    from paper_1809_06360_b200 import _native, synth
    from paper_1809_06360_b200.parallel import raise_for_status, solution_from_outputs

    # 1. the reference's own classes are re-exported
    assert plq.USING_REFERENCE_TYPES
    assert plq.LqrSolution is parlqr.LqrSolution and plq.AffinePolicy is parlqr.AffinePolicy
    assert plq.LqrProblem is parlqr.LqrProblem and plq.Partition is parlqr.parallel.Partition
    assert plq.ParallelDetails is parlqr.parallel.ParallelDetails
    assert plq.make_partition(10, 3) == parlqr.parallel.make_partition(10, 3)

    # 2. results are built as the reference's types
    n, m, T, J = 3, 2, 6, 2
    o = {"x": np.zeros((T + 1, n)), "u": np.zeros((T, m)), "lam": np.zeros((T + 1, n)),
         "K": np.ones((T, m, n)), "k": np.ones((T, m)), "links": np.zeros((1, n)),
         "mu_left": np.zeros((1, n)), "lambda_right": np.zeros((1, n)),
         "vf0": np.zeros((J, 3 * n * n + 2 * n)), "objective": np.array(1.5), "kkt_inf": np.array(0.0),
         "link_mismatch": np.array(0.0), "link_residual": np.array(0.0),
         "feas_rows": np.zeros(J, dtype=np.int32), "feas": np.zeros((J, n, 2 * n + 1)),
         "feas_residual": np.zeros(J)}
    sol = solution_from_outputs(o, plq.make_partition(T, J))
    assert type(sol) is parlqr.LqrSolution
    assert type(sol.details) is parlqr.parallel.ParallelDetails
    assert type(sol.details.partition) is parlqr.parallel.Partition
    assert type(sol.policies[0]) is parlqr.AffinePolicy and sol.policies[0](np.ones(n)).shape == (m,)
    assert sol.details.segment_diagnostics == (None, None)

    # 2b. collect_diagnostics: the reference's StageDiagnostics per endpoint segment, None for the last
    import parlqr.endpoint
    od = dict(o, diag=np.array([[1e-16, 2e-16], [0.0, 0.0]]), diag_rows=np.array([n, 0], dtype=np.int32))
    sd = solution_from_outputs(od, plq.make_partition(T, J)).details.segment_diagnostics
    assert type(sd[0]) is parlqr.endpoint.StageDiagnostics and sd[1] is None
    assert (sd[0].basis_defect, sd[0].projector_defect, sd[0].max_rows) == (1e-16, 2e-16, n)

    # 2c. the oracle's restatement of the diagnostics equals the reference's (endpoint.py:258-299)
    sys.path.insert(0, os.environ["PLQ_REPO_ROOT"])
    from oracle import parlqr_oracle as O
    from parlqr.generate import generate
    for (dn, dm, dT, seed) in [(5, 2, 9, 3), (6, 3, 8, 4), (4, 1, 10, 5)]:
        pr = generate(dn, dm, dT, seed=seed)
        bw = parlqr.endpoint.backward_pass(pr.stages, None, collect_diagnostics=True)
        arr = plq.parallel.stack_problem(pr)
        d = O.endpoint_sweep({f: arr[f] for f in O.STAGE_FIELDS})["diagnostics"]
        assert d["basis_defect"] == bw.diagnostics.basis_defect
        assert d["projector_defect"] == bw.diagnostics.projector_defect
        assert d["max_rows"] == bw.diagnostics.max_rows

    # 3. status codes -> the reference's exception classes
    cases = [(np.array([[0, 3]]), parlqr.errors.CholeskyFailure, "stage", 2),
             (np.array([[_native.PLQ_STATUS_LINK_SINGULAR, 0]]), parlqr.errors.LinkSingular, None, None),
             (np.array([[0, _native.PLQ_STATUS_INFEASIBLE]]), parlqr.errors.Infeasible, "segment", 1)]
    for st, cls, attr, val in cases:
        try:
            raise_for_status(st, np.full(st.shape, 0.5))
        except parlqr.SolverError as exc:
            assert isinstance(exc, cls), (type(exc), cls)
            if attr:
                assert getattr(exc, attr) == val
        else:
            raise AssertionError("no exception")

    # 4. the reference CLI after the INTEGRATION.md monkeypatch: exit codes
    #    3 (numerical failure) and 2 (infeasible) for GPU-reported failures
    a = synth.generate_one(3, 2, 8, seed=1)
    prob = plq.problem_from_arrays(a)
    d = tempfile.mkdtemp()
    pf = os.path.join(d, "p.json")
    parlqr.fileio.save_problem(prob, pf)
    for st, code in ((np.array([[0, 2]]), 3), (np.array([[_native.PLQ_STATUS_LINK_SINGULAR, 0]]), 3),
                     (np.array([[_native.PLQ_STATUS_INFEASIBLE, 0]]), 2)):
        def gpu_solve(problem, J, workers=None, _st=st, **kw):
            raise_for_status(_st, np.full(_st.shape, 0.25))   # what BatchSolver does with the GPU status
        parlqr.solve_parallel = parlqr.parallel.solve_parallel = gpu_solve
        rc = parlqr.cli.main(["solve", "--problem", pf, "--solver", "parallel", "--J", "2",
                              "--out", os.path.join(d, "s.json")])
        assert rc == code, (st, rc, code)
    print("contract ok")
''')


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted (GPU box)")
def test_reference_types_and_error_contract():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF_SRC, ROOT]), PYTHONDONTWRITEBYTECODE="1", PLQ_REPO_ROOT=ROOT)
    env.pop("PLQ_NO_PARLQR", None)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "contract ok" in r.stdout


def test_stand_ins_without_parlqr():
    """Without parlqr the stand-in classes keep the reference's conventions."""
    env = dict(os.environ, PYTHONPATH=ROOT, PLQ_NO_PARLQR="1")
    code = textwrap.dedent('''
        import numpy as np
        import paper_1809_06360_b200 as plq
        from paper_1809_06360_b200 import synth
        assert not plq.USING_REFERENCE_TYPES
        a = synth.generate_one(3, 2, 4, seed=2)
        a["Qxx"][0, 0, 1] += 1e-3                       # asymmetric input is symmetrized
        p = plq.problem_from_arrays(a)
        Q = p.stages[0][0].Qxx
        assert np.array_equal(Q, Q.T) and p.stages[0][0].asymmetry > 0
        assert not Q.flags.writeable
        pol = plq.AffinePolicy.state_feedback(np.ones((2, 3)), np.zeros(2))
        assert np.array_equal(pol(np.ones(3)), [3.0, 3.0])
        try:
            plq.AffinePolicy(np.ones((2, 3)), np.ones((2, 3)), np.zeros(2))(np.ones(3))
        except ValueError:
            pass
        else:
            raise AssertionError
        e = plq.CholeskyFailure(4, segment=2)
        assert isinstance(e, plq.SolverError) and e.stage == 4 and "stage 4" in str(e)
        print("stand-ins ok")
    ''')
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
