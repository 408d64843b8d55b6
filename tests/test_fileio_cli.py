"""JSON problem / solution files and the CLI ``solve`` path
(``parlqr`` fileio.py:1-98, cli.py:26-59), against files the reference
wrote itself (tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err

PROBLEM = os.path.join(GOLDEN, "json_problem_n3_m2_T12.json")
SOLUTION = os.path.join(GOLDEN, "json_solution_parallel_J3.json")


def test_reference_problem_file_round_trips_byte_identical(tmp_path):
    from paper_1809_06360_b200 import fileio
    prob = fileio.load_problem(PROBLEM)
    assert (prob.n, prob.m, prob.T) == (3, 2, 12)
    out = tmp_path / "p.json"
    fileio.save_problem(prob, out)
    assert out.read_bytes() == open(PROBLEM, "rb").read()


def test_declared_dimensions_are_checked(tmp_path):
    from paper_1809_06360_b200 import fileio
    data = json.load(open(PROBLEM))
    data["T"] = 13
    with pytest.raises(ValueError):
        fileio.problem_from_dict(data)


def test_solution_dict_layout():
    from paper_1809_06360_b200 import LqrSolution, fileio
    ref = json.load(open(SOLUTION))
    sol = LqrSolution(states=np.zeros((13, 3)), controls=np.zeros((12, 2)), lambdas=np.zeros((13, 3)),
                      policies=(), objective=1.5, kkt_residual_inf=0.0)
    d = fileio.solution_to_dict(sol, solver="parallel", timing_seconds=0.1)
    assert set(d) == set(ref)


def test_cli_io_and_data_errors(tmp_path):
    from paper_1809_06360_b200 import cli
    assert cli.main(["solve", "--problem", str(tmp_path / "nope.json"), "--out", str(tmp_path / "o")]) == cli.EXIT_IO
    data = json.load(open(PROBLEM))
    data["stages"][4]["Fx"][0][0] = float("nan")
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(data))
    assert cli.main(["solve", "--problem", str(bad), "--solver", "parallel", "--out",
                     str(tmp_path / "o.json")]) == cli.EXIT_NUMERICAL


@pytest.mark.gpu
def test_cli_solve_parallel_matches_reference_solution_file(tmp_path):
    from paper_1809_06360_b200 import cli
    out = tmp_path / "sol.json"
    assert cli.main(["solve", "--problem", PROBLEM, "--solver", "parallel", "--J", "3", "--workers", "1",
                     "--out", str(out)]) == cli.EXIT_OK
    got, ref = json.load(open(out)), json.load(open(SOLUTION))
    assert set(got) == set(ref) and got["solver"] == "parallel"
    assert abs(got["objective"] - ref["objective"]) <= 1e-9 * abs(ref["objective"])
    for key in ("states", "controls", "multipliers"):
        assert rel_err(np.array(got[key]), np.array(ref[key])) <= 1e-9, key
    assert got["kkt_residual"] <= max(10 * ref["kkt_residual"], 1e-9)


@pytest.mark.gpu
def test_cli_solve_with_smoothing(tmp_path):
    from oracle import parlqr_oracle as O
    from paper_1809_06360_b200 import cli, fileio, stack_problem
    out = tmp_path / "sol.json"
    assert cli.main(["solve", "--problem", PROBLEM, "--J", "3", "--smooth", "--out", str(out)]) == cli.EXIT_OK
    a = dict(stack_problem(fileio.load_problem(PROBLEM)))
    ref = O.smooth(a, O.solve(a, J=3))
    got = json.load(open(out))
    assert rel_err(np.array(got["states"]), ref["states"]) <= 1e-9
    assert abs(got["objective"] - ref["objective"]) <= 1e-9 * abs(ref["objective"])
