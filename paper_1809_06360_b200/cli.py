"""Command-line ``solve`` of the partitioned path (``parlqr`` ``cli.py:26-59``,
``build_parser`` ``:97-107``): same flags, same exit codes, same solution
file.  Only ``--solver parallel`` is provided (the serial and dense-KKT
solvers are not part of the B200 path).

Exit codes: 0 success, 1 I/O or parse error, 2 endpoint constraints
infeasible, 3 numerical failure (including invalid problem data).
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import fileio
from .errors import Infeasible, SolverError
from .parallel import smooth, solve_parallel, stack_problem

EXIT_OK = 0
EXIT_IO = 1
EXIT_INFEASIBLE = 2
EXIT_NUMERICAL = 3


def _cmd_solve(args):
    try:
        problem = fileio.load_problem(args.problem)
    except (OSError, ValueError, KeyError, TypeError, json.JSONDecodeError) as exc:
        print(f"error: cannot read problem file: {exc}", file=sys.stderr)
        return EXIT_IO
    # the numeric part of problem.validate (problem.py:298-340) the GPU
    # would otherwise turn into NaNs: non-finite data
    bad = [f for f, v in stack_problem(problem).items() if not np.all(np.isfinite(v))]
    if bad:
        for f in bad:
            print(f"error: non-finite entries in {f}", file=sys.stderr)
        return EXIT_NUMERICAL
    try:
        tic = time.perf_counter()
        solution = solve_parallel(problem, J=args.J, workers=args.workers)
        if args.smooth:
            solution = smooth(problem, solution, workers=args.workers)
        elapsed = time.perf_counter() - tic
    except Infeasible as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INFEASIBLE
    except SolverError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL
    try:
        fileio.save_solution(solution, args.out, solver=args.solver, timing_seconds=elapsed)
    except OSError as exc:
        print(f"error: cannot write solution: {exc}", file=sys.stderr)
        return EXIT_IO
    return EXIT_OK


def build_parser():
    parser = argparse.ArgumentParser(prog="paper_1809_06360_b200",
                                     description="Partition-parallel LQR solve on a B200")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("solve", help="solve a problem file")
    p.add_argument("--problem", required=True)
    p.add_argument("--solver", choices=("parallel",), default="parallel")
    p.add_argument("--J", type=int, default=2)
    p.add_argument("--workers", type=int, default=None)
    p.add_argument("--smooth", action="store_true", help="apply the smoothing pass (parallel.smooth)")
    p.add_argument("--out", required=True)
    p.set_defaults(func=_cmd_solve)
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
