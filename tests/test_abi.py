"""The C-ABI library loads and exports every entry point include/*.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    names = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            names.update(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(plq_\w+)\s*\(", src, re.M))
    return names


def test_header_declares_entry_points():
    names = _declared()
    assert {"plq_solve_parallel", "plq_solve_parallel_host", "plq_workspace_bytes",
            "plq_sweep_segments", "plq_link_solve", "plq_reconstruct_segments",
            "plq_boundary_segments", "plq_finalize"} <= names


def test_library_exports_all_declared_symbols():
    from paper_1809_06360_b200 import build, _native
    build.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.EXPORTS) == _declared()


def test_abi_version_and_struct_layout():
    from paper_1809_06360_b200 import _native
    lib = _native.lib()
    assert lib.plq_abi_version() == 2
    # plq_problem_t: int64 + 5 int32 + 4 pad + 12 pointers + 2 doubles
    assert ctypes.sizeof(_native.PlqProblem) == 8 + 20 + 4 + 12 * 8 + 16
    assert ctypes.sizeof(_native.PlqOutputs) == 21 * 8


def test_argument_errors_without_gpu():
    # invalid shapes are rejected before any CUDA call
    from paper_1809_06360_b200 import _native
    lib = _native.lib()
    P = _native.PlqProblem()
    P.B, P.T, P.n, P.m, P.J, P.max_seg_len = 1, 4, 2, 1, 5, 1   # J > T
    assert lib.plq_workspace_bytes(ctypes.byref(P)) == 0
    assert b"J must be" in lib.plq_last_error()
