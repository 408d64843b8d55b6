"""ctypes binding of the C ABI in ``include/parlqr_b200.h``.

This is the binding a maintainer of the reference would add.
The library is mandatory: there is no CPU fallback, and a missing or stale
``libparlqr_b200.so`` raises at first use.
"""

from __future__ import annotations

import ctypes
import os

LIB_PATH = os.environ.get("PLQ_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                          "libparlqr_b200.so")

PLQ_OK = 0
PLQ_STATUS_DEGENERATE = -1
PLQ_STATUS_LINK_SINGULAR = -2
PLQ_STATUS_INFEASIBLE = -3
PLQ_STATUS_BAD_PARTITION = -4

# every entry point declared in include/parlqr_b200.h
EXPORTS = (
    "plq_abi_version", "plq_last_error", "plq_workspace_bytes", "plq_solve_parallel",
    "plq_host_arena_bytes", "plq_solve_parallel_host", "plq_sweep_segments",
    "plq_link_solve", "plq_reconstruct_segments", "plq_boundary_segments",
    "plq_finalize", "plq_last_launch_count", "plq_smooth", "plq_endpoint_workspace_bytes",
    "plq_endpoint_affine", "plq_endpoint_evaluate", "plq_solve_parallel_sharded",
    "plq_generate_batch",
)

_vp = ctypes.c_void_p


class PlqProblem(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int64), ("T", ctypes.c_int32), ("n", ctypes.c_int32),
        ("m", ctypes.c_int32), ("J", ctypes.c_int32), ("max_seg_len", ctypes.c_int32),
        ("split_times", _vp), ("Qxx", _vp), ("Qux", _vp), ("Quu", _vp), ("qx1", _vp),
        ("qu1", _vp), ("Fx", _vp), ("Fu", _vp), ("f1", _vp), ("QxxT", _vp), ("qx1T", _vp),
        ("x_init", _vp), ("rank_tol", ctypes.c_double), ("feas_tol", ctypes.c_double),
    ]


OUTPUT_FIELDS = ("K", "k", "x", "u", "lam", "links", "mu_left", "lambda_right", "vf0",
                 "Kz", "k1", "objective", "kkt_inf", "link_mismatch", "link_residual",
                 "status", "feas", "feas_rows", "feas_residual", "diag", "diag_rows")


class PlqOutputs(ctypes.Structure):
    _fields_ = [(f, _vp) for f in OUTPUT_FIELDS]


SMOOTH_FIELDS = ("K", "k", "x", "u", "objective", "kkt_inf", "deviation", "status")


class PlqSmoothOutputs(ctypes.Structure):
    _fields_ = [(f, _vp) for f in SMOOTH_FIELDS]


ENDPOINT_FIELDS = ("Kx", "Kz", "k1", "value0", "X", "S", "Lam", "E", "status", "gram_status", "feas", "feas_rows",
                   "diag", "diag_rows")


class PlqEndpointOutputs(ctypes.Structure):
    _fields_ = [(f, _vp) for f in ENDPOINT_FIELDS]


POINT_FIELDS = ("x_init", "x_term", "x", "u", "lam", "mu", "objective", "kkt_inf", "feas_residual")


class PlqEndpointPoint(ctypes.Structure):
    _fields_ = [(f, _vp) for f in POINT_FIELDS]


class PlqRecipe(ctypes.Structure):
    _fields_ = [("a_scale", ctypes.c_double), ("q_eps", ctypes.c_double), ("r_eps", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("first_problem", ctypes.c_int64)]


_LIB = None


def lib():
    """Load (once) and type the shared library; raise if it is missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1809_06360_b200.build` "
            "(the GPU path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(PlqProblem)
    O = ctypes.POINTER(PlqOutputs)
    L.plq_abi_version.restype = ctypes.c_int
    L.plq_last_error.restype = ctypes.c_char_p
    L.plq_last_launch_count.restype = ctypes.c_int
    L.plq_workspace_bytes.restype = ctypes.c_size_t
    L.plq_workspace_bytes.argtypes = [P]
    L.plq_host_arena_bytes.restype = ctypes.c_size_t
    L.plq_host_arena_bytes.argtypes = [P]
    L.plq_solve_parallel.argtypes = [P, O, _vp, ctypes.c_size_t, _vp]
    L.plq_solve_parallel_host.argtypes = [P, O, _vp, ctypes.c_size_t, _vp]
    L.plq_sweep_segments.argtypes = [P, O, ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_size_t, _vp]
    L.plq_link_solve.argtypes = [P, O, _vp, ctypes.c_size_t, _vp]
    L.plq_reconstruct_segments.argtypes = [P, O, ctypes.c_int32, ctypes.c_int32, _vp, _vp,
                                           ctypes.c_size_t, _vp]
    L.plq_boundary_segments.argtypes = [P, O, ctypes.c_int32, ctypes.c_int32, _vp, _vp,
                                        ctypes.c_size_t, _vp]
    L.plq_finalize.argtypes = [P, O, _vp, _vp, ctypes.c_size_t, _vp]
    L.plq_smooth.argtypes = [P, O, ctypes.POINTER(PlqSmoothOutputs), _vp, ctypes.c_size_t, _vp]
    EO = ctypes.POINTER(PlqEndpointOutputs)
    L.plq_endpoint_workspace_bytes.restype = ctypes.c_size_t
    L.plq_endpoint_workspace_bytes.argtypes = [P]
    L.plq_endpoint_affine.argtypes = [P, EO, _vp, ctypes.c_size_t, _vp]
    L.plq_endpoint_evaluate.argtypes = [P, EO, ctypes.POINTER(PlqEndpointPoint), _vp, ctypes.c_size_t, _vp]
    L.plq_generate_batch.argtypes = [P, ctypes.POINTER(PlqRecipe), _vp]
    L.plq_generate_batch.restype = ctypes.c_int
    L.plq_solve_parallel_sharded.argtypes = [P, O, _vp, ctypes.c_size_t, _vp, ctypes.c_int32, ctypes.c_int32, _vp]
    for name in ("plq_solve_parallel", "plq_solve_parallel_host", "plq_sweep_segments", "plq_solve_parallel_sharded",
                 "plq_link_solve", "plq_reconstruct_segments", "plq_boundary_segments",
                 "plq_finalize", "plq_smooth", "plq_endpoint_affine", "plq_endpoint_evaluate"):
        getattr(L, name).restype = ctypes.c_int
    if L.plq_abi_version() != 2:
        raise RuntimeError("libparlqr_b200.so ABI version mismatch; rebuild it")
    _LIB = L
    return L


def check(rc, what):
    if rc != PLQ_OK:
        msg = lib().plq_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")
