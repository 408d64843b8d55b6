"""Per-phase cycle breakdown of the specialized sweep (measurement build).

    python -m paper_1809_06360_b200.build --profile
    PLQ_LIB_PATH=paper_1809_06360_b200/libparlqr_b200_prof.so python tools/phase_profile.py --config 4 [--B 64]

Runs plq_sweep_segments a few times on the config's seeded inputs and prints
the share of group-0 thread-0 cycles spent in each stage phase, summed over
CTAs (clock64 deltas at the phase boundaries of sweep_small_kernel).
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = ["copy wait", "f1 column", "GEMM1", "GEMM2", "tail (QR)", "Cholesky solve", "policy stores",
         "value update", "stage end / prologue", "Cholesky factor (+fused fwd solve)",
         "tail: norms + N = Hx F", "tail: QR (n=64: + Cholesky trailing tiles)", "GEMM2 k-loops (warp 0)",
         "value-update k-loops (warp 0)", "GEMM1 k-loops (warp 0)", "Cholesky diag factor + panel (n=64)"]


GENERIC_NAMES = ["stage start (input staging / loop)", "GEMM1 (+ f1 column)", "GEMM2 (+ w column)",
                 "tail: negate / certificates / row shift (rest of the constrained stage)", "Cholesky factor (+ fused forward solve)", "backward solve",
                 "policy stores", "Y = P + Muu G (constrained stages)", "value update (+ constant column)",
                 "tail: norms + N = Hx F", "tail: stack copy", "tail: Householder QR (gqr8)",
                 "tail: R inverse + back substitution", "-", "-", "-"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--generic", action="store_true", help="the generic sweep's counters (plq_sweep_impl.cuh)")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--B", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_1809_06360_b200 import BatchSolver, _native, synth
    assert "prof" in _native.LIB_PATH, "set PLQ_LIB_PATH to the _prof library"
    cfg = synth.CONFIGS[args.config]
    B = args.B or cfg.B
    cfg = cfg.scaled(B=B)
    dev = torch.device("cuda", 0)
    batch = synth.generate_batch_parallel(cfg, seed=0, count=B)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    s = BatchSolver(B, cfg.T, cfg.n, cfg.m, J=cfg.J, device=dev)
    lib = _native.lib()
    lib.plq_debug_phase_cycles.argtypes = [ctypes.c_void_p]
    lib.plq_debug_phase_cycles.restype = ctypes.c_int
    buf = np.zeros((1024, 16), dtype=np.uint64)
    prob = s._problem_struct(inputs)
    stream = torch.cuda.current_stream(dev)
    run = lambda: lib.plq_sweep_segments(ctypes.byref(prob), ctypes.byref(s._outs), 0, cfg.J,
                                         ctypes.c_void_p(s.workspace.data_ptr()), s.ws_bytes,
                                         ctypes.c_void_p(stream.cuda_stream))
    run()
    torch.cuda.synchronize()
    reader = lib.plq_debug_phase_cycles_generic if args.generic else lib.plq_debug_phase_cycles
    reader.argtypes = [ctypes.c_void_p]
    reader.restype = ctypes.c_int
    reader(ctypes.c_void_p(buf.ctypes.data))   # reset
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.reps):
        _native.check(run(), "sweep")
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.reps
    assert reader(ctypes.c_void_p(buf.ctypes.data)) == 0
    tot = buf.sum(axis=0).astype(np.float64)
    global NAMES
    if args.generic:
        NAMES = GENERIC_NAMES
    ctas = int((buf.sum(axis=1) > 0).sum())   # CTAs >= 1024 fold onto blockIdx % 1024
    stages = B * cfg.T * args.reps
    out = {"config": cfg.name, "B": B, "sweep_ms": ms, "ctas": ctas,
           "cycles_per_stage": float(tot.sum() / stages) * ctas / max(ctas, 1),
           "share": {NAMES[k]: float(tot[k] / tot.sum()) for k in range(16) if tot[k] > 0},
           "cycles_per_stage_by_phase": {NAMES[k]: float(tot[k] / stages) for k in range(16) if tot[k] > 0}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
