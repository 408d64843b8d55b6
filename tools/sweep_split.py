"""Per-stage cost of constrained tail stages vs plain stages in the n=12
sweep: time plq_sweep_segments on the cfg1 batch at J = 8, 4, 2 (same T,
same data) and fit t = a * tail_stages + b * plain_stages."""
import ctypes
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1809_06360_b200 import BatchSolver, _native, synth  # noqa: E402

cfg = synth.CONFIGS[1]
host = synth.generate_batch(cfg, seed=0)
dev = torch.device("cuda", 0)
inputs = {k: torch.from_numpy(v).to(dev) for k, v in host.items()}
lib = _native.lib()
rows = []
for J in (8, 4, 2):
    s = BatchSolver(cfg.B, cfg.T, cfg.n, cfg.m, J=J, device=dev)
    s.run(inputs)
    prob = s._problem_struct(inputs)
    st = torch.cuda.current_stream(dev)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        lib.plq_sweep_segments(ctypes.byref(prob), ctypes.byref(s._outs), 0, J, ctypes.c_void_p(s.workspace.data_ptr()),
                               s.ws_bytes, ctypes.c_void_p(st.cuda_stream))
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = statistics.median(x.elapsed_time(y) for x, y in ts)
    L = cfg.T // J
    tail = (J - 1) * 3                     # n/m = 3 constrained stages per endpoint segment
    plain = (J - 1) * (L - 3) + L          # the rest + the serial last segment
    rows.append((J, ms, tail, plain))
    print(json.dumps({"J": J, "sweep_ms": ms, "tail_stages_per_problem": tail, "plain_stages_per_problem": plain}))
A = np.array([[r[2], r[3]] for r in rows], dtype=float)
y = np.array([r[1] for r in rows])
coef, *_ = np.linalg.lstsq(A, y, rcond=None)
print(json.dumps({"ms_per_tail_stage_per_problem_batch": coef[0], "ms_per_plain_stage": coef[1],
                  "tail_share_at_J8": coef[0] * rows[0][2] / rows[0][1]}))
