"""Run the sweep phase (plq_sweep_segments) of a config a few times -- the
command profiled by ncu (tools/r2_final.sh).

    python tools/run_sweep.py --config 4 --B 148 --reps 2
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--B", type=int, default=None)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--phase", default="sweep", choices=("sweep", "link", "recon", "solve"))
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--J", type=int, default=None)
    args = ap.parse_args()
    import torch

    from paper_1809_06360_b200 import BatchSolver, _native, synth
    cfg = synth.CONFIGS[args.config]
    B = args.B or cfg.B
    cfg = cfg.scaled(B=B, T=args.T or cfg.T, J=args.J or cfg.J)
    dev = torch.device("cuda", 0)
    batch = synth.generate_batch_parallel(cfg, seed=0, count=B)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    s = BatchSolver(B, cfg.T, cfg.n, cfg.m, J=cfg.J, device=dev)
    s.run(inputs)
    lib = _native.lib()
    prob = s._problem_struct(inputs)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    ws = (ctypes.c_void_p(s.workspace.data_ptr()), s.ws_bytes, st)
    calls = {
        "sweep": lambda: lib.plq_sweep_segments(ctypes.byref(prob), ctypes.byref(s._outs), 0, cfg.J, *ws),
        "link": lambda: lib.plq_link_solve(ctypes.byref(prob), ctypes.byref(s._outs), *ws),
        "recon": lambda: lib.plq_reconstruct_segments(ctypes.byref(prob), ctypes.byref(s._outs), 0, cfg.J, None,
                                                      *ws),
        "solve": lambda: s.run(inputs) or 0,
    }
    for _ in range(args.reps):
        _native.check(calls[args.phase](), args.phase)
    torch.cuda.synchronize()
    s.raise_for_status()
    print("ok", cfg.name, B, args.phase)


if __name__ == "__main__":
    main()
