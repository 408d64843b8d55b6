"""One solve of a BASELINE config with a reduced batch / horizon, for ncu
captures: python tools/prof_run.py CFG [B] [T] [J] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1809_06360_b200 import BatchSolver, synth  # noqa: E402


def main():
    cid = int(sys.argv[1])
    cfg = synth.CONFIGS[cid]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.B
    T = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.T
    J = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.J
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    cfg = cfg.scaled(B=B, T=T, J=J)
    host = synth.generate_batch(cfg, seed=0, count=B)
    dev = torch.device("cuda", 0)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in host.items()}
    s = BatchSolver(B, T, cfg.n, cfg.m, J=J, device=dev)
    for _ in range(reps):
        s.run(inputs)
    torch.cuda.synchronize()
    s.raise_for_status()
    print("ok", cfg)


if __name__ == "__main__":
    main()
