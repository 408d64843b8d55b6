"""The phase entry points (plq_sweep_segments ... plq_finalize) driven by the
horizon-sharding orchestration on a real GPU: a world-size-1 NCCL group must
reproduce the one-call solve bitwise."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cfg_id,T,J", [(2, 512, 16), (1, 64, 8), (4, 64, 4)])
def test_phases_equal_one_call_solve(cfg_id, T, J):
    import torch
    import torch.distributed as dist

    from paper_1809_06360_b200 import solve_parallel_batch, synth
    from paper_1809_06360_b200.sharded import sharded_solve_device
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    batch = synth.generate_batch(cfg, seed=5, count=2)
    ref = solve_parallel_batch(batch, J=J)
    dev = torch.device("cuda", 0)
    inputs = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    try:
        solver, res = sharded_solve_device(inputs, J=J, dist=dist)
        torch.cuda.synchronize()
        for k in ("K", "k", "x", "u", "lam", "links", "objective", "kkt_inf", "link_mismatch", "link_residual"):
            a = solver.out[k].cpu().numpy()
            b = ref.out[k].cpu().numpy()
            assert np.array_equal(a, b), k
    finally:
        dist.destroy_process_group()
