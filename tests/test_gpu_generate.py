"""The device-side seeded generator (plq_generate_batch)
against the host restatement of its stream, and a solve of device-generated
problems against the oracle."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import parlqr_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_id,T,count,first", [(1, 16, 3, 0), (4, 8, 2, 5), (3, 3, 1, 2), (2, 9, 2, 1)])
def test_device_generator_matches_host_restatement(cfg_id, T, count, first):
    from paper_1809_06360_b200 import synth
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=1)
    dev = {k: v.cpu().numpy() for k, v in synth.generate_batch_device(cfg, seed=7, count=count, first=first).items()}
    for i in range(count):
        ref = synth.device_stream_reference(cfg, seed=7, problem=first + i)
        for k, v in ref.items():
            assert dev[k][i].shape == v.shape
            # CUDA log / sincospi vs libm: last-bit differences, amplified by the Gram products
            assert np.abs(dev[k][i] - v).max() <= 1e-12 * (1.0 + np.abs(v).max()), k
    for k in ("Qxx", "Quu", "QxxT"):
        assert np.array_equal(dev[k], np.swapaxes(dev[k], -1, -2)), k          # exactly symmetric
    assert np.linalg.eigvalsh(dev["Qxx"][0, 0]).min() > 0 and np.linalg.eigvalsh(dev["Quu"][0, 0]).min() > 0
    assert not dev["Qux"].any()


def test_device_generator_is_launch_shape_independent():
    """Pieces generated with first_problem offsets equal one call, bit for bit;
    another seed gives another batch."""
    from paper_1809_06360_b200 import synth
    cfg = synth.CONFIGS[1].scaled(T=16, J=2)
    whole = synth.generate_batch_device(cfg, seed=3, count=6)
    a = synth.generate_batch_device(cfg, seed=3, count=2, first=0)
    b = synth.generate_batch_device(cfg, seed=3, count=4, first=2)
    other = synth.generate_batch_device(cfg, seed=4, count=6)
    for k in whole:
        w = whole[k].cpu().numpy()
        assert np.array_equal(w[:2], a[k].cpu().numpy()) and np.array_equal(w[2:], b[k].cpu().numpy()), k
        if k != "Qux":
            assert not np.array_equal(w, other[k].cpu().numpy()), k
    g = whole["Fx"].cpu().numpy() - np.eye(cfg.n)
    z = g.ravel() * np.sqrt(cfg.n) / cfg.a_scale               # 6 * 16 * 144 standard normals
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.05


@pytest.mark.parametrize("cfg_id,T,J,count", [(4, 128, 4, 3), (1, 64, 8, 16)])
def test_solve_of_device_generated_batch_matches_oracle(cfg_id, T, J, count):
    from paper_1809_06360_b200 import solve_parallel_batch, synth
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    inputs = synth.generate_batch_device(cfg, seed=1, count=count)
    s = solve_parallel_batch(inputs, J=J)
    host = {k: v.cpu().numpy() for k, v in inputs.items()}
    g = {k: v.cpu().numpy() for k, v in s.out.items() if v is not None}
    for i in (0, count - 1):
        prob = O.problem_slice(host, i)
        ref = O.solve(prob, J=J)
        fl = max(rel_err(O.solve(O.perturbed(prob, 1e-15, 100), J=J)["states"], ref["states"]), 1e-10)
        assert rel_err(g["K"][i], ref["K"]) <= 1e-9
        assert rel_err(g["x"][i], ref["states"]) <= 10 * fl
        assert abs(g["objective"][i] - ref["objective"]) <= 1e-9 * abs(ref["objective"])
