import os
import sys

# the CPU oracle runs many tiny BLAS calls (and fork pools of them):
# multi-threaded OpenBLAS is pathologically slow there
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

try:  # numpy may already be loaded by a plugin: limit its BLAS pool too
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
except Exception:  # noqa: BLE001
    pass
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = float(np.abs(b).max()) if b.size else 0.0
    diff = float(np.abs(a - b).max()) if b.size else 0.0
    return diff / den if den else diff


def load_stored(name):
    """Ragged fixture (tests/golden/make_golden.py:stored_case) -> list of (inputs, outputs, J)."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cases = []
    for i in range(int(z["num"])):
        a = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/in/")}
        o = {k.split("/")[-1]: z[k] for k in z.files if k.startswith(f"{i}/out/")}
        cases.append((a, o, int(z[f"{i}/J"])))
    return cases


def load_synth(name):
    """Seeded-config fixture -> (cfg, batch arrays, golden npz)."""
    from paper_1809_06360_b200 import synth
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = synth.CONFIGS[int(z["cfg_id"])].scaled(T=int(z["T"]), J=int(z["J"]))
    batch = synth.generate_batch(cfg, seed=int(z["seed"]), count=int(z["count"]))
    return cfg, batch, z


SYNTH_FIXTURES = ("cfg0_seed0", "cfg1_first4", "cfg2_shape_T256_J4", "cfg3_shape_T16_J2",
                  "cfg4_shape_T64_J2")


@pytest.fixture(params=["specialized", "generic"])
def kernel_path(request, monkeypatch):
    # PLQ_FORCE_GENERIC=1 routes the config shapes through the generic kernels
    if request.param == "generic":
        monkeypatch.setenv("PLQ_FORCE_GENERIC", "1")
    else:
        monkeypatch.delenv("PLQ_FORCE_GENERIC", raising=False)
    return request.param
