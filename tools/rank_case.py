"""One solve of each reference-written near-threshold rank case
(tests/golden/rank_near.npz): the fast sweeps flag the segment and the
rank-revealing repair pass re-solves it (sanitizer driver)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import load_stored  # noqa: E402

from paper_1809_06360_b200 import Partition, solve_parallel_batch  # noqa: E402

for a, o, J in load_stored("rank_near"):
    sp = tuple(int(s) for s in o["splits"])
    s = solve_parallel_batch({k: v[None] for k, v in a.items()}, partition=Partition(len(sp) - 1, sp))
    assert np.isfinite(s.out["x"].cpu().numpy()).all()
print("rank cases ok")
