"""Horizon sharding across ranks (paper_1809_06360_b200/sharded.py) on CPU:
world-size-2 (and 3) gloo process groups drive the SAME orchestration code
as the NCCL/GPU path, with the CPU oracle as the per-phase backend.  Results
must equal the unsharded oracle solve (links bitwise, scalars to rounding)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import parlqr_oracle as O
from paper_1809_06360_b200 import synth
from paper_1809_06360_b200.sharded import shard_range, solve_sharded


class OracleBackend:
    """Per-phase CPU backend mirroring the C ABI phases' contracts."""

    def __init__(self, prob, splits):
        self.torch = torch
        self.prob, self.splits = prob, tuple(splits)
        self.J = len(splits) - 1
        self.n = n = prob["x_init"].shape[0]
        self.VS = 3 * n * n + 2 * n
        f64 = dict(dtype=torch.float64)
        self.vf0 = torch.zeros((1, self.J, self.VS), **f64)
        self.status = torch.zeros((1, self.J, 1), **f64)
        self.partials = torch.zeros((1, self.J, 3), **f64)
        self.mult = torch.zeros((1, self.J, 2 * n), **f64)
        self.segs, self.recon_out = {}, {}

    def _stage(self, j):
        lo, hi = self.splits[j], self.splits[j + 1]
        return {f: np.array(self.prob[f][lo:hi]) for f in O.STAGE_FIELDS}

    def sweep(self, j0, j1):
        n = self.n
        for j in range(j0, j1):
            if j == self.J - 1:
                seg = O.serial_sweep(self._stage(j), self.prob["QxxT"], self.prob["qx1T"])
                Vxx, vx1 = seg["vf0"]
                row = np.concatenate([Vxx.ravel(), np.zeros(2 * n * n), vx1, np.zeros(n)])
            else:
                seg = O.endpoint_sweep(self._stage(j))
                Vxx, Vzx, Vzz, vx1, vz1 = seg["vf0"]
                row = np.concatenate([Vxx.ravel(), Vzx.ravel(), Vzz.ravel(), vx1, vz1])
                if seg["feas"][0].shape[0]:
                    self.status[0, j, 0] = -1
            self.segs[j] = seg
            self.vf0[0, j] = torch.from_numpy(row)

    def vf0_rows(self, j0, j1):
        return self.vf0[:, j0:j1]

    def status_rows(self, j0, j1):
        return self.status[:, j0:j1]

    def set_vf0(self, vf0):
        self.vf0 = vf0.clone()

    def status_all(self):
        return np.zeros((1, self.J), dtype=np.int32)

    def _vf_tuple(self, j):
        n, nn = self.n, self.n * self.n
        row = self.vf0[0, j].numpy()
        Vxx, vx1 = row[:nn].reshape(n, n), row[3 * nn:3 * nn + n]
        if j == self.J - 1:
            return (Vxx, vx1)
        return (Vxx, row[nn:2 * nn].reshape(n, n), row[2 * nn:3 * nn].reshape(n, n), vx1,
                row[3 * nn + n:])

    def link(self):
        vf = [self._vf_tuple(j) for j in range(self.J)]
        diag, sub, rhs = O.link_system(vf, self.prob["x_init"])
        self.links, self.link_res = O.solve_links(diag, sub, rhs)

    def recon(self, j0, j1):
        p, n = self.prob, self.n
        for j in range(j0, j1):
            seg = dict(self.segs[j])
            seg["vf0"] = self._vf_tuple(j)
            r = O.reconstruct_segment(p, self.splits, j, seg, self.links)
            self.recon_out[j] = r
            lo, hi = self.splits[j], self.splits[j + 1]
            last = j == self.J - 1
            obj, worst = 0.0, 0.0
            lam_next = r["lam_T"] if last else None
            for s in range(hi - lo):
                t = lo + s
                x, u = r["xs"][s], r["us"][s]
                obj += 0.5 * (x @ (p["Qxx"][t] @ x)) + 0.5 * (u @ (p["Quu"][t] @ u))
                obj += u @ (p["Qux"][t] @ x) + p["qx1"][t] @ x + p["qu1"][t] @ u
                if s < hi - lo - 1 or last:
                    ln = r["lam"][s + 1] if s < hi - lo - 1 else lam_next
                    r1 = p["Qxx"][t] @ x + p["Qux"][t].T @ u + p["qx1"][t] + r["lam"][s] - p["Fx"][t].T @ ln
                    r2 = p["Qux"][t] @ x + p["Quu"][t] @ u + p["qu1"][t] - p["Fu"][t].T @ ln
                    worst = max(worst, float(np.abs(r1).max()), float(np.abs(r2).max()))
            if last:
                xT = r["xs"][-1]
                obj += 0.5 * (xT @ (p["QxxT"] @ xT)) + p["qx1T"] @ xT
            else:
                self.mult[0, j, :n] = torch.from_numpy(r["mu"])
            if j:
                self.mult[0, j, n:] = torch.from_numpy(r["lam"][0])
            self.partials[0, j, 0] = obj
            self.partials[0, j, 1] = worst

    def multiplier_rows(self, j0, j1):
        return self.mult[:, j0:j1]

    def set_multiplier_rows(self, rows):
        self.mult = rows.clone()

    def boundary(self, j0, j1):
        p, n = self.prob, self.n
        for j in range(j0, min(j1, self.J - 1)):
            r = self.recon_out[j]
            t = self.splits[j + 1] - 1
            x, u = r["xs"][-2], r["us"][-1]
            ln = self.mult[0, j + 1, n:].numpy()
            r1 = p["Qxx"][t] @ x + p["Qux"][t].T @ u + p["qx1"][t] + r["lam"][-1] - p["Fx"][t].T @ ln
            r2 = p["Qux"][t] @ x + p["Quu"][t] @ u + p["qu1"][t] - p["Fu"][t].T @ ln
            r3 = self.links[j] - r["xs"][-1]
            self.partials[0, j, 2] = max(float(np.abs(v).max()) for v in (r1, r2, r3))

    def partial_rows(self, j0, j1):
        return self.partials[:, j0:j1]

    def set_partials(self, parts):
        self.partials = parts.clone()

    def finalize(self):
        n = self.n
        pr = self.partials[0].numpy()
        self.objective = float(sum(pr[:, 0]))
        self.kkt = float(max(pr[:, 1].max(), pr[:, 2].max()))
        m = self.mult[0].numpy()
        self.mismatch = float(np.abs(m[:-1, :n] + m[1:, n:]).max()) if self.J > 1 else 0.0

    def results(self):
        return {"objective": self.objective, "kkt_inf": self.kkt, "link_mismatch": self.mismatch,
                "link_residual": self.link_res, "links": self.links}


def _worker(rank, world, port, prob, splits, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        be = OracleBackend(prob, splits)
        res = solve_sharded(be, dist)
        j0, j1 = shard_range(be.J, world, rank)
        local = {}
        for j in range(j0, j1):
            local[f"xs{j}"] = be.recon_out[j]["xs"]
            local[f"lam{j}"] = be.recon_out[j]["lam"]
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), objective=res["objective"], kkt=res["kkt_inf"],
                 mismatch=res["link_mismatch"], links=res["links"], **local)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,cfg_id,T,J", [(2, 2, 96, 6), (2, 0, 60, 5), (3, 1, 64, 8)])
def test_sharded_equals_unsharded(world, cfg_id, T, J):
    cfg = synth.CONFIGS[cfg_id].scaled(T=T, J=J)
    prob = O.problem_slice(synth.generate_batch(cfg, seed=31, count=1), 0)
    splits = O.make_partition(T, J)
    ref = O.solve(prob, splits=splits)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), prob, splits, d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    for o in outs:
        # replicated coupling solve: bitwise identical links on every rank
        assert np.array_equal(o["links"], ref["links"])
        assert abs(float(o["objective"]) - ref["objective"]) <= 1e-12 * abs(ref["objective"])
        assert abs(float(o["mismatch"]) - ref["link_mismatch"]) <= 1e-12 * (1 + ref["link_mismatch"])
        assert abs(float(o["kkt"]) - ref["kkt"]) <= 1e-9 * (1 + ref["kkt"])
    assert np.array_equal(outs[0]["links"], outs[-1]["links"])
    for r, o in enumerate(outs):
        j0, j1 = shard_range(J, world, r)
        for j in range(j0, j1):
            lo, hi = splits[j], splits[j + 1]
            assert np.array_equal(o[f"xs{j}"][:-1], ref["states"][lo:hi])
            assert np.array_equal(o[f"lam{j}"], ref["lambdas"][lo:hi])


def test_shard_range_partitions_segments():
    for J in range(1, 40):
        for world in range(1, 9):
            ranges = [shard_range(J, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == J
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1


def _batch_worker(rank, world, port, cfg_id, B, T, J, outdir):
    """Batch sharding as bench.py does it for cfg1 / cfg4: rank r generates and
    solves problems [first, first + count) only; no data-path collective; the
    step time is the max over ranks (an all-reduce of one scalar)."""
    from paper_1809_06360_b200.sharded import batch_shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS[cfg_id].scaled(B=B, T=T, J=J)
        first, count = batch_shard(cfg.B, world, rank)
        batch = synth.generate_batch(cfg, seed=9, count=count, first=first)
        sols = O.solve_batch(batch, J=J)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)       # stand-in for this rank's step time
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        obj = torch.tensor([s["objective"] for s in sols], dtype=torch.float64)
        allobj = torch.empty(world * count, dtype=torch.float64)
        dist.all_gather_into_tensor(allobj, obj)                        # optional gather of outputs
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), first=first, count=count, tmax=float(t),
                 objective=allobj.numpy(), x0=np.stack([s["states"] for s in sols]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_id,B,T,J", [(2, 1, 6, 16, 4), (3, 1, 6, 16, 4)])
def test_batch_sharding_covers_the_batch(world, cfg_id, B, T, J):
    cfg = synth.CONFIGS[cfg_id].scaled(B=B, T=T, J=J)
    ref = O.solve_batch(synth.generate_batch(cfg, seed=9, count=B), J=J)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_batch_worker, args=(world, _free_port(), cfg_id, B, T, J, d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    owned = []
    for r, o in enumerate(outs):
        first, count = int(o["first"]), int(o["count"])
        owned += list(range(first, first + count))
        assert float(o["tmax"]) == float(world)                         # max over ranks, same on every rank
        assert np.array_equal(o["objective"], np.array([s["objective"] for s in ref]))
        for i in range(count):
            assert np.array_equal(o["x0"][i], ref[first + i]["states"])  # same problems as the unsharded batch
    assert owned == list(range(B))                                       # every problem exactly once
    from paper_1809_06360_b200.sharded import batch_shard
    with pytest.raises(ValueError):
        batch_shard(7, 2, 0)
