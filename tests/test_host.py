"""Host-side logic that needs no GPU: partitions (ports of the reference's
partition tests, test_parallel.py:14-44), error mapping, input stacking,
lazy policies, the perf model and the seeded generator."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1809_06360_b200 as plq
from paper_1809_06360_b200 import _native, perfmodel, synth
from paper_1809_06360_b200.parallel import PolicySequence, _check_partition, raise_for_status


class TestPartition:
    def test_balanced_remainder_goes_first(self):
        assert plq.make_partition(10, 3).split_times == (0, 4, 7, 10)

    def test_single_segment(self):
        assert plq.make_partition(5, 1).split_times == (0, 5)

    def test_unit_segments(self):
        assert plq.make_partition(4, 4).split_times == (0, 1, 2, 3, 4)

    def test_out_of_range(self):
        with pytest.raises(ValueError):
            plq.make_partition(5, 0)
        with pytest.raises(ValueError):
            plq.make_partition(5, 6)

    @given(T=st.integers(1, 300), J=st.integers(1, 300))
    @settings(max_examples=200, deadline=None)
    def test_partition_properties(self, T, J):
        if J > T:
            with pytest.raises(ValueError):
                plq.make_partition(T, J)
            return
        splits = plq.make_partition(T, J).split_times
        assert splits[0] == 0 and splits[-1] == T and len(splits) == J + 1
        lengths = np.diff(splits)
        assert lengths.min() >= 1 and lengths.max() - lengths.min() <= 1
        if J > 1:
            assert lengths[:-1].min() >= lengths[-1]

    def test_custom_partition_validation(self):
        # parallel.py:434-440
        with pytest.raises(ValueError, match="cover"):
            _check_partition(plq.Partition(2, (0, 3, 5)), 6)
        with pytest.raises(ValueError, match="increasing"):
            _check_partition(plq.Partition(2, (0, 3, 3, 6)), 6)
        assert _check_partition(plq.Partition(2, (0, 2, 6)), 6).split_times == (0, 2, 6)

    def test_config_partitions_are_balanced(self):
        for cfg in synth.CONFIGS.values():
            lengths = np.diff(plq.make_partition(cfg.T, cfg.J).split_times)
            assert lengths.min() == lengths.max() == cfg.T // cfg.J
            assert (cfg.T // cfg.J) * cfg.m >= cfg.n   # every segment reaches arbitrary endpoints


class TestStatusMapping:
    def test_cholesky_failure_carries_segment_local_stage(self):
        status = np.zeros((2, 4), np.int32)
        status[1, 2] = 1 + 5
        with pytest.raises(plq.CholeskyFailure) as ei:
            raise_for_status(status)
        assert ei.value.stage == 5 and ei.value.segment == 2

    def test_first_failing_segment_wins(self):
        status = np.zeros((1, 4), np.int32)
        status[0, 3] = 1 + 1
        status[0, 1] = 1 + 7
        with pytest.raises(plq.CholeskyFailure) as ei:
            raise_for_status(status)
        assert ei.value.segment == 1 and ei.value.stage == 7

    def test_degenerate_and_link_singular(self):
        status = np.zeros((1, 3), np.int32)
        status[0, 1] = _native.PLQ_STATUS_DEGENERATE
        with pytest.raises(plq.UnsupportedPartition):
            raise_for_status(status)
        status = np.zeros((1, 3), np.int32)
        status[0, 0] = _native.PLQ_STATUS_LINK_SINGULAR
        with pytest.raises(plq.LinkSingular):
            raise_for_status(status)
        raise_for_status(np.zeros((3, 3), np.int32))

    def test_exceptions_share_the_reference_hierarchy(self):
        for exc in (plq.CholeskyFailure(0), plq.LinkSingular(), plq.UnsupportedPartition(0), plq.Infeasible(1.0)):
            assert isinstance(exc, plq.SolverError)


class TestDataModel:
    def test_stack_problem_layout_and_memo(self):
        a = synth.generate_one(3, 2, 5, seed=1)
        prob = plq.problem_from_arrays(a)
        st1 = plq.stack_problem(prob)
        assert st1 is plq.stack_problem(prob)
        for k in a:
            np.testing.assert_array_equal(st1[k], a[k])
        assert st1["Fu"].shape == (5, 3, 2) and st1["Qux"].shape == (5, 2, 3)

    def test_symmetrization_is_a_no_op_on_generated_data(self):
        a = synth.generate_one(6, 2, 4, seed=2)
        prob = plq.problem_from_arrays(a)
        assert all(np.array_equal(c.Qxx, a["Qxx"][t]) for t, (c, _) in enumerate(prob.stages))

    def test_lazy_policies(self):
        K = np.arange(2 * 3 * 4, dtype=float).reshape(2, 3, 4)
        k = np.ones((2, 3))
        pol = PolicySequence(K, k)
        assert len(pol) == 2
        np.testing.assert_array_equal(pol[1].Kx, K[1])
        np.testing.assert_array_equal(pol[1](np.ones(4)), K[1] @ np.ones(4) + 1.0)
        assert len(pol[0:2]) == 2
        assert not np.any(pol[0].Kz)

    def test_problem_validation_errors(self):
        with pytest.raises(ValueError):
            plq.StageCost(np.eye(2), np.zeros((1, 3)), np.eye(1), np.zeros(2), np.zeros(1))
        with pytest.raises(ValueError):
            plq.LqrProblem([], plq.TerminalCost.zero(2), np.zeros(2))


class TestPerfModel:
    def test_flop_counts_match_the_survey(self):
        # flop / knot 27.8k, 30.2k, 432k, 41.3M, 5.17M
        want = {0: 27.8e3, 1: 30.2e3, 2: 432e3, 3: 41.3e6, 4: 5.17e6}
        for cid, w in want.items():
            c = synth.CONFIGS[cid]
            tot, sweep = perfmodel.problem_flops(c.n, c.m, c.T, c.J)
            assert abs(tot / c.T / w - 1) < 0.01
            assert sweep < tot

    def test_bytes_per_knot(self):
        assert perfmodel.knot_bytes(12, 4) == (3424, 640)
        assert sum(perfmodel.knot_bytes(128, 64)) == 428544 + 68608

    def test_fp64_peak_is_measured(self):
        assert 35.0 < perfmodel.fp64_peak_tflops() < 45.0


class TestGenerator:
    def test_seeded_and_reproducible(self):
        a = synth.generate_one(4, 2, 6, seed=11)
        b = synth.generate_one(4, 2, 6, seed=11)
        for k in a:
            np.testing.assert_array_equal(a[k], b[k])

    def test_recipe_statistics(self):
        a = synth.generate_one(32, 8, 512, seed=3)
        G = (a["Fx"] - np.eye(32)) / 0.1
        assert abs(G.std() * np.sqrt(32) - 1) < 0.05            # G ~ N(0, 1/n)
        assert abs(a["Fu"].std() * np.sqrt(32) / 0.1 - 1) < 0.05  # B ~ N(0, 0.01/n)
        assert abs(a["f1"].std() / 0.1 - 1) < 0.05               # c ~ N(0, 0.01)
        assert np.all(np.linalg.eigvalsh(a["Quu"]) > 0.1 - 1e-12)
        assert not np.any(a["Qux"])

    def test_cross_term_option(self):
        base = synth.generate_one(12, 4, 16, seed=3)
        a = synth.generate_one(12, 4, 16, seed=3, cross=0.3)
        for k in base:                       # drawn last: the other fields are unchanged
            if k != "Qux":
                np.testing.assert_array_equal(a[k], base[k])
        assert np.all(np.abs(a["Qux"]).max(axis=(1, 2)) > 0)
        for t in range(16):
            S = a["Qxx"][t] - a["Qux"][t].T @ np.linalg.solve(a["Quu"][t], a["Qux"][t])
            assert np.linalg.eigvalsh(S).min() >= 0.0

    def test_reference_recipe_matches_reference_generator(self):
        """synth.generate_reference_recipe restates parlqr.generate
        (generate.py:14-47): same seed, same problem, byte for byte."""
        import os
        import sys
        src = "/root/reference/pkg/src"
        if not os.path.isdir(src):
            pytest.skip("reference not mounted (GPU box)")
        sys.path.insert(0, src)
        try:
            from parlqr.generate import generate
        finally:
            sys.path.remove(src)
        for n, m, T, seed in ((3, 2, 5, 0), (12, 4, 6, 7), (5, 7, 4, 11)):
            ref = generate(n, m, T, seed)
            a = synth.generate_reference_recipe(n, m, T, seed)
            for f in synth.STAGE_FIELDS:
                want = np.stack([getattr(c if f[0] in "Qq" else d, f) for c, d in ref.stages])
                np.testing.assert_array_equal(a[f], want, err_msg=f)
            np.testing.assert_array_equal(a["QxxT"], ref.terminal.Qxx)
            np.testing.assert_array_equal(a["qx1T"], ref.terminal.qx1)
            np.testing.assert_array_equal(a["x_init"], ref.x_init)
            assert np.any(a["Qux"])

    def test_batch_rows_are_per_problem_seeds(self):
        cfg = synth.CONFIGS[1].scaled(B=3)
        batch = synth.generate_batch(cfg, seed=5, count=3)
        one = synth.generate_one(cfg.n, cfg.m, cfg.T, 5 + 2)
        np.testing.assert_array_equal(batch["Fx"][2], one["Fx"])
        part = synth.generate_batch(cfg, seed=5, count=1, first=2)
        np.testing.assert_array_equal(part["x_init"][0], one["x_init"])


def test_product_path_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    prob = plq.problem_from_arrays(synth.generate_one(3, 1, 6, seed=1))
    with pytest.raises(RuntimeError, match="CUDA"):
        plq.solve_parallel(prob, J=2)


def test_device_generator_stream_restatement():
    """Philox-4x32-10 known answers (the algorithm's published test vectors)
    and the moments of the Box-Muller normals the device generator draws."""
    from paper_1809_06360_b200 import synth
    w = synth._philox4x32_10([0], [0], [0], [0], 0, 0)
    assert [int(x[0]) for x in w] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    w = synth._philox4x32_10([0xFFFFFFFF], [0xFFFFFFFF], [0xFFFFFFFF], [0xFFFFFFFF], 0xFFFFFFFF, 0xFFFFFFFF)
    assert [int(x[0]) for x in w] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    z = synth._device_normals(5, 2, "W", 400_000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01 and abs((z ** 4).mean() - 3) < 0.1
    assert not np.array_equal(z[:100], synth._device_normals(5, 3, "W", 100))
    cfg = synth.CONFIGS[1].scaled(T=4, J=1)
    p = synth.device_stream_reference(cfg, seed=0, problem=1)
    assert p["Qxx"].shape == (4, 12, 12) and np.linalg.eigvalsh(p["Qxx"][0]).min() > 0
