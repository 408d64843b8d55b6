#!/usr/bin/env python
"""Benchmark of the B200 partitioned Riccati solve (BASELINE.json metric:
solved knot-points/s, fp64, including the K_t, k_t policies).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one full ``solve_parallel`` of the configured batch (sweeps, link
solve, reconstruction, objective and KKT diagnostics) with inputs resident in
HBM.  Default workload: BASELINE config 4 (256 independent problems, n=64,
m=32, T=1024, J=32) -- BASELINE.json's metric names no config, so the line
is quoted on the largest configuration that fits one GPU (28.3 GB of
inputs); ``--config 0..3`` select the others.  Batches are sharded across
ranks with no collective on the data path; single horizons (cfg 2, 3) are
segment-sharded with one all-gather of the segment value blocks
(``sharded.py``).  ``--gpus N`` without a torchrun environment re-launches
itself under ``torch.distributed.run`` with N ranks.  Rank 0 prints one JSON
line.  ``--impl reference`` times the CPU oracle port of the reference's path
on the host cores instead (rank 0 only).
"""

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1809_06360_b200 import perfmodel, synth  # noqa: E402

METRIC = "solved knot-points/sec (fp64, incl. K_t,k_t policies)"
L2_BYTES = 126 * 1024 * 1024

NVML_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4, choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-smooth", action="store_true")
    ap.add_argument("--no-endpoint", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--gen", default="device", choices=("device", "host"),
                    help="inputs from the device-side seeded generator (plq_generate_batch) or the numpy one")
    ap.add_argument("--native-sharded", action="store_true",
                    help="horizon-sharded runs through plq_solve_parallel_sharded (library-issued NCCL exchanges) "
                         "instead of the torch.distributed orchestration")
    ap.add_argument("--graph", type=int, default=1, help="replay the solve as one CUDA graph (1) or launch eagerly (0)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler(threading.Thread):
    """NVML clocks / throttle reasons sampled every ~5 ms during the timed region."""

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.nv = None

    def run(self):
        while self.ok and not self._halt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def stop(self):
        self._halt.set()
        self.join(timeout=1.0)

    def report(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        names = [v for k, v in NVML_REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference path (bench's cpu_baseline leg
# and the --impl reference arm; the only places bench.py runs oracle/)

def cpu_sample(cfg, cores, seed):
    """A bounded sample of ``cfg`` for the CPU oracle and how to time it."""
    from oracle import parlqr_oracle as O
    if cfg.B > 1:
        S = max(1, (8 if cfg.n <= 16 else 1) * cores)
        batch = synth.generate_batch(cfg, seed=seed, count=S)
        desc = (f"first {S} of {cfg.B} problems (T={cfg.T}, J={cfg.J}), problem-level fork pool "
                f"of {cores} workers around the reference's per-problem solve (it has no batch API)")
        return (lambda: O.solve_batch(batch, J=cfg.J, workers=cores)), S * cfg.T, desc, cores
    if cfg.T <= 4096 and cfg.n <= 16:
        prob = synth.generate_batch(cfg, seed=seed, count=1)
        prob = O.problem_slice(prob, 0)
        w = min(cfg.J, cores)
        desc = f"full problem, segment fork pool of {w} workers (reference default min(J, cores))"
        return (lambda: O.solve(prob, J=cfg.J, workers=w)), cfg.T, desc, w
    L = cfg.T // cfg.J
    Js = 2 * cores
    sub = cfg.scaled(T=L * Js, J=Js)
    prob = O.problem_slice(synth.generate_batch(sub, seed=seed, count=1), 0)
    desc = (f"sub-horizon T={sub.T} with the config's segment length L={L} (J={Js}), segment fork pool "
            f"of {cores} workers (reference default)")
    return (lambda: O.solve(prob, J=Js, workers=cores)), sub.T, desc, cores


def time_cpu(cfg, seed, steps, warmup):
    from oracle import parlqr_oracle as O
    cores = O.host_cores()
    fn, knots, desc, used = cpu_sample(cfg, cores, seed)
    for _ in range(warmup):
        fn()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return {"value": knots / statistics.mean(times), "unit": "knots/s", "cores": used, "kind": "port",
            "sample": desc, "sample_seconds_mean": statistics.mean(times), "steps": steps}


def time_cpu_smooth(cfg, seed, budget_s=4.0):
    """Oracle smooth() (parallel.py:567-633) on a bounded sample, one core,
    parent solves precomputed (only the smoothing pass is timed)."""
    from oracle import parlqr_oracle as O
    if cfg.B > 1:
        batch = synth.generate_batch(cfg, seed=seed, count=min(cfg.B, 8))
        probs = [O.problem_slice(batch, i) for i in range(batch["qx1"].shape[0])]
        J, desc = cfg.J, "problems of the config"
    else:
        L = cfg.T // cfg.J
        Js = min(cfg.J, 16)
        sub = cfg.scaled(T=L * Js, J=Js)
        probs = [O.problem_slice(synth.generate_batch(sub, seed=seed, count=1), 0)]
        J, desc = Js, f"sub-horizon T={sub.T} (segment length {L}, J={Js})"
    sols = [O.solve(p, J=J) for p in probs]
    done, knots, t0 = 0, 0, time.perf_counter()
    while True:
        i = done % len(probs)
        O.smooth(probs[i], sols[i])
        done += 1
        knots += probs[i]["qx1"].shape[0]
        el = time.perf_counter() - t0
        if el >= budget_s or done >= 4 * len(probs):
            break
    return {"value": knots / el, "unit": "knots/s", "cores": 1, "kind": "port",
            "sample": f"{done} smoothing passes over {desc}, parent solves precomputed"}


def time_cpu_endpoint(cfg, seed, budget_s=4.0):
    """Oracle solve_endpoint_affine + evaluate (endpoint.py:603-653) on a
    bounded sample of the config's problems, one core."""
    from oracle import parlqr_oracle as O
    batch = synth.generate_batch(cfg, seed=seed, count=min(cfg.B, 4))
    probs = [O.problem_slice(batch, i) for i in range(batch["qx1"].shape[0])]
    zs = np.random.default_rng(seed).standard_normal((len(probs), cfg.n))
    done, knots, t0 = 0, 0, time.perf_counter()
    while True:
        i = done % len(probs)
        aff = O.solve_endpoint_affine(probs[i])
        O.evaluate_endpoint(probs[i], aff, probs[i]["x_init"], zs[i])
        done += 1
        knots += cfg.T
        el = time.perf_counter() - t0
        if el >= budget_s or done >= 4 * len(probs):
            break
    return {"value": knots / el, "unit": "knots/s", "cores": 1, "kind": "port",
            "sample": f"{done} two-point-boundary solves of the config's problems"}


def parity_sample(cfg, host, out, B_loc, stages=None):
    """A sample of the solved problems against the CPU oracle, computed
    outside the timed region (the oracle is the checker here, never the
    thing measured), with the SURVEY.md 8(c) gates: every output within
    max(1e-9, 10 x floor), floor = the oracle's own relative change under a
    1e-15 relative input perturbation of the same problem (two draws)."""
    from oracle import parlqr_oracle as O
    picks = [0] if B_loc == 1 else sorted({0, B_loc // 2, B_loc - 1})
    probs = [{k: v[i].numpy() for k, v in host.items()} for i in picks]
    w = O.host_cores()
    t0 = time.perf_counter()
    pert = [O.perturbed(p, 1e-15, 100 + s) for p in probs for s in range(2)]
    if B_loc == 1:
        ww = min(w, cfg.J)
        refs = [O.solve(probs[0], J=cfg.J, workers=ww)]
        prefs = [O.solve(p, J=cfg.J, workers=ww) for p in pert]
    else:
        stack = lambda ps: {k: np.stack([p[k] for p in ps]) for k in ps[0]}
        refs = O.solve_batch(stack(probs), J=cfg.J, workers=w)
        prefs = O.solve_batch(stack(pert), J=cfg.J, workers=w)

    def rel(a, b):
        d = float(np.abs(b).max())
        return float(np.abs(a - b).max()) / d if d else float(np.abs(a - b).max())

    errs, floors, ok = {}, {}, True
    lo, hi = stages if stages is not None else (0, cfg.T)   # this rank's stages (horizon sharding)
    keys = (("K", "K"), ("k", "k"), ("x", "states"), ("u", "controls"), ("lam", "lambdas"))
    for pi, (i, ref) in enumerate(zip(picks, refs)):
        fl = {}
        for pr in prefs[2 * pi:2 * pi + 2]:
            for key, rk in keys:
                fl[key] = max(fl.get(key, 0.0), rel(pr[rk][lo:hi], ref[rk][lo:hi]))
            fl["objective"] = max(fl.get("objective", 0.0), rel(np.array([pr["objective"]]),
                                                                np.array([ref["objective"]])))
        e = {key: rel(out[key][i][lo:hi].cpu().numpy(), ref[rk][lo:hi]) for key, rk in keys}
        e["objective"] = rel(out["objective"][i:i + 1].cpu().numpy(), np.array([ref["objective"]]))
        for key, v in e.items():
            errs[key] = max(errs.get(key, 0.0), v)
            floors[key] = max(floors.get(key, 0.0), fl[key])
            ok = ok and v <= max(1e-9, 10.0 * fl[key])
    return {"problems": picks, "stages": [int(lo), int(hi)], "max_rel_err": errs, "oracle_floor": floors,
            "gate": "max(1e-9, 10 x floor) per output (SURVEY.md 8c)", "pass": ok,
            "oracle": "oracle/parlqr_oracle.py (the reference's call sequence restated)",
            "oracle_seconds": time.perf_counter() - t0}


# ---------------------------------------------------------------------------

def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    cb = time_cpu(cfg, args.seed, max(1, args.steps), max(0, args.warmup))
    line = {
        "metric": METRIC, "value": cb["value"], "unit": "knots/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * cb["sample_seconds_mean"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json recipe, seeded)", "impl": "reference",
        "config": {"workload": cfg.name, "B": cfg.B, "n": cfg.n, "m": cfg.m, "T": cfg.T, "J": cfg.J},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "knots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    from paper_1809_06360_b200 import BatchSolver, HostSolver, _native
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = synth.CONFIGS[args.config]
    sharded = cfg.B == 1 and world > 1
    if cfg.B > 1:
        from paper_1809_06360_b200.sharded import batch_shard
        try:
            first, B_loc = batch_shard(cfg.B, world, rank)
        except ValueError as exc:
            raise SystemExit(str(exc))
    else:
        B_loc, first = 1, 0          # single horizon: segments sharded across ranks
    scaling = "strong"
    # seeded host inputs (fork-pool generator), pinned once: the e2e leg reads
    # them as its host buffers, the device-resident leg copies them to HBM
    device_gen = args.gen == "device" and not sharded
    gen = None if device_gen else synth.generate_batch_parallel(cfg, seed=args.seed, count=B_loc, first=first)
    solver = BatchSolver(B_loc, cfg.T, cfg.n, cfg.m, J=cfg.J, device=dev, degenerate=not sharded)
    j0, j1, t0 = 0, cfg.J, 0
    full = None
    if device_gen:
        # the batch is generated in HBM (plq_generate_batch: same recipe, counter-based stream) and
        # copied once to pinned host memory for the e2e leg and the oracle parity sample
        inputs = synth.generate_batch_device(cfg, seed=args.seed, count=B_loc, first=first, device=dev)
        host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v) for k, v in inputs.items()}
    elif sharded:
        # horizon sharding: this rank uploads and holds only its segments'
        # stages (shifted pointers, DeviceBackend(t0=...))
        from paper_1809_06360_b200.sharded import shard_range, stage_window
        j0, j1 = shard_range(cfg.J, world, rank)
        full = gen if rank == 0 else None       # rank 0 keeps the whole problem for the parity check
        gen, t0 = stage_window(gen, solver.partition.split_times, j0, j1)
    if not device_gen:
        host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in gen.items()}
        del gen
        inputs = {k: v.to(dev) for k, v in host.items()}
    stream = torch.cuda.current_stream(dev)
    if sharded:
        from paper_1809_06360_b200.sharded import DeviceBackend, raise_sharded_status, solve_sharded
        backend = DeviceBackend(solver, inputs, t0=t0)
        if args.native_sharded:
            from paper_1809_06360_b200.sharded import NcclComm, solve_sharded_native
            comm = NcclComm(dist)

        def one_step_native():
            solve_sharded_native(solver, inputs, comm, t0=t0, check=False)

        def one_step():
            # no host synchronization inside the step: status rows travel
            # with the value blocks and are checked after the timed region
            solve_sharded(backend, dist, check=False)
            solver.launches = backend.launches
    elif args.graph:
        # the whole solve captured once into a CUDA graph, replayed per step
        graph = solver.capture(inputs)
        launches_per_graph = solver.launches

        def one_step():
            graph.replay()
            solver.launches = launches_per_graph
    else:
        def one_step():
            solver.run(inputs)
    if sharded and args.native_sharded:
        one_step = one_step_native

    def check_status():
        if sharded and args.native_sharded:
            solver.raise_for_status()
        elif sharded:
            raise_sharded_status(backend)
        else:
            solver.raise_for_status()

    for _ in range(max(args.warmup, 1)):
        one_step()
    check_status()
    in_bytes = sum(v.numel() * 8 for v in inputs.values())
    flush = None
    if in_bytes < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    sampler = ClockSampler(dev.index if world == 1 else local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    for i in range(args.steps):
        if flush is not None:
            flush.zero_()
        ev[i][0].record(stream)
        one_step()
        ev[i][1].record(stream)
        launches += solver.launches
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    knots = cfg.B * cfg.T
    value = knots / (ms_per_step / 1000.0)
    check_status()

    # ---- dominant kernel (the segment sweep) timed on its own stream, and the other phases
    import ctypes
    lib = _native.lib()
    prob = solver._problem_struct(inputs, t0=t0)
    phase_ms = {}
    phases = {
        "sweep": lambda: lib.plq_sweep_segments(ctypes.byref(prob), ctypes.byref(solver._outs), j0, j1,
                                                ctypes.c_void_p(solver.workspace.data_ptr()), solver.ws_bytes,
                                                ctypes.c_void_p(stream.cuda_stream)),
        "link": lambda: lib.plq_link_solve(ctypes.byref(prob), ctypes.byref(solver._outs),
                                           ctypes.c_void_p(solver.workspace.data_ptr()), solver.ws_bytes,
                                           ctypes.c_void_p(stream.cuda_stream)),
        "recon": lambda: lib.plq_reconstruct_segments(ctypes.byref(prob), ctypes.byref(solver._outs), j0, j1,
                                                      None, ctypes.c_void_p(solver.workspace.data_ptr()),
                                                      solver.ws_bytes, ctypes.c_void_p(stream.cuda_stream)),
    }
    reps = max(3, min(args.steps, 20))
    for name, fn in phases.items():
        es = []
        for _ in range(reps):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _native.check(fn(), name)
            b.record(stream)
            es.append((a, b))
        torch.cuda.synchronize()
        phase_ms[name] = statistics.mean(x.elapsed_time(y) for x, y in es)
    # algorithmic work of this rank's sweep launch (all segments, or the
    # rank's segment range when the horizon is sharded)
    Fe, Fs, _, _ = perfmodel.stage_flops(cfg.n, cfg.m)
    L = cfg.T / cfg.J
    n_end = min(j1, cfg.J - 1) - j0
    sweep_fl = L * (n_end * Fe + (Fs if j1 == cfg.J else 0.0))
    peak_f64 = perfmodel.fp64_peak_tflops()
    achieved = B_loc * sweep_fl / (phase_ms["sweep"] / 1000.0) / 1e12
    hbm_peak, hbm_src = perfmodel.hbm_peak_gbs(ROOT)
    sweep_b = B_loc * perfmodel.sweep_bytes(cfg.n, cfg.m, cfg.T, cfg.J) * (j1 - j0) / cfg.J
    kernel = perfmodel.sweep_kernel_name(cfg.n, cfg.m)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh).get(cfg.name)
        if isinstance(tj, dict) and tj.get("kernel") == kernel:
            # ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch
            # of the whole-config sweep (B_loc = the batch the capture ran)
            traffic = tj["bytes"] * B_loc / tj.get("B", B_loc)
            traffic_src = tj.get("source")

    # ---- parity of a sample of this rank's problems against the CPU oracle
    # (outside the timed region; the tests gate every output at the floor)
    parity = None
    if not args.no_parity and rank == 0:
        if sharded:
            parity = parity_sample(cfg, {k: torch.from_numpy(v) for k, v in full.items()}, solver.out, 1,
                                   stages=(t0, solver.partition.split_times[j1]))
        else:
            parity = parity_sample(cfg, host, solver.out, B_loc)
    # whole-job algorithmic rates (all ranks) against world x the peaks
    total_fl, _ = perfmodel.problem_flops(cfg.n, cfg.m, cfg.T, cfg.J)
    bin_, bout = perfmodel.knot_bytes(cfg.n, cfg.m)
    sec = ms_per_step / 1000.0
    whole = {
        "fp64_tflops": cfg.B * total_fl / sec / 1e12,
        "fp64_frac": cfg.B * total_fl / sec / 1e12 / (peak_f64 * world),
        "hbm_gbs": cfg.B * cfg.T * (bin_ + bout) / sec / 1e9,
    }
    whole["hbm_frac"] = whole["hbm_gbs"] / (hbm_peak * world)

    # ---- end-to-end: host buffers through plq_solve_parallel_host
    e2e = None
    if not args.no_e2e:
        if sharded:
            # horizon-sharded end to end: each rank copies its window of
            # stages in, runs the phases with the exchanges, and copies its
            # stages' K, k, x, u, lam back (pinned buffers, host wall clock)
            lo_t, hi_t = t0, solver.partition.split_times[j1]
            outs_h = {k: torch.empty(tuple(solver.out[k][0, lo_t:hi_t].shape), dtype=torch.float64).pin_memory()
                      for k in ("K", "k", "x", "u", "lam")}

            class _ShardedE2E:
                h2d_bytes = sum(v.numel() * 8 for v in host.values())
                d2h_bytes = sum(v.numel() * 8 for v in outs_h.values())

                def run(self, pinned_in):
                    for k, v in pinned_in.items():
                        inputs[k].copy_(v, non_blocking=True)
                    solve_sharded(backend, dist, check=False)
                    for k, v in outs_h.items():
                        v.copy_(solver.out[k][0, lo_t:hi_t], non_blocking=True)
                    torch.cuda.synchronize()
            hs = _ShardedE2E()
            e2e_api = "sharded phases (pinned window in -> this rank's K, k, x, u, lam out)"
        else:
            hs = HostSolver(B_loc, cfg.T, cfg.n, cfg.m, J=cfg.J, device=dev, pin=True)
            e2e_api = "plq_solve_parallel_host (pinned host inputs -> host LqrSolution arrays)"
        pinned = host
        for _ in range(max(1, min(args.warmup, 3))):
            hs.run(pinned)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e_steps = max(3, min(args.steps, 10))
        per = []
        for _ in range(e_steps):
            tic = time.perf_counter()
            hs.run(pinned)                 # synchronizes on the result copy
            per.append(time.perf_counter() - tic)
        if sharded:
            raise_sharded_status(backend)
        # host wall clock per step (the copies are the host's): median, so a
        # stall of the shared VM host does not stand for the path
        el = statistics.median(per)
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        # the copy roofline of this leg: pinned H2D / D2H bandwidth measured here
        probe = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
        dprobe = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        bw = {}
        for name, dst, src in (("h2d", dprobe, probe), ("d2h", probe, dprobe)):
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record()
            for _ in range(4):
                dst.copy_(src, non_blocking=True)
            b_.record()
            torch.cuda.synchronize()
            bw[name] = 4 * probe.numel() / (a_.elapsed_time(b_) / 1000.0) / 1e9
        del probe, dprobe
        copy_floor = max(hs.h2d_bytes / (bw["h2d"] * 1e9), hs.d2h_bytes / (bw["d2h"] * 1e9))
        e2e = {"value": knots / el, "unit": "knots/s", "h2d_bytes_per_step": int(hs.h2d_bytes) * world,
               "d2h_bytes_per_step": int(hs.d2h_bytes) * world, "ms_per_step": el * 1000.0,
               "ms_per_step_min_mean_max": [1000 * min(per), 1000 * statistics.mean(per), 1000 * max(per)],
               "steps": e_steps, "statistic": "median of per-step host wall clock",
               "api": e2e_api,
               "copy_roofline": {"h2d_gbs": bw["h2d"], "d2h_gbs": bw["d2h"],
                                 "floor_ms": 1000.0 * copy_floor, "frac": copy_floor / el,
                                 "note": "pinned-copy bandwidth measured in this run; floor = max(H2D, D2H) "
                                         "time of the step's bytes (the directions overlap)"}}
        del hs, pinned
        torch.cuda.empty_cache()

    # ---- smoothing pass (parallel.smooth, §8f row 1) over this solve: device time
    smooth = None
    # (single-GPU runs only: the whole-job throughput of N ranks would need a
    # max-over-ranks time for these legs as well)
    if world == 1 and not args.no_smooth and cfg.J > 1:
        solver.run(inputs)
        solver.smooth(inputs)
        torch.cuda.synchronize()
        es = []
        for _ in range(max(3, min(args.steps, 20))):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            solver.smooth(inputs)
            b.record(stream)
            es.append((a, b))
        torch.cuda.synchronize()
        sm_ms = statistics.mean(x.elapsed_time(y) for x, y in es)
        smooth = {"metric": "smoothed_knots_per_s", "value": knots / (sm_ms / 1000.0), "unit": "knots/s",
                  "ms_per_step": sm_ms, "gpu_launches": solver.launches,
                  "what": "plq_smooth: J-1 conditioned serial sweeps + rollout/objective/KKT, "
                          "parent solve resident"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            smooth["cpu_baseline"] = time_cpu_smooth(cfg, args.seed)
        solver.raise_for_status()

    # ---- two-point-boundary solve (§8f row 3) on the config's problems
    endpoint = None
    if world == 1 and not args.no_endpoint and cfg.T <= 1024 and cfg.n <= 64:
        from paper_1809_06360_b200 import EndpointBatch
        eb = EndpointBatch(B_loc, cfg.T, cfg.n, cfg.m, device=dev)
        zs = torch.from_numpy(np.random.default_rng(args.seed).standard_normal((B_loc, cfg.n))).to(dev)
        def ep_step():
            eb.affine(inputs)
            n_aff = eb.launches
            eb.evaluate(zs)
            return n_aff + eb.launches
        ep_step()
        torch.cuda.synchronize()
        eb.raise_for_status()
        es = []
        for _ in range(max(3, min(args.steps, 10))):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            nl = ep_step()
            b.record(stream)
            es.append((a, b))
        torch.cuda.synchronize()
        ep_ms = statistics.mean(x.elapsed_time(y) for x, y in es)
        endpoint = {"metric": "endpoint_knots_per_s", "value": knots / (ep_ms / 1000.0), "unit": "knots/s",
                    "ms_per_step": ep_ms, "gpu_launches": nl,
                    "what": "plq_endpoint_affine + plq_endpoint_evaluate: terminal-seeded endpoint sweep, "
                            "forward maps, multiplier normal equations, evaluation at x_term"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            endpoint["cpu_baseline"] = time_cpu_endpoint(cfg, args.seed)
        del eb

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = time_cpu(cfg, args.seed, steps=3, warmup=1)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "knots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (BASELINE.json recipe, seeded; generated on the device by plq_generate_batch, "
                     "Philox-4x32-10 + Box-Muller)" if device_gen else
                     "synthetic (BASELINE.json recipe, seeded numpy generator, see synth.py)"),
            "config": {"workload": cfg.name, "B": cfg.B, "n": cfg.n, "m": cfg.m, "T": cfg.T, "J": cfg.J,
                       "global_batch": cfg.B,
                       "parallelism": (f"batch-shard x{world}" if cfg.B > 1 else f"segment-shard x{world}"),
                       "l2": "inputs exceed L2" if flush is None else "L2 flushed between steps",
                       "launch": "CUDA graph replay" if (args.graph and not sharded) else "eager"},
            "gpu_launches": launches,
            "roofline": {"bound": "tensor", "kernel": kernel + " (K1 segment sweep, DMMA.8x8x4 fp64)",
                         "achieved": achieved, "peak": peak_f64, "unit": "TFLOP/s",
                         "frac": achieved / peak_f64, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": "FP64 (DFMA / DMMA) peak measured on this pool's B200 by "
                                        "tools/fp64_peak.cu (profiles/fp64_peak.json); MEASURED_PEAKS.json "
                                        "has no FP64 entry",
                         "algorithmic_flops_per_launch": B_loc * sweep_fl,
                         "algorithmic_bytes_per_launch": sweep_b,
                         "hbm_frac": sweep_b / (phase_ms["sweep"] / 1000.0) / 1e9 / hbm_peak,
                         "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src},
            "whole_solve": whole,
            "phases_ms": phase_ms,
            "clocks": sampler.report(),
            "parity_checked": parity,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "smooth": smooth,
            "endpoint": endpoint,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def spawn_ranks(args):
    """``--gpus N`` outside torchrun: re-launch this script with N ranks
    (one process per GPU, rendezvous on 127.0.0.1); returns the exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                raise SystemExit(f"--gpus {args.gpus}: only {have} CUDA device(s) visible (one rank per GPU)")
        raise SystemExit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
