#!/usr/bin/env python
"""PDHG iterations/s of the B200 PDCS engine (BASELINE.json metric) on the
north-star workload C5: the 50M-nnz synthetic LP (m = 10M, n = 20M).

One "step" is one PDHG iteration of the real solve loop (default options:
adaptive steps, reflected Halpern, duality-gap restarts with checks every
2000 iterations -- the timed region includes whatever checks and restarts
fall inside it).  `value` is device-timed (CUDA events on the engine stream)
with the instance resident in HBM; `e2e` is the same metric through the
public `solve()` API from host numpy buffers (upload, device
preconditioning, iterations, download all inside the wall-clock region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5]
  python bench.py --impl reference ...   # the CPU oracle port of the reference

Multi-GPU (torchrun, one rank per GPU): one solve with G's rows sharded over
the ranks (cone-block-aligned cuts, NCCL all-reduces inside the CUDA graph),
scaling "strong"; value = iterations / max-over-ranks device time.
`--replicas` instead runs an independent copy per rank (scaling "weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "PDHG iters/sec and time-to-1e-6 KKT at 1/2/4/8 B200; SpMV HBM GB/s vs peak"

WORKLOADS = {
    "C1": ("C1: lp_random m=2000 n=4000 density=0.01 seed=0 (NONNEG rows, box [-2,2])",
           lambda I: I.lp_random(2000, 4000, 0.01, 0)),
    "C2": ("C2: group_robust_regression 10k SOC(11) blocks, m=200k n=100k",
           lambda I: I.group_robust_regression()),
    "C3": ("C3: entropy_max 1M exponential-cone blocks, m=3.001M n=2M",
           lambda I: I.entropy_max()),
    "C4": ("C4: markowitz_rsoc N=500k k=40 (one RSOC block of 500,042 rows)",
           lambda I: I.markowitz_rsoc()),
    "C5": ("C5: lp_large m=10,000,000 n=20,000,000 5 nnz/row (30% ZERO rows, NONNEG rest), box [-2,2]",
           lambda I: I.lp_large()),
    # primal cone blocks at scale (not BASELINE configurations)
    "C3p": ("C3p: entropy_max_primal 1M PRIMAL exponential-cone blocks, n=3M m=1.001M",
            lambda I: I.entropy_max_primal()),
    "C2p": ("C2p: group_regression_primal 10k PRIMAL SOC(11) blocks (rescaled), n=155k m=100k",
            lambda I: I.group_regression_primal()),
    # C5's pattern at 1/10 (single-panel SpMVs; launch-variant sweeps only)
    "C5s": ("C5s: lp_large m=1,000,000 n=2,000,000 5 nnz/row (C5 pattern at 1/10)",
            lambda I: I.lp_large(m=1_000_000, n=2_000_000)),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-runs", type=int, default=3, help="whole solves timed for e2e (median)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-reps", type=int, default=5)
    ap.add_argument("--ttt", action="store_true", help="also solve to 1e-6 and report time-to-tolerance")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: every rank solves its own copy instead of one row-sharded solve")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded engine even on one GPU (NCCL in-graph path)")
    ap.add_argument("--selfcheck", action="store_true",
                    help="with --sharded on one GPU: also run the N>1 trajectory self-check")
    ap.add_argument("--no-ttt-c1", action="store_true",
                    help="skip the C1 time-to-1e-6 solve (both arms run it by default)")
    ap.add_argument("--no-sustained", action="store_true",
                    help="skip the sustained it/s over one whole check interval")
    ap.add_argument("--batch", type=int, default=0,
                    help="also time B concurrent solves of the workload (solve_many) and report the "
                         "aggregate iterations/s (small configurations)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.tmp,
                stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.tmp.flush()
        self.tmp.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.tmp.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.tmp.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_traffic(config: str, stage: str):
    """DRAM bytes (read + write) per launch of a stage from the committed ncu
    capture of the same configuration (profiles/traffic_<config>.json), or None."""
    path = os.path.join(REPO, "profiles", f"traffic_{config}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f).get("stages", {}).get(stage)


def kernel_bytes(problem, stage: str) -> int:
    """Algorithmic bytes of one launch of the fused kernels (values + indices
    + row pointers once, gathered vector once, each streamed vector once)."""
    import numpy as np

    n, m, nnz = problem.n, problem.m, problem.G.nnz
    nb = int(np.sum(np.isfinite(problem.l) | np.isfinite(problem.u)))
    if stage == "step_y_spmv":
        # CSR(G^) + gather x~ + y-space: read y, y_hat, y_anchor, y_bar, gx, gx_hat, gx_anchor, h;
        # write y, y_bar, gx, gx_hat, y_hat
        return 12 * nnz + 4 * (m + 1) + 8 * n + 8 * 13 * m
    if stage == "step_t_spmv":
        # CSR(G^T) + gather y_hat + read c (+ l, u on finite-bound coordinates) + write gth
        return 12 * nnz + 4 * (n + 1) + 8 * m + 8 * (2 * n + 2 * nb)
    if stage == "step_x":
        # read x, x_hat, x_anchor, x_bar, gty, gth, gty_anchor, c (+ l, u); write x, x_bar, gty, x_hat, x~
        return 8 * (13 * n + 2 * nb)
    return 0


def workload_config(args, problem) -> dict:
    """The `config` dict both arms emit (identical for the same workload)."""
    return {"workload": WORKLOADS[args.config][0], "nnz": int(problem.G.nnz), "m": int(problem.m),
            "n": int(problem.n),
            "options": "defaults except rel/abs tol 1e-12 (no early exit)",
            "l2": "inputs larger than L2 (1.3 GB CSR of G and G^T vs 126 MB L2); no flush needed"}


def host_info() -> dict:
    """CPU model, core count and the numpy/scipy versions."""
    import numpy
    import scipy

    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = os.cpu_count()
    return {"cpu_model": model, "nproc": os.cpu_count(), "cpus_available": avail,
            "numpy": numpy.__version__, "scipy": scipy.__version__}


def blas_threads() -> int | None:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else None
    except Exception:  # noqa: BLE001
        return None


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle port of conic_pdhg (pinned to the
    reference's golden outputs, tests/test_oracle_golden.py) on the box's host
    cores, rank 0 only, BLAS left at all the threads it can use.  scipy's
    csr_matvec and the per-block projections are single-threaded whatever the
    thread count, so the SpMV-bound iteration runs on one core in practice."""
    if rank != 0:
        return
    from oracle import pdcs_oracle as oracle
    from paper_2603_15504_b200 import instances

    desc, make = WORKLOADS[args.config]
    t0 = time.monotonic()
    problem = make(instances)
    gen_s = time.monotonic() - t0
    iters = 3 if args.config in ("C3", "C4", "C5") else min(max(args.steps, 3), 200)
    med, setup = oracle.time_iterations(problem, iters)
    value = 1.0 / med
    host = host_info()
    threads = blas_threads()
    cores = host["cpus_available"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": args.gpus,
        # the iterations actually timed (a bounded sample: C5 runs ~2.5 s per iteration on one core)
        "steps": iters, "steps_requested": args.steps, "warmup": 0, "warmup_requested": args.warmup,
        "ms_per_step": 1000.0 * med,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, problem),
        "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "kind": "port",
                         "sample": f"{iters} PDHG iterations of {args.config} by the numpy/scipy oracle "
                                   f"restatement of conic_pdhg (identity scaling, restarts off; "
                                   f"marginal it/s = 1/median iteration time); setup {setup:.1f}s, "
                                   f"instance generation {gen_s:.1f}s; BLAS threads {threads} of "
                                   f"{cores} host cores, scipy csr_matvec and the projections are "
                                   "single-threaded"},
        "host": host,
        "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if not args.no_ttt_c1:
        # C1 to 1e-6 by the same port: the time-to-tolerance the GPU arm's
        # "time_to_1e-6_C1" is compared with (reference: 46.1 s)
        from paper_2603_15504_b200 import instances as I

        p1 = I.lp_random(2000, 4000, 0.01, 0)
        t0 = time.perf_counter()
        r = oracle.solve(p1, oracle.options_from(None, rel_tol=1e-6, abs_tol=1e-6, time_limit=1e4))
        line["time_to_1e-6_C1"] = {"status": r["status"], "iterations": int(r["iterations"]),
                                   "wall_s": time.perf_counter() - t0, "p_obj": float(r["p_obj"])}
    emit(line)


def selfcheck_sharded(problem, rank, world, k=20, tol=1e-9):
    """N>1 correctness gate of the sharded engine: every rank runs the row-
    sharded solve for k iterations, rank 0 re-runs the same k iterations on
    one GPU, and the returned iterates must agree to `tol` (relative to their
    max-abs).  The sharded column statistics of the preconditioner and the
    reduce-scattered G^T y sums add in another order, so agreement is to
    rounding, not bit for bit (<= 1e-11 at k <= 20)."""
    import numpy as np
    import torch.distributed as dist

    from paper_2603_15504_b200 import SolverOptions, solve
    from paper_2603_15504_b200.distributed import solve_sharded

    opts = dict(max_iter=k, rel_tol=1e-14, abs_tol=1e-14, time_limit=1e9)
    t0 = time.perf_counter()
    rs = solve_sharded(problem, SolverOptions(**opts))
    out = {"k": k, "tol": tol, "iterations": rs.iterations}
    ok = 1.0
    if rank == 0:
        r1 = solve(problem, SolverOptions(**opts))
        dx = float(np.max(np.abs(rs.x - r1.x)) / max(1.0, float(np.max(np.abs(r1.x)))))
        dy = float(np.max(np.abs(rs.y - r1.y)) / max(1.0, float(np.max(np.abs(r1.y)))))
        ok = float(rs.iterations == r1.iterations and dx <= tol and dy <= tol)
        out.update(max_rel_diff_x=dx, max_rel_diff_y=dy, single_iterations=r1.iterations)
    import torch

    t = torch.tensor([ok], device="cuda", dtype=torch.float64)
    dist.broadcast(t, src=0)
    out["pass"] = bool(t.item() == 1.0)
    out["wall_s"] = time.perf_counter() - t0
    return out


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2603_15504_b200 import SolverOptions, instances, solve
    from paper_2603_15504_b200._native import launch_count
    from paper_2603_15504_b200.distributed import sharded_loop_class, solve_sharded
    from paper_2603_15504_b200.engine import _Loop

    torch.cuda.set_device(local)
    dist = None
    sharded = (world > 1 and not args.replicas) or args.sharded
    if world > 1 or sharded:
        import torch.distributed as dist  # noqa: F811

        if "MASTER_ADDR" in os.environ:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            import socket

            sock = socket.socket()
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
            sock.close()
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
    desc, make = WORKLOADS[args.config]
    t_gen = time.monotonic()
    problem = make(instances)
    gen_s = time.monotonic() - t_gen
    selfcheck = None
    if sharded and (world > 1 or args.selfcheck):
        selfcheck = selfcheck_sharded(problem, rank, world)
        torch.cuda.empty_cache()
    opts = SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=10**9, time_limit=1e9)

    t_setup = time.monotonic()
    loop = sharded_loop_class()(problem, opts) if sharded else _Loop(problem, opts)
    state, ex = loop._start()
    setup_s = time.monotonic() - t_setup
    launch_info = loop.dev.info()
    ex = loop._advance(state, ex, until=args.warmup)
    stream = loop.dev.stream
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = launch_count()
    k0 = state.k_bar
    ev0.record(stream)
    ex = loop._advance(state, ex, until=args.warmup + args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = launch_count() - l0
    clk = clocks.stop()
    iters = state.k_bar - k0
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        it = torch.tensor([iters], device="cuda", dtype=torch.float64)
        dist.all_reduce(it, op=dist.ReduceOp.SUM)
        # one sharded solve: every rank advanced the same iterations
        total_iters = iters if sharded else int(it.item())
    else:
        total_iters = iters
    value = total_iters / (ms / 1000.0)

    # sustained rate over one whole check interval: from the
    # current k_bar through the next check (termination + restart scan, gap
    # search, possible restart) to the same position one interval later
    sustained = None
    if not args.no_sustained:
        freq = loop.check_freq if hasattr(loop, "check_freq") else 2000
        kb0 = state.k_bar
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        s0.record(stream)
        ex = loop._advance(state, ex, until=kb0 + freq)
        s1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        sms = s0.elapsed_time(s1)
        if dist:
            t = torch.tensor([sms, wall], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sms, wall = float(t[0].item()), float(t[1].item())
        its = state.k_bar - kb0
        sustained = {"iterations": its, "checks": 1, "device_ms": sms, "wall_s": wall,
                     "value": its / (sms / 1000.0), "value_wall": its / wall, "unit": "it/s",
                     "iteration_roofline_frac": instances.algorithmic_bytes(problem) * its / (sms / 1000.0)
                     / 1e9 / peaks()[0],
                     "note": "one whole check interval (k_bar %d -> %d) incl. the termination / restart "
                             "check, gap search and any restart" % (kb0, state.k_bar)}

    # per-stage device times of eager trials (live, CUDA events on the engine stream)
    stages = []
    if args.profile_reps > 0:
        loop.dev.flush()
        loop._prepare_batch(state, state.k_bar + 10 * args.profile_reps + 100)
        stages = loop.dev.profile_slot(args.profile_reps)
    peak, peak_kind = peaks()
    b_alg = instances.algorithmic_bytes(problem)
    iter_gbs = b_alg * (iters / (ms / 1000.0)) / 1e9
    dom = max(stages, key=lambda s: s[1]) if stages else ("step_y_spmv", None)
    dom_bytes = kernel_bytes(problem, dom[0])
    # no per-stage profile (--profile-reps 0): no kernel roofline (null, not NaN)
    dom_gbs = dom_bytes / (dom[1] / 1000.0) / 1e9 if dom[1] else None
    slot_ms = sum(s[1] for s in stages)
    loop.close()
    del loop
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        n, m, nnz = problem.n, problem.m, problem.G.nnz
        h2d = 4 * (m + 1) + 4 * nnz + 8 * nnz + 8 * (n + m + 2 * problem.num_box)
        d2h = 8 * (2 * n + 2 * m)
        e2e_iters = args.steps
        e2e_opts = SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=e2e_iters, time_limit=1e9)
        # the median of --e2e-runs whole solves: a solve's setup is ~0.1-0.2 s and
        # its device-pool growth occasionally stalls (profiles/r02_e2e_spread.txt)
        walls = []
        for _ in range(max(1, args.e2e_runs)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = solve_sharded(problem, e2e_opts) if sharded else solve(problem, e2e_opts)
            walls.append(time.perf_counter() - t0)
        wall = sorted(walls)[len(walls) // 2]
        e2e = {"value": r.iterations / wall, "unit": "it/s",
               "h2d_bytes_per_step": h2d / max(r.iterations, 1), "d2h_bytes_per_step": d2h / max(r.iterations, 1),
               "iterations": r.iterations, "wall_s": wall, "walls_s": walls, "h2d_bytes": h2d, "d2h_bytes": d2h,
               "note": "public solve() from host numpy: upload, device Ruiz+PC, iterations with checks, "
                       "download; median wall of %d solves" % len(walls)}

    batched = None
    if args.batch > 1 and not sharded:
        from paper_2603_15504_b200.batch import solve_many

        probs = [problem] * args.batch
        b_opts = SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=args.steps, time_limit=1e9)
        batched = {}
        for mode in ("graph", "threads"):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = solve_many(probs, b_opts, batched=(mode == "graph"))
            wall = time.perf_counter() - t0
            total = sum(r.iterations for r in res)
            batched[mode] = {"instances": args.batch, "iterations_total": total, "wall_s": wall,
                             "value": total / wall, "unit": "it/s"}
        batched["note"] = ("solve_many wall clock incl. upload/setup/download; graph = one CUDA graph "
                           "per replay advancing every instance (pdcs_batch_run), threads = an engine, "
                           "stream and graph per instance on a thread pool")

    ttt = None
    if args.ttt:
        t0 = time.perf_counter()
        tt_opts = SolverOptions(rel_tol=1e-6, abs_tol=1e-6, time_limit=3600.0)
        r = solve_sharded(problem, tt_opts) if sharded else solve(problem, tt_opts)
        ttt = {"status": r.exit_status, "iterations": r.iterations, "wall_s": time.perf_counter() - t0,
               "solve_time_s": r.solve_time_s, "p_obj": r.p_obj}

    ttt_c1 = None
    if not args.no_ttt_c1 and not sharded and args.config != "C1":
        # C1 (2000 x 4000 LP) to 1e-6 through the public solve(): the reference
        # takes 54,000 iterations / 46.1 s (the reference
        # arm re-times its port on this box as "time_to_1e-6_C1")
        p1 = instances.lp_random(2000, 4000, 0.01, 0)
        t0 = time.perf_counter()
        r1 = solve(p1, SolverOptions(rel_tol=1e-6, abs_tol=1e-6))
        ttt_c1 = {"status": r1.exit_status, "iterations": r1.iterations, "wall_s": time.perf_counter() - t0,
                  "solve_time_s": r1.solve_time_s, "p_obj": r1.p_obj,
                  "reference": {"iterations": 54000, "wall_s": 46.1, "p_obj": -5063.1994466,
                                "source": "BASELINE.md section 2 (reference conic_pdhg, survey host)"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits

        from oracle import pdcs_oracle as oracle

        it_cpu = 2 if args.config in ("C3", "C4", "C5") else 20
        with threadpool_limits(limits=1):
            med, setup = oracle.time_iterations(problem, it_cpu)
        cpu = {"value": 1.0 / med, "unit": "it/s", "cores": 1, "kind": "port",
               "sample": f"{it_cpu} PDHG iterations of {args.config} by the numpy/scipy oracle restatement "
                         f"(identity scaling, restarts off; 1/median iteration time; setup {setup:.1f}s; "
                         "BLAS pinned to 1 thread)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / max(iters, 1), "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(args, problem),
            "parallelism": (f"sharded x{world}: rows of G and x-slices, in-graph NCCL all-gather of x~ + "
                            "reduce-scatter of G^T y" if sharded else ("replicas" if world > 1 else "single")),
            "run": {"iterations_timed": iters, "restarts_so_far": state.t, "setup_s": setup_s,
                    "instance_gen_s": gen_s, "launch": launch_info, "tune": os.environ.get("PDCS_TUNE", ""),
                    "host": host_info()},
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": dom_gbs, "peak": peak,
                         "unit": "GB/s", "frac": dom_gbs / peak if dom_gbs is not None else None,
                         "traffic": measured_traffic(args.config, dom[0]),
                         "bytes_per_launch": dom_bytes, "launch_ms": dom[1], "peak_source": peak_kind},
            "iteration_roofline": {"B_alg_bytes": b_alg, "achieved": iter_gbs, "peak": peak, "unit": "GB/s",
                                   "frac": iter_gbs / peak},
            "stages_ms": {k: v for k, v in stages}, "slot_ms": slot_ms,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        if ttt:
            line["time_to_1e-6"] = ttt
        if ttt_c1:
            line["time_to_1e-6_C1"] = ttt_c1
        if sustained:
            line["sustained"] = sustained
        if selfcheck:
            line["selfcheck"] = selfcheck
        ttt_path = os.path.join(REPO, "profiles", "r02_ttt.jsonl")
        if os.path.exists(ttt_path):
            # long time-to-tolerance solves (minutes each) recorded by tools/ttt.py in a
            # separate run on a B200; labelled as recorded, not measured in this run
            with open(ttt_path) as f:
                line["recorded_time_to_tolerance"] = {
                    "source": "profiles/r02_ttt.jsonl (tools/ttt.py, separate run, public solve())",
                    "runs": [json.loads(x) for x in f if x.strip()]}
        if batched:
            line["batched"] = batched
        emit(line)
    if dist:
        dist.destroy_process_group()
    if selfcheck and not selfcheck["pass"]:
        sys.stderr.write(f"sharded self-check FAILED: {selfcheck}\n")
        sys.exit(3)


_OUT = None


def emit(line: dict) -> None:
    """The one JSON line on the real stdout (library banners such as NCCL's
    version print are diverted to stderr, see main)."""
    _OUT.write(json.dumps(line) + "\n")
    _OUT.flush()


def main():
    global _OUT
    # keep stdout for the JSON line only: fd 1 -> stderr for everything else
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
