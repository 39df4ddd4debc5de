"""Many independent solves on one GPU at once.

A C1-class instance (thousands of variables) leaves a B200 mostly idle: each
PDHG trial is a handful of tiny kernels, bound by launch latency.  Running
several solves concurrently -- one engine and one CUDA stream per instance,
driven from host threads (ctypes releases the GIL inside libpdcs, where the
CUDA-graph replays and synchronisations happen) -- overlaps their device
loops.  Every solve is still the deterministic single-instance solve: results
are bit-identical to calling `solve` one by one.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

from .engine import SolveResult, SolverOptions, solve


def solve_many(problems, options: SolverOptions | None = None,
               max_workers: int | None = None) -> list[SolveResult]:
    """Solve a list of instances concurrently; results in input order."""
    problems = list(problems)
    if not problems:
        return []
    if options is not None and options.iteration_callback is not None:
        raise ValueError("solve_many does not support iteration callbacks")
    workers = max_workers or min(16, len(problems))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(lambda p: solve(p, options), problems))
