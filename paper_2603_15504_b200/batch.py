"""Many independent solves on one GPU at once.

A C1-class instance (thousands of variables) leaves a B200 mostly idle: each
PDHG trial is a handful of tiny kernels, bound by launch latency.  The
reference solves one problem per call (engine.py:683-689); here

* `solve_many(problems, options)` (default, ``batched=True``) builds one
  engine per instance and advances ALL of them with one CUDA graph per
  replay (libpdcs `pdcs_batch_run`: the graph forks into every engine's
  stream, each branch runs that engine's line-search trials, then joins).
  Each instance keeps its own host loop -- the reference's check, restart and
  termination logic of `engine._Loop`, run on a host thread -- and a
  coordinator launches the shared graph whenever every unfinished instance
  is waiting for device iterations.  Instances stopped at a check (or done)
  are gated off inside the graph.
* ``batched=False`` is the plain thread pool: one engine, one stream and its
  own graph replays per instance.

Either way every member runs the graph-path kernels of a single solve, so
results are bit-identical to `solve` calls on the graph path (`PDCS_TUNE=
persist=0`); a lone small solve runs the persistent kernel instead, whose
reductions are grouped differently (equal to rounding).
"""

from __future__ import annotations

import ctypes as C
import threading
from concurrent.futures import ThreadPoolExecutor

from . import _native as N
from .engine import SolveResult, SolverOptions, _adopt, _Loop, solve
from .model import ConicProblem


class _BatchCoordinator:
    """Launches the shared batch graph when every unfinished member waits."""

    def __init__(self, loops):
        import torch

        self.lib = N.lib()
        self.loops = loops
        self.stream = torch.cuda.Stream()
        handles = (C.c_void_p * len(loops))(*[lp.dev.handle.value for lp in loops])
        h = C.c_void_p()
        N.check(self.lib.pdcs_batch_create(handles, len(loops), C.c_void_p(self.stream.cuda_stream),
                                           C.byref(h)), "pdcs_batch_create")
        self.handle = h
        self.cv = threading.Condition()
        self.waiting: dict[int, int] = {}
        self.active = set(range(len(loops)))
        self.generation = 0
        self.error: BaseException | None = None
        self.launches = 0

    def close(self):
        if self.handle is not None and self.handle.value:
            self.lib.pdcs_batch_destroy(self.handle)
            self.handle = None

    def _launch_locked(self):
        slots = max(self.waiting.values())
        try:
            N.check(self.lib.pdcs_batch_run(self.handle, int(slots)), "pdcs_batch_run")
        except BaseException as exc:  # noqa: BLE001 - handed to every waiting member
            self.error = exc
        self.launches += 1
        self.waiting.clear()
        self.generation += 1
        self.cv.notify_all()

    def run_inner(self, idx: int, slots: int) -> None:
        with self.cv:
            if self.error is not None:
                raise self.error
            self.waiting[idx] = slots
            gen = self.generation
            if set(self.waiting) >= self.active:
                self._launch_locked()
            else:
                while self.generation == gen and self.error is None:
                    self.cv.wait()
            if self.error is not None:
                raise self.error

    def finish(self, idx: int) -> None:
        """Member idx is done (or failed): keep its device loop stopped and
        stop waiting for it."""
        dev = self.loops[idx].dev
        c = dev.get_ctrl()
        c.stop = 1
        dev.set_ctrl(c)
        with self.cv:
            self.active.discard(idx)
            self.waiting.pop(idx, None)
            if self.waiting and set(self.waiting) >= self.active:
                self._launch_locked()


def solve_many(problems, options: SolverOptions | None = None, max_workers: int | None = None,
               batched: bool = True) -> list[SolveResult]:
    """Solve a list of instances concurrently; results in input order."""
    problems = list(problems)
    if not problems:
        return []
    if options is None:
        options = SolverOptions()
    if options.iteration_callback is not None:
        raise ValueError("solve_many does not support iteration callbacks")
    options.validate()
    if not batched:
        from .device import _thread_opts

        def one(p):
            # concurrent solves stay on the graph path (a persistent cooperative
            # launch of a small solve would occupy the whole GPU)
            _thread_opts.no_persist = True
            return solve(p, options)

        workers = max_workers or min(16, len(problems))
        with ThreadPoolExecutor(max_workers=workers) as pool:
            return list(pool.map(one, problems))

    probs = [p if isinstance(p, ConicProblem) else _adopt(p) for p in problems]
    # engines (upload, transpose, panels, preconditioning) on a pool of threads
    workers = max_workers or min(16, len(probs))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        loops = list(pool.map(lambda p: _Loop(p, options), probs))
    coord = _BatchCoordinator(loops)
    for i, lp in enumerate(loops):
        lp.dev.run_inner = (lambda i: lambda slots: coord.run_inner(i, slots))(i)

    def member(i):
        try:
            return loops[i].run()
        finally:
            coord.finish(i)

    try:
        # one host thread per member: each blocks in the coordinator while the
        # shared graph runs (ctypes releases the GIL inside libpdcs)
        with ThreadPoolExecutor(max_workers=len(loops)) as pool:
            out = list(pool.map(member, range(len(loops))))
    finally:
        coord.close()
        for lp in loops:
            lp.close()
    return out
