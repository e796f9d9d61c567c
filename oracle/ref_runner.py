"""The genuine reference pipeline on the host cores -- BASELINE
INFRASTRUCTURE ONLY (bench.py's reference arm and cpu_baseline legs).

Runs the unmodified reference (`seriesaug` from oracle/_ref, plus the
BASELINE-only kinds as reference plugins, oracle/extras_ref.py) the three ways
SURVEY.md §8(d) lists:

  serial     Pipeline(parallel=False).run        (reference pipeline.py:129-141)
  threads    Pipeline(parallel=True).run          (its thread pool, core.py:146-174)
  processes  a process pool over every host core, each process running the
             reference's per-sample loop -- stage.augment_one(x,
             SeedContext(seed, j, i_global)) for every stage j of series i --
             on its own contiguous range of series (pipeline.py:143-157; bitwise
             the standard mode's result)

This module imports neither torch nor the product package, so the spawned
worker processes stay light and the reference arm never loads the B200
library.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np

_STATE: dict = {}


def walks(n: int, L: int, seed: int) -> np.ndarray:
    """Gaussian random walks with N(0, 1) steps (the distribution of the
    reference's synthetic_batch, bench.py:217-221), seeded per block."""
    return np.cumsum(np.random.default_rng(seed).normal(0.0, 1.0, (n, L)), axis=1)


def reference_pipeline(config: dict):
    from oracle.refpkg import import_reference

    ref = import_reference()
    import oracle.extras_ref  # noqa: F401  (registers the BASELINE-only kinds)

    return ref.Pipeline.parse(config)


def _prepare(task) -> int:
    """Build the task's pipeline and input block in this process (untimed).
    A task is one (config, L, first, rows, seed) block or a list of them."""
    if isinstance(task, list):
        for t in task:
            _prepare(t)
        return os.getpid()
    cfg, L, first, rows, seed = task
    if cfg not in _STATE:
        _STATE[cfg] = reference_pipeline(json.loads(cfg))
    if (rows, L, seed) not in _STATE:
        _STATE[(rows, L, seed)] = walks(rows, L, seed)
    return os.getpid()


def _work(task: tuple) -> tuple[int, float]:
    """One task = (config JSON, L, first global series index, rows, input
    seed): the reference's per-sample loop over `rows` random walks; returns
    (output points, checksum).  Pipelines and inputs are cached per process,
    so a repeated task times the augmentation only."""
    from seriesaug.core import SeedContext

    if isinstance(task, list):
        res = [_work(t) for t in task]
        return sum(r[0] for r in res), sum(r[1] for r in res)
    cfg, L, first, rows, seed = task
    _prepare(task)
    pipe, x = _STATE[cfg], _STATE[(rows, L, seed)]
    ms = pipe.master_seed
    pts, chk = 0, 0.0
    for q in range(rows):
        y = x[q]
        for j, stage in enumerate(pipe.stages):
            y = stage.augment_one(y, SeedContext(ms, j, first + q))
        pts += y.size
        chk += float(y[0])
    return pts, chk


def _worker_main(cmd_q, res_q, barrier) -> None:
    task = None
    while True:
        cmd = cmd_q.get()
        if cmd[0] == "task":
            task = cmd[1]
            _prepare(task)
            res_q.put(("ready", os.getpid()))
        elif cmd[0] == "run":
            barrier.wait()
            t0 = time.perf_counter()
            pts, chk = _work(task)
            res_q.put(("done", pts, time.perf_counter() - t0))
        else:
            return


class ProcessPool:
    """`cores` persistent spawn-context worker processes, one block of series
    each.  run() releases all workers through one barrier and returns the
    points they produced and the slowest worker's time: the wall time of
    the parallel pass (inputs and pipelines are built before the barrier)."""

    def __init__(self, cores: int | None = None):
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        self.cores = cores or os.cpu_count() or 1
        self.barrier = ctx.Barrier(self.cores)
        self.res_q = ctx.Queue()
        self.cmd_q = [ctx.Queue() for _ in range(self.cores)]
        self.procs = [ctx.Process(target=_worker_main, args=(q, self.res_q, self.barrier), daemon=True)
                      for q in self.cmd_q]
        for p in self.procs:
            p.start()

    def assign(self, tasks: list) -> None:
        """Give worker w task w (one per worker) and wait until all are built."""
        assert len(tasks) == self.cores
        for q, t in zip(self.cmd_q, tasks):
            q.put(("task", t))
        for _ in tasks:
            assert self.res_q.get()[0] == "ready"

    def run(self) -> tuple[int, float]:
        for q in self.cmd_q:
            q.put(("run",))
        res = [self.res_q.get() for _ in range(self.cores)]
        return sum(r[1] for r in res), max(r[2] for r in res)

    def close(self) -> None:
        for q in self.cmd_q:
            q.put(("stop",))
        for p in self.procs:
            p.join(timeout=10)


def config_tasks(config: dict, L: int, rows_per_core: int, cores: int, first: int = 0, seed: int = 5) -> list:
    """One contiguous block of series per core (global indices from `first`)."""
    cfg = json.dumps(config, sort_keys=True)
    return [(cfg, L, first + w * rows_per_core, rows_per_core, seed * 1_000_003 + w) for w in range(cores)]


def time_pipeline(config: dict, n: int, L: int, parallel: bool, seed: int = 5) -> tuple[int, float]:
    """The reference's own Pipeline.run (standard mode) on an n x L batch."""
    from oracle.refpkg import import_reference

    ref = import_reference()
    pipe = reference_pipeline(dict(config, parallel=parallel))
    b = ref.Batch(walks(n, L, seed))
    t0 = time.perf_counter()
    out = pipe.run(b)
    return out.values.size, time.perf_counter() - t0
