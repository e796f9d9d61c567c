"""The genuine reference pipeline on all host cores -- BASELINE
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

This module imports neither torch nor the product package, so spawned worker
processes stay light and the reference arm never loads the B200 library.
"""

from __future__ import annotations

import os
import time

import numpy as np

_STATE: dict = {}


def walks(n: int, L: int, seed: int) -> np.ndarray:
    """Gaussian random walks with N(0, 1) steps (the distribution of the
    reference's synthetic_batch, bench.py:217-221), seeded per block."""
    return np.cumsum(np.random.default_rng(seed).normal(0.0, 1.0, (n, L)), axis=1)


def pipeline_from_config(config: dict):
    from oracle.refpkg import import_reference

    ref = import_reference()
    import oracle.extras_ref  # noqa: F401  (registers the BASELINE-only kinds)

    return ref.Pipeline.parse(config)


def _init(config: dict, rows: int, L: int, seed: int) -> None:
    _STATE["pipe"] = pipeline_from_config(config)
    _STATE["rows"], _STATE["L"], _STATE["seed"] = rows, L, seed


def _work(task: tuple[int, int]) -> tuple[int, float]:
    """Per-sample reference loop over `rows` series whose global indices start
    at `first`; returns (output points, checksum)."""
    from seriesaug.core import SeedContext

    first, block = task
    pipe = _STATE["pipe"]
    x = _STATE.get(("x", block))
    if x is None:
        x = walks(_STATE["rows"], _STATE["L"], _STATE["seed"] * 1_000_003 + block)
        _STATE[("x", block)] = x
    seed = pipe.master_seed
    pts, chk = 0, 0.0
    for q in range(x.shape[0]):
        y = x[q]
        for j, stage in enumerate(pipe.stages):
            y = stage.augment_one(y, SeedContext(seed, j, first + q))
        pts += y.size
        chk += float(y[0])
    return pts, chk


class ProcessPoolRun:
    """A spawn-context pool of `cores` processes, each holding `rows` input
    series; run(step) times one pass of every process over its series."""

    def __init__(self, config: dict, rows: int, L: int, cores: int | None = None, seed: int = 5):
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        self.cores = cores or os.cpu_count() or 1
        self.rows, self.L = rows, L
        self.ex = ProcessPoolExecutor(self.cores, mp_context=mp.get_context("spawn"), initializer=_init,
                                      initargs=(config, rows, L, seed))
        # every worker imports the reference and generates its block (untimed)
        list(self.ex.map(_work, [(w * rows, w) for w in range(self.cores)]))

    def run(self) -> tuple[int, float]:
        t0 = time.perf_counter()
        res = list(self.ex.map(_work, [(w * self.rows, w) for w in range(self.cores)]))
        dt = time.perf_counter() - t0
        return sum(p for p, _ in res), dt

    def close(self):
        self.ex.shutdown()


def time_serial(config: dict, n: int, L: int, parallel: bool, seed: int = 5) -> tuple[int, float]:
    """The reference's own Pipeline.run (standard mode) on an n x L batch."""
    from oracle.refpkg import import_reference

    ref = import_reference()
    cfg = dict(config, parallel=parallel)
    pipe = pipeline_from_config(cfg)
    b = ref.Batch(walks(n, L, seed))
    t0 = time.perf_counter()
    out = pipe.run(b)
    return out.values.size, time.perf_counter() - t0
