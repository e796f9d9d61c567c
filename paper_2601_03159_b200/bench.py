"""Wall-time and peak-memory reports for augmenters and pipelines, on the
device backend (reference: bench.py, the
`make_report` route).

Same protocol and report schema as the reference: one warm-up call, then
`repeats` timed calls of the public (host-buffer) API, each sample the wall
time of a call that has returned its host result -- so every sample includes
the H2D copy, the fused kernel and the D2H copy.  The checksum of the last
output is kept; peak memory is the process RSS above baseline sampled on a
watcher thread (host memory; device memory is not RSS).  `environment_note`
names the GPU.  Timings are wall clock of the API, not kernel events: for
kernel-level numbers use the repo's root `bench.py`.
"""

from __future__ import annotations

import csv
import io
import json
import os
import platform
import threading
import time
from dataclasses import dataclass
from typing import Any, Callable

import numpy as np

from .basic import Drift, Jitter, Reverse, Scale
from .core import Augmenter, Batch, SeedContext, derive_stream
from .errors import InvalidParameterError, UnsupportedPlatformError
from .freqaugment import AmplitudePhasePerturb, FrequencyMask
from .pipeline import Pipeline
from .warp import TimeWarp

_MB = 1 << 20


@dataclass(frozen=True)
class TimingRecord:
    label: str
    samples_ms: tuple[float, ...]
    median_ms: float
    min_ms: float
    checksum: float

    @property
    def repeats(self) -> int:
        return len(self.samples_ms)


@dataclass(frozen=True)
class BenchReport:
    dataset_name: str
    n_series: int
    series_len: int
    stage_timings: tuple[TimingRecord, ...]
    pipeline_timing: TimingRecord
    peak_rss_mb: float | None
    repeats: int
    environment: str

    def __post_init__(self) -> None:
        if self.repeats < 3:
            raise InvalidParameterError(f"a bench report needs repeats >= 3, got {self.repeats}")


def _time_runs(fn: Callable[[], Batch], repeats: int, label: str) -> TimingRecord:
    if repeats < 1:
        raise InvalidParameterError(f"repeats must be >= 1, got {repeats}")
    fn()  # warm-up (also loads the kernels)
    samples = []
    out = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        out = fn()
        samples.append((time.perf_counter() - t0) * 1e3)
    return TimingRecord(label=label, samples_ms=tuple(samples), median_ms=float(np.median(samples)),
                        min_ms=min(samples), checksum=float(np.sum(out.values)))


def bench_augmenter(aug: Augmenter, batch: Batch, repeats: int = 3, master_seed: int = 0,
                    parallel: bool = False, augmenter_index: int = 0) -> TimingRecord:
    """Median/min wall time of augment_batch (one fused launch) (bench.py:84-97)."""
    return _time_runs(lambda: aug.augment_batch(batch, master_seed, parallel, augmenter_index), repeats,
                      aug.kind)


def bench_pipeline(pipe: Pipeline, batch: Batch, repeats: int = 3) -> TimingRecord:
    """Median/min wall time of a full pipeline run (bench.py:100-102)."""
    return _time_runs(lambda: pipe.run(batch), repeats, "pipeline")


def measure_peak_memory(work: Callable[[], Any]) -> float:
    """Peak process RSS above baseline during `work`, in MB (bench.py:105-141)."""
    try:
        import psutil
    except ImportError:
        raise UnsupportedPlatformError("peak-RSS sampling needs psutil, which failed to import") from None
    proc = psutil.Process()
    baseline = proc.memory_info().rss
    peak = baseline
    stop = threading.Event()

    def watch() -> None:
        nonlocal peak
        while not stop.is_set():
            peak = max(peak, proc.memory_info().rss)
            stop.wait(0.005)

    watcher = threading.Thread(target=watch, daemon=True)
    watcher.start()
    try:
        work()
    finally:
        stop.set()
        watcher.join()
    peak = max(peak, proc.memory_info().rss)
    return (peak - baseline) / _MB


def environment_note() -> str:
    gpu = "no GPU"
    try:
        import torch

        if torch.cuda.is_available():
            gpu = torch.cuda.get_device_name(torch.cuda.current_device())
    except Exception:  # pragma: no cover - informational only
        pass
    return (f"{platform.platform()}; Python {platform.python_version()}; numpy {np.__version__}; "
            f"{os.cpu_count()} cpus; {gpu} (paper_2601_03159_b200 device backend)")


def make_report(pipe: Pipeline, batch: Batch, repeats: int = 3, dataset_name: str = "unnamed") -> BenchReport:
    """Each stage on its true intermediate input, then the whole pipeline,
    then peak RSS over one more run (bench.py:151-179)."""
    if repeats < 3:
        raise InvalidParameterError(f"a bench report needs repeats >= 3, got {repeats}")
    stage_timings = []
    current = batch
    for j, stage in enumerate(pipe.stages):
        stage_timings.append(bench_augmenter(stage, current, repeats, pipe.master_seed, pipe.parallel, j))
        current = stage.augment_batch(current, pipe.master_seed, pipe.parallel, j)
    pipeline_timing = bench_pipeline(pipe, batch, repeats)
    try:
        peak = measure_peak_memory(lambda: pipe.run(batch))
    except UnsupportedPlatformError:
        peak = None
    return BenchReport(dataset_name=dataset_name, n_series=batch.n, series_len=batch.length,
                       stage_timings=tuple(stage_timings), pipeline_timing=pipeline_timing, peak_rss_mb=peak,
                       repeats=repeats, environment=environment_note())


def _record(t: TimingRecord) -> dict[str, Any]:
    return {"label": t.label, "samples_ms": list(t.samples_ms), "median_ms": t.median_ms, "min_ms": t.min_ms,
            "checksum": t.checksum}


def report_json(report: BenchReport) -> str:
    doc = {"dataset_name": report.dataset_name, "n_series": report.n_series, "series_len": report.series_len,
           "repeats": report.repeats, "stages": [_record(t) for t in report.stage_timings],
           "pipeline": _record(report.pipeline_timing), "peak_rss_mb": report.peak_rss_mb,
           "environment": report.environment}
    return json.dumps(doc, indent=2) + "\n"


def report_csv(report: BenchReport) -> str:
    """One row per stage plus a final pipeline-total row (bench.py:205-214)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["stage", "label", "median_ms", "min_ms", "checksum"])
    for j, t in enumerate(report.stage_timings):
        w.writerow([j, t.label, repr(t.median_ms), repr(t.min_ms), repr(t.checksum)])
    p = report.pipeline_timing
    w.writerow(["total", p.label, repr(p.median_ms), repr(p.min_ms), repr(p.checksum)])
    return buf.getvalue()


def synthetic_batch(n: int, length: int, seed: int = 0) -> Batch:
    """Seeded Gaussian random walks: cumsum of the normals of stream
    SeedContext(seed) (bench.py:217-221)."""
    rng = derive_stream(SeedContext(seed))
    return Batch(np.cumsum(rng.normal(0.0, 1.0, (n, length)), axis=1))


def default_chain() -> tuple[Augmenter, ...]:
    """The seven length-preserving stages of the CLI default (bench.py:224-234)."""
    return (Jitter(sigma=0.1), Scale(sigma_factor=0.1), Drift(max_drift=0.5, n_points=6),
            TimeWarp(n_knots=4, intensity=0.5), AmplitudePhasePerturb(sigma_amp=0.5, sigma_phase=0.2),
            FrequencyMask(width=10), Reverse())


def power_law_exponent(sizes, times) -> float:
    """Least-squares slope of log(time) against log(size) (bench.py:237-245)."""
    sizes = np.asarray(sizes, dtype=np.float64)
    times = np.asarray(times, dtype=np.float64)
    if sizes.shape != times.shape or sizes.size < 2:
        raise InvalidParameterError(
            f"need two or more (size, time) pairs, got {sizes.size} and {times.size}")
    return float(np.polyfit(np.log(sizes), np.log(times), 1)[0])
