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
from typing import Any, Callable, Sequence

import numpy as np

from .basic import Drift, Jitter, Reverse, Scale
from .core import Augmenter, Batch, SeedContext, derive_stream
from .errors import InvalidParameterError, UnsupportedPlatformError
from .freqaugment import AmplitudePhasePerturb, FrequencyMask
from .pipeline import Pipeline
from .warp import TimeWarp

_MB = float(1 << 20)
_RSS_PERIOD_S = 0.005


# ---------------------------------------------------------------- report schema (reference bench.py:23-62)
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

    def as_dict(self) -> dict[str, Any]:
        return {"label": self.label, "samples_ms": list(self.samples_ms), "median_ms": self.median_ms,
                "min_ms": self.min_ms, "checksum": self.checksum}

    def csv_cells(self) -> list:
        return [self.label, repr(self.median_ms), repr(self.min_ms), repr(self.checksum)]


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
        _need_report_repeats(self.repeats)


def _need_report_repeats(repeats: int) -> None:
    if repeats < 3:
        raise InvalidParameterError(f"a bench report needs repeats >= 3, got {repeats}")


# ---------------------------------------------------------------- timing
def _timed(call: Callable[[], Batch], repeats: int, label: str) -> TimingRecord:
    """The reference's protocol (bench.py:65-81): one untimed warm-up call
    (it also loads the kernels), then `repeats` wall-clock samples of calls
    that return their host result; the last result's sum is the checksum."""
    if repeats < 1:
        raise InvalidParameterError(f"repeats must be >= 1, got {repeats}")
    call()
    samples = np.empty(repeats)
    result = None
    for k in range(repeats):
        t = time.perf_counter()
        result = call()
        samples[k] = (time.perf_counter() - t) * 1e3
    return TimingRecord(label, tuple(float(v) for v in samples), float(np.median(samples)), float(samples.min()),
                        float(np.sum(result.values)))


def bench_augmenter(aug: Augmenter, batch: Batch, repeats: int = 3, master_seed: int = 0,
                    parallel: bool = False, augmenter_index: int = 0) -> TimingRecord:
    """augment_batch (one fused kernel launch per call) (bench.py:84-97)."""
    return _timed(lambda: aug.augment_batch(batch, master_seed, parallel, augmenter_index), repeats, aug.kind)


def bench_pipeline(pipe: Pipeline, batch: Batch, repeats: int = 3) -> TimingRecord:
    """Pipeline.run (one fused kernel launch per call) (bench.py:100-102)."""
    return _timed(lambda: pipe.run(batch), repeats, "pipeline")


class _RssPeak:
    """Context manager: the process RSS is sampled every 5 ms on a daemon
    thread while the body runs; `mb` is the peak above the entry value."""

    def __init__(self) -> None:
        try:
            import psutil
        except ImportError:
            raise UnsupportedPlatformError("peak-RSS sampling needs psutil, which failed to import") from None
        self._proc = psutil.Process()
        self._done = threading.Event()
        self.mb = 0.0

    def _sample(self) -> None:
        self._peak = max(self._peak, self._proc.memory_info().rss)

    def _loop(self) -> None:
        while not self._done.is_set():
            self._sample()
            self._done.wait(_RSS_PERIOD_S)

    def __enter__(self) -> "_RssPeak":
        self._base = self._peak = self._proc.memory_info().rss
        self._thread = threading.Thread(target=self._loop, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc) -> None:
        self._done.set()
        self._thread.join()
        self._sample()
        self.mb = (self._peak - self._base) / _MB


def measure_peak_memory(work: Callable[[], Any]) -> float:
    """Peak process RSS above baseline while `work` runs, in MB (bench.py:105-141)."""
    with _RssPeak() as peak:
        work()
    return peak.mb


def environment_note() -> str:
    try:
        import torch

        gpu = torch.cuda.get_device_name(torch.cuda.current_device()) if torch.cuda.is_available() else "no GPU"
    except Exception:  # pragma: no cover - informational only
        gpu = "no GPU"
    parts = (platform.platform(), f"Python {platform.python_version()}", f"numpy {np.__version__}",
             f"{os.cpu_count()} cpus", f"{gpu} (paper_2601_03159_b200 device backend)")
    return "; ".join(parts)


def make_report(pipe: Pipeline, batch: Batch, repeats: int = 3, dataset_name: str = "unnamed") -> BenchReport:
    """Every stage timed on the input it really sees (the previous stage's
    output), then the whole pipeline, then peak RSS over one more run
    (bench.py:151-179)."""
    _need_report_repeats(repeats)
    per_stage = []
    seen = batch
    for index, stage in enumerate(pipe.stages):
        per_stage.append(bench_augmenter(stage, seen, repeats, pipe.master_seed, pipe.parallel, index))
        seen = stage.augment_batch(seen, pipe.master_seed, pipe.parallel, index)
    total = bench_pipeline(pipe, batch, repeats)
    try:
        peak: float | None = measure_peak_memory(lambda: pipe.run(batch))
    except UnsupportedPlatformError:
        peak = None
    return BenchReport(dataset_name, batch.n, batch.length, tuple(per_stage), total, peak, repeats,
                       environment_note())


# ---------------------------------------------------------------- serialisation
def report_json(report: BenchReport) -> str:
    fields = (("dataset_name", report.dataset_name), ("n_series", report.n_series),
              ("series_len", report.series_len), ("repeats", report.repeats),
              ("stages", [t.as_dict() for t in report.stage_timings]), ("pipeline", report.pipeline_timing.as_dict()),
              ("peak_rss_mb", report.peak_rss_mb), ("environment", report.environment))
    return json.dumps(dict(fields), indent=2) + "\n"


def report_csv(report: BenchReport) -> str:
    """Header, one row per stage, a final `total` row (bench.py:205-214)."""
    rows: list[Sequence] = [("stage", "label", "median_ms", "min_ms", "checksum")]
    rows += [[index] + t.csv_cells() for index, t in enumerate(report.stage_timings)]
    rows.append(["total"] + report.pipeline_timing.csv_cells())
    out = io.StringIO()
    csv.writer(out, lineterminator="\n").writerows(rows)
    return out.getvalue()


# ---------------------------------------------------------------- inputs and fits
def synthetic_batch(n: int, length: int, seed: int = 0) -> Batch:
    """Seeded Gaussian random walks: cumulative sums of the normals drawn
    from stream SeedContext(seed) (bench.py:217-221)."""
    steps = derive_stream(SeedContext(seed)).normal(0.0, 1.0, (n, length))
    return Batch(np.cumsum(steps, axis=1))


def default_chain() -> tuple[Augmenter, ...]:
    """The CLI's built-in seven-stage length-preserving chain (bench.py:224-234)."""
    return (Jitter(sigma=0.1), Scale(sigma_factor=0.1), Drift(max_drift=0.5, n_points=6),
            TimeWarp(n_knots=4, intensity=0.5), AmplitudePhasePerturb(sigma_amp=0.5, sigma_phase=0.2),
            FrequencyMask(width=10), Reverse())


def power_law_exponent(sizes, times) -> float:
    """Slope of the least-squares line through (log size, log time) (bench.py:237-245)."""
    x, y = (np.asarray(v, dtype=np.float64) for v in (sizes, times))
    if x.size < 2 or x.shape != y.shape:
        raise InvalidParameterError(f"need two or more (size, time) pairs, got {x.size} and {y.size}")
    return float(np.polyfit(np.log(x), np.log(y), 1)[0])
