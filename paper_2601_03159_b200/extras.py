"""BASELINE.json operators that the reference does not implement.

SURVEY.md §8(a) rows M2-M6: Dropout, Pool, Convolve, a speed-change
TimeWarp with cubic resampling, and an additive random-phase sinusoid in the
frequency domain.  They are written as ordinary ``Augmenter`` /
``SpectralAugmenter`` subclasses in the reference's plugin style (frozen
dataclass, ``kind`` registration, gate-first draw order, reference
core.py:177-237), so ``Pipeline`` / JSON configs treat them like the
reference's own kinds.  Their semantics are defined here and restated in the
C oracle (oracle/sa_oracle.c); parity for them is oracle-vs-device only
("parity unpinned by the reference's tests").

Draw order per series (after the gate draw):
  dropout          L doubles u_t; y_t = fill if u_t < rate else x_t
  pool             no draws; block reducer over consecutive `size` samples
  convolve         no draws; edge-replicated, scipy get_window(fftbins=False)
                   taps normalised by their sum
  speed_warp       n_speed_change + 1 uniforms in [1, max_speed_ratio]
  random_sinusoid  bin = integers(min_bin, L//2 + 1), then phase = 2*pi*random()
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import ClassVar

import numpy as np

from . import _abi
from .core import Augmenter
from .errors import InvalidParameterError
from .freqaugment import SpectralAugmenter

POOL_REDUCERS = ("mean", "max", "min")
WINDOWS = ("hann", "hamming", "triang", "flat")
INTERPOLATIONS = ("linear", "cubic")
MAX_CONVOLVE_TAPS = 257


@dataclass(frozen=True)
class Dropout(Augmenter):
    """Replace each sample with `fill` with probability `rate` (BASELINE M2)."""

    rate: float
    fill: float = 0.0
    probability: float = 1.0
    kind: ClassVar[str] = "dropout"

    def _validate(self) -> None:
        if not 0.0 <= self.rate <= 1.0:
            raise InvalidParameterError(f"{self.kind}: rate must lie in [0, 1], got {self.rate}")
        if not math.isfinite(self.fill):
            raise InvalidParameterError(f"{self.kind}: fill must be finite")

    def _lower(self, index, aux):
        return _abi.make_stage(
            _abi.SA_OP_DROPOUT, index, self.probability, f=(self.rate, self.fill)
        )


@dataclass(frozen=True)
class Pool(Augmenter):
    """Length-preserving block pooling: every run of `size` consecutive
    samples is replaced by its mean / max / min (BASELINE M3)."""

    size: int
    reducer: str = "mean"
    probability: float = 1.0
    kind: ClassVar[str] = "pool"

    def _validate(self) -> None:
        if self.size < 1:
            raise InvalidParameterError(f"{self.kind}: size must be >= 1")
        if self.reducer not in POOL_REDUCERS:
            raise InvalidParameterError(
                f"{self.kind}: reducer must be one of {POOL_REDUCERS}, got {self.reducer!r}"
            )

    def _lower(self, index, aux):
        return _abi.make_stage(
            _abi.SA_OP_POOL, index, self.probability,
            i=(self.size, POOL_REDUCERS.index(self.reducer)),
        )


def window_taps(window: str, size: int) -> np.ndarray:
    """The smoothing kernel: scipy.signal.get_window(window, size,
    fftbins=False) -- the symmetric window of filter design ("flat" is
    scipy's "boxcar") -- normalised by its sum.  Computed on the host once per
    stage and uploaded with the stage table."""
    from scipy.signal import get_window

    w = get_window("boxcar" if window == "flat" else window, size, fftbins=False)
    return w / w.sum()


@dataclass(frozen=True)
class Convolve(Augmenter):
    """Smooth with a normalised window, edges replicated (BASELINE M4):
    y[t] = sum_k taps[k] * x[clamp(t + k - size//2)], summed in k order."""

    window: str = "hann"
    size: int = 7
    probability: float = 1.0
    kind: ClassVar[str] = "convolve"

    def _validate(self) -> None:
        if self.window not in WINDOWS:
            raise InvalidParameterError(
                f"{self.kind}: window must be one of {WINDOWS}, got {self.window!r}"
            )
        if not 1 <= self.size <= MAX_CONVOLVE_TAPS:
            raise InvalidParameterError(
                f"{self.kind}: size must lie in [1, {MAX_CONVOLVE_TAPS}], got {self.size}"
            )
        from scipy.signal import get_window

        if not get_window("boxcar" if self.window == "flat" else self.window, self.size, fftbins=False).sum() > 0:
            raise InvalidParameterError(
                f"{self.kind}: the {self.window} window of size {self.size} is all zeros"
            )

    def taps(self) -> np.ndarray:
        return window_taps(self.window, self.size)

    def _lower(self, index, aux):
        off = len(aux)
        aux.extend(float(v) for v in self.taps())
        return _abi.make_stage(
            _abi.SA_OP_CONVOLVE, index, self.probability, aux_off=off, aux_len=self.size
        )


@dataclass(frozen=True)
class SpeedWarp(Augmenter):
    """tsaug-style time warp (BASELINE M5): the series is cut into
    n_speed_change + 1 equal segments, each replayed at a random speed in
    [1, max_speed_ratio]; the cumulative time map is rescaled to end at L-1
    and the series is resampled along it (Catmull-Rom cubic or linear)."""

    n_speed_change: int = 3
    max_speed_ratio: float = 3.0
    interpolation: str = "cubic"
    probability: float = 1.0
    kind: ClassVar[str] = "speed_warp"

    def _validate(self) -> None:
        if self.n_speed_change < 0:
            raise InvalidParameterError(f"{self.kind}: n_speed_change must be >= 0")
        if not self.max_speed_ratio >= 1.0 or not math.isfinite(self.max_speed_ratio):
            raise InvalidParameterError(f"{self.kind}: max_speed_ratio must be >= 1")
        if self.interpolation not in INTERPOLATIONS:
            raise InvalidParameterError(
                f"{self.kind}: interpolation must be one of {INTERPOLATIONS}"
            )

    def validate_for_length(self, length: int) -> None:
        if length < 2:
            raise InvalidParameterError(f"{self.kind}: input length must be >= 2")

    def _lower(self, index, aux):
        return _abi.make_stage(
            _abi.SA_OP_SPEED_WARP, index, self.probability,
            f=(self.max_speed_ratio,),
            i=(self.n_speed_change, INTERPOLATIONS.index(self.interpolation)),
        )


@dataclass(frozen=True)
class RandomSinusoid(SpectralAugmenter):
    """Add amplitude * cos(2*pi*b*t/L + phase) at a random bin b >= min_bin
    with a uniform random phase, applied on the half spectrum (BASELINE M6)."""

    amplitude: float
    min_bin: int = 1
    probability: float = 1.0
    kind: ClassVar[str] = "random_sinusoid"

    def _validate(self) -> None:
        if not math.isfinite(self.amplitude):
            raise InvalidParameterError(f"{self.kind}: amplitude must be finite")
        if self.min_bin < 0:
            raise InvalidParameterError(f"{self.kind}: min_bin must be >= 0")

    def validate_for_length(self, length: int) -> None:
        if self.min_bin > length // 2:
            raise InvalidParameterError(
                f"{self.kind}: min_bin={self.min_bin} exceeds the last bin {length // 2}"
            )

    def _is_noop(self) -> bool:
        return self.amplitude == 0

    def _lower(self, index, aux):
        return _abi.make_stage(
            _abi.SA_OP_SINUSOID, index, self.probability, f=(self.amplitude,), i=(self.min_bin,)
        )
