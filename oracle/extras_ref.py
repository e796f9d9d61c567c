"""BASELINE-only operators as plugins of the GENUINE reference -- TEST /
BASELINE INFRASTRUCTURE ONLY.

BASELINE.json names five operators the reference does not implement (SURVEY.md
§8(a) M2-M6).  Here each is written the way the reference's own plugin API
asks (reference core.py:177-237: a frozen dataclass subclass of `Augmenter`
with a `kind`, a per-series `_apply(series, rng)` drawing from the stream
after the gate; reference freqaugment.py:24-47: a `SpectralAugmenter` with
`_perturb_row(re, im, original_len, rng)` on the reference's own rfft/irfft
plumbing), in numpy, on top of the reference package imported unmodified
(oracle/refpkg.py).  Registering them puts their kinds in the reference's
AUGMENTER_REGISTRY, so the reference's own `Pipeline.parse(...).run(...)`
executes every stage of BASELINE config 5 -- these goldens
(tests/golden/make_golden.py) and bench.py's reference arm come from it.

Semantics (the product's paper_2601_03159_b200/extras.py implements the same
on the device; the C oracle restates them in sa_oracle.c):
  dropout          L doubles u_t = random(); y_t = fill if u_t < rate else x_t
  pool             consecutive blocks of `size` samples (the last one may be
                   shorter) replaced by their mean (summed left to right, then
                   divided by the block length) / max / min
  convolve         taps = scipy.signal.get_window(window, size, fftbins=False)
                   normalised by their sum ("flat" = "boxcar"); edges
                   replicated: y_t = sum_k taps[k] x[clip(t + k - size//2)],
                   accumulated from 0.0 in k order
  speed_warp       n_speed_change + 1 speeds = uniform(1, max_speed_ratio);
                   segment m = [(mL + K)//(K+1), ((m+1)L + K)//(K+1)), K =
                   n_speed_change; tau_t = cumulative segment bases + speed_m
                   (t - start_m), rescaled by (L-1)/tau_{L-1}, tau_{L-1} = L-1;
                   y_t = Catmull-Rom (or linear) interpolation of x at tau_t
  random_sinusoid  b = min_bin + integers(0, L//2 + 1 - min_bin), phase =
                   2 pi random(); adds amplitude cos(2 pi b t / L + phase):
                   bin b += (A L / 2) e^{i phase} (DC / Nyquist: re += A L cos)
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass
from typing import ClassVar

import numpy as np

from oracle.refpkg import import_reference

sa = import_reference()
from seriesaug.core import Augmenter  # noqa: E402
from seriesaug.errors import InvalidParameterError  # noqa: E402
from seriesaug.freqaugment import SpectralAugmenter  # noqa: E402

POOL_REDUCERS = ("mean", "max", "min")
WINDOWS = ("hann", "hamming", "triang", "flat")
INTERPOLATIONS = ("linear", "cubic")


@functools.lru_cache(maxsize=64)
def window_taps(window: str, size: int) -> np.ndarray:
    from scipy.signal import get_window

    w = get_window("boxcar" if window == "flat" else window, size, fftbins=False)
    return w / w.sum()


@dataclass(frozen=True)
class Dropout(Augmenter):
    rate: float
    fill: float = 0.0
    probability: float = 1.0
    kind: ClassVar[str] = "dropout"

    def _validate(self) -> None:
        if not 0.0 <= self.rate <= 1.0:
            raise InvalidParameterError(f"{self.kind}: rate must lie in [0, 1], got {self.rate}")

    def _apply(self, x, rng):
        if self.rate == 0.0:
            return x.copy()
        u = rng.random(x.size)
        return np.where(u < self.rate, self.fill, x)


@dataclass(frozen=True)
class Pool(Augmenter):
    size: int
    reducer: str = "mean"
    probability: float = 1.0
    kind: ClassVar[str] = "pool"

    def _validate(self) -> None:
        if self.size < 1 or self.reducer not in POOL_REDUCERS:
            raise InvalidParameterError(f"{self.kind}: bad parameters")

    def _apply(self, x, rng):
        P, L = self.size, x.size
        if P == 1:
            return x.copy()
        y = np.empty_like(x)
        for b0, b1 in ((0, L - L % P), (L - L % P, L)):
            if b1 <= b0:
                continue
            n = min(P, b1 - b0)
            blk = x[b0:b1].reshape(-1, n)
            if self.reducer == "mean":
                acc = np.zeros(blk.shape[0])
                for k in range(n):
                    acc = acc + blk[:, k]
                v = acc / float(n)
            else:
                v = blk[:, 0].copy()
                for k in range(1, n):
                    c = blk[:, k]
                    v = np.where(c > v, c, v) if self.reducer == "max" else np.where(c < v, c, v)
            y[b0:b1] = np.repeat(v, n)
        return y


@dataclass(frozen=True)
class Convolve(Augmenter):
    window: str = "hann"
    size: int = 7
    probability: float = 1.0
    kind: ClassVar[str] = "convolve"

    def _validate(self) -> None:
        if self.window not in WINDOWS or self.size < 1:
            raise InvalidParameterError(f"{self.kind}: bad parameters")

    def _apply(self, x, rng):
        taps = window_taps(self.window, self.size)
        S, h, L = self.size, self.size // 2, x.size
        xp = np.concatenate([np.full(h, x[0]), x, np.full(S - 1 - h, x[-1])])
        acc = np.zeros(L)
        for k in range(S):
            acc = acc + taps[k] * xp[k:k + L]
        return acc


def speed_map(L: int, speeds: np.ndarray) -> np.ndarray:
    K = speeds.size - 1
    starts = np.array([(m * L + K) // (K + 1) for m in range(K + 1)], dtype=np.int64)
    base = np.zeros(K + 1)
    for m in range(K):  # sequential, as the cumulative time is built
        base[m + 1] = base[m] + speeds[m] * float(starts[m + 1] - starts[m])
    t = np.arange(L)
    m = np.searchsorted(starts[1:], t, side="right")
    tau = base[m] + speeds[m] * (t - starts[m]).astype(np.float64)
    tau = tau * ((float(L) - 1.0) / tau[L - 1])
    tau[L - 1] = float(L) - 1.0
    return tau


def resample(x: np.ndarray, tau: np.ndarray, cubic: bool) -> np.ndarray:
    L = x.size
    j = np.clip(np.floor(tau).astype(np.int64), 0, L - 2)
    f = tau - j.astype(np.float64)
    p1, p2 = x[j], x[j + 1]
    if cubic:
        p0 = x[np.maximum(j - 1, 0)]
        p3 = x[np.minimum(j + 2, L - 1)]
        a = ((-0.5 * p0 + 1.5 * p1) - 1.5 * p2) + 0.5 * p3
        b = ((p0 - 2.5 * p1) + 2.0 * p2) - 0.5 * p3
        c = -0.5 * p0 + 0.5 * p2
        y = ((a * f + b) * f + c) * f + p1
    else:
        y = p1 + (p2 - p1) * f
    y = np.where(tau <= 0.0, x[0], y)
    return np.where(tau >= float(L - 1), x[L - 1], y)


@dataclass(frozen=True)
class SpeedWarp(Augmenter):
    n_speed_change: int = 3
    max_speed_ratio: float = 3.0
    interpolation: str = "cubic"
    probability: float = 1.0
    kind: ClassVar[str] = "speed_warp"

    def _validate(self) -> None:
        if self.n_speed_change < 0 or not self.max_speed_ratio >= 1.0 or self.interpolation not in INTERPOLATIONS:
            raise InvalidParameterError(f"{self.kind}: bad parameters")

    def validate_for_length(self, length: int) -> None:
        if length < 2:
            raise InvalidParameterError(f"{self.kind}: input length must be >= 2")

    def _apply(self, x, rng):
        if self.n_speed_change == 0 or self.max_speed_ratio == 1.0:
            return x.copy()
        speeds = rng.uniform(1.0, self.max_speed_ratio, self.n_speed_change + 1)
        return resample(x, speed_map(x.size, speeds), self.interpolation == "cubic")


@dataclass(frozen=True)
class RandomSinusoid(SpectralAugmenter):
    amplitude: float
    min_bin: int = 1
    probability: float = 1.0
    kind: ClassVar[str] = "random_sinusoid"

    def _validate(self) -> None:
        if not math.isfinite(self.amplitude) or self.min_bin < 0:
            raise InvalidParameterError(f"{self.kind}: bad parameters")

    def validate_for_length(self, length: int) -> None:
        if self.min_bin > length // 2:
            raise InvalidParameterError(f"{self.kind}: min_bin exceeds the last bin")

    def _is_noop(self) -> bool:
        return self.amplitude == 0

    def _perturb_row(self, re, im, original_len, rng):
        bins = re.size
        b = self.min_bin + int(rng.integers(0, bins - self.min_bin))
        phi = 2.0 * np.pi * rng.random()
        A = self.amplitude
        if b == 0 or (original_len % 2 == 0 and b == bins - 1):
            re[b] = re[b] + (A * float(original_len)) * math.cos(phi)
        else:
            h = (A * float(original_len)) * 0.5
            re[b] = re[b] + h * math.cos(phi)
            im[b] = im[b] + h * math.sin(phi)
        return re, im


EXTRA_KINDS = ("dropout", "pool", "convolve", "speed_warp", "random_sinusoid")
