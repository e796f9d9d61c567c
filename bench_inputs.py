"""Seeded synthetic inputs and pipelines for the five BASELINE.json configs.

The paper's aeon corpus is not available (no network); these generators
stand in for it with the shapes, sizes and value distributions BASELINE.json
names.  Measurement infrastructure, not product code.

  1  1,000 x 512     sum of 3 sinusoids (periods U[8,128], amplitudes U(0.5,2),
                     phases U[0,2pi)) + N(0, 0.1^2), seed 0
  2  10,000 x 1,024  Gaussian random walks, N(0,1) steps, seed 1 (the
                     reference's synthetic_batch construction, bench.py:217-221)
  3  50,000 x 2,048  AR(2), phi = (0.6, -0.2), unit noise, zero init, seed 2
  4  100,000 x 1,500 random walk + sinusoid (period 200, amplitude 3), seed 3
  5  1,000,000 x 1,024 random walks (8.2 GB), generated on the GPU from a
                     seeded torch generator (a numpy stream of 1e9 normals
                     would take minutes on the host), seed 5
"""

from __future__ import annotations

import numpy as np

CONFIG_SHAPES = {1: (1000, 512), 2: (10_000, 1024), 3: (50_000, 2048), 4: (100_000, 1500), 5: (1_000_000, 1024)}


def config1_input(n: int = 1000, L: int = 512, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    t = np.arange(L)
    x = np.zeros((n, L))
    for _ in range(3):
        per = rng.uniform(8, 128, (n, 1))
        amp = rng.uniform(0.5, 2.0, (n, 1))
        ph = rng.uniform(0, 2 * np.pi, (n, 1))
        x += amp * np.sin(2 * np.pi * t / per + ph)
    return x + rng.normal(0, 0.1, (n, L))


def synthetic_walks(n: int, L: int, seed: int) -> np.ndarray:
    """The reference's synthetic_batch(n, L, seed): cumsum of the normals of
    stream SeedContext(seed) (reference bench.py:217-221)."""
    from paper_2601_03159_b200.core import SeedContext, derive_stream

    rng = derive_stream(SeedContext(seed))
    return np.cumsum(rng.normal(0.0, 1.0, (n, L)), axis=1)


def ar2_input(n: int = 50_000, L: int = 2048, seed: int = 2, phi=(0.6, -0.2)) -> np.ndarray:
    from scipy.signal import lfilter

    e = np.random.default_rng(seed).normal(0.0, 1.0, (n, L))
    return lfilter([1.0], [1.0, -phi[0], -phi[1]], e, axis=1)


def walk_sine_input(n: int = 100_000, L: int = 1500, seed: int = 3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = np.cumsum(rng.normal(0.0, 1.0, (n, L)), axis=1)
    return x + 3.0 * np.sin(2 * np.pi * np.arange(L) / 200.0)


def device_walks(n: int, L: int, seed: int, device, row0: int = 0):
    """Random walks generated on the GPU (config 5); rows are a pure function
    of (seed, global row) chunk so shards are reproducible."""
    import torch

    out = torch.empty((n, L), dtype=torch.float64, device=device)
    chunk = 65536
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + (row0 + a) // chunk)
        steps = torch.randn((b - a, L), dtype=torch.float64, device=device, generator=g)
        torch.cumsum(steps, dim=1, out=out[a:b])
    return out


def host_input(cfg: int, n: int | None = None) -> np.ndarray:
    N, L = CONFIG_SHAPES[cfg]
    n = N if n is None else n
    if cfg == 1:
        return config1_input(n, L)
    if cfg == 2:
        return synthetic_walks(n, L, 1)
    if cfg == 3:
        return ar2_input(n, L)
    if cfg == 4:
        return walk_sine_input(n, L)
    return synthetic_walks(n, L, 5)


def pipeline(cfg: int):
    """The pipeline each BASELINE config names, in the reference's plugin
    API (SURVEY.md §8(d) mapping; geometry ops at p=1 per core.py:207-211)."""
    from paper_2601_03159_b200 import (AmplitudePhasePerturb, Convolve, Crop, Drift, Dropout, FrequencyMask,
                                       GaussianNoise, InjectNoise, Jitter, PermuteSegments, Pipeline, Pool,
                                       Quantize, RandomSinusoid, Resize, Reverse, Rotate, Scale, SlopeTrendNoise,
                                       SpeedWarp, SpikeNoise, TimeWarp, UniformNoise, WindowWarp)

    if cfg == 1:
        stages = (Jitter(sigma=0.05),)
        seed = 0
    elif cfg == 2:
        stages = (Crop(819), Drift(0.5, 5, probability=0.5), Quantize(16, probability=0.5),
                  Dropout(0.05, probability=0.5), Pool(4, probability=0.5), Reverse(probability=0.5))
        seed = 1
    elif cfg == 3:
        stages = (FrequencyMask(102), RandomSinusoid(1.0))  # 10% of the 1,025 bins of L = 2,048
        seed = 2
    elif cfg == 4:
        stages = (SpeedWarp(3, 3.0, "cubic"), Resize(1500), Convolve("hann", 7))
        seed = 3
    else:
        p = 0.5
        stages = (Jitter(0.05, probability=p), Scale(0.1, probability=p), Rotate(probability=p),
                  PermuteSegments(4, probability=p), Reverse(probability=p), Quantize(16, probability=p),
                  Drift(0.5, 5, probability=p), InjectNoise(UniformNoise(0.1), probability=p),
                  InjectNoise(GaussianNoise(0.1), probability=p), InjectNoise(SpikeNoise(5, 2.0), probability=p),
                  InjectNoise(SlopeTrendNoise(0.5), probability=p),
                  AmplitudePhasePerturb(0.1, 0.1, probability=p), FrequencyMask(51, probability=p),
                  TimeWarp(5, 0.5, probability=p), WindowWarp(128, 4, 0.5, probability=p),
                  Dropout(0.05, probability=p), Pool(4, probability=p), Convolve("hann", 7, probability=p),
                  RandomSinusoid(0.5, probability=p), SpeedWarp(3, 3.0, probability=p))
        seed = 5
    return Pipeline(stages=stages, master_seed=seed)


def sweep_datasets(count: int = 100, seed: int = 2026):
    """BASELINE config 5's sweep: `count` synthetic datasets with series
    counts log-uniform in [20, 24000] and lengths log-uniform in [24, 2900]
    (random walks, seed = dataset id).  Returns [(id, n, L)]."""
    rng = np.random.default_rng(seed)
    n = np.exp(rng.uniform(np.log(20), np.log(24_000), count)).astype(int)
    L = np.exp(rng.uniform(np.log(24), np.log(2_900), count)).astype(int)
    return [(i, int(a), int(b)) for i, (a, b) in enumerate(zip(n, L))]


def sweep_pipeline(L: int, seed: int):
    """The config-5 chain with length-scaled parameters:
    mask width ~5% of the bins, window = min(128, L), segments <= L."""
    from paper_2601_03159_b200 import (AmplitudePhasePerturb, Convolve, Drift, Dropout, FrequencyMask,
                                       GaussianNoise, InjectNoise, Jitter, PermuteSegments, Pipeline, Pool,
                                       Quantize, RandomSinusoid, Reverse, Rotate, Scale, SlopeTrendNoise,
                                       SpeedWarp, SpikeNoise, TimeWarp, UniformNoise, WindowWarp)

    p = 0.5
    bins = L // 2 + 1
    stages = (Jitter(0.05, probability=p), Scale(0.1, probability=p), Rotate(probability=p),
              PermuteSegments(min(4, L), probability=p), Reverse(probability=p), Quantize(16, probability=p),
              Drift(0.5, 5, probability=p), InjectNoise(UniformNoise(0.1), probability=p),
              InjectNoise(GaussianNoise(0.1), probability=p),
              InjectNoise(SpikeNoise(min(5, L), 2.0), probability=p),
              InjectNoise(SlopeTrendNoise(0.5), probability=p), AmplitudePhasePerturb(0.1, 0.1, probability=p),
              FrequencyMask(max(1, int(0.05 * bins)), probability=p), TimeWarp(5, 0.5, probability=p),
              WindowWarp(min(128, L), 4, 0.5, probability=p), Dropout(0.05, probability=p),
              Pool(4, probability=p), Convolve("hann", 7, probability=p),
              RandomSinusoid(0.5, min_bin=min(1, L // 2), probability=p), SpeedWarp(3, 3.0, probability=p))
    return Pipeline(stages=stages, master_seed=seed)
