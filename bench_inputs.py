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


_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream(seed: int, j: int = 0, i: int = 0) -> np.random.Generator:
    """The reference's derive_stream(SeedContext(seed, j, i)) (core.py:40-82),
    computed here in plain Python so input generation never loads the
    product library."""
    g = 0x9E3779B97F4A7C15
    st = _mix64(_mix64(_mix64(seed) + g + j & _M64) + g + i & _M64)
    return np.random.Generator(np.random.Philox(key=_mix64(st) | (_mix64(st + g & _M64) << 64)))


def synthetic_walks(n: int, L: int, seed: int) -> np.ndarray:
    """The reference's synthetic_batch(n, L, seed): cumsum of the normals of
    stream SeedContext(seed) (reference bench.py:217-221)."""
    return np.cumsum(stream(seed).normal(0.0, 1.0, (n, L)), axis=1)


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


def _st(kind, p=1.0, **params):
    return {"kind": kind, "probability": p, "params": params}


def pipeline_config(cfg: int) -> dict:
    """The pipeline each BASELINE config names, as the reference's JSON config
    (pipeline.py:159-201; SURVEY.md §8(d) mapping; geometry ops at p=1 per
    core.py:207-211).  Both arms build from it: the product's Pipeline.parse
    and the reference's (with the BASELINE-only kinds as plugins)."""
    if cfg == 1:
        stages, seed = [_st("jitter", sigma=0.05)], 0
    elif cfg == 2:
        stages = [_st("crop", size=819), _st("drift", 0.5, max_drift=0.5, n_points=5),
                  _st("quantize", 0.5, n_levels=16), _st("dropout", 0.5, rate=0.05), _st("pool", 0.5, size=4),
                  _st("reverse", 0.5)]
        seed = 1
    elif cfg == 3:  # mask 10% of the 1,025 bins of L = 2,048, then the random-phase sinusoid
        stages, seed = [_st("frequency_mask", width=102), _st("random_sinusoid", amplitude=1.0)], 2
    elif cfg == 4:
        stages = [_st("speed_warp", n_speed_change=3, max_speed_ratio=3.0, interpolation="cubic"),
                  _st("resize", target_len=1500), _st("convolve", window="hann", size=7)]
        seed = 3
    else:
        stages, seed = chain5_stages(1024, mask_width=51), 5
    return {"master_seed": seed, "parallel": False, "mode": "standard", "stages": stages}


def chain5_stages(L: int, mask_width: int | None = None) -> list:
    """Config 5's chain of all 20 length-preserving kinds at p = 0.5; for the
    sweep its length-dependent parameters scale with L:
    mask width ~5% of the bins, window = min(128, L), segments <= L."""
    p = 0.5
    bins = L // 2 + 1
    if mask_width is None:
        mask_width = max(1, int(0.05 * bins))
    return [_st("jitter", p, sigma=0.05), _st("scale", p, sigma_factor=0.1), _st("rotate", p),
            _st("permute_segments", p, n_segments=min(4, L)), _st("reverse", p), _st("quantize", p, n_levels=16),
            _st("drift", p, max_drift=0.5, n_points=5),
            _st("inject_noise", p, noise={"kind": "uniform", "half_width": 0.1}),
            _st("inject_noise", p, noise={"kind": "gaussian", "sigma": 0.1}),
            _st("inject_noise", p, noise={"kind": "spike", "count": min(5, L), "magnitude": 2.0}),
            _st("inject_noise", p, noise={"kind": "slope_trend", "max_offset": 0.5}),
            _st("amplitude_phase_perturb", p, sigma_amp=0.1, sigma_phase=0.1),
            _st("frequency_mask", p, width=mask_width),
            _st("time_warp", p, n_knots=5, intensity=0.5),
            _st("time_warp_window", p, window_size=min(128, L), n_knots=4, intensity=0.5),
            _st("dropout", p, rate=0.05), _st("pool", p, size=4), _st("convolve", p, window="hann", size=7),
            _st("random_sinusoid", p, amplitude=0.5, min_bin=min(1, L // 2)),
            _st("speed_warp", p, n_speed_change=3, max_speed_ratio=3.0, interpolation="cubic")]


def pipeline(cfg: int):
    """The product Pipeline for a BASELINE config."""
    from paper_2601_03159_b200 import Pipeline

    return Pipeline.parse(pipeline_config(cfg))


def sweep_datasets(count: int = 100, seed: int = 2026):
    """BASELINE config 5's sweep: `count` synthetic datasets with series
    counts log-uniform in [20, 24000] and lengths log-uniform in [24, 2900]
    (random walks, seed = dataset id).  Returns [(id, n, L)]."""
    rng = np.random.default_rng(seed)
    n = np.exp(rng.uniform(np.log(20), np.log(24_000), count)).astype(int)
    L = np.exp(rng.uniform(np.log(24), np.log(2_900), count)).astype(int)
    return [(i, int(a), int(b)) for i, (a, b) in enumerate(zip(n, L))]


def sweep_config(L: int, seed: int) -> dict:
    return {"master_seed": seed, "parallel": False, "mode": "standard", "stages": chain5_stages(L)}


def sweep_pipeline(L: int, seed: int):
    """The config-5 chain with length-scaled parameters for one sweep dataset."""
    from paper_2601_03159_b200 import Pipeline

    return Pipeline.parse(sweep_config(L, seed))
