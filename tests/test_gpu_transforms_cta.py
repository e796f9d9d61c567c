"""CTA-cooperative transform kernels (csrc/sa_fft_cta.cuh: rfft / irfft /
DCT-II / DCT-III for power-of-two complex lengths N = L/2 in [256, 2048])
against numpy / scipy pocketfft directly (the reference's own calls,
freqtransform.py:47-116; the C oracle's O(L^2) DFT is too slow at L = 8192) and against the warp-per-row kernels
(SA_CTA_FFT=0).  Batch sizes cover one row, fewer rows than CTAs, and several
rows per CTA (grid-stride)."""

import numpy as np
import pytest

import scipy.fft
from paper_2601_03159_b200 import Batch, DctBatch, dct_forward, dct_inverse, fft_forward, fft_inverse
from sa_testutil import spectral_tol

pytestmark = pytest.mark.gpu


def walks(n, L, seed):
    return np.cumsum(np.random.default_rng(seed).normal(0.0, 1.0, (n, L)), axis=1)


@pytest.mark.parametrize("L", [256, 512, 1024, 2048, 4096, 8192])
@pytest.mark.parametrize("n", [1, 37, 3000])
def test_cta_transforms_vs_oracle(L, n):
    x = walks(n, L, L + n)
    sb = fft_forward(Batch(x))
    rows = slice(0, n) if n < 100 else np.r_[0:20, n - 20:n]
    X = np.fft.rfft(x[rows], axis=1)
    re, im = X.real, X.imag
    tol = spectral_tol(re)
    assert np.abs(sb.re[rows] - re).max() <= tol and np.abs(sb.im[rows] - im).max() <= tol
    assert np.all(sb.im[:, 0] == 0.0) and np.all(sb.im[:, -1] == 0.0)
    assert np.abs(fft_inverse(sb).values - x).max() <= spectral_tol(x)
    d = dct_forward(Batch(x))
    want = scipy.fft.dct(x[rows], type=2, norm="ortho", axis=1)
    assert np.abs(d.coeffs[rows] - want).max() <= 1e-10 * max(1.0, np.abs(x).max() * L)
    assert np.abs(dct_inverse(d).values - x).max() <= spectral_tol(x)


@pytest.mark.parametrize("L", [512, 2048, 4096])
def test_cta_matches_warp_kernels(L, monkeypatch):
    x = walks(200, L, 7)
    spec = np.random.default_rng(1).normal(0, 1, (200, L // 2 + 1)) * 50
    spec_im = np.random.default_rng(2).normal(0, 1, (200, L // 2 + 1)) * 50
    spec_im[:, 0] = spec_im[:, -1] = 0.0

    def run():
        sb = fft_forward(Batch(x))
        from paper_2601_03159_b200 import SpectrumBatch

        inv = fft_inverse(SpectrumBatch(spec, spec_im, L)).values
        d = dct_forward(Batch(x)).coeffs
        di = dct_inverse(DctBatch(x)).values
        return sb.re, sb.im, inv, d, di

    a = run()
    monkeypatch.setenv("SA_CTA_FFT", "0")
    b = run()
    for u, v in zip(a, b):
        assert np.abs(u - v).max() <= 1e-12 * max(1.0, np.abs(v).max())


# ---------------------------------------------------------------- spectral-only chains
def _spectral_chains(L):
    from paper_2601_03159_b200 import FrequencyMask, Pipeline, RandomSinusoid

    bins = L // 2 + 1
    return [
        Pipeline(stages=(FrequencyMask(L // 20, probability=0.5), RandomSinusoid(0.5, probability=0.5)),
                 master_seed=3),  # BASELINE config 3's shape
        Pipeline(stages=(RandomSinusoid(1.0, min_bin=0), FrequencyMask(0), RandomSinusoid(0.3, min_bin=bins - 2),
                         FrequencyMask(bins, probability=0.3), RandomSinusoid(2.0, probability=0.7)),
                 master_seed=11),  # DC / Nyquist bins, a no-op mask, a mask over every bin
        Pipeline(stages=(FrequencyMask(7),), master_seed=5),
    ]


@pytest.mark.parametrize("L", [512, 1024, 2048, 4096])
def test_cta_spectral_chain_vs_oracle(L):
    import torch

    from oracle import oracle as O

    x = walks(300, L, L)
    for pipe in _spectral_chains(L):
        got = pipe.run_device(torch.from_numpy(x).cuda(), series_offset=17).cpu().numpy()
        want = O.run_pipeline(pipe, x[:64], series_offset=17)
        assert np.abs(got[:64] - want).max() <= spectral_tol(want), pipe.stages
        # rows whose stages all stay off are copied bitwise
        same = np.flatnonzero(np.all(want == x[:64], axis=1))
        assert np.array_equal(got[same], x[same])


@pytest.mark.parametrize("L", [512, 2048])
def test_cta_spectral_chain_matches_warp_chain(L, monkeypatch):
    import torch

    x = torch.from_numpy(walks(500, L, 3)).cuda()
    for pipe in _spectral_chains(L):
        a = pipe.run_device(x).cpu().numpy()
        monkeypatch.setenv("SA_CTA_CHAIN", "0")
        b = pipe.run_device(x).cpu().numpy()
        monkeypatch.delenv("SA_CTA_CHAIN")
        assert np.abs(a - b).max() <= 1e-11 * max(1.0, np.abs(b).max())


def test_cta_spectral_chain_nonfinite_input():
    import torch

    from paper_2601_03159_b200 import InvalidInputError

    x = walks(40, 1024, 1)
    x[13, 100] = np.nan
    with pytest.raises(InvalidInputError):
        _spectral_chains(1024)[0].run_device(torch.from_numpy(x).cuda())
