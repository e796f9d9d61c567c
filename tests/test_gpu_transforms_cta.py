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
