"""Shared test helpers (tolerances, comparisons)."""

import numpy as np


def spectral_tol(expected: np.ndarray) -> float:
    """Absolute tolerance for FFT-bearing results: 1e-10 x row scale, the
    reference's own transform bound (test_freqtransform.py:63-70 uses 1e-9 on
    unit-scale data) tightened by 10x."""
    return 1e-10 * max(1.0, float(np.abs(expected).max()))


def assert_matches(got: np.ndarray, want: np.ndarray, exact: bool, what: str = ""):
    assert got.shape == want.shape, (what, got.shape, want.shape)
    if exact:  # bitwise: identical float64 bit patterns, sign of zero included
        bad = np.flatnonzero(np.ascontiguousarray(got).view(np.uint64) != np.ascontiguousarray(want).view(np.uint64))
        assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]}"
    else:
        err = float(np.abs(got - want).max()) if got.size else 0.0
        assert err <= spectral_tol(want), f"{what}: max abs err {err:.3e}"
