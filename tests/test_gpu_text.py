"""Device number codec vs CPython (the reference's own repr/float calls,
datafiles.py:63,133): bit-exact on every case."""

import numpy as np
import pytest

from text_cases import interesting_doubles, parse_cases, py_float

pytestmark = pytest.mark.gpu


def test_repr_matches_cpython():
    from paper_2601_03159_b200 import textcodec
    import torch

    x = interesting_doubles(400_000)
    got = textcodec.repr_values(torch.from_numpy(x).cuda())
    want = [repr(float(v)) for v in x]
    bad = [(float(v), g, w) for v, g, w in zip(x, got, want) if g != w]
    assert not bad, bad[:10]


def test_repr_specials():
    from paper_2601_03159_b200 import textcodec
    import torch

    x = np.array([np.inf, -np.inf, np.nan, 0.0, -0.0])
    assert textcodec.repr_values(torch.from_numpy(x).cuda()) == ["inf", "-inf", "nan", "0.0", "-0.0"]


def test_parse_matches_cpython():
    from paper_2601_03159_b200 import textcodec

    cases = parse_cases(400_000)
    vals, ok = textcodec.parse_values(cases)
    bad = []
    for s, v, k in zip(cases, vals, ok):
        w, wk = py_float(s)
        if bool(k) != wk or (wk and np.float64(w).view(np.uint64) != np.float64(v).view(np.uint64)
                             and not (np.isnan(w) and np.isnan(v)
                                      and np.signbit(w) == np.signbit(v))):
            bad.append((s[:80], v, k, w, wk))
    assert not bad, bad[:10]


def test_repr_parse_roundtrip_random_bits():
    """Size-independent property at scale: parse(repr(x)) == x bitwise."""
    from paper_2601_03159_b200 import textcodec
    import torch

    rng = np.random.default_rng(11)
    u = rng.integers(0, 2**64, 1_000_000, dtype=np.uint64)
    x = u.view(np.float64)
    x = x[np.isfinite(x)]
    s = textcodec.repr_values(torch.from_numpy(x).cuda())
    v, ok = textcodec.parse_values(s)
    assert ok.all()
    assert np.array_equal(v.view(np.uint64), x.view(np.uint64))
