"""The warp ziggurat walk (sa_rng.cuh normals()) on crafted word streams.

normals() parses a 128-word window in one pass (slow-run parity -> heads,
parallel wedge tests, warp scan of accepted heads).  Real Philox streams are
99.3% fast-path words, so runs of slow words across lanes, all-slow lanes and a
slow head on the window's last word are rare there; tests/csrc/rng_probe.cu
builds the same walk over a caller-supplied word array and this file compares
it with the C oracle's sequential numpy random_standard_normal on the same
words: stream positions after every call exact, values bitwise (tail values
included: they go through sa_log1p, the restatement of the reference libm's
log1p, tests/test_log1p_pin.py).
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from zig_streams import crafted, pattern

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tests", "_build", "librngprobe.so")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def probe():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "csrc")], check=True)
    L = ctypes.CDLL(LIB)
    vp = ctypes.c_void_p
    L.rngprobe_normals.argtypes = [vp, ctypes.c_int64, vp, ctypes.c_int, ctypes.c_int, vp, vp]
    return L


def run_probe(L, words, counts, mode):
    w = np.ascontiguousarray(words, dtype=np.uint64)
    c = np.ascontiguousarray(counts, dtype=np.int32)
    out = np.empty(int(c.sum()))
    pos = np.empty(len(c), dtype=np.int64)
    assert L.rngprobe_normals(w.ctypes.data, w.size, c.ctypes.data, len(c), mode, out.ctypes.data,
                              pos.ctypes.data) == 0
    return out, pos


def check(L, words, counts, mode):
    got, pos = run_probe(L, words, counts, mode)
    skip = 1 if mode == 1 else 0
    want, _ = O.normals_words(words, int(sum(counts)), skip)
    cum = np.cumsum(counts)
    want_pos = [O.normals_words(words, int(n), skip)[1] for n in cum]
    assert list(pos) == want_pos
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


CALLS = [[1000], [1, 2, 3, 127, 128, 129, 5, 500], [97] * 11, [4, 1, 1, 300]]


@pytest.mark.parametrize("p_slow,p_tail", [(0.007, 0.04), (0.05, 0.1), (0.3, 0.0), (0.3, 0.3), (0.6, 0.05),
                                           (0.95, 0.0), (0.95, 0.5)])
@pytest.mark.parametrize("mode", [0, 1])
def test_crafted_streams(probe, p_slow, p_tail, mode):
    for seed, counts in enumerate(CALLS):
        words = crafted(12_000, p_slow, p_tail, seed=seed + int(1000 * p_slow) + int(100 * p_tail))
        check(probe, words, counts, mode)


@pytest.mark.parametrize("spec", [
    "f" * 127 + "w" + "u" + "f" * 300,           # wedge head on the window's last word
    "f" * 126 + "ww" + "u" + "f" * 300,          # wedge run straddling the window end
    "f" * 4 + "wwww" + "f" * 300,                # an all-slow lane
    "f" * 3 + "w" * 9 + "f" * 300,               # a slow run across three lanes
    "f" * 5 + "w" * 12 + "t" + "uuuuuu" + "f" * 300,
    "tuuuu" * 40 + "f" * 300,                    # tails back to back
    "fffw" + "u" + "f" * 300,                    # wedge on the cached gate block's last word
    "ftuu" + "f" * 300,                          # tail inside the cached gate block
    "w" * 300 + "f" * 300,                       # alternating heads / uniforms for a long run
])
@pytest.mark.parametrize("mode", [0, 1])
def test_patterns(probe, spec, mode):
    words = pattern(spec)
    for counts in ([200], [1] * 150, [3, 64, 64, 60]):
        check(probe, words, counts, mode)
