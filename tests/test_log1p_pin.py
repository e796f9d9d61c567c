"""Pin of sa_log1p (paper_2601_03159_b200/csrc/sa_log1p.h) to the C library's
log1p -- the function numpy's ziggurat tail calls (random_standard_normal,
idx 0).  With it the device's tail normals are bitwise the reference's.

CPU: the header compiled by gcc vs libm on 2e7 seeded arguments per domain.
GPU: the same header compiled by nvcc for sm_100a (tests/csrc/rng_probe.cu)
vs libm through ctypes.
"""

import ctypes
import ctypes.util
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "_build")


def test_log1p_restatement_matches_libm_cpu(tmp_path):
    exe = tmp_path / "log1p_pin"
    subprocess.run(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "csrc", "log1p_pin.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), "20000000"], check=True, capture_output=True, text=True).stdout
    rows = [ln.split() for ln in out.strip().splitlines()]
    assert len(rows) == 4
    for name, bad, cnt in rows:
        assert int(cnt) > 1_000_000 and int(bad) == 0, (name, bad, cnt)


@pytest.mark.gpu
def test_log1p_restatement_matches_libm_device():
    lib = os.path.join(BUILD, "librngprobe.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "csrc")], check=True)
    P = ctypes.CDLL(lib)
    P.rngprobe_log1p.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    m = ctypes.CDLL(ctypes.util.find_library("m"))
    m.log1p.restype = ctypes.c_double
    m.log1p.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(11)
    u = (rng.integers(0, 1 << 53, 400_000, dtype=np.uint64).astype(np.float64)) * 2.0 ** -53
    x = np.concatenate([-u, u * 64.0, (u - 0.5) * 1e-6 * u * u, -u ** 4])
    y = np.empty_like(x)
    assert P.rngprobe_log1p(x.ctypes.data, y.ctypes.data, x.size) == 0
    want = np.array([m.log1p(float(v)) for v in x])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))
