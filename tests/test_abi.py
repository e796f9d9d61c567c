"""The C ABI boundary (CPU-only checks, no compute calls).

* every constant of include/seriesaug_b200.h matches the ctypes mirror;
* struct sa_stage has the same size and field offsets on both sides;
* the built library loads and exports every function the header declares;
* the host-only entry points that need no device work (version, key
  derivation) behave.
"""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2601_03159_b200 import _abi, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seriesaug_b200.h")


def header_text():
    with open(HEADER) as fh:
        return fh.read()


def test_constants_match_header():
    defs = dict(re.findall(r"#define\s+(SA_[A-Z0-9_]+)\s+(-?\w+)", header_text()))
    checked = 0
    for name, val in defs.items():
        if name in ("SERIESAUG_B200_H",):
            continue
        v = int(val.rstrip("u"), 0)
        assert getattr(_abi, name) == v, name
        checked += 1
    assert checked >= 30


def declared_functions():
    return re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(sa_\w+)\s*\(", header_text(), re.M)


def test_header_declares_expected_entry_points():
    fns = set(declared_functions())
    for fn in ("sa_init", "sa_pipeline_launch", "sa_pipeline_run", "sa_pipeline_run_host", "sa_fft_forward",
               "sa_fft_inverse", "sa_augment_spectrum", "sa_derive_key", "sa_last_error", "sa_abi_version"):
        assert fn in fns


def test_struct_layout_matches_c():
    """Compile a probe against the header and compare sizeof/offsetof."""
    src = r"""
    #include <stddef.h>
    #include <stdio.h>
    #include "seriesaug_b200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(sa_stage), offsetof(sa_stage, op),
             offsetof(sa_stage, index), offsetof(sa_stage, probability), offsetof(sa_stage, f),
             offsetof(sa_stage, i), offsetof(sa_stage, aux_off), offsetof(sa_stage, aux_len));
      return 0;
    }
    """
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        c = os.path.join(td, "probe.c")
        exe = os.path.join(td, "probe")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    S = _abi.SaStage
    want = [ctypes.sizeof(S), S.op.offset, S.index.offset, S.probability.offset, S.f.offset, S.i.offset,
            S.aux_off.offset, S.aux_len.offset]
    assert got == want


def test_library_exports_every_declared_symbol():
    lib = _native.lib()  # raises if the .so is missing
    for fn in declared_functions():
        assert hasattr(lib, fn), fn
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for fn in declared_functions():
        assert re.search(rf"\bT {fn}\b", out), fn


def test_library_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_side_entry_points():
    lib = _native.lib()
    assert lib.sa_abi_version() == _abi.SA_ABI_VERSION
    from oracle import oracle as O

    for ctx in [(0, 0, 0), (5, 7, 123), (2**64 - 1, 3, 2**40)]:
        assert _native.derive_key(*ctx) == O.derive_key(*ctx)


def test_no_cpu_fallback_without_device():
    """On a machine without a CUDA device the product raises instead of
    computing anything on the host."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np

    from paper_2601_03159_b200 import Batch, Jitter, UnsupportedPlatformError

    with pytest.raises(UnsupportedPlatformError):
        Jitter(0.1).augment_batch(Batch(np.zeros((2, 4))), 1)


def test_entry_points_reject_bad_arguments_before_device_work():
    """Null buffers and negative sizes come back as SA_ERR_INVALID_ARG (no
    device needed: the checks run before any CUDA call)."""
    L = _native.lib()
    E = _abi.SA_ERR_INVALID_ARG
    null = None
    st = (_abi.SaStage * 1)()
    assert L.sa_derive_key(1, 2, 3, None, None) == E
    for fn in (L.sa_pipeline_run, L.sa_pipeline_run_host):
        extra = [None] if fn is L.sa_pipeline_run else []
        assert fn(st, 1, None, 0, 0, 0, null, 4, 8, null, 8, *extra) == E       # null batch
        assert fn(None, 1, None, 0, 0, 0, null, 0, 8, null, 8, *extra) == E      # stage table missing
        assert fn(st, 1, None, 3, 0, 0, null, 0, 8, null, 8, *extra) == E        # aux table missing
        assert fn(st, 1, None, 0, 0, 0, null, -1, 8, null, 8, *extra) == E       # n < 0
    assert L.sa_pipeline_launch(st, 1, None, 0, 0, 0, null, 0, 8, null, 8, None, None) == E  # flags
    assert L.sa_fft_forward(None, 2, 8, None, None, None) == E
    assert L.sa_fft_inverse(None, None, 2, 8, None, None) == E
    assert L.sa_dct_forward(None, 2, 8, None, None) == E
    assert L.sa_dct_inverse(None, 2, 0, None, None) == E
    assert L.sa_fft_forward_host(None, 2, 8, None, None) == E
    assert L.sa_fft_inverse_host(None, None, 2, 8, None) == E
    assert L.sa_dct_forward_host(None, 2, 8, None) == E
    assert L.sa_dct_inverse_host(None, 2, 8, None) == E
    assert L.sa_dtw_batch(None, None, 2, 8, 8, None, None) == E
    assert L.sa_dtw_batch_host(None, None, 2, 8, 8, None) == E
    assert L.sa_dtw_path(None, 8, None, 8, None, None, None, None, None) == E
    assert L.sa_repr_values(None, 3, None, None, None) == E
    assert L.sa_parse_values(None, None, 3, None, None, None, None) == E
    assert L.sa_augment_spectrum(None, 0, 0, None, None, 1, 8, None, None, None) == E
    assert L.sa_host_copy(None, None, 16) == E
    assert L.sa_host_alloc(None, 16) == E
    assert b"null" in L.sa_last_error() or b"bad" in L.sa_last_error()
