"""ctypes binding of the C ABI (include/seriesaug_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2601_03159_b200/csrc``) into ``paper_2601_03159_b200/_lib``.
There is deliberately no fallback: if the library or a CUDA device is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _abi
from .errors import (
    InvalidConfigError,
    InvalidInputError,
    UnsupportedPlatformError,
)

# SA_LIB_PATH: an alternative build of the same backend (A/B timing, tools/ab_timing.py)
LIB_PATH = os.environ.get("SA_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                         "libseriesaug_b200.so")

_lock = threading.Lock()
_lib = None
_inited: set[int] = set()

_i32, _i64, _u64, _f64p, _vp = (
    ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p
)
_stp = ctypes.POINTER(_abi.SaStage)


def lib() -> ctypes.CDLL:
    """Load (once) and return the backend library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise UnsupportedPlatformError(
                f"CUDA backend not built: {LIB_PATH} is missing "
                "(run __graft_entry__.build() or make -C paper_2601_03159_b200/csrc)"
            )
        L = ctypes.CDLL(LIB_PATH)
        L.sa_abi_version.restype = ctypes.c_int
        L.sa_last_error.restype = ctypes.c_char_p
        L.sa_launch_count.restype = _i64
        L.sa_init.argtypes = [_i32]
        L.sa_derive_key.argtypes = [_u64, _u64, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]
        pipe = [_stp, _i32, _f64p, _i32, _u64, _i64, _vp, _i64, _i64, _vp, _i64]
        L.sa_pipeline_launch.argtypes = pipe + [_vp, _vp]
        L.sa_pipeline_run.argtypes = pipe + [_vp]
        L.sa_pipeline_run_host.argtypes = pipe
        L.sa_fft_forward.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp]
        L.sa_fft_inverse.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
        L.sa_dct_forward.argtypes = [_vp, _i64, _i64, _vp, _vp]
        L.sa_dct_inverse.argtypes = [_vp, _i64, _i64, _vp, _vp]
        L.sa_dtw_batch.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp, _vp]
        L.sa_dtw_path.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
        L.sa_augment_spectrum.argtypes = [_stp, _u64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp]
        L.sa_fft_forward_host.argtypes = [_vp, _i64, _i64, _vp, _vp]
        L.sa_fft_inverse_host.argtypes = [_vp, _vp, _i64, _i64, _vp]
        L.sa_dct_forward_host.argtypes = [_vp, _i64, _i64, _vp]
        L.sa_dct_inverse_host.argtypes = [_vp, _i64, _i64, _vp]
        L.sa_dtw_batch_host.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp]
        L.sa_repr_values.argtypes = [_vp, _i64, _vp, _vp, _vp]
        L.sa_parse_values.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, _vp]
        _infop = ctypes.POINTER(_abi.SaDatasetInfo)
        L.sa_dataset_open.argtypes = [_vp, _i64, _i32, _i32, ctypes.POINTER(ctypes.c_void_p), _infop, _vp]
        L.sa_dataset_values.argtypes = [_vp, _vp, _infop]
        L.sa_dataset_labels.argtypes = [_vp, _vp]
        L.sa_dataset_headers.argtypes = [_vp, _vp]
        L.sa_dataset_close.argtypes = [_vp]
        L.sa_dataset_format_size.argtypes = [_vp, _i64, _i64, _i32, _vp, _i64, _vp, ctypes.POINTER(_i64), _vp]
        L.sa_dataset_format_write.argtypes = [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]
        L.sa_host_copy.argtypes = [_vp, _vp, _i64]
        L.sa_host_alloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), _i64]
        L.sa_host_free.argtypes = [_vp]
        L.sa_host_all_finite.argtypes = [_vp, _i64, _vp]
        for fn in ("sa_init", "sa_derive_key", "sa_pipeline_launch", "sa_pipeline_run",
                   "sa_pipeline_run_host", "sa_fft_forward", "sa_fft_inverse",
                   "sa_augment_spectrum", "sa_host_alloc", "sa_host_free", "sa_dct_forward",
                   "sa_dct_inverse", "sa_dtw_batch", "sa_dtw_path", "sa_repr_values", "sa_parse_values", "sa_dataset_open",
                   "sa_dataset_values", "sa_dataset_labels", "sa_dataset_headers", "sa_dataset_close",
                   "sa_dataset_format_size", "sa_dataset_format_write", "sa_fft_forward_host", "sa_fft_inverse_host",
                   "sa_dct_forward_host", "sa_dct_inverse_host", "sa_dtw_batch_host", "sa_host_copy",
                   "sa_host_all_finite"):
            getattr(L, fn).restype = ctypes.c_int
        if L.sa_abi_version() != _abi.SA_ABI_VERSION:
            raise UnsupportedPlatformError("backend library ABI version mismatch")
        _lib = L
        return _lib


def last_error() -> str:
    msg = lib().sa_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a C ABI status onto the reference's exception taxonomy."""
    if rc == _abi.SA_OK:
        return
    msg = last_error() or what
    if rc == _abi.SA_ERR_NONFINITE:
        raise InvalidInputError("batch contains non-finite values (NaN or Inf)")
    if rc == _abi.SA_ERR_INVALID_ARG:
        raise InvalidConfigError(msg)
    if rc == _abi.SA_ERR_NO_DEVICE:
        raise UnsupportedPlatformError(msg)
    raise RuntimeError(msg)


def ensure_device(device: int) -> None:
    if device in _inited:
        return
    check(lib().sa_init(device), "sa_init")
    _inited.add(device)


def current_device() -> int:
    import torch

    if not torch.cuda.is_available():
        raise UnsupportedPlatformError("no CUDA device: the B200 backend has no CPU fallback")
    dev = torch.cuda.current_device()
    ensure_device(dev)
    return dev


def derive_key(seed: int, j: int, i: int) -> tuple[int, int]:
    lo, hi = _u64(), _u64()
    check(lib().sa_derive_key(seed, j, i, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def launch_count() -> int:
    return int(lib().sa_launch_count())
