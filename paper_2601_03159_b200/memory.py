"""Page-locked host batches for the host-buffer path.

``Pipeline.run`` / ``augment_batch`` accept any C-contiguous float64 array;
with ordinary (pageable) numpy memory the host-to-device copies are staged
by the driver and run at host-memory speed (measured ~6 GB/s on the GPU
boxes).  Arrays from ``pinned_empty`` are page-locked (sa_host_alloc), so the
chunked three-stream pipeline streams them at PCIe speed (~93 GB/s
H2D + D2H concurrently on B200).
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _native


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (freed with the array)."""
    _native.current_device()
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    ptr = ctypes.c_void_p()
    _native.check(_native.lib().sa_host_alloc(ctypes.byref(ptr), max(nbytes, 1)), "sa_host_alloc")
    buf = (ctypes.c_char * max(nbytes, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)
    weakref.finalize(buf, _native.lib().sa_host_free, ptr.value)
    return arr


def pinned_copy(values: np.ndarray) -> np.ndarray:
    """Page-locked copy of `values` (float64, C-contiguous)."""
    out = pinned_empty(values.shape)
    out[...] = values
    return out
