"""Element-wise number text codec on the device (reference datafiles.py:63,133).

The reference writes every value as ``repr(float(v))`` (shortest round-trip
decimal) and reads every field with ``float(f)``.  These are the same two
operations as CUDA kernels (csrc/sa_text.cuh), bit-exact with CPython:

* ``repr_values(values)`` -- CUDA float64 tensor -> list of repr strings;
* ``parse_values(fields)`` -- strings -> (float64 array, ok mask), where
  ``ok[i]`` is False exactly where ``float(fields[i])`` raises ValueError.

The dataset-level codec (datafiles.py) uses the same device functions fused
into its line/field kernels; these entry points exist for direct use and
for parity testing.
"""

from __future__ import annotations

import numpy as np

from . import _native

SLOT = 32  # bytes per formatted value (the longest repr is 24)


def _stream(torch, dev):
    return ctypes_ptr(torch.cuda.current_stream(dev).cuda_stream)


def ctypes_ptr(x):
    import ctypes

    return ctypes.c_void_p(int(x))


def repr_values(values) -> list[str]:
    """[repr(float(v)) for v in values] for a 1-D CUDA float64 tensor."""
    import torch

    dev = _native.current_device()
    v = values.to(device=f"cuda:{dev}", dtype=torch.float64).contiguous().reshape(-1)
    n = v.numel()
    out = torch.empty((max(n, 1), SLOT), dtype=torch.uint8, device=v.device)
    lens = torch.empty(max(n, 1), dtype=torch.int32, device=v.device)
    _native.check(_native.lib().sa_repr_values(ctypes_ptr(v.data_ptr()), n, ctypes_ptr(out.data_ptr()),
                                              ctypes_ptr(lens.data_ptr()), _stream(torch, dev)))
    buf = out[:n].cpu().numpy()
    ln = lens[:n].cpu().numpy()
    return [bytes(buf[i, :ln[i]]).decode("ascii") for i in range(n)]


def parse_values(fields) -> tuple[np.ndarray, np.ndarray]:
    """(float(f) or 0.0, parsed-ok) for each string; bit-exact with float()."""
    import torch

    dev = _native.current_device()
    enc = [f.encode("utf-8", "surrogatepass") for f in fields]
    off = np.zeros(len(enc) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(e) for e in enc])
    blob = b"".join(enc)
    text = torch.frombuffer(bytearray(blob or b"\0"), dtype=torch.uint8).to(f"cuda:{dev}")
    scratch = torch.empty_like(text)
    d_off = torch.from_numpy(off).to(text.device)
    n = len(enc)
    out = torch.empty(max(n, 1), dtype=torch.float64, device=text.device)
    ok = torch.empty(max(n, 1), dtype=torch.int32, device=text.device)
    _native.check(_native.lib().sa_parse_values(ctypes_ptr(text.data_ptr()), ctypes_ptr(d_off.data_ptr()), n,
                                               ctypes_ptr(out.data_ptr()), ctypes_ptr(ok.data_ptr()),
                                               ctypes_ptr(scratch.data_ptr()), _stream(torch, dev)))
    return out[:n].cpu().numpy(), ok[:n].cpu().numpy().astype(bool)
