"""Host orchestration between the reference-shaped API and the C ABI.

Lowers augmenters to ``sa_stage`` descriptors (pipeline.lower_stages) and calls
the fused kernel either on host buffers (sa_pipeline_run_host: chunked H2D ->
kernel -> D2H, overlapped on two streams) or on device tensors
(sa_pipeline_run on torch's current stream).  torch is used only for device
memory and streams.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _abi, _native
from .errors import InvalidInputError
from .pipeline import lower_stages


def _row_factor(stages, repeat_rows: bool) -> int:
    for s in stages:
        if s.kind == "repeat" and s.expands():
            return s.r if repeat_rows else 1
    return 1


_LOWERED: dict = {}


def _lower(stages, first_index, repeat_rows):
    """Stage table + aux taps of a stage tuple, cached per (stages, first
    index, repeat mode): augmenters are frozen dataclasses, so a pipeline
    called repeatedly (a training loop, the bench protocol) lowers once.
    The cached ctypes table is only read by the library."""
    try:
        key = (tuple(stages), int(first_index), bool(repeat_rows))
        hit = _LOWERED.get(key)
    except TypeError:  # an unhashable user-defined stage: lower every call
        return _lower_uncached(stages, first_index, repeat_rows)
    if hit is None:
        if len(_LOWERED) >= 256:
            _LOWERED.clear()
        hit = _LOWERED[key] = _lower_uncached(stages, first_index, repeat_rows)
    return hit


def _lower_uncached(stages, first_index, repeat_rows):
    arr, aux = lower_stages(stages, first_index)
    if not repeat_rows:  # Repeat's per-series form is the identity (basic.py:396-397)
        for j in range(len(stages)):
            if arr[j].op == _abi.SA_OP_REPEAT:
                arr[j].probability = 0.0
    return arr, aux


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def devices_for(parallel: bool) -> list[int]:
    """The GPUs a host-buffer call uses: the current one, or -- for the
    reference's ``parallel=True`` -- every visible one (SA_DEVICES, a comma
    list, overrides; repeats are allowed and only exercise the sharding)."""
    env = os.environ.get("SA_DEVICES")
    if env:
        return [int(d) for d in env.split(",") if d.strip()]
    dev = _native.current_device()
    if not parallel:
        return [dev]
    import torch

    return list(range(torch.cuda.device_count())) or [dev]


def run_host(stages, values: np.ndarray, seed: int, first_index: int = 0, series_offset: int = 0,
             len_out: int | None = None, check_finite: bool = True, repeat_rows: bool = True,
             out: np.ndarray | None = None, devices: list[int] | None = None) -> np.ndarray:
    """Run `stages` over a host (n, L) float64 batch; returns a new array.
    With several `devices` the rows are split into contiguous ranges, one
    host thread per range, each passing its global first row as the series
    offset (sharding.py) -- bitwise the single-device result."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    n, L = values.shape
    _native.current_device()
    arr, aux = _lower(stages, first_index, repeat_rows)
    r = _row_factor(stages, repeat_rows)
    rows = n * r
    L_out = L if len_out is None else int(len_out)
    if out is None:
        from .memory import output_array

        out = output_array((rows, L_out))
    elif out.shape != (rows, L_out) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float64 array of shape {(rows, L_out)}")
    devices = devices or [_native.current_device()]
    aux_p = aux.ctypes.data_as(ctypes.c_void_p)

    def shard(k: int) -> int:
        from .sharding import shard_range

        lo, hi = shard_range(n, k, len(devices))
        if hi == lo:
            return _abi.SA_OK
        if len(devices) > 1:
            import torch

            torch.cuda.set_device(devices[k])
            _native.ensure_device(devices[k])
        return _native.lib().sa_pipeline_run_host(
            arr, len(stages), aux_p, aux.size, int(seed), int(series_offset) + lo,
            _ptr(values) + 8 * lo * L, hi - lo, L, _ptr(out) + 8 * lo * r * L_out, L_out,
        )

    if len(devices) == 1:
        rcs = [shard(0)]
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(len(devices)) as ex:
            rcs = list(ex.map(shard, range(len(devices))))
    for rc in rcs:
        if rc == _abi.SA_ERR_NONFINITE and not check_finite:
            continue
        _native.check(rc, "sa_pipeline_run_host")
    return out


def run_device(stages, values, seed: int, series_offset: int = 0, len_out: int | None = None,
               first_index: int = 0, out=None):
    """Run `stages` over a CUDA float64 tensor (n, L); returns the output tensor."""
    import torch

    if not (values.is_cuda and values.dtype == torch.float64 and values.dim() == 2):
        raise TypeError("run_device expects a 2-D float64 CUDA tensor")
    values = values.contiguous()
    n, L = values.shape
    with torch.cuda.device(values.device):
        _native.ensure_device(values.device.index)
        arr, aux = _lower(stages, first_index, True)
        rows = n * _row_factor(stages, True)
        L_out = L if len_out is None else int(len_out)
        if out is None:
            out = torch.empty((rows, L_out), dtype=torch.float64, device=values.device)
        stream = torch.cuda.current_stream(values.device).cuda_stream
        rc = _native.lib().sa_pipeline_run(
            arr, len(stages), aux.ctypes.data_as(ctypes.c_void_p), aux.size, int(seed),
            int(series_offset), values.data_ptr(), n, L, out.data_ptr(), L_out, stream,
        )
        _native.check(rc, "sa_pipeline_run")
    return out


def launch_device(stages, values, out, flags, seed: int, series_offset: int = 0, first_index: int = 0,
                  stream=None, lowered=None):
    """Asynchronous launch (no sync, no status read): flags is a 1-element
    int32 CUDA tensor that receives SA_FLAG_* bits.  Used by bench.py."""
    import torch

    arr, aux = lowered if lowered is not None else _lower(stages, first_index, True)
    n, L = values.shape
    st = stream if stream is not None else torch.cuda.current_stream(values.device).cuda_stream
    rc = _native.lib().sa_pipeline_launch(
        arr, len(stages), aux.ctypes.data_as(ctypes.c_void_p), aux.size, int(seed), int(series_offset),
        values.data_ptr(), n, L, out.data_ptr(), out.shape[1], flags.data_ptr(), st,
    )
    _native.check(rc, "sa_pipeline_launch")


class GraphedRun:
    """A fused-chain launch captured in a CUDA graph (launch-bound small
    batches: one graph launch instead of a host-planned kernel launch per
    step).  ``values`` is the captured input buffer -- refill it in place
    between replays; ``out`` receives every replay's result.  ``check()``
    reads the device flags (one sync) and raises like ``run_device``."""

    def __init__(self, graph, values, out, flags):
        self.graph, self.values, self.out, self.flags = graph, values, out, flags

    def replay(self):
        self.graph.replay()
        return self.out

    def check(self):
        f = int(self.flags.item())
        if f & _abi.SA_FLAG_NONFINITE:
            raise InvalidInputError("batch contains non-finite values (NaN or Inf)")
        if f & _abi.SA_FLAG_WARP_MONOTONE:
            raise RuntimeError("warp map failed to stay strictly increasing")
        return self.out


def capture_device(stages, values, seed: int, series_offset: int = 0, len_out: int | None = None,
                   first_index: int = 0) -> GraphedRun:
    """Capture one fused-chain launch over the CUDA tensor ``values`` in a
    CUDA graph.  The first launch runs eagerly (device tables, plan and
    stream-ordered scratch pool are set up outside the capture) and is
    checked; the captured graph is the same sa_pipeline_launch."""
    import torch

    if not (values.is_cuda and values.dtype == torch.float64 and values.dim() == 2 and values.is_contiguous()):
        raise TypeError("capture_device expects a contiguous 2-D float64 CUDA tensor")
    dev = values.device
    n, L = values.shape
    with torch.cuda.device(dev):
        _native.ensure_device(dev.index)
        low = _lower(stages, first_index, True)
        out = torch.empty((n * _row_factor(stages, True), L if len_out is None else int(len_out)),
                          dtype=torch.float64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            launch_device(stages, values, out, flags, seed, series_offset, first_index, side.cuda_stream, low)
        torch.cuda.current_stream(dev).wait_stream(side)
        run = GraphedRun(None, values, out, flags)
        run.check()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            flags.zero_()
            launch_device(stages, values, out, flags, seed, series_offset, first_index,
                          torch.cuda.current_stream(dev).cuda_stream, low)
        run.graph = graph
    return run


def fft_forward_host(values: np.ndarray):
    """rfft of each row: host arrays through sa_fft_forward_host (staged)."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    n, L = x.shape
    _native.current_device()
    bins = L // 2 + 1
    from .memory import output_array

    re = output_array((n, bins))
    im = output_array((n, bins))
    _native.check(_native.lib().sa_fft_forward_host(_ptr(x), n, L, _ptr(re), _ptr(im)), "sa_fft_forward_host")
    return re, im


def fft_inverse_host(re: np.ndarray, im: np.ndarray, L: int) -> np.ndarray:
    """irfft(n=L) of each half spectrum (sa_fft_inverse_host)."""
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    _native.current_device()
    n = re.shape[0]
    from .memory import output_array

    out = output_array((n, L))
    _native.check(_native.lib().sa_fft_inverse_host(_ptr(re), _ptr(im), n, L, _ptr(out)), "sa_fft_inverse_host")
    return out


def augment_spectrum_host(stage, seed: int, re: np.ndarray, im: np.ndarray, L: int):
    import torch

    dev = _native.current_device()
    tre = torch.from_numpy(np.ascontiguousarray(re)).to(f"cuda:{dev}")
    tim = torch.from_numpy(np.ascontiguousarray(im)).to(f"cuda:{dev}")
    n = tre.shape[0]
    ore, oim = torch.empty_like(tre), torch.empty_like(tim)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(_native.lib().sa_augment_spectrum(
        ctypes.byref(stage), int(seed), 0, tre.data_ptr(), tim.data_ptr(), n, L,
        ore.data_ptr(), oim.data_ptr(), st,
    ))
    return ore.cpu().numpy(), oim.cpu().numpy()


def dct_host(values: np.ndarray, inverse: bool) -> np.ndarray:
    """Orthonormal DCT-II (inverse: DCT-III) of each row (sa_dct_*_host)."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    n, L = x.shape
    _native.current_device()
    from .memory import output_array

    out = output_array((n, L))
    fn = _native.lib().sa_dct_inverse_host if inverse else _native.lib().sa_dct_forward_host
    _native.check(fn(_ptr(x), n, L, _ptr(out)), "sa_dct_host")
    return out
