"""Dataset files in the reference's two layouts, parsed and formatted on the
GPU (reference: datafiles.py).

CSV-rows: one series per line, comma-separated decimals, every line the same
field count.  TS-style: '@'-prefixed header lines (kept verbatim), then one
series per line with a class label after the last ':'.  The format is
detected from the first non-blank line ('@' means TS) and can be forced.
Numbers are written as ``repr(float(v))`` (shortest round trip) and read with
``float()`` semantics -- both bit-exact on the device (csrc/sa_text.cuh).

The text itself is split, stripped, classified, checked and converted by the
kernels of csrc/sa_dataset.cuh through the C ABI (sa_dataset_*); the host
only moves bytes and turns the kernels' status into the reference's
exception messages.  ``parse_dataset_device`` / ``format_dataset_device``
keep the batch in HBM for device-resident flows (``augment_file``).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _abi, _native
from .core import Batch
from .errors import InvalidInputError

FORMATS = ("csv", "ts")
_FMT_CODE = {"csv": _abi.SA_FORMAT_CSV, "ts": _abi.SA_FORMAT_TS}


@dataclass(frozen=True)
class DatasetFile:
    """A parsed dataset (reference datafiles.py:24-56)."""

    batch: Batch
    format: str                            # "csv" | "ts"
    header_lines: tuple[str, ...] = ()     # ts only, kept verbatim
    labels: Optional[tuple[str, ...]] = None  # ts only, one per series

    def __post_init__(self) -> None:
        if self.format not in FORMATS:
            raise InvalidInputError(f"format must be one of {FORMATS}, got {self.format!r}")
        if self.labels is not None and len(self.labels) != self.batch.n:
            raise InvalidInputError(f"{len(self.labels)} labels for {self.batch.n} series")
        if self.format == "csv" and (self.header_lines or self.labels is not None):
            raise InvalidInputError("csv datasets carry no header lines or labels")

    def with_batch(self, batch: Batch) -> "DatasetFile":
        """Carry format and labels over to an augmented batch; a batch grown
        to a whole multiple of N (repeat) replicates each label consecutively
        (datafiles.py:43-56)."""
        labels = self.labels
        if labels is not None and batch.n != self.batch.n:
            if batch.n % self.batch.n != 0:
                raise InvalidInputError(f"cannot carry {len(labels)} labels onto {batch.n} series")
            r = batch.n // self.batch.n
            labels = tuple(lab for lab in labels for _ in range(r))
        return replace(self, batch=batch, labels=labels)


@dataclass(frozen=True)
class DeviceDataset:
    """A parsed dataset whose (n, L) float64 batch stays on the GPU."""

    values: object                         # torch.Tensor, cuda, float64
    format: str
    header_lines: tuple[str, ...] = ()
    labels: Optional[tuple[str, ...]] = None


def _vp(x) -> ctypes.c_void_p:
    return ctypes.c_void_p(int(x))


def _cur_stream(torch, dev):
    return _vp(torch.cuda.current_stream(dev).cuda_stream)


_staging: dict = {}
_staging_lock = threading.Lock()


def _staging_buffer(nbytes: int) -> np.ndarray:
    """A grow-only page-locked host buffer (one per process): file bytes are
    read into it and text is copied out of it at PCIe speed without a
    page-locked allocation per call.  Callers hold _staging_lock."""
    from .memory import pinned_empty

    buf = _staging.get("buf")
    if buf is None or buf.size < nbytes:
        cap = max(nbytes, 1 << 20)
        if buf is not None:
            cap = max(cap, 2 * buf.size)
        buf = pinned_empty((cap,), np.uint8)
        _staging["buf"] = buf
    return buf


def _to_device_bytes(data, dev):
    """Host bytes -> (cuda uint8 tensor, nbytes) through the pinned staging
    buffer (or straight from `data` when it already is that buffer)."""
    import torch

    mv = memoryview(data).cast("B")
    n = mv.nbytes
    d = torch.empty(max(n, 1), dtype=torch.uint8, device=f"cuda:{dev}")
    if n == 0:
        return d, 0
    with _staging_lock:
        host = _staging_buffer(n)
        src = np.frombuffer(mv, dtype=np.uint8)
        if not np.shares_memory(src, host):
            _copy(host[:n], src)
            src = host[:n]
        d.copy_(torch.from_numpy(src), non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    return d, n


def _copy(dst: np.ndarray, src: np.ndarray) -> None:
    """Host memcpy on the runtime's copy threads (sa_host_copy)."""
    _native.check(_native.lib().sa_host_copy(_vp(dst.ctypes.data), _vp(src.ctypes.data), src.nbytes),
                  "sa_host_copy")


def _to_numpy(t) -> np.ndarray:
    """A CUDA tensor -> a fresh numpy array: D2H into the pinned staging
    buffer, then a parallel host copy (a pageable D2H runs at a few GB/s)."""
    import torch

    n = t.numel() * t.element_size()
    out = np.empty(tuple(t.shape), dtype=np.dtype(str(t.dtype).replace("torch.", "")))
    if n == 0:
        return out
    with _staging_lock:
        host = _staging_buffer(n)
        torch.from_numpy(host[:n]).copy_(t.contiguous().view(torch.uint8).reshape(-1), non_blocking=True)
        torch.cuda.current_stream(t.device.index).synchronize()
        _copy(out.reshape(-1).view(np.uint8), host[:n])
    return out


def _to_cuda(a: np.ndarray, dev: int):
    """A host array -> a CUDA tensor through the pinned staging buffer."""
    import torch

    a = np.ascontiguousarray(a)
    d = torch.empty(a.shape, dtype=getattr(torch, a.dtype.name), device=f"cuda:{dev}")
    n = a.nbytes
    if n == 0:
        return d
    with _staging_lock:
        host = _staging_buffer(n)
        _copy(host[:n], a.reshape(-1).view(np.uint8))
        d.view(torch.uint8).reshape(-1).copy_(torch.from_numpy(host[:n]), non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
    return d


def _split_joined(buf: bytes, count: int) -> tuple[str, ...]:
    """'\\n'-terminated items -> tuple of str."""
    if count == 0:
        return ()
    items = buf.decode("utf-8", "surrogatepass").split("\n")
    return tuple(items[:count])


def _raise_status(info, host_bytes) -> None:
    st = info.status
    k = info.err_line
    if st == _abi.SA_DS_EMPTY:
        raise InvalidInputError("dataset file is empty")
    if st == _abi.SA_DS_HEADER_AFTER_DATA:
        raise InvalidInputError(f"line {k}: header after first data row")
    if st == _abi.SA_DS_MISSING_LABEL:
        raise InvalidInputError(f"line {k}: missing ':label' separator")
    if st == _abi.SA_DS_NOT_A_NUMBER:
        field = bytes(host_bytes[info.err_begin:info.err_end]).decode("utf-8", "surrogatepass")
        raise InvalidInputError(f"line {k}: not a number: {field.strip()!r}")
    if st == _abi.SA_DS_RAGGED:
        raise InvalidInputError(
            f"line {k}: {info.err_fields} fields, but line {info.err_ref_line} has {info.err_ref_fields}")
    if st == _abi.SA_DS_NO_DATA:
        raise InvalidInputError("dataset file has headers but no data rows")
    if st == _abi.SA_DS_NONFINITE:
        raise InvalidInputError("batch contains non-finite values (NaN or Inf)")
    if st == _abi.SA_DS_BAD_UTF8:
        raw = host_bytes.tobytes() if hasattr(host_bytes, "tobytes") else bytes(host_bytes)
        raw.decode("utf-8")  # raises the decoder's own UnicodeDecodeError
    raise RuntimeError(f"dataset parse: unexpected status {st}")


def _timed(events, fn):
    """Run fn(); if `events` is a list, bracket it with CUDA events on the
    current stream (bench.py times the dominant kernel this way)."""
    if events is None:
        return fn()
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn()
    b.record()
    events.append((a, b))
    return r


def _parse_device(d_text, nbytes: int, host_bytes, fmt, validate: bool, events=None) -> DeviceDataset:
    import torch

    if fmt is not None and fmt not in FORMATS:
        code = _abi.SA_FORMAT_AUTO
    else:
        code = _abi.SA_FORMAT_AUTO if fmt is None else _FMT_CODE[fmt]
    dev = d_text.device.index
    L = _native.lib()
    stream = _cur_stream(torch, dev)
    info = _abi.SaDatasetInfo()
    handle = ctypes.c_void_p()
    _native.check(L.sa_dataset_open(_vp(d_text.data_ptr()), nbytes, code, 1 if validate else 0,
                                    ctypes.byref(handle), ctypes.byref(info), stream), "sa_dataset_open")
    try:
        if fmt is not None and fmt not in FORMATS:
            if info.status in (_abi.SA_DS_EMPTY, _abi.SA_DS_BAD_UTF8):  # checked before the format (:71-79)
                _raise_status(info, host_bytes)
            raise InvalidInputError(f"format must be one of {FORMATS}, got {fmt!r}")
        values = None
        if info.status == _abi.SA_DS_OK:
            values = torch.empty((info.n_series, info.length), dtype=torch.float64, device=d_text.device)
            _native.check(_timed(events, lambda: L.sa_dataset_values(handle, _vp(values.data_ptr()),
                                                                     ctypes.byref(info))), "sa_dataset_values")
        if info.status != _abi.SA_DS_OK:
            _raise_status(info, host_bytes)
        fmt_name = FORMATS[info.format]
        hb, lb = info.header_bytes, info.label_bytes
        d_hdr = torch.empty(max(hb, 1), dtype=torch.uint8, device=d_text.device)
        d_lab = torch.empty(max(lb, 1), dtype=torch.uint8, device=d_text.device)
        _native.check(L.sa_dataset_headers(handle, _vp(d_hdr.data_ptr())), "sa_dataset_headers")
        _native.check(L.sa_dataset_labels(handle, _vp(d_lab.data_ptr())), "sa_dataset_labels")
        headers = ()
        if hb:
            headers = tuple(d_hdr[:hb].cpu().numpy().tobytes().decode("utf-8", "surrogatepass").split("\n")[:-1])
        labels = None
        if fmt_name == "ts":
            labels = _split_joined(d_lab[:lb].cpu().numpy().tobytes(), info.n_series)
        return DeviceDataset(values=values, format=fmt_name, header_lines=headers, labels=labels)
    finally:
        L.sa_dataset_close(handle)


def parse_dataset_device(data, fmt: Optional[str] = None, *, validate_utf8: bool = True) -> DeviceDataset:
    """Parse UTF-8 dataset bytes on the current GPU; the batch stays there."""
    dev = _native.current_device()
    d_text, n = _to_device_bytes(data, dev)
    return _parse_device(d_text, n, memoryview(data).cast("B"), fmt, validate_utf8)


def parse_dataset(text: str, fmt: Optional[str] = None) -> DatasetFile:
    """Reference datafiles.py:70-116 -- same result, same first error."""
    data = text.encode("utf-8", "surrogatepass")
    dd = parse_dataset_device(data, fmt, validate_utf8=False)
    return _to_host(dd)


def _to_host(dd: DeviceDataset) -> DatasetFile:
    values = _to_numpy(dd.values)
    return DatasetFile(batch=Batch._from_device_checked(values), format=dd.format,
                       header_lines=dd.header_lines, labels=dd.labels)


def read_dataset(path, fmt: Optional[str] = None) -> DatasetFile:
    """Reference datafiles.py:119-124: errors are prefixed with the path."""
    try:
        dd = _read_device(path, fmt)
    except InvalidInputError as exc:
        raise InvalidInputError(f"{path}: {exc}") from None
    return _to_host(dd)


def _read_device(path, fmt) -> DeviceDataset:
    """File -> pinned staging (one read) -> HBM -> device parse."""
    import torch

    with open(path, "rb") as fh:  # I/O errors first, as the reference's open()
        dev = _native.current_device()
        size = fh.seek(0, 2)
        fh.seek(0)
        with _staging_lock:
            host = _staging_buffer(max(size, 1))
            got = fh.readinto(memoryview(host)[:size]) if size else 0
            d = torch.empty(max(got, 1), dtype=torch.uint8, device=f"cuda:{dev}")
            if got:
                d.copy_(torch.from_numpy(host[:got]), non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
            # the host copy is needed only to word an error; keep the bytes
            # only if the parse fails
    try:
        return _parse_device(d, got, _LazyHostBytes(d, got), fmt, True)
    finally:
        del d


class _LazyHostBytes:
    """Host view of device text, fetched only when an error message needs it."""

    def __init__(self, d, n):
        self.d, self.n = d, n

    def __getitem__(self, sl):
        return self.d[: self.n].cpu().numpy().tobytes()[sl]

    def tobytes(self):
        return self.d[: self.n].cpu().numpy().tobytes()


# ------------------------------------------------------------------ format
def _label_blob(labels, n: int):
    """(label bytes without separators, int64 offsets[n+1]) or (None, None)."""
    if labels is None:
        return None, None
    joined = "\n".join(labels)
    blob = joined.encode("utf-8", "surrogatepass")
    arr = np.frombuffer(blob, dtype=np.uint8)
    nl = np.flatnonzero(arr == 10)
    if len(nl) == n - 1:
        ends = np.append(nl, len(arr)).astype(np.int64)
        starts = np.concatenate([[0], nl + 1]).astype(np.int64)
        lens = ends - starts
        data = arr[arr != 10] if len(nl) else arr
    else:  # labels that themselves hold '\n'
        enc = [lab.encode("utf-8", "surrogatepass") for lab in labels]
        lens = np.array([len(e) for e in enc], dtype=np.int64)
        data = np.frombuffer(b"".join(enc), dtype=np.uint8)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return data, off


def format_dataset_device(values, fmt: str = "csv", header_lines=(), labels=None) -> bytes:
    """The file bytes of format_dataset for an (n, L) CUDA float64 tensor."""
    out = format_dataset_to_device(values, fmt, header_lines, labels)
    return _fetch(out, lambda mv: bytes(mv))


def _fetch(d_out, consume):
    """D2H of a device byte buffer through the pinned staging buffer; the
    bytes are handed to `consume(memoryview)` while the staging is held."""
    import torch

    n = int(d_out.numel())
    with _staging_lock:
        host = _staging_buffer(max(n, 1))
        if n:
            torch.from_numpy(host[:n]).copy_(d_out, non_blocking=True)
            torch.cuda.current_stream(d_out.device.index).synchronize()
        return consume(memoryview(host)[:n])


def format_dataset_to_device(values, fmt: str = "csv", header_lines=(), labels=None, events=None):
    """format_dataset's bytes as a CUDA uint8 tensor (no host copy)."""
    import torch

    if fmt not in FORMATS:
        raise InvalidInputError(f"format must be one of {FORMATS}, got {fmt!r}")
    dev = values.device.index
    values = values.contiguous()
    n, length = int(values.shape[0]), int(values.shape[1])
    L = _native.lib()
    stream = _cur_stream(torch, dev)
    head = "".join(h + "\n" for h in header_lines).encode("utf-8", "surrogatepass") if fmt == "ts" else b""
    d_lab = d_off = None
    if fmt == "ts" and labels is not None:
        data, off = _label_blob(labels, n)
        d_lab = torch.from_numpy(np.ascontiguousarray(data) if len(data) else np.zeros(1, np.uint8)).to(values.device)
        d_off = torch.from_numpy(off).to(values.device)
    row_off = torch.empty(n, dtype=torch.int64, device=values.device)
    total = ctypes.c_int64()
    _native.check(L.sa_dataset_format_size(_vp(values.data_ptr()), n, length, _FMT_CODE[fmt],
                                           _vp(d_off.data_ptr()) if d_off is not None else None, len(head),
                                           _vp(row_off.data_ptr()), ctypes.byref(total), stream),
                  "sa_dataset_format_size")
    out = torch.empty(total.value, dtype=torch.uint8, device=values.device)
    if head:
        out[:len(head)].copy_(torch.frombuffer(bytearray(head), dtype=torch.uint8))
    _native.check(_timed(events, lambda: L.sa_dataset_format_write(
        _vp(values.data_ptr()), n, length, _FMT_CODE[fmt], _vp(d_lab.data_ptr()) if d_lab is not None else None,
        _vp(d_off.data_ptr()) if d_off is not None else None, _vp(row_off.data_ptr()), _vp(out.data_ptr()),
        stream)), "sa_dataset_format_write")
    return out


def format_dataset(ds: DatasetFile) -> str:
    """Reference datafiles.py:127-138."""
    import torch

    dev = _native.current_device()
    values = _to_cuda(ds.batch.values, dev)
    labels = ds.labels
    out = format_dataset_to_device(values, ds.format, ds.header_lines, labels)
    return _fetch(out, lambda mv: str(mv, "utf-8", "surrogatepass"))


def write_dataset(path, ds: DatasetFile) -> None:
    """Reference datafiles.py:141-143."""
    import torch

    dev = _native.current_device()
    values = _to_cuda(ds.batch.values, dev)
    _write_device(path, format_dataset_to_device(values, ds.format, ds.header_lines, ds.labels), ds)


def _write_device(path, d_out, ds_like) -> None:
    try:  # the reference's text-mode write fails on unencodable labels/headers
        for s in tuple(ds_like.header_lines) + tuple(ds_like.labels or ()):
            s.encode("utf-8")
    except UnicodeEncodeError:
        text = _fetch(d_out, lambda mv: str(mv, "utf-8", "surrogatepass"))
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
        return

    def write(mv):
        with open(path, "wb") as fh:
            fh.write(mv)

    _fetch(d_out, write)


def augment_file(src, dst, pipeline, fmt: Optional[str] = None) -> DeviceDataset:
    """The reference's `seriesaug augment` data path (cli.py:48-54) with the
    batch resident in HBM: read -> parse -> pipeline -> format -> write, one
    H2D of the input text and one D2H of the output text."""
    try:
        dd = _read_device(src, fmt)
    except InvalidInputError as exc:
        raise InvalidInputError(f"{src}: {exc}") from None
    out = pipeline.run_device(dd.values)
    labels = dd.labels
    if labels is not None and out.shape[0] != dd.values.shape[0]:
        r = out.shape[0] // dd.values.shape[0]
        labels = tuple(lab for lab in labels for _ in range(r))
    res = DeviceDataset(values=out, format=dd.format, header_lines=dd.header_lines, labels=labels)
    _write_device(dst, format_dataset_to_device(out, dd.format, dd.header_lines, labels), res)
    return res
