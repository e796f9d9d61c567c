"""Dynamic time warping on the device (reference: dtw.py).

Same API: ``dtw_distance`` (distance + one optimal path, ties broken in the
reference's order), ``dtw_similarity`` and ``mean_similarity`` (row-wise
over two batches).  The accumulated-cost matrix is computed by the warp
wavefront in csrc/sa_dtw.cuh (sa_dtw_batch / sa_dtw_path); every cell is one
addition of its cost to a min of final neighbours, so distances equal the
reference bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import Batch
from .errors import InvalidInputError


def _as_series(name: str, values) -> np.ndarray:
    x = np.ascontiguousarray(values, dtype=np.float64)
    if x.ndim != 1 or x.size == 0:
        raise InvalidInputError(f"{name} must be a non-empty 1-D sequence")
    if not np.all(np.isfinite(x)):
        raise InvalidInputError(f"{name} must contain only finite values")
    return x


@dataclass(frozen=True)
class DtwResult:
    distance: float
    path: list  # [(i, j), ...] from (0, 0) to (L1-1, L2-1)
    similarity: float

    @property
    def path_length(self) -> int:
        return len(self.path)


def similarity_from_distance(distance: float, len_a: int, len_b: int) -> float:
    """dtw.py:88-89."""
    return 1.0 / (1.0 + distance / max(len_a, len_b))


def dtw_distance(a, b) -> DtwResult:
    """Full DTW between two series with one optimal path (dtw.py:40-85)."""
    import torch

    from . import _native

    a = _as_series("a", a)
    b = _as_series("b", b)
    n, m = a.size, b.size
    dev = _native.current_device()
    ta = torch.from_numpy(a).to(f"cuda:{dev}")
    tb = torch.from_numpy(b).to(f"cuda:{dev}")
    acc = torch.empty(n * m, dtype=torch.float64, device=ta.device)
    path = torch.empty(2 * (n + m), dtype=torch.int32, device=ta.device)
    plen = torch.empty(1, dtype=torch.int32, device=ta.device)
    dist = torch.empty(1, dtype=torch.float64, device=ta.device)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(_native.lib().sa_dtw_path(ta.data_ptr(), n, tb.data_ptr(), m, acc.data_ptr(), path.data_ptr(),
                                            plen.data_ptr(), dist.data_ptr(), st))
    k = int(plen.item())
    pairs = path[: 2 * k].view(k, 2).cpu().tolist()
    distance = float(dist.item())
    return DtwResult(distance, [tuple(p) for p in pairs], similarity_from_distance(distance, n, m))


def dtw_similarity(a, b) -> float:
    """Length-normalized similarity in (0, 1]; 1 means identical (dtw.py:92-94)."""
    return dtw_distance(a, b).similarity


def dtw_distances(a: Batch, b: Batch) -> np.ndarray:
    """Row-wise DTW distances of two batches (one warp per pair), host
    arrays through the staging runtime (sa_dtw_batch_host)."""
    from . import _native

    if a.n != b.n:
        raise InvalidInputError(
            f"batches must have the same number of series, got {a.n} and {b.n}"
        )
    _native.current_device()
    va = np.ascontiguousarray(a.values)
    vb = np.ascontiguousarray(b.values)
    dist = np.empty(a.n, dtype=np.float64)
    _native.check(_native.lib().sa_dtw_batch_host(va.ctypes.data, vb.ctypes.data, a.n, a.length, b.length,
                                                  dist.ctypes.data), "sa_dtw_batch_host")
    return dist


def mean_similarity(a: Batch, b: Batch) -> float:
    """Mean row-wise DTW similarity between two batches of equal N (dtw.py:97-106)."""
    d = dtw_distances(a, b)
    total = 0.0
    for i in range(a.n):
        total += similarity_from_distance(float(d[i]), a.length, b.length)
    return total / a.n
