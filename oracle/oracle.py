"""ctypes wrapper of the C oracle -- TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs, as the checker / baseline -- never by the product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libsaoracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        vp, i64, u64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32
        L.sao_pipeline_run.argtypes = [vp, i32, vp, u64, i64, vp, i64, i64, vp, i64, i32]
        L.sao_augment_spectrum.argtypes = [vp, u64, i64, vp, vp, i64, i64, vp, vp]
        L.sao_fft_forward.argtypes = [vp, i64, i64, vp, vp]
        L.sao_fft_inverse.argtypes = [vp, vp, i64, i64, vp]
        L.sao_dct.argtypes = [vp, i64, i64, vp, i32]
        L.sao_dtw.argtypes = [vp, i64, vp, i64, vp, vp]
        L.sao_dtw.restype = ctypes.c_double
        L.sao_derive_key.argtypes = [u64, u64, u64, vp]
        L.sao_raw.argtypes = [u64, u64, u64, i64, vp]
        L.sao_normals.argtypes = [u64, u64, u64, i64, ctypes.c_double, ctypes.c_double, vp]
        L.sao_doubles.argtypes = [u64, u64, u64, i64, vp]
        L.sao_normals_words.argtypes = [vp, i64, i64, i64, vp, vp]
        L.sao_script.argtypes = [u64, u64, u64, i64, vp, vp, vp]
        L.sao_permutation.argtypes = [u64, u64, u64, i64, vp]
        L.sao_choice.argtypes = [u64, u64, u64, i64, i64, vp]
        L.sao_pairwise_sum.argtypes = [vp, i64]
        L.sao_pairwise_sum.restype = ctypes.c_double
        L.sao_std.argtypes = [vp, i64]
        L.sao_std.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}")
        self.code = code


def run_stages(stage_arr, n_stages: int, aux: np.ndarray, seed: int, values: np.ndarray,
               len_out: int, rows_out: int, series_offset: int = 0, threads: int = 1) -> np.ndarray:
    """Run a lowered stage table (pipeline.lower_stages) over a host batch."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    n, L = values.shape
    out = np.empty((rows_out, len_out), dtype=np.float64)
    aux = np.ascontiguousarray(aux, dtype=np.float64)
    rc = lib().sao_pipeline_run(ctypes.addressof(stage_arr), n_stages, _p(aux) if aux.size else None,
                                seed, series_offset, _p(values), n, L, _p(out), len_out, threads)
    if rc:
        raise OracleError(rc)
    return out


def run_pipeline(pipe, values: np.ndarray, threads: int = 1, series_offset: int = 0) -> np.ndarray:
    """Oracle result of product Pipeline `pipe` on `values` (same lowering)."""
    from paper_2601_03159_b200.pipeline import lower_stages

    arr, aux = lower_stages(pipe.stages, 0)
    L_out = pipe.projected_length(values.shape[1])
    rows = values.shape[0] * pipe.row_factor()
    return run_stages(arr, len(pipe.stages), aux, pipe.master_seed, values, L_out, rows,
                      series_offset=series_offset, threads=threads)


def fft_forward(values: np.ndarray):
    values = np.ascontiguousarray(values, dtype=np.float64)
    n, L = values.shape
    re = np.empty((n, L // 2 + 1))
    im = np.empty_like(re)
    lib().sao_fft_forward(_p(values), n, L, _p(re), _p(im))
    return re, im


def fft_inverse(re: np.ndarray, im: np.ndarray, L: int) -> np.ndarray:
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    out = np.empty((re.shape[0], L))
    lib().sao_fft_inverse(_p(re), _p(im), re.shape[0], L, _p(out))
    return out


def augment_spectrum(stage, seed: int, re: np.ndarray, im: np.ndarray, L: int):
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    ro, io = np.empty_like(re), np.empty_like(im)
    lib().sao_augment_spectrum(ctypes.addressof(stage), seed, 0, _p(re), _p(im), re.shape[0], L,
                               _p(ro), _p(io))
    return ro, io


def derive_key(seed, j, i):
    out = np.zeros(2, dtype=np.uint64)
    lib().sao_derive_key(seed, j, i, _p(out))
    return int(out[0]), int(out[1])


def raw(seed, j, i, n):
    out = np.empty(n, dtype=np.uint64)
    lib().sao_raw(seed, j, i, n, _p(out))
    return out


def normals(seed, j, i, n, loc=0.0, scale=1.0):
    out = np.empty(n)
    lib().sao_normals(seed, j, i, n, loc, scale, _p(out))
    return out


def normals_words(words: np.ndarray, n: int, skip: int = 0):
    """numpy's ziggurat on a crafted word stream: (n normals, position after)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    out = np.empty(n)
    pos = ctypes.c_int64(0)
    lib().sao_normals_words(_p(w), w.size, skip, n, _p(out), ctypes.byref(pos))
    return out, pos.value


def doubles(seed, j, i, n):
    out = np.empty(n)
    lib().sao_doubles(seed, j, i, n, _p(out))
    return out


def script(seed, j, i, ops, args):
    ops = np.ascontiguousarray(ops, dtype=np.int32)
    args = np.ascontiguousarray(args, dtype=np.int64)
    out = np.empty(len(ops))
    lib().sao_script(seed, j, i, len(ops), _p(ops), _p(args), _p(out))
    return out


def permutation(seed, j, i, n):
    out = np.empty(n, dtype=np.int64)
    lib().sao_permutation(seed, j, i, n, _p(out))
    return out


def choice(seed, j, i, pop, k):
    out = np.empty(max(k, 1), dtype=np.int64)
    lib().sao_choice(seed, j, i, pop, k, _p(out))
    return out[:k]


def pairwise_sum(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().sao_pairwise_sum(_p(a), a.size)


def std(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().sao_std(_p(a), a.size)


def dct(values: np.ndarray, inverse: bool = False) -> np.ndarray:
    values = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty_like(values)
    lib().sao_dct(_p(values), values.shape[0], values.shape[1], _p(out), int(inverse))
    return out


def dtw(a, b):
    """(distance, path) of dtw.py:40-85."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    path = np.empty(2 * (a.size + b.size), dtype=np.int32)
    plen = np.zeros(1, dtype=np.int32)
    d = lib().sao_dtw(_p(a), a.size, _p(b), b.size, _p(path), _p(plen))
    k = int(plen[0])
    return d, [tuple(int(v) for v in path[2 * q:2 * q + 2]) for q in range(k)]
