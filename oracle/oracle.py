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


class OStage(ctypes.Structure):
    """struct sa_stage (include/seriesaug_b200.h), declared here so the oracle
    lowers configs without the product package."""

    _fields_ = [("op", ctypes.c_int32), ("index", ctypes.c_int32), ("probability", ctypes.c_double),
                ("f", ctypes.c_double * 6), ("i", ctypes.c_int64 * 6),
                ("aux_off", ctypes.c_int32), ("aux_len", ctypes.c_int32)]


# kind -> (op code, int params, float params); the header's SA_OP_* codes
_OPS = {
    "jitter": (1, [], ["sigma"]), "scale": (2, [], ["sigma_factor"]), "rotate": (3, [], []),
    "permute_segments": (4, ["n_segments"], []), "crop": (5, ["size"], []), "reverse": (6, [], []),
    "resize": (7, ["target_len"], []), "quantize": (8, ["n_levels"], []),
    "drift": (9, ["n_points"], ["max_drift"]), "repeat": (14, ["r"], []),
    "amplitude_phase_perturb": (15, [], ["sigma_amp", "sigma_phase"]), "frequency_mask": (16, ["width"], []),
    "time_warp": (17, ["n_knots"], ["intensity"]), "time_warp_window": (18, ["window_size", "n_knots"], ["intensity"]),
    "dropout": (19, [], ["rate", "fill"]), "pool": (20, ["size", "reducer"], []), "convolve": (21, [], []),
    "speed_warp": (22, ["n_speed_change", "interpolation"], ["max_speed_ratio"]),
    "random_sinusoid": (23, ["min_bin"], ["amplitude"]),
}
_NOISE = {"uniform": (10, "half_width"), "gaussian": (11, "sigma"), "spike": (12, "magnitude"),
          "slope_trend": (13, "max_offset")}
_ENUMS = {"reducer": ("mean", "max", "min"), "interpolation": ("linear", "cubic")}
_DEFAULTS = {"dropout": {"fill": 0.0}, "pool": {"reducer": "mean"}, "convolve": {"window": "hann", "size": 7},
             "speed_warp": {"n_speed_change": 3, "max_speed_ratio": 3.0, "interpolation": "cubic"},
             "random_sinusoid": {"min_bin": 1}, "time_warp": {"n_knots": 4, "intensity": 0.5},
             "drift": {"n_points": 6}, "time_warp_window": {"n_knots": 4, "intensity": 0.5}}


def lower_config(config: dict, first_index: int = 0):
    """A reference JSON pipeline config -> (stage table, aux table)."""
    stages = config["stages"]
    arr = (OStage * max(1, len(stages)))()
    aux: list = []
    for j, rec in enumerate(stages):
        kind, p = rec["kind"], dict(_DEFAULTS.get(rec["kind"], {}), **rec.get("params", {}))
        st = arr[j]
        st.index, st.probability = first_index + j, float(rec.get("probability", 1.0))
        if kind == "inject_noise":
            nz = p["noise"]
            st.op, name = _NOISE[nz["kind"]]
            st.f[0] = nz[name]
            st.i[0] = nz.get("count", 0)
            continue
        st.op, ints, flts = _OPS[kind]
        for k, name in enumerate(ints):
            st.i[k] = _ENUMS[name].index(p[name]) if name in _ENUMS else int(p[name])
        for k, name in enumerate(flts):
            st.f[k] = float(p[name])
        if kind == "convolve":
            from scipy.signal import get_window

            w = get_window("boxcar" if p["window"] == "flat" else p["window"], p["size"], fftbins=False)
            taps = w / w.sum()
            st.aux_off, st.aux_len = len(aux), len(taps)
            aux.extend(float(v) for v in taps)
    return arr, np.ascontiguousarray(aux, dtype=np.float64)


def geometry(config: dict, L: int) -> tuple[int, int]:
    """(rows out per row in, final length): Repeat / Crop / Resize at p = 1."""
    r, out = 1, L
    for rec in config["stages"]:
        if float(rec.get("probability", 1.0)) != 1.0:
            continue
        p = rec.get("params", {})
        if rec["kind"] == "crop":
            out = int(p["size"])
        elif rec["kind"] == "resize":
            out = int(p["target_len"])
        elif rec["kind"] == "repeat":
            r = int(p["r"])
    return r, out


def run_config(config: dict, values: np.ndarray, threads: int = 1, series_offset: int = 0,
               first_index: int = 0) -> np.ndarray:
    """Oracle result of a reference JSON pipeline config on `values`."""
    arr, aux = lower_config(config, first_index)
    r, L_out = geometry(config, values.shape[1])
    return run_stages(arr, len(config["stages"]), aux, int(config.get("master_seed", 0)), values, L_out,
                      values.shape[0] * r, series_offset=series_offset, threads=threads)


def run_pipeline(pipe, values: np.ndarray, threads: int = 1, series_offset: int = 0) -> np.ndarray:
    """Oracle result of a Pipeline (any object with the reference's
    describe()) on `values`: lowered from its JSON config by the oracle."""
    return run_config(pipe.describe(), values, threads=threads, series_offset=series_offset)


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
