"""ctypes mirror of include/seriesaug_b200.h (the C ABI).

Op codes and status codes must match the header; tests/test_abi.py parses the
header and checks every constant and the struct layout.
"""

from __future__ import annotations

import ctypes

SA_ABI_VERSION = 1

SA_OK = 0
SA_ERR_INVALID_ARG = -1
SA_ERR_NONFINITE = -2
SA_ERR_WARP_MONOTONE = -3
SA_ERR_CUDA = -4
SA_ERR_UNSUPPORTED = -5
SA_ERR_NO_DEVICE = -6

SA_FLAG_NONFINITE = 1
SA_FLAG_WARP_MONOTONE = 2

SA_OP_JITTER = 1
SA_OP_SCALE = 2
SA_OP_ROTATE = 3
SA_OP_PERMUTE = 4
SA_OP_CROP = 5
SA_OP_REVERSE = 6
SA_OP_RESIZE = 7
SA_OP_QUANTIZE = 8
SA_OP_DRIFT = 9
SA_OP_NOISE_UNIFORM = 10
SA_OP_NOISE_GAUSSIAN = 11
SA_OP_NOISE_SPIKE = 12
SA_OP_NOISE_SLOPE = 13
SA_OP_REPEAT = 14
SA_OP_APP = 15
SA_OP_FREQ_MASK = 16
SA_OP_TIME_WARP = 17
SA_OP_WINDOW_WARP = 18
SA_OP_DROPOUT = 19
SA_OP_POOL = 20
SA_OP_CONVOLVE = 21
SA_OP_SPEED_WARP = 22
SA_OP_SINUSOID = 23
SA_OP_MAX = 24

SA_MAX_STAGES = 64

# dataset files (include/seriesaug_b200.h, reference datafiles.py)
SA_FORMAT_AUTO = -1
SA_FORMAT_CSV = 0
SA_FORMAT_TS = 1
SA_DS_OK = 0
SA_DS_EMPTY = 1
SA_DS_HEADER_AFTER_DATA = 2
SA_DS_MISSING_LABEL = 3
SA_DS_NOT_A_NUMBER = 4
SA_DS_RAGGED = 5
SA_DS_NO_DATA = 6
SA_DS_NONFINITE = 7
SA_DS_BAD_UTF8 = 8


class SaDatasetInfo(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("status", ctypes.c_int32), ("n_lines", ctypes.c_int64),
                ("n_series", ctypes.c_int64), ("length", ctypes.c_int64), ("header_bytes", ctypes.c_int64),
                ("label_bytes", ctypes.c_int64), ("err_line", ctypes.c_int64), ("err_ref_line", ctypes.c_int64),
                ("err_fields", ctypes.c_int64), ("err_ref_fields", ctypes.c_int64), ("err_begin", ctypes.c_int64),
                ("err_end", ctypes.c_int64)]


class SaStage(ctypes.Structure):
    """struct sa_stage: one lowered {kind, probability, params} record."""

    _fields_ = [
        ("op", ctypes.c_int32),
        ("index", ctypes.c_int32),
        ("probability", ctypes.c_double),
        ("f", ctypes.c_double * 6),
        ("i", ctypes.c_int64 * 6),
        ("aux_off", ctypes.c_int32),
        ("aux_len", ctypes.c_int32),
    ]


def make_stage(op: int, index: int, probability: float, f=(), i=(), aux_off=0, aux_len=0) -> SaStage:
    st = SaStage()
    st.op = op
    st.index = index
    st.probability = float(probability)
    for k, v in enumerate(f):
        st.f[k] = float(v)
    for k, v in enumerate(i):
        st.i[k] = int(v)
    st.aux_off = aux_off
    st.aux_len = aux_len
    return st
