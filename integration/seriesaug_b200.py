"""seriesaug/_b200.py -- the binding a reference maintainer adds to route the
reference's augmentation path to the B200 C ABI (include/seriesaug_b200.h).

It is written against the reference package (relative imports of its own
modules), kept here so it can be executed: tests/test_integration_binding.py
loads it as `seriesaug._b200` inside the unmodified reference (oracle/_ref),
installs it, and checks the patched reference against the reference's own
CPU results.  INTEGRATION.md §2 walks through it.

Entry points it binds (the reference interface each replaces):
  sa_pipeline_run_host   Pipeline.run (reference pipeline.py:129-157) and
                         Augmenter.augment_batch (core.py:239-259)
  sa_last_error          the message of a failed call
"""

import ctypes
import os

import numpy as np

from .errors import InvalidConfigError, InvalidInputError
from .pipeline import stage_to_dict

LIB_ENV = "SERIESAUG_B200_LIB"
_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(os.environ.get(LIB_ENV, "libseriesaug_b200.so"))
        _lib.sa_last_error.restype = ctypes.c_char_p
    return _lib


class SaStage(ctypes.Structure):  # struct sa_stage
    _fields_ = [("op", ctypes.c_int32), ("index", ctypes.c_int32), ("probability", ctypes.c_double),
                ("f", ctypes.c_double * 6), ("i", ctypes.c_int64 * 6),
                ("aux_off", ctypes.c_int32), ("aux_len", ctypes.c_int32)]


# kind -> (op code, int params, float params), include/seriesaug_b200.h SA_OP_*
OPS = {
    "jitter": (1, [], ["sigma"]),
    "scale": (2, [], ["sigma_factor"]),
    "rotate": (3, [], []),
    "permute_segments": (4, ["n_segments"], []),
    "crop": (5, ["size"], []),
    "reverse": (6, [], []),
    "resize": (7, ["target_len"], []),
    "quantize": (8, ["n_levels"], []),
    "drift": (9, ["n_points"], ["max_drift"]),
    "repeat": (14, ["r"], []),
    "amplitude_phase_perturb": (15, [], ["sigma_amp", "sigma_phase"]),
    "frequency_mask": (16, ["width"], []),
    "time_warp": (17, ["n_knots"], ["intensity"]),
    "time_warp_window": (18, ["window_size", "n_knots"], ["intensity"]),
    # BASELINE-only kinds (added to the reference as plugins)
    "dropout": (19, [], ["rate", "fill"]),
    "pool": (20, ["size", "reducer"], []),
    "convolve": (21, [], []),
    "speed_warp": (22, ["n_speed_change", "interpolation"], ["max_speed_ratio"]),
    "random_sinusoid": (23, ["min_bin"], ["amplitude"]),
}
NOISE = {"uniform": (10, "half_width"), "gaussian": (11, "sigma"), "spike": (12, "magnitude"),
         "slope_trend": (13, "max_offset")}
ENUMS = {"reducer": ("mean", "max", "min"), "interpolation": ("linear", "cubic")}


def convolve_taps(window, size):
    from scipy.signal import get_window

    w = get_window("boxcar" if window == "flat" else window, size, fftbins=False)
    return w / w.sum()


def lower(j, stage, aux):
    rec = stage_to_dict(stage)
    p, kind = rec["params"], rec["kind"]
    st = SaStage(index=j, probability=rec["probability"])
    if kind == "inject_noise":
        nz = p["noise"]
        st.op, name = NOISE[nz["kind"]]
        st.f[0] = nz[name]
        st.i[0] = nz.get("count", 0)
        return st
    if kind not in OPS:
        raise InvalidConfigError(f"augmenter kind {kind!r} has no B200 kernel")
    st.op, ints, flts = OPS[kind]
    for n, name in enumerate(ints):
        v = p[name]
        st.i[n] = ENUMS[name].index(v) if name in ENUMS else v
    for n, name in enumerate(flts):
        st.f[n] = p[name]
    if kind == "convolve":
        taps = convolve_taps(p["window"], p["size"])
        st.aux_off, st.aux_len = len(aux), len(taps)
        aux.extend(float(v) for v in taps)
    return st


def lower_all(stages, first_index=0):
    aux = []
    arr = (SaStage * max(1, len(stages)))(*[lower(first_index + j, s, aux) for j, s in enumerate(stages)])
    return arr, np.ascontiguousarray(aux, dtype=np.float64)


def run_stages(stages, values, seed, first_index, L_out, rows):
    arr, aux = lower_all(stages, first_index)
    values = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty((rows, L_out))
    rc = lib().sa_pipeline_run_host(arr, len(stages), aux.ctypes.data_as(ctypes.c_void_p), ctypes.c_int32(aux.size),
                                    ctypes.c_uint64(seed), ctypes.c_int64(0),
                                    values.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(values.shape[0]),
                                    ctypes.c_int64(values.shape[1]), out.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.c_int64(L_out))
    if rc == -2:
        raise InvalidInputError("batch contains non-finite values (NaN or Inf)")
    if rc != 0:
        raise RuntimeError(lib().sa_last_error().decode())
    return out


def _rows(stages, n):
    for s in stages:
        if s.kind == "repeat" and s.probability == 1.0:
            return n * s.r
    return n


def run_pipeline(pipe, batch):
    """Pipeline.run on the device (validation stays in the reference)."""
    L_out = pipe.projected_length(batch.length)
    return run_stages(pipe.stages, batch.values, pipe.master_seed, 0, L_out, _rows(pipe.stages, batch.n))


def augment_batch(stage, batch, master_seed, augmenter_index=0):
    """Augmenter.augment_batch on the device (core.py:239-259)."""
    stage.validate_for_length(batch.length)
    L_out = stage.output_length(batch.length) if stage.probability == 1.0 else batch.length
    return run_stages((stage,), batch.values, master_seed, augmenter_index, L_out, _rows((stage,), batch.n))


def install():
    """The opt-in switch: Pipeline.run and augment_batch call the device."""
    from .core import Augmenter, Batch
    from .pipeline import Pipeline

    Pipeline.run = lambda self, batch: Batch(run_pipeline(self, batch))
    Augmenter.augment_batch = lambda self, batch, master_seed, parallel=False, augmenter_index=0: Batch(
        augment_batch(self, batch, master_seed, augmenter_index))
