"""Host-side API mirror vs the reference (CPU only, no device needed).

The drop-in promise is that user code written against seriesaug keeps
working: same classes, fields, defaults, validation errors, config JSON, and
stage lowering.  Tests that compare with the reference itself skip when it is
absent (it is only mounted in the build container).
"""

import ctypes
import json

import numpy as np
import pytest

import paper_2601_03159_b200 as sa
from paper_2601_03159_b200 import _abi
from paper_2601_03159_b200.pipeline import lower_stages

GOOD = [
    ("jitter", {"sigma": 0.1}), ("scale", {"sigma_factor": 0.2}), ("rotate", {}),
    ("permute_segments", {"n_segments": 3}), ("crop", {"size": 5}), ("reverse", {}),
    ("resize", {"target_len": 9}), ("quantize", {"n_levels": 4}), ("drift", {"max_drift": 0.5, "n_points": 4}),
    ("inject_noise", {"noise": {"kind": "spike", "count": 2, "magnitude": 1.5}}),
    ("inject_noise", {"noise": {"kind": "uniform", "half_width": 0.3}}),
    ("repeat", {"r": 2}), ("amplitude_phase_perturb", {"sigma_amp": 0.1, "sigma_phase": 0.2}),
    ("frequency_mask", {"width": 3}), ("time_warp", {"n_knots": 5, "intensity": 0.4}),
    ("time_warp_window", {"window_size": 6, "n_knots": 3, "intensity": 0.3}),
]

BAD = [
    ("jitter", {"sigma": -1.0}), ("scale", {"sigma_factor": -0.1}), ("permute_segments", {"n_segments": 0}),
    ("crop", {"size": 0}), ("resize", {"target_len": 1}), ("quantize", {"n_levels": 1}),
    ("drift", {"max_drift": -1.0}), ("drift", {"max_drift": 1.0, "n_points": 1}), ("repeat", {"r": 0}),
    ("amplitude_phase_perturb", {"sigma_amp": -1.0, "sigma_phase": 0.0}), ("frequency_mask", {"width": -1}),
    ("time_warp", {"n_knots": 1}), ("time_warp", {"intensity": -0.5}),
    ("time_warp_window", {"window_size": 1}),
]


def test_registry_covers_reference_kinds(reference):
    assert set(reference.AUGMENTER_REGISTRY) <= set(sa.AUGMENTER_REGISTRY)
    extras = set(sa.AUGMENTER_REGISTRY) - set(reference.AUGMENTER_REGISTRY)
    assert extras == {"dropout", "pool", "convolve", "speed_warp", "random_sinusoid"}


def test_public_names_cover_reference_augmentation_api(reference):
    wanted = {"Batch", "SeedContext", "derive_stream", "Augmenter", "AUGMENTER_REGISTRY", "Pipeline", "Mode",
              "parse_mode", "stage_from_dict", "stage_to_dict", "SpectrumBatch", "fft_forward", "fft_inverse",
              "InvalidParameterError", "InvalidInputError", "InvalidConfigError", "SeriesAugError",
              "UnsupportedPlatformError"} | {c.__name__ for c in reference.AUGMENTER_REGISTRY.values()}
    assert wanted <= set(dir(sa))


@pytest.mark.parametrize("kind,params", GOOD)
def test_config_roundtrip_matches_reference(reference, kind, params):
    rec = {"kind": kind, "probability": 1.0, "params": params}
    ours = sa.stage_to_dict(sa.stage_from_dict(rec))
    theirs = reference.stage_to_dict(reference.stage_from_dict(rec))
    assert json.loads(json.dumps(ours)) == json.loads(json.dumps(theirs))


@pytest.mark.parametrize("kind,params", BAD)
def test_validation_errors_match_reference(reference, kind, params):
    rec = {"kind": kind, "probability": 1.0, "params": params}
    with pytest.raises(Exception) as theirs:
        reference.stage_from_dict(rec)
    with pytest.raises(Exception) as ours:
        sa.stage_from_dict(rec)
    assert type(ours.value).__name__ == type(theirs.value).__name__
    assert str(ours.value) == str(theirs.value)


def test_geometry_probability_rule(reference):
    for mod in (reference, sa):
        with pytest.raises(mod.InvalidParameterError, match="probability must be 0 or 1"):
            mod.Crop(size=3, probability=0.5)


def test_projected_length_errors_match_reference(reference):
    cfg = {"stages": [{"kind": "crop", "params": {"size": 8}}, {"kind": "crop", "params": {"size": 9}}]}
    with pytest.raises(reference.InvalidConfigError) as theirs:
        reference.Pipeline.parse(cfg).projected_length(10)
    with pytest.raises(sa.InvalidConfigError) as ours:
        sa.Pipeline.parse(cfg).projected_length(10)
    assert str(ours.value) == str(theirs.value)
    assert sa.Pipeline.parse(cfg | {"stages": cfg["stages"][:1]}).projected_length(10) == 8


def test_pipeline_rules_match_reference(reference):
    for mod in (reference, sa):
        with pytest.raises(mod.InvalidConfigError):
            mod.Pipeline(stages=(mod.Repeat(r=2), mod.Repeat(r=3)))
        with pytest.raises(mod.InvalidConfigError):
            mod.Pipeline(stages=(mod.Repeat(r=2),), mode=mod.Mode.PER_SAMPLE)
        with pytest.raises(mod.InvalidConfigError):
            mod.Pipeline.parse({"stages": [], "bogus": 1})
        with pytest.raises(mod.InvalidParameterError):
            mod.Pipeline(master_seed=-1)


def test_default_chain_describe_matches(reference):
    pipe = reference.Pipeline(stages=reference.default_chain(), master_seed=41)
    d = pipe.describe()
    assert sa.Pipeline.parse(d).describe() == d


def test_derive_stream_matches_reference(reference):
    for ctx in [(0, 0, 0), (7, 3, 11), (2**64 - 1, 17, 123456789)]:
        a = reference.derive_stream(reference.SeedContext(*ctx)).bit_generator.random_raw(8)
        b = sa.derive_stream(sa.SeedContext(*ctx)).bit_generator.random_raw(8)
        assert np.array_equal(a, b)


def test_batch_validation_matches_reference(reference):
    for bad in (np.zeros(3), np.zeros((0, 3)), np.array([[1.0, np.nan]])):
        with pytest.raises(reference.InvalidInputError) as theirs:
            reference.Batch(bad)
        with pytest.raises(sa.InvalidInputError) as ours:
            sa.Batch(bad)
        assert str(ours.value) == str(theirs.value)
    b = sa.Batch(np.arange(6.0).reshape(2, 3))
    assert b.n == 2 and b.length == 3 and b == sa.Batch.from_sequences([[0, 1, 2], [3, 4, 5]])


def test_spectrum_batch_validation():
    with pytest.raises(sa.InvalidInputError, match="DC bin"):
        sa.SpectrumBatch(np.ones((1, 3)), np.ones((1, 3)), 4)
    with pytest.raises(sa.InvalidInputError, match="implies"):
        sa.SpectrumBatch(np.ones((1, 3)), np.zeros((1, 3)), 7)


def test_lowering_op_codes_and_params():
    pipe = sa.Pipeline(stages=(
        sa.Jitter(0.1), sa.InjectNoise(sa.SpikeNoise(3, 2.0), probability=0.25), sa.WindowWarp(8, 5, 0.3),
        sa.Convolve("hann", 5), sa.Pool(3, "max"), sa.SpeedWarp(2, 2.5, "linear"), sa.RandomSinusoid(0.5, 2)))
    arr, aux = lower_stages(pipe.stages, first_index=4)
    ops = [arr[j].op for j in range(7)]
    assert ops == [_abi.SA_OP_JITTER, _abi.SA_OP_NOISE_SPIKE, _abi.SA_OP_WINDOW_WARP, _abi.SA_OP_CONVOLVE,
                   _abi.SA_OP_POOL, _abi.SA_OP_SPEED_WARP, _abi.SA_OP_SINUSOID]
    assert [arr[j].index for j in range(7)] == [4, 5, 6, 7, 8, 9, 10]
    assert arr[1].probability == 0.25 and arr[1].i[0] == 3 and arr[1].f[0] == 2.0
    assert (arr[2].i[0], arr[2].i[1], arr[2].f[0]) == (8, 5, 0.3)
    assert arr[3].aux_len == 5 and np.isclose(aux[arr[3].aux_off:arr[3].aux_off + 5].sum(), 1.0)
    assert (arr[4].i[0], arr[4].i[1]) == (3, 1)
    assert (arr[5].i[0], arr[5].i[1], arr[5].f[0]) == (2, 0, 2.5)


def test_extras_validation():
    with pytest.raises(sa.InvalidParameterError):
        sa.Dropout(rate=1.5)
    with pytest.raises(sa.InvalidParameterError):
        sa.Pool(size=0)
    with pytest.raises(sa.InvalidParameterError):
        sa.Pool(size=2, reducer="median")
    with pytest.raises(sa.InvalidParameterError):
        sa.Convolve("gauss", 5)
    with pytest.raises(sa.InvalidParameterError):
        sa.SpeedWarp(max_speed_ratio=0.5)
    with pytest.raises(sa.InvalidConfigError):
        sa.Pipeline(stages=(sa.RandomSinusoid(1.0, min_bin=9),)).projected_length(8)
    taps = sa.Convolve("triang", 7).taps()
    assert np.isclose(taps.sum(), 1.0) and (taps > 0).all() and np.allclose(taps, taps[::-1])
    # hann: scipy's symmetric window (zero end taps), normalised by its sum
    hann = sa.Convolve("hann", 7).taps()
    assert hann[0] == 0.0 == hann[-1] and np.allclose(hann, np.array([0, 1, 3, 4, 3, 1, 0]) / 12.0, rtol=0, atol=1e-15)
    with pytest.raises(sa.InvalidParameterError):
        sa.Convolve("hann", 2)


def test_custom_augmenter_without_kernel_fails_loudly():
    from dataclasses import dataclass
    from typing import ClassVar

    import numpy as np

    @dataclass(frozen=True)
    class Mine(sa.Augmenter):
        probability: float = 1.0
        kind: ClassVar[str] = "mine_test"

        def _apply(self, series, rng):
            return series + 1.0

    @dataclass(frozen=True)
    class MySpectral(sa.SpectralAugmenter):
        probability: float = 1.0
        kind: ClassVar[str] = "my_spectral_test"

        def _perturb_row(self, re, im, original_len, rng):
            return re, im

    @dataclass(frozen=True)
    class MyJitter(sa.Jitter):  # overriding a built-in's hook drops its kernel
        def _apply(self, series, rng):
            return series

    @dataclass(frozen=True)
    class NoHook(sa.Augmenter):
        probability: float = 1.0
        kind: ClassVar[str] = "no_hook_test"

    # the reference refuses to instantiate an operator without _apply (ABC)
    with pytest.raises(TypeError):
        NoHook()
    # kernel-less operators are rejected when the pipeline is built
    for op in (Mine(), MySpectral(), MyJitter(0.1)):
        with pytest.raises(sa.InvalidConfigError, match="no B200 kernel"):
            sa.Pipeline(stages=(sa.Jitter(0.1), op))
        with pytest.raises(sa.InvalidConfigError, match="no B200 kernel"):
            lower_stages((op,))
    # built-ins run on the device only: their Python hook refuses
    with pytest.raises(sa.InvalidConfigError, match="not available"):
        sa.Jitter(0.1)._apply(np.zeros(4), None)
    assert sa.Pipeline(stages=(sa.Jitter(0.1), sa.FrequencyMask(3), sa.Dropout(0.1))).stages


@pytest.mark.parametrize("where", [0, 12345, (1 << 20) + 7, -1])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_batch_native_finiteness_scan(where, bad):
    """Large batches are validated by the library's multi-threaded scan
    (sa_host_all_finite): same predicate as np.isfinite(...).all()."""
    from paper_2601_03159_b200 import Batch, InvalidInputError
    from paper_2601_03159_b200.core import _NATIVE_SCAN_MIN

    x = np.random.default_rng(0).normal(size=(64, (_NATIVE_SCAN_MIN + 4096) // 64))
    Batch(x)
    x.reshape(-1)[where] = bad
    with pytest.raises(InvalidInputError):
        Batch(x)
    x.reshape(-1)[where] = np.finfo(np.float64).max  # largest finite: accepted
    Batch(x)
    x.reshape(-1)[where] = 5e-324  # subnormal: accepted
    Batch(x)


def test_output_cache_policy(monkeypatch):
    """memory.output_array: first request of a size -> numpy memory, a repeat
    -> a page-locked block that returns to the cache with its array."""
    import gc

    from paper_2601_03159_b200 import memory

    calls = []

    class FakeLib:
        def sa_host_alloc(self, pp, size):
            buf = ctypes.create_string_buffer(size)
            calls.append(("alloc", size, buf))
            pp._obj.value = ctypes.addressof(buf)
            return 0

        def sa_host_free(self, ptr):
            calls.append(("free", ptr))
            return 0

    monkeypatch.setattr(memory._native, "lib", lambda: FakeLib())
    monkeypatch.setattr(memory, "_outputs", memory._OutputCache())
    memory._outputs.cap = 64 << 20
    small = memory.output_array((10, 10))
    assert isinstance(small.base, type(None)) or not calls  # below the threshold: numpy
    a = memory.output_array((1024, 1024))  # 8 MB, first request of this size
    assert not calls and a.flags.owndata
    b = memory.output_array((1024, 1024))  # repeat: page-locked block
    assert len(calls) == 1 and calls[0][1] == 8 << 20 and b.shape == (1024, 1024) and not b.flags.owndata
    b[...] = 1.0
    ptr = b.ctypes.data
    del b
    gc.collect()
    c = memory.output_array((1024, 1024))  # reused from the cache
    assert len(calls) == 1 and c.ctypes.data == ptr
    d = memory.output_array((1024, 1024))  # second live block
    assert len(calls) == 2
    memory._outputs.cap = 20 << 20  # no room for a third
    e = memory.output_array((1024, 1024))
    assert len(calls) == 2 and e.flags.owndata
