"""Pin the C oracle against the reference's own outputs (tests/golden).

Each golden case is a reference pipeline config run by the reference itself
(tests/golden/make_golden.py).  Here the same JSON is parsed by the product's
Pipeline.parse, lowered to the C-ABI stage table, and executed by the oracle:
this pins both the oracle's semantics and the product's lowering.  Non-FFT
cases must match bitwise; FFT cases within tests/conftest.spectral_tol.
"""

import numpy as np

from oracle import oracle as O
from paper_2601_03159_b200 import Jitter, Pipeline, stage_from_dict
from paper_2601_03159_b200.pipeline import lower_stages
from sa_testutil import assert_matches, spectral_tol


def _cases(golden, kinds):
    meta, _ = golden
    return [c for c in meta["cases"] if c["kind"] in kinds]


def run_case_oracle(case, x):
    cfg = case["config"]
    pipe = Pipeline.parse(cfg)
    first = case["augmenter_index"] or 0
    arr, aux = lower_stages(pipe.stages, first)
    L_out = pipe.projected_length(x.shape[1])
    rows = x.shape[0] * pipe.row_factor()
    return O.run_stages(arr, len(pipe.stages), aux, cfg["master_seed"], x, L_out, rows)


def test_pipeline_cases(golden):
    meta, arrays = golden
    cases = _cases(golden, ("pipeline", "augment_batch"))
    assert len(cases) >= 50
    for case in cases:
        x = arrays[case["input"]]
        got = run_case_oracle(case, x)
        assert_matches(got, arrays[case["output"]], case["exact"], case["name"])


def test_fft_cases(golden):
    meta, arrays = golden
    for case in _cases(golden, ("fft",)):
        x = arrays[case["input"]]
        re, im = O.fft_forward(x)
        assert np.abs(re - arrays[case["re"]]).max() <= spectral_tol(arrays[case["re"]]), case["name"]
        assert np.abs(im - arrays[case["im"]]).max() <= spectral_tol(arrays[case["re"]]), case["name"]
        back = O.fft_inverse(arrays[case["re"]], arrays[case["im"]], x.shape[1])
        assert np.abs(back - arrays[case["inverse"]]).max() <= spectral_tol(x), case["name"]


def test_spectrum_cases(golden):
    meta, arrays = golden
    for case in _cases(golden, ("spectrum",)):
        x = arrays[case["input"]]
        re, im = O.fft_forward(x)
        stage = stage_from_dict(case["stage"])._lower(case["augmenter_index"], [])
        ro, io = O.augment_spectrum(stage, case["seed"], re, im, x.shape[1])
        tol = spectral_tol(arrays[case["re"]])
        assert np.abs(ro - arrays[case["re"]]).max() <= tol, case["name"]
        assert np.abs(io - arrays[case["im"]]).max() <= tol, case["name"]
        # masked / real bins are exact zeros (test_freqaugment.py:111-125)
        assert np.array_equal(io[:, 0], np.zeros(x.shape[0]))


def test_gate_pin(golden):
    """'p=0.5 fired 5016/10000' (reference test_output.txt:21)."""
    meta, _ = golden
    pin = meta["gate_pin"]
    pipe = Pipeline(stages=(Jitter(sigma=pin["sigma"], probability=pin["probability"]),),
                    master_seed=pin["seed"])
    x = np.ones(pin["shape"])
    out = O.run_pipeline(pipe, x)
    fired = int(np.sum(np.any(out != 1.0, axis=1)))
    assert fired == pin["fired"] == 5016


def _one(aug, x, seed=0):
    pipe = Pipeline(stages=(aug,), master_seed=seed)
    return O.run_pipeline(pipe, np.asarray(x, dtype=np.float64)[None, :])[0]


def test_reference_known_answers():
    """Known answers from the reference's unit tests (test_basic.py)."""
    from paper_2601_03159_b200 import (Drift, InjectNoise, PermuteSegments, Quantize, Resize,
                                       SlopeTrendNoise)

    assert np.array_equal(_one(PermuteSegments(n_segments=2), [1.0, 2.0, 3.0, 4.0], seed=1),
                          [3.0, 4.0, 1.0, 2.0])  # test_basic.py:88-91
    assert np.array_equal(_one(Resize(target_len=3), [0.0, 2.0]), [0.0, 1.0, 2.0])
    assert np.array_equal(_one(Quantize(n_levels=2), [0.0, 0.5, 1.0]), [0.0, 0.0, 1.0])
    for seed in range(8):  # test_basic.py:220-225
        assert np.abs(_one(Drift(max_drift=0.7, n_points=5), np.zeros(64), seed=seed)).max() == 0.7
    x = np.random.default_rng(11).normal(0, 1, 40)
    ramp = _one(InjectNoise(noise=SlopeTrendNoise(max_offset=1.5)), x, seed=6) - x
    assert ramp[0] == 0.0 and abs(ramp[-1]) == 1.5


def test_standard_equals_per_sample_and_sharding(golden):
    """Series-range sharding with a global series_offset reproduces the
    unsharded result bit for bit."""
    meta, arrays = golden
    case = next(c for c in meta["cases"] if c["name"] == "cfg5_time_domain")
    pipe = Pipeline.parse(case["config"])
    x = arrays[case["input"]]
    full = O.run_pipeline(pipe, x)
    parts = [O.run_pipeline(pipe, x[a:b], series_offset=a) for a, b in ((0, 1), (1, 3))]
    assert np.array_equal(np.concatenate(parts), full)
    assert np.array_equal(O.run_pipeline(pipe, x, threads=3), full)


def test_dct_cases(golden):
    """Orthonormal DCT-II / III vs scipy via the reference (freqtransform.py:91-98)."""
    meta, arrays = golden
    cases = [c for c in meta["cases"] if c["kind"] == "dct"]
    assert len(cases) >= 7
    for case in cases:
        x = arrays[case["input"]]
        assert np.abs(O.dct(x) - arrays[case["coeffs"]]).max() <= spectral_tol(x), case["name"]
        back = O.dct(arrays[case["coeffs"]], inverse=True)
        assert np.abs(back - arrays[case["inverse"]]).max() <= spectral_tol(x), case["name"]


def test_dtw_cases(golden):
    """dtw.py:40-85: distance bitwise, path exactly (tie order included)."""
    meta, arrays = golden
    cases = [c for c in meta["cases"] if c["kind"] == "dtw"]
    assert len(cases) >= 8
    for case in cases:
        d, path = O.dtw(arrays[case["a"]], arrays[case["b"]])
        assert d == case["distance"], case["name"]
        assert [list(p) for p in path] == case["path"], case["name"]


def test_similarity_ordering_criterion10(golden):
    """Acceptance criterion 10 (test_acceptance.py:334-369) through the
    oracle: recorded scores 0.998 / 0.964 / 0.901 / 0.722 (test_output.txt:29)."""
    meta, arrays = golden
    case = next(c for c in meta["cases"] if c["kind"] == "similarity")
    base = arrays[case["base"]]
    for name, rec in case["augmented"].items():
        pipe = Pipeline.parse({"master_seed": 99, "stages": [rec["stage"]]})
        out = O.run_pipeline(pipe, base)
        sims = [1.0 / (1.0 + O.dtw(base[i], out[i])[0] / base.shape[1]) for i in range(base.shape[0])]
        score = sum(sims) / len(sims)
        assert abs(score - case["augmented"][name]["score"]) < 1e-9, name


def test_oracle_lowering_equals_product(golden):
    """The oracle lowers JSON configs itself (oracle.lower_config, no product
    code); for every golden config it must produce the product's stage table
    byte for byte (so oracle results check the product's lowering too)."""
    import dataclasses

    from paper_2601_03159_b200 import AUGMENTER_REGISTRY

    for case in _cases(golden, ("pipeline", "augment_batch")):
        first = case["augmenter_index"] or 0
        a1, x1 = O.lower_config(case["config"], first)
        a2, x2 = lower_stages(Pipeline.parse(case["config"]).stages, first)
        n = len(case["config"]["stages"])
        assert bytes(a1)[:n * 120] == bytes(a2)[:n * 120], case["name"]
        assert np.array_equal(x1, x2), case["name"]
    # the oracle's parameter defaults (for configs that omit them) are the product's
    for kind, dflt in O._DEFAULTS.items():
        fields = {f.name: f.default for f in dataclasses.fields(AUGMENTER_REGISTRY[kind])}
        for name, v in dflt.items():
            assert fields[name] == v, (kind, name)
