"""INTEGRATION.md §2's reference-side binding (integration/seriesaug_b200.py),
executed: loaded as `seriesaug._b200` inside the unmodified reference
(oracle/_ref, installed by build()), lowering checked against the product's
(CPU), then installed so the reference's own Pipeline.run / augment_batch
call sa_pipeline_run_host, and compared with the reference's CPU results
(GPU): bitwise for exact chains, the spectral tolerance for FFT chains."""

import ctypes
import importlib.util
import os

import numpy as np
import pytest

from sa_testutil import assert_matches

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binding():
    from oracle.refpkg import import_reference, location

    if location() is None:
        pytest.skip("reference package not installed")
    ref = import_reference()
    import oracle.extras_ref  # noqa: F401  (BASELINE-only kinds as reference plugins)

    spec = importlib.util.spec_from_file_location("seriesaug._b200", os.path.join(ROOT, "integration",
                                                                                  "seriesaug_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    os.environ.setdefault(mod.LIB_ENV, os.path.join(ROOT, "paper_2601_03159_b200", "_lib", "libseriesaug_b200.so"))
    return ref, mod


def _pipeline_cases(golden):
    meta, arrays = golden
    return [c for c in meta["cases"] if c["kind"] in ("pipeline", "augment_batch")]


def test_binding_lowering_equals_product(binding, golden):
    """The binding lowers every golden config (all 23 op codes) to the same
    sa_stage bytes and aux table as the product's lower_stages."""
    from paper_2601_03159_b200 import Pipeline as PPipeline
    from paper_2601_03159_b200.pipeline import lower_stages

    ref, mod = binding
    ops = set()
    for case in _pipeline_cases(golden):
        first = case["augmenter_index"] or 0
        rp = ref.Pipeline.parse(case["config"])
        a1, x1 = mod.lower_all(rp.stages, first)
        a2, x2 = lower_stages(PPipeline.parse(case["config"]).stages, first)
        assert bytes(a1) == bytes(a2), case["name"]
        assert np.array_equal(x1, x2), case["name"]
        ops.update(a1[j].op for j in range(len(rp.stages)))
    assert ops == set(range(1, 24))


@pytest.mark.gpu
def test_installed_binding_matches_reference_cpu(binding, golden):
    ref, mod = binding
    meta, arrays = golden
    cases = [c for c in _pipeline_cases(golden) if c["config"]["mode"] == "standard"]
    want = {}
    for case in cases:  # the reference's own CPU results first
        x = arrays[case["input"]]
        if case["kind"] == "pipeline":
            want[case["name"]] = ref.Pipeline.parse(case["config"]).run(ref.Batch(x)).values
        else:
            st = ref.stage_from_dict(case["config"]["stages"][0])
            want[case["name"]] = st.augment_batch(ref.Batch(x), case["config"]["master_seed"],
                                                  augmenter_index=case["augmenter_index"]).values
    run0, ab0 = ref.Pipeline.run, ref.Augmenter.augment_batch
    mod.install()
    try:
        before = mod.lib()
        for case in cases:
            x = arrays[case["input"]]
            if case["kind"] == "pipeline":
                got = ref.Pipeline.parse(case["config"]).run(ref.Batch(x)).values
            else:
                st = ref.stage_from_dict(case["config"]["stages"][0])
                got = st.augment_batch(ref.Batch(x), case["config"]["master_seed"],
                                       augmenter_index=case["augmenter_index"]).values
            assert_matches(got, want[case["name"]], case["exact"], case["name"])
        assert before is mod.lib()
    finally:
        ref.Pipeline.run, ref.Augmenter.augment_batch = run0, ab0
    with pytest.raises(ref.InvalidInputError):
        mod.run_stages(ref.Pipeline.parse({"stages": [{"kind": "reverse"}]}).stages,
                       np.array([[1.0, np.nan]]), 0, 0, 2, 1)
