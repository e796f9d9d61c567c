"""Generate tests/golden/reference_cases.{json,npz} by running the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every case is a seriesaug pipeline config (the reference's own JSON schema,
pipeline.py:159-201) or a transform call, run through the reference's public
API on a small seeded input (the BASELINE-only kinds -- dropout, pool,
convolve, speed_warp, random_sinusoid -- as the reference plugins of
oracle/extras_ref.py); inputs and outputs are stored so the tests can
replay them against the C oracle (CPU) and the CUDA backend (GPU) without the
reference present.  numpy / scipy versions are recorded in the JSON.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def st(kind, p=1.0, **params):
    return {"kind": kind, "probability": p, "params": params}


def sinusoids(n, L, seed):
    """BASELINE config 1 input: sum of 3 sinusoids, periods U[8,128],
    amplitudes U(0.5,2), phases U[0,2pi), plus N(0, 0.1^2) noise."""
    rng = np.random.default_rng(seed)
    t = np.arange(L)
    x = np.zeros((n, L))
    for _ in range(3):
        per = rng.uniform(8, 128, (n, 1))
        amp = rng.uniform(0.5, 2.0, (n, 1))
        ph = rng.uniform(0, 2 * np.pi, (n, 1))
        x += amp * np.sin(2 * np.pi * t / per + ph)
    return x + rng.normal(0, 0.1, (n, L))


def main() -> None:
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import scipy
    from scipy.signal import lfilter

    from oracle.refpkg import import_reference

    ref = import_reference()
    import oracle.extras_ref  # noqa: F401  (registers the BASELINE-only kinds as reference plugins)

    arrays: dict[str, np.ndarray] = {}
    cases: list[dict] = []

    def inp(name, arr):
        arrays["in_" + name] = np.ascontiguousarray(arr, dtype=np.float64)
        return "in_" + name

    rng = np.random.default_rng(20260101)
    inputs = {
        "w64": inp("w64", np.cumsum(rng.normal(0, 1, (5, 64)), axis=1)),
        "w100": inp("w100", np.cumsum(rng.normal(0, 1, (4, 100)), axis=1)),
        "w128": inp("w128", np.cumsum(rng.normal(0, 1, (4, 128)), axis=1)),
        "w7": inp("w7", rng.normal(0, 1, (3, 7))),
        "w15": inp("w15", rng.normal(0, 1, (3, 15))),
        "w2": inp("w2", rng.normal(0, 1, (3, 2))),
        "w1": inp("w1", rng.normal(0, 1, (3, 1))),
        "w1024": inp("w1024", ref.synthetic_batch(3, 1024, seed=1).values),
        "const": inp("const", np.full((2, 16), 2.5)),
        "zeros64": inp("zeros64", np.zeros((8, 64))),
        "sin512": inp("sin512", sinusoids(6, 512, seed=0)),
        "w1500": inp("w1500", np.cumsum(rng.normal(0, 1, (2, 1500)), axis=1)
                     + 3 * np.sin(2 * np.pi * np.arange(1500) / 200.0)),
        "ar2048": inp("ar2048", lfilter([1.0], [1.0, -0.6, 0.2], rng.normal(0, 1, (3, 2048)), axis=1)),
    }

    def case(name, stages, inkey, seed=7, mode="standard", exact=True, index=None):
        cfg = {"master_seed": seed, "parallel": False, "mode": mode, "stages": stages}
        batch = ref.Batch(arrays[inkey])
        if index is None:
            out = ref.Pipeline.parse(cfg).run(batch).values
        else:
            aug = ref.stage_from_dict(stages[0])
            out = aug.augment_batch(batch, seed, augmenter_index=index).values
        arrays["out_" + name] = out
        cases.append({"name": name, "kind": "pipeline" if index is None else "augment_batch",
                      "config": cfg, "input": inkey, "output": "out_" + name,
                      "augmenter_index": index, "exact": exact})

    I = inputs
    # --- pointwise family
    case("jitter", [st("jitter", sigma=0.05)], I["sin512"], seed=0)
    case("jitter_p05", [st("jitter", 0.5, sigma=1.0)], I["w64"], seed=3)
    case("jitter_zero", [st("jitter", sigma=0.0)], I["w64"])
    case("jitter_idx5", [st("jitter", sigma=0.3)], I["w100"], index=5)
    case("scale", [st("scale", sigma_factor=0.2)], I["w64"])
    case("scale_zero", [st("scale", sigma_factor=0.0)], I["w7"])
    case("rotate", [st("rotate")], I["w15"])
    case("reverse", [st("reverse", 0.5)], I["w100"])
    case("quantize16", [st("quantize", n_levels=16)], I["w128"])
    case("quantize2", [st("quantize", n_levels=2)], I["w7"])
    case("quantize_const", [st("quantize", n_levels=4)], I["const"])
    case("drift", [st("drift", max_drift=0.5, n_points=5)], I["w100"])
    case("drift_peak", [st("drift", max_drift=0.7, n_points=5)], I["zeros64"], seed=3)
    case("drift_two", [st("drift", max_drift=1.3, n_points=2)], I["w15"])
    case("drift_len1", [st("drift", max_drift=1.0)], I["w1"])
    case("drift_zero", [st("drift", max_drift=0.0)], I["w7"])
    case("noise_uniform", [st("inject_noise", noise={"kind": "uniform", "half_width": 0.3})], I["w64"])
    case("noise_gaussian", [st("inject_noise", noise={"kind": "gaussian", "sigma": 0.2})], I["w64"])
    case("noise_spike", [st("inject_noise", noise={"kind": "spike", "count": 3, "magnitude": 2.0})], I["w100"])
    case("noise_spike_all", [st("inject_noise", noise={"kind": "spike", "count": 15, "magnitude": 1.0})], I["w15"])
    case("noise_spike_big", [st("inject_noise", noise={"kind": "spike", "count": 90, "magnitude": 0.5})], I["w128"])
    case("noise_spike_const", [st("inject_noise", noise={"kind": "spike", "count": 4, "magnitude": 1.0})], I["const"])
    case("noise_spike_1024", [st("inject_noise", noise={"kind": "spike", "count": 40, "magnitude": 3.0})], I["w1024"])
    case("noise_slope", [st("inject_noise", noise={"kind": "slope_trend", "max_offset": 1.5})], I["w64"])
    # --- gather / interpolation family (G1-G7)
    case("crop", [st("crop", size=51)], I["w64"])
    case("crop_full", [st("crop", size=64)], I["w64"])
    case("crop_one", [st("crop", size=1)], I["w7"])
    case("crop_p0", [st("crop", 0.0, size=3)], I["w7"])
    case("resize_up", [st("resize", target_len=29)], I["w15"])
    case("resize_down", [st("resize", target_len=37)], I["w100"])
    case("resize_same", [st("resize", target_len=64)], I["w64"])
    case("resize_two", [st("resize", target_len=3)], I["w2"])
    case("permute2", [st("permute_segments", n_segments=2)], I["w64"])
    case("permute4", [st("permute_segments", n_segments=4)], I["w100"])
    case("permute_all", [st("permute_segments", n_segments=7)], I["w7"])
    case("permute_odd", [st("permute_segments", n_segments=3)], I["w100"])
    case("time_warp", [st("time_warp", n_knots=4, intensity=0.5)], I["w100"])
    case("time_warp_2knots", [st("time_warp", n_knots=2, intensity=0.5)], I["w64"])
    case("time_warp_wild", [st("time_warp", n_knots=10, intensity=5.0)], I["w128"])
    case("time_warp_zero", [st("time_warp", n_knots=4, intensity=0.0)], I["w15"])
    case("time_warp_len2", [st("time_warp", n_knots=3, intensity=1.0)], I["w2"])
    case("window_warp", [st("time_warp_window", window_size=16, n_knots=4, intensity=0.5)], I["w100"])
    case("window_warp_full", [st("time_warp_window", window_size=64, n_knots=5, intensity=0.5)], I["w64"])
    case("repeat", [st("jitter", sigma=0.1), st("repeat", r=3), st("scale", 0.5, sigma_factor=0.3)], I["w15"])
    case("repeat_p0", [st("repeat", 0.0, r=3), st("jitter", sigma=0.1)], I["w15"])
    # --- spectral family (F1-F4): pocketfft vs our FFT -> tolerance
    case("app", [st("amplitude_phase_perturb", sigma_amp=0.5, sigma_phase=0.2)], I["w64"], exact=False)
    case("app_amp_only", [st("amplitude_phase_perturb", sigma_amp=0.3, sigma_phase=0.0)], I["w128"], exact=False)
    case("app_noop", [st("amplitude_phase_perturb", sigma_amp=0.0, sigma_phase=0.0)], I["w64"])
    case("app_odd", [st("amplitude_phase_perturb", sigma_amp=0.5, sigma_phase=0.2)], I["w15"], exact=False)
    case("fmask", [st("frequency_mask", width=10)], I["w64"], exact=False)
    case("fmask_all", [st("frequency_mask", width=33)], I["w64"], exact=False)
    case("fmask_1024", [st("frequency_mask", width=51)], I["w1024"], exact=False)
    case("fmask_zero", [st("frequency_mask", width=0)], I["w64"])
    # --- chains: default_chain and the BASELINE configs' reference-mappable parts
    dchain = [ref.stage_to_dict(s) for s in ref.default_chain()]
    case("default_chain", dchain, I["w128"], seed=41, exact=False)
    case("default_chain_per_sample", dchain, I["w64"], seed=41, mode="per-sample", exact=False)
    case("cfg1_jitter", [st("jitter", sigma=0.05)], I["sin512"], seed=0)
    case("cfg2_mappable", [st("crop", size=819), st("drift", 0.5, max_drift=0.5, n_points=5),
                           st("quantize", 0.5, n_levels=16), st("reverse", 0.5)], I["w1024"], seed=1)
    case("cfg4_mappable", [st("time_warp", n_knots=5, intensity=0.5), st("resize", target_len=1500)],
         I["w1500"], seed=3)
    cfg5 = [st("jitter", .5, sigma=0.05), st("scale", .5, sigma_factor=0.1), st("rotate", .5),
            st("permute_segments", .5, n_segments=4), st("reverse", .5), st("quantize", .5, n_levels=16),
            st("drift", .5, max_drift=0.5, n_points=5),
            st("inject_noise", .5, noise={"kind": "uniform", "half_width": 0.1}),
            st("inject_noise", .5, noise={"kind": "gaussian", "sigma": 0.1}),
            st("inject_noise", .5, noise={"kind": "spike", "count": 5, "magnitude": 2.0}),
            st("inject_noise", .5, noise={"kind": "slope_trend", "max_offset": 0.5}),
            st("time_warp", .5, n_knots=5, intensity=0.5),
            st("time_warp_window", .5, window_size=128, n_knots=4, intensity=0.5)]
    case("cfg5_time_domain", cfg5, I["w1024"], seed=5)
    case("cfg5_full", cfg5[:11] + [st("amplitude_phase_perturb", .5, sigma_amp=0.1, sigma_phase=0.1),
                                    st("frequency_mask", .5, width=51)] + cfg5[11:],
         I["w1024"], seed=5, exact=False)
    cfg5_all = (cfg5[:11] + [st("amplitude_phase_perturb", .5, sigma_amp=0.1, sigma_phase=0.1),
                             st("frequency_mask", .5, width=51)] + cfg5[11:]
                + [st("dropout", .5, rate=0.05), st("pool", .5, size=4), st("convolve", .5, window="hann", size=7),
                   st("random_sinusoid", .5, amplitude=0.5), st("speed_warp", .5, n_speed_change=3,
                                                                max_speed_ratio=3.0)])
    case("cfg5_all20", cfg5_all, I["w1024"], seed=5, exact=False)
    case("cfg5_all20_per_sample", cfg5_all, I["w128"], seed=6, mode="per-sample", exact=False)

    # --- BASELINE-only operators (M2-M6) as reference plugins (oracle/extras_ref.py),
    #     run by the reference's own Pipeline
    case("dropout", [st("dropout", rate=0.05)], I["w1024"])
    case("dropout_half_fill", [st("dropout", 0.5, rate=0.5, fill=-1.0)], I["w100"], seed=4)
    case("dropout_zero", [st("dropout", rate=0.0)], I["w15"])
    case("dropout_all", [st("dropout", rate=1.0, fill=2.5)], I["w7"])
    case("pool_mean4", [st("pool", size=4)], I["w1024"])
    case("pool_mean4_partial", [st("pool", 0.5, size=4)], I["w15"], seed=2)
    case("pool_max5", [st("pool", size=5, reducer="max")], I["w64"])
    case("pool_min3", [st("pool", size=3, reducer="min")], I["w7"])
    case("pool_big", [st("pool", size=40)], I["w15"])
    case("pool_one", [st("pool", size=1)], I["w15"])
    case("convolve_hann7", [st("convolve", window="hann", size=7)], I["w1024"])
    case("convolve_flat4", [st("convolve", window="flat", size=4)], I["w64"])
    case("convolve_triang31", [st("convolve", window="triang", size=31)], I["w100"])
    case("convolve_hamming6", [st("convolve", 0.5, window="hamming", size=6)], I["w15"], seed=3)
    case("convolve_wide", [st("convolve", window="hann", size=25)], I["w7"])
    case("convolve_one", [st("convolve", window="flat", size=1)], I["w15"])
    case("speed_warp", [st("speed_warp", n_speed_change=3, max_speed_ratio=3.0)], I["w1500"])
    case("speed_warp_1024", [st("speed_warp", 0.5, n_speed_change=3, max_speed_ratio=3.0)], I["w1024"])
    case("speed_warp_linear", [st("speed_warp", n_speed_change=7, max_speed_ratio=1.5,
                                  interpolation="linear")], I["w100"])
    case("speed_warp_len2", [st("speed_warp", n_speed_change=3, max_speed_ratio=2.0)], I["w2"])
    case("speed_warp_many", [st("speed_warp", n_speed_change=10, max_speed_ratio=4.0)], I["w7"])
    case("speed_warp_noop", [st("speed_warp", n_speed_change=0)], I["w15"])
    case("sinusoid", [st("random_sinusoid", amplitude=1.0)], I["w1024"], exact=False)
    case("sinusoid_bin0", [st("random_sinusoid", amplitude=0.5, min_bin=0)], I["w64"], exact=False)
    case("sinusoid_odd", [st("random_sinusoid", amplitude=2.0)], I["w15"], exact=False)
    case("sinusoid_zero", [st("random_sinusoid", amplitude=0.0)], I["w64"])
    # --- BASELINE configs 2-5 in full (every stage), through the reference's Pipeline
    case("cfg2_full", [st("crop", size=819), st("drift", 0.5, max_drift=0.5, n_points=5),
                       st("quantize", 0.5, n_levels=16), st("dropout", 0.5, rate=0.05),
                       st("pool", 0.5, size=4), st("reverse", 0.5)], I["w1024"], seed=1)
    case("cfg3_full", [st("frequency_mask", width=102), st("random_sinusoid", amplitude=1.0)], I["ar2048"],
         seed=2, exact=False)
    case("cfg4_full", [st("speed_warp", n_speed_change=3, max_speed_ratio=3.0), st("resize", target_len=1500),
                       st("convolve", window="hann", size=7)], I["w1500"], seed=3)

    # --- transforms (F5)
    for key in ("w1", "w2", "w15", "w64", "w100", "w128", "w1024"):
        sb = ref.fft_forward(ref.Batch(arrays[I[key]]))
        arrays["fftre_" + key], arrays["fftim_" + key] = sb.re, sb.im
        arrays["ifft_" + key] = ref.fft_inverse(sb).values
        cases.append({"name": "fft_" + key, "kind": "fft", "input": I[key],
                      "re": "fftre_" + key, "im": "fftim_" + key, "inverse": "ifft_" + key})
    # --- DCT (next-1: freqtransform.py:91-98)
    for key in ("w1", "w2", "w7", "w15", "w64", "w100", "w1024"):
        db = ref.dct_forward(ref.Batch(arrays[I[key]]))
        arrays["dct_" + key] = db.coeffs
        arrays["idct_" + key] = ref.dct_inverse(db).values
        cases.append({"name": "dct_" + key, "kind": "dct", "input": I[key], "coeffs": "dct_" + key,
                      "inverse": "idct_" + key})
    # --- DTW (next-2: dtw.py:40-106)
    drng = np.random.default_rng(77)
    for q, (n1, n2) in enumerate([(1, 1), (1, 5), (6, 1), (3, 4), (17, 23), (64, 64), (100, 37), (33, 129)]):
        a1 = np.round(drng.normal(0, 2, n1), 1) if q < 4 else drng.normal(0, 1, n1).cumsum()
        b1 = np.round(drng.normal(0, 2, n2), 1) if q < 4 else drng.normal(0, 1, n2).cumsum()
        r = ref.dtw_distance(a1, b1)
        arrays[f"dtw_a{q}"], arrays[f"dtw_b{q}"] = a1, b1
        cases.append({"name": f"dtw_{q}", "kind": "dtw", "a": f"dtw_a{q}", "b": f"dtw_b{q}",
                      "distance": r.distance, "path": [list(p) for p in r.path], "similarity": r.similarity})
    # criterion 10 (test_acceptance.py:334-369): scores recorded as 0.998/0.964/0.901/0.722
    crng = ref.derive_stream(ref.SeedContext(2026))
    n_c, len_c = 24, 128
    tt = np.arange(len_c)
    rows = []
    for _ in range(n_c):
        center = len_c / 2 + crng.normal(0.0, 1.5)
        width = len_c / 8 * (1.0 + 0.15 * crng.normal())
        amp = 2.0 + 0.3 * crng.normal()
        rows.append(amp * np.exp(-0.5 * ((tt - center) / width) ** 2) + 0.05 * crng.normal(0.0, 1.0, len_c))
    base = np.array(rows)
    arrays["crit10_base"] = base
    crit = {}
    for name, rec in (("window_warp", st("time_warp_window", window_size=16, n_knots=4, intensity=0.5)),
                      ("reverse", st("reverse")), ("drift", st("drift", max_drift=0.6, n_points=6)),
                      ("app", st("amplitude_phase_perturb", sigma_amp=5.0, sigma_phase=2.0))):
        aug = ref.stage_from_dict(rec)
        out = aug.augment_batch(ref.Batch(base), 99)
        arrays["crit10_" + name] = out.values
        crit[name] = {"stage": rec, "score": ref.mean_similarity(ref.Batch(base), out)}
    cases.append({"name": "criterion10", "kind": "similarity", "base": "crit10_base", "augmented": crit})
    # --- augment_spectrum (F2)
    for name, rec in (("spec_app", st("amplitude_phase_perturb", sigma_amp=0.5, sigma_phase=0.2)),
                      ("spec_fmask", st("frequency_mask", 0.5, width=7))):
        sb = ref.fft_forward(ref.Batch(arrays[I["w64"]]))
        out = ref.stage_from_dict(rec).augment_spectrum(sb, 9, augmenter_index=2)
        arrays[name + "_re"], arrays[name + "_im"] = out.re, out.im
        cases.append({"name": name, "kind": "spectrum", "stage": rec, "seed": 9, "augmenter_index": 2,
                      "input": I["w64"], "re": name + "_re", "im": name + "_im"})

    # --- single-series known answers from the reference's tests (test_basic.py)
    gate = ref.Jitter(sigma=0.5, probability=0.5).augment_batch(ref.Batch(np.ones((10_000, 8))), 12345)
    fired = int(np.sum(np.any(gate.values != 1.0, axis=1)))

    meta = {
        "numpy": np.__version__,
        "scipy": scipy.__version__,
        "reference": "seriesaug " + ref.__version__,
        "plugins": "oracle/extras_ref.py (BASELINE-only kinds as reference Augmenter subclasses)",
        "gate_pin": {"seed": 12345, "sigma": 0.5, "probability": 0.5, "shape": [10000, 8], "fired": fired},
        "cases": cases,
    }
    np.savez_compressed(os.path.join(HERE, "reference_cases.npz"), **arrays)
    with open(os.path.join(HERE, "reference_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{len(cases)} cases, gate fired {fired}/10000, "
          f"{os.path.getsize(os.path.join(HERE, 'reference_cases.npz')) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
