"""Front ends on the device backend vs the reference's recorded CLI and
worker outputs (tests/golden/frontends_cases.json)."""

import contextlib
import io
import json
import os

import numpy as np
import pytest

from oracle import datafiles_oracle as O
from sa_testutil import spectral_tol

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "frontends_cases.json")
FFT_KINDS = {"frequency_mask", "amplitude_phase_perturb"}


def golden():
    with open(GOLDEN, encoding="utf-8") as fh:
        return json.load(fh)


def run(argv):
    from paper_2601_03159_b200.cli import main

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("case", golden()["augment"],
                         ids=lambda c: f"{c['format_hint']}-{'default' if c['config'] is None else len(c['config']['stages'])}-{'_'.join(c['flags'])}")
def test_augment_matches_reference(case, tmp_path):
    src = tmp_path / f"in.{case['format_hint']}"
    src.write_text(case["input"])
    argv = ["augment", str(src), "-o", str(tmp_path / "out")] + case["flags"]
    exact = True
    if case["config"] is not None:
        cfg = tmp_path / "c.json"
        cfg.write_text(json.dumps(case["config"]))
        argv += ["--config", str(cfg)]
        exact = not any(s["kind"] in FFT_KINDS for s in case["config"]["stages"])
    else:
        exact = False  # default chain: APP + frequency mask
    rc, _, err = run(argv)
    assert rc == case["rc"], err
    got = (tmp_path / "out").read_text()
    if exact:
        assert got == case["output"]
    else:
        g, w = O.parse(got), O.parse(case["output"])
        assert g[:3] == w[:3]
        assert g[3].shape == w[3].shape
        assert np.abs(g[3] - w[3]).max() <= spectral_tol(w[3])


def test_augment_error_message(tmp_path):
    case = golden()["errors"][0]
    bad = tmp_path / "bad.csv"
    bad.write_text(case["input"])
    rc, _, err = run(["augment", str(bad), "-o", str(tmp_path / "o")])
    assert rc == case["rc"]
    assert err == case["stderr"].replace("TMP", str(tmp_path))


@pytest.mark.parametrize("k", range(3))
def test_quality_matches_reference(k, tmp_path):
    case = golden()["quality"][k]
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    a.write_text(case["a"])
    b.write_text(case["b"])
    rc, out, _ = run(["quality", str(a), str(b)])
    assert rc == case["rc"]
    assert out == case["stdout"]


@pytest.mark.parametrize("case", [c for c in golden()["serve"] if json.loads(c["response"])["ok"]],
                         ids=lambda c: c["request"][:40])
def test_worker_matches_reference(case):
    from paper_2601_03159_b200.serve import handle_line

    assert json.loads(handle_line(case["request"])) == json.loads(case["response"])


def test_roundtrip_and_bench_commands(tmp_path):
    rng = np.random.default_rng(0)
    p = tmp_path / "in.csv"
    p.write_text(O.format_rows(rng.normal(0, 1, (6, 20))))
    for transform in ("fft", "dct"):
        rc, out, _ = run(["roundtrip", str(p), transform])
        assert rc == 0 and float(out.strip()) <= 1e-8
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"stages": [{"kind": "jitter", "params": {"sigma": 0.1}},
                                          {"kind": "reverse", "params": {}}]}))
    rc, out, err = run(["bench", "--synthetic", "16", "32", "--config", str(cfg)])
    assert rc == 0
    doc = json.loads(out)
    assert doc["dataset_name"] == "synthetic-16x32" and doc["n_series"] == 16 and doc["series_len"] == 32
    assert doc["repeats"] == 3 and len(doc["stages"]) == 2 and "pipeline median" in err
    rep = tmp_path / "rep.csv"
    assert run(["bench", str(p), "--config", str(cfg), "--report", str(rep)])[0] == 0
    assert len(rep.read_text().strip().splitlines()) == 1 + 2 + 1


def test_ts_labels_and_repeat_through_cli(tmp_path):
    from paper_2601_03159_b200 import read_dataset

    src = tmp_path / "in.ts"
    src.write_text("@problemName toy\n@data\n1.0,2.0,3.0:a\n4.0,5.0,6.0:b\n")
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"stages": [{"kind": "reverse", "params": {}}, {"kind": "repeat",
                                                                           "params": {"r": 2}}]}))
    assert run(["augment", str(src), "-o", str(tmp_path / "o.ts"), "--config", str(cfg)])[0] == 0
    ds = read_dataset(tmp_path / "o.ts")
    assert ds.labels == ("a", "a", "b", "b") and ds.header_lines == ("@problemName toy", "@data")
    assert np.array_equal(ds.batch.values[0], [3.0, 2.0, 1.0])
