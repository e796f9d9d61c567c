"""CPU: front-end behaviour that needs no device (argument handling, exit
codes, worker error responses), against the reference's recorded outputs
(tests/golden/frontends_cases.json) and its test suite's expectations
(test_cli.py / test_serve.py / test_bench.py)."""

import io
import json
import os

import numpy as np
import pytest

from paper_2601_03159_b200 import __version__
from paper_2601_03159_b200.bench import power_law_exponent, synthetic_batch, default_chain, measure_peak_memory
from paper_2601_03159_b200.cli import main
from paper_2601_03159_b200.errors import InvalidParameterError
from paper_2601_03159_b200.serve import handle_line, serve_forever

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "frontends_cases.json")


def golden():
    with open(GOLDEN, encoding="utf-8") as fh:
        return json.load(fh)


# the worker's error cases never reach the device
ERROR_IDS = {8, 9, 10, 11, 12, 13, None}


@pytest.mark.parametrize("case", [c for c in golden()["serve"] if json.loads(c["response"])["id"] in ERROR_IDS
                                  or json.loads(c["response"])["result" if json.loads(c["response"])["ok"]
                                                                   else "error"] == {"version": "0.1.0"}],
                         ids=lambda c: c["request"][:30])
def test_worker_errors_match_reference(case):
    got = json.loads(handle_line(case["request"]))
    want = json.loads(case["response"])
    assert got["id"] == want["id"] and got["ok"] == want["ok"]
    if want["ok"]:
        assert got["result"] == want["result"]
        return
    assert got["error"]["type"] == want["error"]["type"]
    if want["error"]["message"].startswith("unknown augmenter kind"):
        # the registry also holds the BASELINE-only kinds (extras.py), so the
        # list of expected kinds is a superset of the reference's
        head = want["error"]["message"].split(", expected")[0]
        assert got["error"]["message"].startswith(head)
        listed = got["error"]["message"].split("expected one of ")[1]
        for kind in json.loads(want["error"]["message"].split("expected one of ")[1].replace("'", '"')):
            assert repr(kind) in listed
    else:
        assert got["error"]["message"] == want["error"]["message"]


def test_serve_forever_skips_blank_lines_and_answers_each():
    src = io.StringIO('{"id": 1, "op": "version"}\n\n   \n{"id": 2, "op": "nope"}\n')
    out = io.StringIO()
    assert serve_forever(src, out) == 0
    replies = [json.loads(x) for x in out.getvalue().splitlines()]
    assert [r["id"] for r in replies] == [1, 2]
    assert replies[0]["result"] == {"version": __version__} and not replies[1]["ok"]


class TestCliNoDevice:
    def test_version(self, capsys):
        with pytest.raises(SystemExit) as exc:
            main(["--version"])
        assert exc.value.code == 0
        assert capsys.readouterr().out.startswith("seriesaug ")

    def test_no_command_usage_error(self):
        with pytest.raises(SystemExit) as exc:
            main([])
        assert exc.value.code == 2

    def test_unknown_transform_usage_error(self, tmp_path):
        with pytest.raises(SystemExit) as exc:
            main(["roundtrip", str(tmp_path / "x.csv"), "wavelet"])
        assert exc.value.code == 2

    def test_missing_input_exits_two(self, tmp_path, capsys):
        rc = main(["augment", str(tmp_path / "nope.csv"), "-o", str(tmp_path / "o.csv")])
        assert rc == 2
        assert "I/O error:" in capsys.readouterr().err
        assert main(["roundtrip", str(tmp_path / "gone.csv"), "fft"]) == 2

    def test_bench_argument_errors(self, tmp_path, capsys):
        assert main(["bench", "--synthetic", "4", "8", "--repeats", "1"]) == 1
        assert "repeats" in capsys.readouterr().err
        p = tmp_path / "d.csv"
        p.write_text("1.0,2.0\n")
        assert main(["bench", str(p), "--synthetic", "4", "8"]) == 1
        assert "exactly one" in capsys.readouterr().err
        assert main(["bench"]) == 1
        assert main(["bench", "--synthetic", "0", "8"]) == 1


class TestBenchHost:
    def test_synthetic_batch_is_the_reference_walk(self):
        b = synthetic_batch(3, 50, seed=4)
        assert b.values.shape == (3, 50)
        assert np.array_equal(b.values, synthetic_batch(3, 50, seed=4).values)
        steps = np.diff(b.values, axis=1)
        assert abs(steps.mean()) < 0.5 and 0.5 < steps.std() < 1.5

    def test_default_chain_shape(self):
        kinds = [s.kind for s in default_chain()]
        assert kinds == ["jitter", "scale", "drift", "time_warp", "amplitude_phase_perturb", "frequency_mask",
                         "reverse"]

    def test_power_law(self):
        assert power_law_exponent([100, 1000, 10000], [1.0, 10.0, 100.0]) == pytest.approx(1.0, abs=1e-12)
        assert power_law_exponent([10, 100, 1000], [1.0, 100.0, 10000.0]) == pytest.approx(2.0, abs=1e-12)
        with pytest.raises(InvalidParameterError):
            power_law_exponent([100], [1.0])

    def test_peak_memory(self):
        assert measure_peak_memory(lambda: None) < 20.0

        def work():
            block = np.ones((100, 1024, 1024), dtype=np.uint8)
            block += 1
            return block.sum()

        assert measure_peak_memory(work) >= 60.0
