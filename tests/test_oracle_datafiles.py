"""CPU: the dataset-format oracle pinned against the reference's own outputs
(tests/golden/datafiles_cases.json, made by make_golden_datafiles.py), and
the host-side DatasetFile logic (reference test_datafiles.py TestWithBatch /
TestValidation)."""

import json
import os

import numpy as np
import pytest

from oracle import datafiles_oracle as O
from paper_2601_03159_b200 import Batch, DatasetFile, InvalidInputError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "datafiles_cases.json")


def golden():
    with open(GOLDEN, encoding="utf-8") as fh:
        return json.load(fh)


def unhex(rows):
    return np.array([[float.fromhex(v) for v in row] for row in rows], dtype=np.float64)


@pytest.mark.parametrize("case", golden()["parse"], ids=lambda c: repr(c["text"][:24]))
def test_oracle_parse_matches_reference(case):
    if case["ok"]:
        fmt, headers, labels, values = O.parse(case["text"], case["fmt"])
        assert fmt == case["format"]
        assert list(headers) == case["headers"]
        assert (None if labels is None else list(labels)) == case["labels"]
        want = unhex(case["values"])
        assert values.shape == want.shape
        assert np.array_equal(values.view(np.uint64), want.view(np.uint64))
    else:
        with pytest.raises(ValueError) as exc:
            O.parse(case["text"], case["fmt"])
        assert str(exc.value) == case["error"]


@pytest.mark.parametrize("case", golden()["format"], ids=lambda c: c["format"])
def test_oracle_format_matches_reference(case):
    text = O.format_rows(unhex(case["values"]), case["format"], case["headers"], case["labels"])
    assert text == case["text"]


def test_random_datasets_round_trip_in_oracle():
    from text_cases import random_dataset

    for seed in range(20):
        text, values, labels, headers = random_dataset(seed, 7, 5, ts=bool(seed % 2))
        fmt, h, lab, v = O.parse(text)
        assert fmt == ("ts" if seed % 2 else "csv")
        assert np.array_equal(v.view(np.uint64), values.view(np.uint64))
        if labels is not None:
            assert list(lab) == [x.strip() for x in labels]


class TestDatasetFileHost:
    """Pure host logic, mirrors reference test_datafiles.py:127-170."""

    def ds(self):
        return DatasetFile(batch=Batch(np.arange(6.0).reshape(2, 3)), format="ts", labels=("a", "b"))

    def test_same_count_keeps_labels(self):
        out = self.ds().with_batch(Batch(np.zeros((2, 3))))
        assert out.labels == ("a", "b") and out.format == "ts"

    def test_repeat_replicates_labels(self):
        out = self.ds().with_batch(Batch(np.zeros((6, 3))))
        assert out.labels == ("a", "a", "a", "b", "b", "b")

    def test_non_multiple_growth_rejected(self):
        with pytest.raises(InvalidInputError):
            self.ds().with_batch(Batch(np.zeros((5, 3))))

    def test_csv_growth_needs_no_labels(self):
        ds = DatasetFile(batch=Batch(np.zeros((2, 3))), format="csv")
        assert ds.with_batch(Batch(np.zeros((6, 3)))).labels is None

    def test_label_count_mismatch(self):
        with pytest.raises(InvalidInputError, match="1 labels for 2 series"):
            DatasetFile(batch=Batch(np.zeros((2, 3))), format="ts", labels=("only-one",))

    def test_unknown_format(self):
        with pytest.raises(InvalidInputError, match="format must be one of"):
            DatasetFile(batch=Batch(np.zeros((1, 2))), format="parquet")

    def test_csv_headers_rejected(self):
        with pytest.raises(InvalidInputError, match="csv datasets carry no header lines or labels"):
            DatasetFile(batch=Batch(np.zeros((1, 2))), format="csv", header_lines=("@x",))
