"""Device dataset codec vs the reference (golden fixtures) and vs the oracle
(random datasets and corruptions): same values bit for bit, same labels and
header lines, same first error message."""

import json
import os

import numpy as np
import pytest

from oracle import datafiles_oracle as O
from text_cases import corrupt_dataset, random_dataset

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "datafiles_cases.json")


def golden():
    with open(GOLDEN, encoding="utf-8") as fh:
        return json.load(fh)


def unhex(rows):
    return np.array([[float.fromhex(v) for v in row] for row in rows], dtype=np.float64)


def same_bits(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def outcome_device(text, fmt=None):
    from paper_2601_03159_b200 import InvalidInputError, parse_dataset

    try:
        ds = parse_dataset(text, fmt)
    except InvalidInputError as exc:
        return ("err", str(exc))
    return ("ok", ds.format, tuple(ds.header_lines), ds.labels, ds.batch.values)


def outcome_oracle(text, fmt=None):
    try:
        fmt, headers, labels, values = O.parse(text, fmt)
    except ValueError as exc:
        return ("err", str(exc))
    return ("ok", fmt, tuple(headers), labels, values)


def assert_same(got, want, what=""):
    assert got[0] == want[0], (what, got[:2], want[:2])
    if got[0] == "err":
        assert got[1] == want[1], what
    else:
        assert got[1:4] == want[1:4], what
        assert same_bits(got[4], want[4]), what


@pytest.mark.parametrize("case", golden()["parse"], ids=lambda c: repr(c["text"][:24]))
def test_parse_matches_reference(case):
    got = outcome_device(case["text"], case["fmt"])
    if case["ok"]:
        want = ("ok", case["format"], tuple(case["headers"]),
                None if case["labels"] is None else tuple(case["labels"]), unhex(case["values"]))
    else:
        want = ("err", case["error"])
    assert_same(got, want)


@pytest.mark.parametrize("case", golden()["format"], ids=lambda c: c["format"])
def test_format_matches_reference(case):
    from paper_2601_03159_b200 import Batch, DatasetFile, format_dataset

    ds = DatasetFile(batch=Batch(unhex(case["values"])), format=case["format"],
                     header_lines=tuple(case["headers"]),
                     labels=None if case["labels"] is None else tuple(case["labels"]))
    assert format_dataset(ds) == case["text"]


@pytest.mark.parametrize("seed", range(40))
def test_random_datasets_match_oracle(seed):
    ts = bool(seed % 2)
    n, L = [(1, 1), (3, 7), (40, 33), (200, 5), (7, 300)][seed % 5]
    text, values, labels, headers = random_dataset(seed, n, L, ts)
    got, want = outcome_device(text), outcome_oracle(text)
    assert want[0] == "ok"
    assert_same(got, want, seed)
    assert same_bits(got[4], values)


@pytest.mark.parametrize("seed", range(60))
def test_corrupted_datasets_same_first_error(seed):
    text, *_ = random_dataset(1000 + seed, 30, 6, ts=bool(seed % 3 == 0))
    bad = corrupt_dataset(text, seed)
    assert_same(outcome_device(bad), outcome_oracle(bad), seed)


def test_large_dataset_round_trip():
    """Size-independent property at scale: format -> parse is the identity
    (bitwise) and the text equals the oracle's formatting."""
    import torch

    from paper_2601_03159_b200 import format_dataset_device, parse_dataset_device

    rng = np.random.default_rng(5)
    x = np.cumsum(rng.normal(0, 1, (2000, 1024)), axis=1)
    labels = tuple(f"c{r % 7}" for r in range(2000))
    data = format_dataset_device(torch.from_numpy(x).cuda(), "ts", ("@problemName big", "@data"), labels)
    assert data.decode() == O.format_rows(x, "ts", ("@problemName big", "@data"), labels)
    dd = parse_dataset_device(data)
    assert dd.format == "ts" and dd.labels == labels and dd.header_lines == ("@problemName big", "@data")
    assert same_bits(dd.values.cpu().numpy(), x)


def test_file_io_and_read_error_names_path(tmp_path):
    from paper_2601_03159_b200 import Batch, DatasetFile, InvalidInputError, read_dataset, write_dataset

    b = Batch(np.random.default_rng(2).normal(0, 1, (3, 5)))
    path = tmp_path / "data.csv"
    write_dataset(path, DatasetFile(batch=b, format="csv"))
    assert read_dataset(path).batch == b
    bad = tmp_path / "bad.csv"
    bad.write_text("1.0,zzz\n")
    with pytest.raises(InvalidInputError, match=r"bad\.csv: line 1: not a number: 'zzz'"):
        read_dataset(bad)


def test_invalid_utf8_raises_decode_error(tmp_path):
    from paper_2601_03159_b200 import read_dataset

    p = tmp_path / "x.csv"
    p.write_bytes(b"1.0,2.0\n3.0,\xff4.0\n")
    with pytest.raises(UnicodeDecodeError) as exc:
        read_dataset(p)
    with pytest.raises(UnicodeDecodeError) as ref:
        open(p, encoding="utf-8").read()
    assert str(exc.value) == str(ref.value)
    for blob in (b"\xc0\x80", b"\xed\xa0\x80", b"\xf4\x90\x80\x80", b"\xe2\x82", b"\x80", b"\xf0\x9f\x98"):
        p.write_bytes(b"1,2:" + blob + b"\n")
        with pytest.raises(UnicodeDecodeError):
            read_dataset(p)
    p.write_bytes("@data\n1,2:\U0001f600 ok\n".encode())
    assert read_dataset(p).labels == ("\U0001f600 ok",)


def test_augment_file_matches_host_flow(tmp_path):
    """The device-resident augment flow (cli.py:48-54) writes the same bytes
    as read_dataset -> Pipeline.run -> write_dataset."""
    import bench_inputs
    from paper_2601_03159_b200 import (Batch, DatasetFile, Repeat, Pipeline, augment_file, read_dataset,
                                       write_dataset)

    x = bench_inputs.host_input(2, 300)
    labels = tuple(f"k{r % 3}" for r in range(300))
    src = tmp_path / "in.ts"
    write_dataset(src, DatasetFile(batch=Batch(x), format="ts", header_lines=("@data",), labels=labels))
    pipe = bench_inputs.pipeline(2)
    pipe = Pipeline(stages=pipe.stages + (Repeat(2),), master_seed=pipe.master_seed)
    augment_file(src, tmp_path / "dev.ts", pipe)
    ds = read_dataset(src)
    write_dataset(tmp_path / "host.ts", ds.with_batch(pipe.run(ds.batch)))
    assert (tmp_path / "dev.ts").read_bytes() == (tmp_path / "host.ts").read_bytes()
