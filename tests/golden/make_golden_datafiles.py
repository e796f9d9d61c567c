"""Generate tests/golden/datafiles_cases.json by running the REFERENCE's
parse_dataset / format_dataset (datafiles.py:70-143) in this container.

    python tests/golden/make_golden_datafiles.py

Each parse case stores the input text, the forced format (or null), and
either the parsed result (format, header lines, labels, values as float hex
strings) or the reference's exact error message.  Each format case stores a
batch (float hex) with format/headers/labels and the reference's text.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def hexrows(values):
    return [[float(v).hex() for v in row] for row in np.asarray(values)]


def parse_cases():
    rng = np.random.default_rng(7)
    walk = np.cumsum(rng.normal(0, 1, (6, 9)), axis=1)
    csv_walk = "\n".join(",".join(repr(float(v)) for v in row) for row in walk) + "\n"
    ts_walk = "@problemName walk\n@timeStamps false\n@classLabel true a b\n@data\n" + "\n".join(
        ",".join(repr(float(v)) for v in row) + (":a" if r % 2 else ":b") for r, row in enumerate(walk)) + "\n"
    cases = [
        ("1.0,2.0,3.0\n4.0,5.5,-6.0\n", None),
        ("@problemName toy\n@timeStamps false\n@data\n1.0,2.0,3.0:a\n4.0,5.5,-6.0:b\n", None),
        ("1.0,2.0\n\n3.0,4.0\n\n", None),
        (" 1.0 , 2.0 \n3.0,4.0\n", None),
        ("1.0,2.0\n1.0,oops\n", None),
        ("1.0,2.0,3.0\n1.0,2.0\n", None),
        ("", None),
        ("\n\n", None),
        ("   \n\t\n", None),
        ("@data\n1.0,2.0:my label\n", None),
        ("@data\n1.0:2.0:x\n", None),
        ("@data\n1.0,2.0\n", None),
        ("@data\n1.0:a\n@late true\n", None),
        ("@data\n", None),
        ("@a\n@b\n\n", None),
        (csv_walk, None),
        (ts_walk, None),
        (csv_walk, "ts"),
        (ts_walk, "csv"),
        ("1,2\n3,4\n", "parquet"),
        ("", "parquet"),
        ("1.0,2.0\r\n3.0,4.0\r\n", None),
        ("1.0,2.0\r3.0,4.0\r", None),
        ("1.0,2.0\x0b3.0,4.0\x0c5,6\x1c7,8\x1d9,10\x1e11,12", None),
        ("1.0,2.0\x853.0,4.0\u20285,6\u20297,8\n", None),
        ("1.0,2.0\n3.0,4.0", None),
        ("\xa0 1.0,2.0\u3000\n3.0,4.0\u2003\n", None),
        ("1.0,2.0\x1f\n3.0,4.0\n", None),
        ("1.0,\x1f2.0\n3.0,4.0\n", None),
        ("1_0,2e1_0\n3.,.5\n", None),
        ("\u0661\u0662,\u0663\n1,2\n", None),
        ("1,2\n3,inf\n", None),
        ("1,2\n3,nan\n", None),
        ("1,2\n3,1e400\n", None),
        ("1,2\n3,-0.0\n", None),
        ("1,,2\n", None),
        (",\n", None),
        ("1,2,\n", None),
        ("@data\n1,2:\n3,4:  spaced label  \n", None),
        ("@data\n1,2:a:b\n", None),
        ("@data\n1,2:a,b\n3,4:c\n", None),
        ("@data\n1,2 :a\n3 , 4: b\n", None),
        ("@data\n:a\n", None),
        ("@data\n1,2:x\n1,2,3:y\n", None),
        ("@data\n1,2:x\n1,zz:y\n1:y\n", None),
        ("@data\n1,2:x\n1,2,3:y\n@h\n", None),
        ("@data\n1,2:x\n1,2\n", None),
        ("@data\n1,2:x\nzz\n", None),
        ("1,2\n@x\n", None),
        ("@x\n1,2\n", "csv"),
        ("1,2:a\n", "ts"),
        ("@data\n1,2:\u03bb label\n3,4:\u65e5\u672c\n", None),
        ("x,1\n", None),
        ("1.5e-324,2\n", None),
        ("0.1," + "9" * 400 + "\n", None),
        ("2.4703282292062327e-324,2.4703282292062328e-324\n", None),
        ("1,2\n3,4\n5,6,7\n8\n", None),
        ("1;2\n", None),
        ("\ufeff1,2\n", None),
        ("1 2,3\n", None),
        ("+1,-2\n", None),
        ("  @data\n 1,2:a\n", None),
        ("@data\n\n\n1,2:a\n\n", None),
        ("1,2\n" * 50, None),
    ]
    return cases


def format_cases():
    rng = np.random.default_rng(8)
    out = []
    b = rng.normal(0, 1, (5, 9))
    out.append((b, "csv", (), None))
    out.append((b, "ts", ("@problemName x", "@data"), tuple("pqrst")))
    out.append((b, "ts", (), None))
    out.append((np.array([[0.1, 1e-300, 1.7976931348623157e308, -0.0, 5e-324, 1e16, 1e17, 123.0, 1e-5]]), "csv",
                (), None))
    out.append((np.array([[1.0, 2.0], [3.0, 4.0]]), "ts", ("@h",), ("\u03bb", "")))
    out.append((rng.integers(-1000, 1000, (3, 4)).astype(np.float64), "csv", (), None))
    return out


def main():
    sys.path.insert(0, REF)
    import seriesaug
    from seriesaug import Batch, DatasetFile, InvalidInputError, format_dataset, parse_dataset

    parse_out = []
    for text, fmt in parse_cases():
        rec = {"text": text, "fmt": fmt}
        try:
            ds = parse_dataset(text, fmt)
            rec.update(ok=True, format=ds.format, headers=list(ds.header_lines),
                       labels=None if ds.labels is None else list(ds.labels), values=hexrows(ds.batch.values))
        except InvalidInputError as exc:
            rec.update(ok=False, error=str(exc))
        parse_out.append(rec)
    fmt_out = []
    for values, fmt, headers, labels in format_cases():
        ds = DatasetFile(batch=Batch(values), format=fmt, header_lines=headers, labels=labels)
        fmt_out.append({"values": hexrows(values), "format": fmt, "headers": list(headers),
                        "labels": None if labels is None else list(labels), "text": format_dataset(ds)})
    doc = {"generator": "tests/golden/make_golden_datafiles.py", "reference": "seriesaug " +
           getattr(seriesaug, "__version__", "?"), "parse": parse_out, "format": fmt_out}
    with open(os.path.join(HERE, "datafiles_cases.json"), "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=1, ensure_ascii=True)
        fh.write("\n")
    print(len(parse_out), "parse cases,", len(fmt_out), "format cases")


if __name__ == "__main__":
    main()
