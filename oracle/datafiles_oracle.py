"""CPU restatement of the reference's dataset formats -- TEST INFRASTRUCTURE ONLY.

May be imported only by tests/ and bench.py's CPU baseline legs, as the
checker / baseline -- never by the product package.

Restates reference datafiles.py:70-143 (parse_dataset / format_dataset) with
Python's own str.splitlines / str.strip / float / repr, which ARE the
reference's number and line semantics; pinned against fixtures produced by
running the reference itself (tests/golden/make_golden_datafiles.py).

Returns plain values instead of DatasetFile objects:
    parse(text, fmt) -> (fmt, headers, labels or None, values (n, L) float64)
and raises ValueError(message) with the reference's exact message text.
"""

from __future__ import annotations

import numpy as np


def parse(text: str, fmt=None):
    # datafiles.py:71-72 -- numbered non-blank lines, stripped
    numbered = [(k + 1, ln.strip()) for k, ln in enumerate(text.splitlines())]
    numbered = [(k, ln) for k, ln in numbered if ln]
    if not numbered:
        raise ValueError("dataset file is empty")
    if fmt is None:  # :74-75 -- '@' on the first non-blank line means TS
        fmt = "ts" if numbered[0][1][:1] == "@" else "csv"
    if fmt not in ("csv", "ts"):
        raise ValueError(f"format must be one of ('csv', 'ts'), got {fmt!r}")
    headers, labels, rows = [], [], []
    width = None
    for k, ln in numbered:  # :84-110
        if fmt == "ts" and ln[:1] == "@":
            if rows:
                raise ValueError(f"line {k}: header after first data row")
            headers.append(ln)
            continue
        if fmt == "ts":
            cut = ln.rfind(":")
            if cut < 0:
                raise ValueError(f"line {k}: missing ':label' separator")
            part, label = ln[:cut], ln[cut + 1:]
            labels.append(label.strip())
        else:
            part = ln
        row = []
        for field in part.split(","):  # :62-67
            try:
                row.append(float(field))
            except ValueError:
                raise ValueError(f"line {k}: not a number: {field.strip()!r}") from None
        if width is None:
            width = (len(row), k)
        elif len(row) != width[0]:
            raise ValueError(f"line {k}: {len(row)} fields, but line {width[1]} has {width[0]}")
        rows.append(row)
    if not rows:
        raise ValueError("dataset file has headers but no data rows")
    values = np.array(rows, dtype=np.float64)
    if not np.isfinite(values).all():  # Batch.__post_init__, core.py:104-105
        raise ValueError("batch contains non-finite values (NaN or Inf)")
    return fmt, tuple(headers), (tuple(labels) if fmt == "ts" else None), values


def format_rows(values, fmt: str = "csv", headers=(), labels=None) -> str:
    """datafiles.py:127-138."""
    lines = list(headers) if fmt == "ts" else []
    if fmt == "ts" and labels is None:
        labels = [""] * len(values)
    for r, row in enumerate(np.asarray(values, dtype=np.float64)):
        body = ",".join(repr(float(v)) for v in row)
        lines.append(body + (":" + labels[r] if fmt == "ts" else ""))
    return "\n".join(lines) + "\n"
