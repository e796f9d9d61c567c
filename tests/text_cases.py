"""Seeded number-text cases for the device codec (CPython's repr/float are
the oracle: they ARE the reference's calls, datafiles.py:63,133)."""

from __future__ import annotations

import math
import struct
from decimal import Decimal, getcontext

import numpy as np


def bits_to_f64(u: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(u, dtype=np.uint64).view(np.float64)


def interesting_doubles(n_random: int, seed: int = 0) -> np.ndarray:
    """Random bit patterns over the whole finite range plus the classes that
    stress shortest formatting: subnormals, powers of two and ten and their
    neighbours, integers, short decimals, extremes, signed zero."""
    rng = np.random.default_rng(seed)
    parts = []
    u = rng.integers(0, 2**64, n_random, dtype=np.uint64)
    parts.append(bits_to_f64(u))
    parts.append(bits_to_f64(rng.integers(1, 2**52, n_random // 8, dtype=np.uint64)))  # subnormals
    parts.append(rng.normal(0, 1, n_random // 8))
    parts.append(rng.uniform(0, 1, n_random // 8))
    parts.append(np.round(rng.uniform(-1e6, 1e6, n_random // 8), rng.integers(0, 8)))
    parts.append(rng.integers(-2**53, 2**53, n_random // 16).astype(np.float64))
    p2 = np.ldexp(1.0, np.arange(-1074, 1024))
    parts.append(p2)
    parts.append(np.nextafter(p2, np.inf))
    parts.append(np.nextafter(p2, 0))
    p10 = np.array([float(f"1e{k}") for k in range(-323, 309)])
    parts.append(p10)
    parts.append(np.nextafter(p10, np.inf))
    parts.append(np.nextafter(p10, 0))
    parts.append(np.array([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 2.225073858507201e-308,
                           1.7976931348623157e308, -1.7976931348623157e308, 0.1, 0.2, 0.3, 1 / 3, 2 / 3,
                           1e16, 1e17, 9007199254740993.0, 123456789012345678.0, 1e-4, 1e-5, 0.0001234,
                           1e22, 1e23, 5e-324 * 3, 9.5, 0.5, 1.5, 2.5]))
    x = np.concatenate(parts)
    x = np.concatenate([x, -x])
    return x[np.isfinite(x)]


def _halfway_strings(rng, count: int) -> list[str]:
    """Exact decimal expansions of midpoints between adjacent doubles (round
    half even decides) and their one-unit-in-the-last-digit neighbours."""
    getcontext().prec = 1200
    out = []
    for _ in range(count):
        bits = int(rng.integers(1, 0x7FEFFFFFFFFFFFFF))
        a = struct.unpack("<d", struct.pack("<Q", bits))[0]
        b = math.nextafter(a, math.inf)
        mid = (Decimal(a) + Decimal(b)) / 2
        s = format(mid, "f") if abs(mid.adjusted()) < 30 else format(mid, "e")
        out.append(s)
        k = int(rng.integers(17, 40))
        digits = format(mid, f".{k}e")
        out.append(digits)
    return out


def decimal_strings(n: int, seed: int = 1) -> list[str]:
    """Random float() inputs: 1-60 digits, exponents across the whole range
    and beyond, signs, '.', 'e'/'E', '_' separators, padding."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        nd = int(rng.integers(1, 60)) if rng.random() < 0.3 else int(rng.integers(1, 20))
        digits = "".join(str(int(d)) for d in rng.integers(0, 10, nd))
        if rng.random() < 0.2:
            digits = "0" * int(rng.integers(1, 30)) + digits
        pos = int(rng.integers(0, nd + 1))
        mant = digits[:pos] + "." + digits[pos:] if rng.random() < 0.7 else digits
        if mant in (".",):
            mant = "0."
        e = ""
        if rng.random() < 0.8:
            ex = int(rng.integers(-360, 330))
            e = ("e" if rng.random() < 0.5 else "E") + (("+" if rng.random() < 0.3 else "") if ex >= 0 else "") \
                + str(ex)
        sign = ["", "-", "+"][int(rng.integers(0, 3))]
        out.append(sign + mant + e)
    return out


def underscore_and_odd_strings() -> list[str]:
    base = ["1_0", "1_000.000_1", "1e1_0", "1_0e-1_0", "_1", "1_", "1__0", "1_.0", "1._0", "1e_1", "1_e1",
            "0_0", "in_f", "1.", ".5", "1.e5", ".e5", ".", "", " ", "e5", "1e", "1e+", "-", "+", "--1", "+-1",
            "1.2.3", "0x10", "1e5.5", "nan", "NaN", "-nan", "+nan", "inf", "-inf", "+Inf", "infinity", "-Infinity",
            "iNfInItY", "infinit", "nan(1)", "nanx", "1\x00", " 1 ", "\t1\n", "\x0b1\x0c", "1\x1f", "\x1c1",
            "1 2", "1\xa0", " 1", "1　", "١٢", "١.٢e٣", "１２",
            "١_٢", "1²", "½", "1 ", "x", "1e999999999999", "-1e999999999999",
            "1e-999999999999", "0e999999999999", "0." + "0" * 400 + "1e400", "1" + "0" * 400 + "e-400",
            "4.9406564584124654e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
            "2.2250738585072011e-308", "2.2250738585072012e-308", "1.7976931348623157e308",
            "1.7976931348623158e308", "1.7976931348623159e308", "179769313486231580793728971405301e276",
            "9007199254740993", "9007199254740992.5", "9007199254740993.0000000000000000000001",
            "0.1", "-0", "-0.0", "+0e-5", "00000000000000000000000000001", "1" * 800, "0." + "9" * 800,
            "1.00000000000000011102230246251565404236316680908203125",
            "1.00000000000000011102230246251565404236316680908203124",
            "1.00000000000000011102230246251565404236316680908203126",
            "7.2057594037927933e16", "7.2057594037927932e16", "3.5e-324", "2.5e-324"]
    return base


def parse_cases(n: int, seed: int = 3) -> list[str]:
    rng = np.random.default_rng(seed)
    vals = interesting_doubles(max(8, n // 4), seed)
    reprs = [repr(float(v)) for v in vals[: n // 2]]
    return reprs + decimal_strings(n // 2, seed) + _halfway_strings(rng, max(1, n // 40)) \
        + underscore_and_odd_strings()


def py_float(s: str):
    try:
        return float(s), True
    except ValueError:
        return 0.0, False


# ------------------------------------------------------------------ datasets
_BREAKS = ["\n"] * 8 + ["\r\n", "\r", "\x0b", "\x0c", "\x1c", "\x1d", "\x1e", "\x85", "\u2028", "\u2029"]
_PADS = ["", "", "", " ", "\t", "  ", "\xa0", "\u3000", "\u2003"]
_LABELS = ["a", "b", "class 1", "", "  spaced  ", "\u03bb", "\u65e5\u672c", "x,y", "7"]


def _field_text(rng, v: float) -> str:
    r = rng.random()
    if r < 0.6:
        s = repr(float(v))
    elif r < 0.75:
        s = "%.17g" % v
    elif r < 0.85:
        s = "%.6e" % v
    elif r < 0.9:
        s = "%.3f" % v
    elif r < 0.95 and abs(v) >= 1000 and float(int(v)) == v:
        s = f"{int(v):_}"
    else:
        s = repr(float(v)).upper()
    if rng.random() < 0.05:
        s = _PADS[int(rng.integers(0, len(_PADS)))] + s + _PADS[int(rng.integers(0, len(_PADS)))]
    return s


def random_dataset(seed: int, n: int, L: int, ts: bool):
    """(text, values, labels, headers): a valid dataset with mixed number
    spellings, padding, blank lines and every str.splitlines() break;
    values are float() of the spelled fields."""
    rng = np.random.default_rng(seed)
    pool = interesting_doubles(2000, seed)
    pool = pool[np.abs(pool) < 1e300]  # '%.3f' of huge values stays finite
    values = pool[rng.integers(0, len(pool), (n, L))]
    spelled = [[_field_text(rng, v) for v in row] for row in values]
    values = np.array([[float(f) for f in row] for row in spelled], dtype=np.float64).reshape(n, L)
    headers = [f"@problemName set{seed}", "@timeStamps false", "@data"] if ts else []
    labels = [_LABELS[int(rng.integers(0, len(_LABELS)))] for _ in range(n)] if ts else None
    lines = list(headers)
    for r in range(n):
        body = ",".join(spelled[r])
        if ts:
            body += ":" + labels[r]
        lines.append(body)
        if rng.random() < 0.05:
            lines.append(_PADS[int(rng.integers(0, len(_PADS)))])
    text = ""
    for ln in lines:
        text += ln + _BREAKS[int(rng.integers(0, len(_BREAKS)))]
    if rng.random() < 0.3:
        text = text.rstrip("\n")
    return text, values, labels, headers


def corrupt_dataset(text: str, seed: int) -> str:
    """One random corruption (bad number, ragged row, late header, missing
    label separator, non-finite value) at a random line."""
    rng = np.random.default_rng(seed)
    lines = text.split("\n")
    k = int(rng.integers(0, len(lines)))
    kind = int(rng.integers(0, 6))
    ln = lines[k]
    if kind == 0 and "," in ln:
        parts = ln.split(",")
        j = int(rng.integers(0, len(parts)))
        parts[j] = ["zz", "", "1..2", "1e", "--1", "0x1p3", "1_", "١x"][int(rng.integers(0, 8))]
        ln = ",".join(parts)
    elif kind == 1 and "," in ln:
        ln = ln.replace(",", "", 1)
    elif kind == 2:
        ln = ln + ",1.5"
    elif kind == 3:
        ln = "@late header"
    elif kind == 4:
        ln = ln.replace(":", ";")
    else:
        ln = ln.replace(",", ",inf,", 1) if rng.random() < 0.5 else ln.replace(",", ",1e999,", 1)
    lines[k] = ln
    return "\n".join(lines)
