"""Crafted 64-bit word streams for the ziggurat walk (test helper).

numpy's random_standard_normal reads a word w as idx = w & 0xff, sign = bit 8,
rabs = bits 9..60; it is a fast-path normal iff rabs < ki[idx], else a wedge
(idx != 0: the next word is its uniform) or a tail (idx 0: log1p loop).
Real Philox streams are 99.3% fast; these streams raise the slow share so the
parallel window parse meets long slow runs, slow heads on window boundaries
and all-slow lanes.
"""

import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M52 = (1 << 52) - 1


def ki_table() -> np.ndarray:
    src = open(os.path.join(ROOT, "paper_2601_03159_b200", "csrc", "zig_tables.h")).read()
    body = src[src.index("SA_ZIG_KI_DOUBLE_INIT"):]
    body = body[: body.index("}")]
    return np.array([int(v, 16) for v in re.findall(r"0x([0-9a-fA-F]+)ULL", body)], dtype=np.uint64)


def word(idx: int, rabs: int, sign: int) -> int:
    return (idx & 0xFF) | ((sign & 1) << 8) | ((rabs & M52) << 9)


def crafted(n: int, p_slow: float, p_tail: float, seed: int) -> np.ndarray:
    """n words: each is slow with probability p_slow (a tail word with
    probability p_tail of those), else a fast word; a slow word's successor is
    random (it may be consumed as a uniform)."""
    ki = ki_table()
    rng = np.random.default_rng(seed)
    out = np.empty(n, dtype=np.uint64)
    for k in range(n):
        sign = int(rng.integers(0, 2))
        u = rng.random()
        if u < p_slow:
            idx = 0 if rng.random() < p_tail else int(rng.integers(1, 256))
            lo = int(ki[idx])
            rabs = lo + int(rng.integers(0, (M52 + 1) - lo))
        else:
            idx = int(rng.integers(2, 256))
            rabs = int(rng.integers(0, int(ki[idx])))
        out[k] = word(idx, rabs, sign)
    return out


def pattern(spec: str) -> np.ndarray:
    """Deterministic stream from a letter per word: f fast, w wedge (idx 1,
    always slow), t tail (idx 0, rabs max), u a uniform-like word."""
    ki = ki_table()
    rng = np.random.default_rng(len(spec))
    out = []
    for ch in spec:
        if ch == "f":
            out.append(word(7, int(ki[7]) // 3, 0))
        elif ch == "w":
            out.append(word(1, int(rng.integers(0, M52)), int(rng.integers(0, 2))))
        elif ch == "t":
            out.append(word(0, M52, 1))
        else:
            out.append(int(rng.integers(0, 2**63)) * 2 + 1)
    return np.array(out, dtype=np.uint64)
