"""Pin the C oracle's numpy-compatible streams against numpy itself.

The reference draws everything through np.random.Generator(Philox) (reference
core.py:71-82); these tests check our restatement of that third-party
arithmetic (numpy 2.3.5) bit for bit: raw words, random(), the ziggurat
normal (all three paths), Lemire integers with numpy's buffered 32-bit half,
permutation, choice (Floyd and tail shuffle), pairwise summation and std.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

MASK = (1 << 64) - 1
G = 0x9E3779B97F4A7C15


def mix(z):
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return (z ^ (z >> 31)) & MASK


def ref_key(seed, j, i):  # restates reference core.py:77-82
    s = mix(seed)
    s = mix((s + G + j) & MASK)
    s = mix((s + G + i) & MASK)
    return mix(s), mix((s + G) & MASK)


def gen(seed, j, i):
    lo, hi = ref_key(seed, j, i)
    return np.random.Generator(np.random.Philox(key=lo | (hi << 64)))


CTX = [(0, 0, 0), (7, 3, 11), (2**64 - 1, 17, 123456789), (12345, 0, 9999)]


@pytest.mark.parametrize("ctx", CTX)
def test_key_and_raw_words(ctx):
    assert O.derive_key(*ctx) == ref_key(*ctx)
    assert np.array_equal(O.raw(*ctx, 37), gen(*ctx).bit_generator.random_raw(37))


@pytest.mark.parametrize("ctx", CTX)
def test_doubles(ctx):
    assert np.array_equal(O.doubles(*ctx, 1001), gen(*ctx).random(1001))


@pytest.mark.parametrize("seed", range(6))
def test_normals_bitwise_all_paths(seed):
    # 300k normals cover ~80 tail and ~2000 wedge evaluations per seed
    z = gen(seed, 1, 2).normal(0.0, 1.0, 300_000)
    assert np.array_equal(O.normals(seed, 1, 2, 300_000), z)
    assert np.array_equal(O.normals(seed, 1, 2, 500, 0.5, 0.1), gen(seed, 1, 2).normal(0.5, 0.1, 500))


def test_mixed_draw_script():
    """32-bit draws share numpy's buffered upper half across 64-bit draws."""
    rng = np.random.default_rng(0)
    for trial in range(40):
        ops = rng.integers(0, 4, 60)
        args = rng.integers(1, 3000, 60)
        args[rng.random(60) < 0.1] = 1  # integers(0, 1): no draw
        g = gen(trial, 2, 5)
        want = []
        for op, a in zip(ops, args):
            if op == 0:
                want.append(g.random())
            elif op == 1:
                want.append(g.standard_normal())
            elif op == 2:
                want.append(float(g.integers(0, a)))
            else:
                want.append(float(g.integers(0, 2**32, dtype=np.uint64)))
        got = O.script(trial, 2, 5, ops, args)
        assert np.array_equal(got, np.array(want)), trial


def test_integers_rejection_branch():
    """Bounds close to 2^32 exercise Lemire's rejection loop."""
    for bound in (3_000_000_000, 2**32 - 7, 4_000_000_001):
        g = gen(9, 9, bound)
        want = [float(g.integers(0, bound)) for _ in range(300)]
        got = O.script(9, 9, bound, np.full(300, 2), np.full(300, bound))
        assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 17, 64, 1000])
def test_permutation(n):
    for s in range(5):
        assert np.array_equal(O.permutation(s, 4, n, n), gen(s, 4, n).permutation(n))


@pytest.mark.parametrize("pop,k", [(10, 0), (10, 3), (10, 10), (1024, 40), (1024, 1024),
                                   (9000, 500), (12000, 200), (12000, 241), (20000, 900)])
def test_choice_floyd_and_tail(pop, k):
    for s in range(3):
        want = gen(s, 6, pop).choice(pop, size=k, replace=False)
        assert np.array_equal(O.choice(s, 6, pop, pop, k), want)


def test_pairwise_sum_and_std():
    rng = np.random.default_rng(3)
    for n in list(range(1, 40)) + [127, 128, 129, 255, 256, 1000, 1024, 2900, 5000]:
        a = rng.normal(0, 1, n) * 10 ** rng.uniform(-3, 3)
        assert O.pairwise_sum(a) == np.sum(a)
        assert O.std(a) == a.std()


def test_ziggurat_tables_match_numpy():
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(here, "tools", "gen_ziggurat_tables.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("ctx", CTX)
def test_normals_on_word_stream_hook(ctx):
    # the crafted-stream hook (tests/test_gpu_rng_probe.py) reads words from an
    # array: on the Philox words of a stream it must give that stream's normals
    raw = O.raw(*ctx, 50_000)
    z, pos = O.normals_words(raw, 40_000)
    assert np.array_equal(z, O.normals(*ctx, 40_000)) and pos < raw.size


def test_crafted_stream_classes():
    from zig_streams import crafted, ki_table

    ki = ki_table()
    assert ki.size == 256 and ki[1] == 0
    w = crafted(4000, 0.5, 0.2, seed=1)
    idx = (w & np.uint64(0xFF)).astype(np.int64)
    rabs = (w >> np.uint64(9)) & np.uint64((1 << 52) - 1)
    slow = rabs >= ki[idx]
    assert 0.45 < slow.mean() < 0.55 and (slow & (idx == 0)).sum() > 200
