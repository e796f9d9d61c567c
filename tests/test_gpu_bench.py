"""The driver's bench.py contract: one JSON line per arm with every key the
round-end harness reads (metric / value / roofline / cpu_baseline / e2e /
clocks / gpu_launches), on a small config so the test stays quick."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--config", "2", "--steps", "3", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0 and d["higher_is_better"]
    assert d["config"]["workload"] and d["dtype"] == "f64" and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 10_000 * 1024 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("port", "reference") and c["sample"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--config", "2", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_two_ranks_shard_bitwise(tmp_path):
    """`bench.py --gpus 2` launches its own two ranks (no torchrun env), each
    on its contiguous series range with its global series_offset; here both
    ranks share cuda:0 and synchronise over gloo (no kernel waits on another
    rank: the ranks only meet at the barrier and the max-reduce).  The two
    shards concatenated must equal the single-rank output bit for bit."""
    env = dict(os.environ, SA_BENCH_DEVICE="0", SA_BENCH_BACKEND="gloo")
    common = ["--config", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"]

    def run(n, d):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), *common,
                              "--check-out", str(d)], cwd=ROOT, capture_output=True, text=True, timeout=600,
                             env=env)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, out.stdout
        return json.loads(lines[0])

    import numpy as np

    one = run(1, tmp_path / "one")
    two = run(2, tmp_path / "two")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["n_series"] == one["config"]["n_series"] == 10_000
    a = np.load(tmp_path / "one" / "rank0_of1.npy")
    b = np.concatenate([np.load(tmp_path / "two" / f"rank{r}_of2.npy") for r in range(2)])
    assert a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
