"""Pipeline.capture_device: the fused chain captured in a CUDA graph.

Replays must equal eager run_device results bitwise on the captured buffers
(refilled in place between replays), and the device flags must still raise
the reference's InvalidInputError for non-finite data (core.py:104-105).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _pipe():
    from paper_2601_03159_b200 import Crop, Drift, Dropout, Jitter, Pipeline, Pool, Quantize, Reverse

    return Pipeline(stages=(Crop(200), Jitter(0.05, probability=0.5), Drift(0.5, 5, probability=0.5),
                            Quantize(16, probability=0.5), Dropout(0.05, probability=0.5),
                            Pool(4, probability=0.5), Reverse(probability=0.5)), master_seed=11)


@pytest.mark.parametrize("rows", [700, 6000])  # 6000: the fire-pattern sort kernels are captured too
def test_graph_replay_matches_eager(rows):
    pipe = _pipe()
    rng = np.random.default_rng(rows)
    a = torch.from_numpy(np.cumsum(rng.normal(size=(rows, 256)), axis=1)).cuda()
    b = torch.from_numpy(np.cumsum(rng.normal(size=(rows, 256)), axis=1)).cuda()
    want_a = pipe.run_device(a).clone()
    want_b = pipe.run_device(b).clone()
    buf = a.clone()
    run = pipe.capture_device(buf)
    assert torch.equal(run.check(), want_a)  # the eager warm-up launch
    for src, want in ((b, want_b), (a, want_a), (b, want_b)):
        buf.copy_(src)
        got = run.replay()
        torch.cuda.synchronize()
        assert torch.equal(run.check(), want) and got.data_ptr() == run.out.data_ptr()


def test_graph_replay_flags_nonfinite():
    from paper_2601_03159_b200 import InvalidInputError, Jitter, Pipeline

    pipe = Pipeline(stages=(Jitter(0.05),), master_seed=1)
    x = torch.ones((64, 128), dtype=torch.float64, device="cuda")
    run = pipe.capture_device(x)
    x[3, 7] = float("nan")
    run.replay()
    with pytest.raises(InvalidInputError):
        run.check()
    x[3, 7] = 1.0
    run.replay()
    assert torch.equal(run.check(), pipe.run_device(x))
