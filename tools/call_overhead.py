"""Per-call cost of the drop-in Pipeline.run on sweep datasets (steady state):
Python lowering vs the C ABI call vs the device time.  Usage: python tools/call_overhead.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_inputs as B  # noqa: E402
from paper_2601_03159_b200 import Batch, _engine  # noqa: E402

ds = sorted(B.sweep_datasets(), key=lambda d: d[1] * d[2])
pick = [ds[0], ds[10], ds[50], ds[90], ds[-1]]
for i, n, L in pick:
    pipe = B.sweep_pipeline(L, i)
    b = Batch(B.synthetic_walks(n, L, i))
    for _ in range(3):
        pipe.run(b)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        pipe.run(b)
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    for _ in range(20):
        _engine._lower(pipe.stages, 0, True)
    tl = (time.perf_counter() - t0) / 20
    x = torch.from_numpy(b.values).cuda()
    out = torch.empty_like(x)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    low = _engine._lower(pipe.stages, 0, True)
    for _ in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
    e.record()
    torch.cuda.synchronize()
    print(f"ds {i:3d} n={n:6d} L={L:5d}: Pipeline.run median {1e3 * np.median(ts):8.3f} ms, lowering {1e3 * tl:6.3f} ms, "
          f"device {a.elapsed_time(e) / 10:7.3f} ms", flush=True)
