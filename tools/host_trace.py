"""Pipeline.run on config 5 with SA_HOST_TRACE=1: where the host pipeline's
loop time goes (pageable in, page-locked out).  Usage: python tools/host_trace.py"""
import os
import sys
import time

os.environ.setdefault("SA_HOST_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench_inputs  # noqa: E402
from paper_2601_03159_b200 import Batch, pinned_empty  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
pipe = bench_inputs.pipeline(5)
x = bench_inputs.device_walks(n, 1024, 5, torch.device("cuda")).cpu().numpy()
b = Batch._from_device_checked(x)
o = pinned_empty(x.shape)
xp = pinned_empty(x.shape)
xp[...] = x
bp = Batch._from_device_checked(xp)
for label, bb in (("pageable in, pinned out", b), ("pinned in, pinned out", bp)):
    for _ in range(3):
        t0 = time.perf_counter()
        pipe.run(bb, out=o)
        print(f"{label}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
