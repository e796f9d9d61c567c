import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench_inputs
from paper_2601_03159_b200 import Batch
pipe = bench_inputs.pipeline(5)
n = 250_000
x = bench_inputs.device_walks(n, 1024, 5, torch.device("cuda")).cpu().numpy()
b = Batch._from_device_checked(x)
pipe.run(b)
t = time.perf_counter(); out = pipe.run(b); dt = time.perf_counter() - t
print(f"Pipeline.run pageable numpy {n}x1024: {dt*1e3:.0f} ms -> {n*1024/dt/1e9:.2f} Gpts/s ({2*x.nbytes/dt/1e9:.1f} GB/s moved)")
# second call: output pages already touched? (fresh output array each call)
t = time.perf_counter(); out = pipe.run(b); dt = time.perf_counter() - t
print(f"Pipeline.run pageable numpy (2nd) {dt*1e3:.0f} ms -> {n*1024/dt/1e9:.2f} Gpts/s")
from paper_2601_03159_b200 import pinned_empty
o = pinned_empty(x.shape)
pipe.run(b, out=o)
t = time.perf_counter(); pipe.run(b, out=o); dt = time.perf_counter() - t
print(f"Pipeline.run pageable in, pinned out: {dt*1e3:.0f} ms -> {n*1024/dt/1e9:.2f} Gpts/s")
