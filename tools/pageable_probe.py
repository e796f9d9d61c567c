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
