import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench_inputs
from oracle import oracle as O
from paper_2601_03159_b200 import Pipeline
i, n, L = [d for d in bench_inputs.sweep_datasets() if d[0] == 88][0]
pipe = bench_inputs.sweep_pipeline(L, seed=i)
x = bench_inputs.synthetic_walks(min(n, 64), L, seed=i)
want = O.run_pipeline(pipe, x)
got = pipe.run_device(torch.from_numpy(x).cuda()).cpu().numpy()
r = int(np.argmax(np.abs(got - want).max(axis=1)))
pre = O.run_pipeline(Pipeline(stages=pipe.stages[:11], master_seed=pipe.master_seed), x[r:r+1], series_offset=r)
# APP alone on the oracle's pre-state: same stream (stage index 11, series r)
app = Pipeline(stages=pipe.stages[:12], master_seed=pipe.master_seed)
import dataclasses
stages = list(pipe.stages[:12])
for j in range(11):
    stages[j] = dataclasses.replace(stages[j], probability=0.0)
only = Pipeline(stages=tuple(stages), master_seed=pipe.master_seed)
w = O.run_pipeline(only, pre, series_offset=r)
g = only.run_device(torch.from_numpy(pre.copy()).cuda(), series_offset=r).cpu().numpy()
print("row", r, "APP-only err", np.abs(g - w).max())
re, im = O.fft_forward(pre)
mag = np.hypot(re, im)[0]
print("smallest |X| bins:", np.argsort(mag)[:5], np.sort(mag)[:5], "median", np.median(mag))
Xw = np.fft.rfft(w[0]); Xg = np.fft.rfft(g[0])
d = np.abs(Xw - Xg)
print("bins with largest output spectral diff:", np.argsort(d)[-5:], np.sort(d)[-5:])
