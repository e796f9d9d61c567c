import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, dataclasses
import bench_inputs
from oracle import oracle as O
from paper_2601_03159_b200 import Pipeline
bad = 0
for i, n, L in bench_inputs.sweep_datasets():
    pipe = bench_inputs.sweep_pipeline(L, seed=i)
    x = bench_inputs.synthetic_walks(min(n, 64), L, seed=i)
    want = O.run_pipeline(pipe, x)
    got = pipe.run_device(torch.from_numpy(x).cuda()).cpu().numpy()
    err = np.abs(got - want).max(axis=1)
    scale = max(1.0, float(np.abs(want).max()))
    if err.max() > 1e-9 * scale:
        bad += 1
        rows = np.flatnonzero(err > 1e-9 * scale)
        # find the first stage where this row diverges
        r = int(rows[0])
        first = None
        for j in range(1, len(pipe.stages) + 1):
            sub = Pipeline(stages=pipe.stages[:j], master_seed=pipe.master_seed)
            w = O.run_pipeline(sub, x[r:r+1], series_offset=r)
            g = sub.run_device(torch.from_numpy(x[r:r+1].copy()).cuda(), series_offset=r).cpu().numpy()
            if np.abs(g - w).max() > 1e-9 * scale:
                first = (j - 1, pipe.stages[j - 1].kind, float(np.abs(g - w).max()))
                break
        print(f"dataset {i} n={n} L={L}: {rows.size} rows bad, max err {err.max():.3e} (scale {scale:.1f}); first divergence {first}", flush=True)
print("bad datasets", bad)
