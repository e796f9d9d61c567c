"""Device time of single sweep datasets (median of 7 launches, ms), one
subprocess per environment variant: python tools/ds_time.py 73,35 SA_CTA_WARPS=4 SA_CTA_WARPS=8"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import bench_inputs as B
    from paper_2601_03159_b200 import _engine

    res = {}
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    for i in [int(v) for v in sys.argv[2].split(",")]:
        _, n, L = B.sweep_datasets()[i]
        pipe = B.sweep_pipeline(L, i)
        x = torch.from_numpy(B.synthetic_walks(n, L, i)).cuda()
        out = torch.empty_like(x)
        low = _engine._lower(pipe.stages, 0, True)
        for _ in range(2):
            _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[i] = float(np.median(ts))
    print(json.dumps(res))
    sys.exit(0)
ids = sys.argv[1]
for var in sys.argv[2:] or ["BASE=1"]:
    k, v = var.split("=")
    o = subprocess.run([sys.executable, __file__, "--child", ids], env=dict(os.environ, **{k: v}), capture_output=True,
                       text=True)
    print(var, o.stdout.strip() or o.stderr[-500:], flush=True)
