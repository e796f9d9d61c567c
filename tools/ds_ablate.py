"""Device time of sweep datasets with stage subsets (median of 7 launches, ms):
python tools/ds_ablate.py 73,35,74   -> full chain, without spectral stages, spectral stages only"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_inputs as B  # noqa: E402
from paper_2601_03159_b200 import Pipeline, _engine  # noqa: E402

SPEC = ("amplitude_phase_perturb", "frequency_mask", "random_sinusoid")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")


def timed(stages, x, out, seed):
    low = _engine._lower(stages, 0, True)
    for _ in range(2):
        _engine.launch_device(stages, x, out, flags, seed, lowered=low)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _engine.launch_device(stages, x, out, flags, seed, lowered=low)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


res = {}
for i in [int(v) for v in sys.argv[1].split(",")]:
    _, n, L = B.sweep_datasets()[i]
    pipe = B.sweep_pipeline(L, i)
    x = torch.from_numpy(B.synthetic_walks(n, L, i)).cuda()
    out = torch.empty_like(x)
    st = pipe.stages
    r = {"n": n, "L": L, "full": timed(st, x, out, pipe.master_seed)}
    r["no_spec"] = timed(tuple(s for s in st if s.kind not in SPEC), x, out, pipe.master_seed)
    r["spec_only"] = timed(tuple(s for s in st if s.kind in SPEC), x, out, pipe.master_seed)
    r["app_only"] = timed(tuple(s for s in st if s.kind == "amplitude_phase_perturb"), x, out, pipe.master_seed)
    res[i] = r
    print(i, json.dumps(r), flush=True)
