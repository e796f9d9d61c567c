import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2601_03159_b200 import *
x = np.cumsum(np.random.default_rng(0).normal(0, 1, (64, 256)), axis=1)
ops = {"fm": FrequencyMask(12), "sin": RandomSinusoid(1.0), "app": AmplitudePhasePerturb(0.1, 0.1), "rev": Reverse(), "jit": Jitter(0.1)}
for combo in (["fm"], ["sin"], ["app"], ["fm", "sin"], ["sin", "app"], ["fm", "app"], ["fm", "sin", "app"], ["rev", "fm"], ["jit", "app"], ["app", "rev"], ["app", "app"], ["fm", "fm"]):
    pipe = Pipeline(stages=tuple(ops[c] for c in combo), master_seed=4)
    g = pipe.run_device(torch.from_numpy(x).cuda()).cpu().numpy()
    w = O.run_pipeline(pipe, x)
    e = np.abs(g - w).max(axis=1)
    print(combo, "max %.2e" % e.max(), "bad rows", np.flatnonzero(e > 1e-9)[:10], flush=True)
