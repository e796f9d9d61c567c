"""Per-op spectral error probe (GPU vs oracle)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2601_03159_b200 import *
for L in (4, 8, 16, 32, 64, 256, 1024):
    x = np.cumsum(np.random.default_rng(0).normal(0, 1, (8, L)), axis=1)
    re, im = O.fft_forward(x)
    sb = fft_forward(Batch(x))
    e1 = max(np.abs(sb.re - re).max(), np.abs(sb.im - im).max())
    back = fft_inverse(SpectrumBatch(re, im, L)).values
    e2 = np.abs(back - x).max()
    errs = []
    for aug in (FrequencyMask(2), RandomSinusoid(1.0), AmplitudePhasePerturb(0.1, 0.0), AmplitudePhasePerturb(0.0, 0.1)):
        pipe = Pipeline(stages=(aug,), master_seed=4)
        g = pipe.run_device(torch.from_numpy(x).cuda()).cpu().numpy()
        w = O.run_pipeline(pipe, x)
        errs.append(float(np.abs(g - w).max()))
    print(L, "rfft %.2e irfft %.2e" % (e1, e2), "ops", ["%.2e" % e for e in errs], flush=True)
