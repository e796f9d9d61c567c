"""Sanitizer target for the odd-length real transforms: paired columns (composite), Bluestein on
the half range of bins (large prime factors), shared-memory and global-scratch row buffers,
the standalone transforms and DCT.  compute-sanitizer --tool memcheck python tools/sanitize_odd.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench_inputs
from paper_2601_03159_b200 import *
for L in (9, 45, 121, 219, 541, 909, 997, 1361, 2369):
    x = bench_inputs.synthetic_walks(40, L, L)
    pipe = bench_inputs.sweep_pipeline(L, 3)
    for mode in ("0", "1"):
        os.environ["SA_FORCE_GLOBAL"] = mode
        pipe.run_device(torch.from_numpy(x).cuda())
    os.environ["SA_FORCE_GLOBAL"] = "0"
    b = Batch(x)
    fft_inverse(fft_forward(b)); dct_inverse(dct_forward(b))
    Pipeline(stages=(AmplitudePhasePerturb(0.1, 0.1),), master_seed=2).run(b)
torch.cuda.synchronize()
print("ok")
