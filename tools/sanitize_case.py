"""Small workload touching every operator, FFT lengths and DTW (sanitizer target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench_inputs
from paper_2601_03159_b200 import *
for L in (64, 97, 1024):
    pipe = bench_inputs.sweep_pipeline(L, 3)
    x = torch.from_numpy(bench_inputs.synthetic_walks(300, L, 1)).cuda()
    pipe.run_device(x)
pipe = bench_inputs.pipeline(2)
pipe.run(Batch(bench_inputs.synthetic_walks(200, 1024, 2)))
p4 = Pipeline(stages=(Repeat(2), SpeedWarp(3, 3.0), Resize(300), Convolve("hann", 7), Crop(100)), master_seed=1)
p4.run(Batch(bench_inputs.synthetic_walks(50, 256, 3)))
b = Batch(np.random.default_rng(0).normal(0, 1, (8, 45)))
dct_inverse(dct_forward(b)); fft_inverse(fft_forward(b))
dtw_distance(b.values[0], b.values[1][:30]); mean_similarity(b, b)
torch.cuda.synchronize()
print("ok")
