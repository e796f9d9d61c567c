"""Launch one pipeline (a bench config or a single op) a few times: the ncu target."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import bench_inputs
from bench_inputs import device_walks
from paper_2601_03159_b200 import *
from paper_2601_03159_b200 import _engine
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sweep-ds", type=int, default=-1, help="profile sweep dataset i instead of a config")
a = ap.parse_args()
if a.sweep_ds >= 0:
    _, a.n, L = bench_inputs.sweep_datasets()[a.sweep_ds]
    pipe = bench_inputs.sweep_pipeline(L, a.sweep_ds)
else:
    N, L = bench_inputs.CONFIG_SHAPES[a.config]
    pipe = bench_inputs.pipeline(a.config)
x = device_walks(a.n, L, 5, torch.device("cuda"))
out = torch.empty((a.n * pipe.row_factor(), pipe.projected_length(L)), dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
low = _engine._lower(pipe.stages, 0, True)
for _ in range(a.reps):
    _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
torch.cuda.synchronize()
assert int(flags.item()) == 0
print("ok")
