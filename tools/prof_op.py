"""Single-op pipeline launcher for ncu (python tools/prof_op.py jitter)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench_inputs import device_walks
from paper_2601_03159_b200 import *
from paper_2601_03159_b200 import _engine
OPS = {"jitter": Jitter(0.05), "app": AmplitudePhasePerturb(0.1, 0.1), "spike": InjectNoise(SpikeNoise(5, 2.0)),
       "drift": Drift(0.5, 5), "resize": Resize(1500), "fmask": FrequencyMask(51), "time_warp": TimeWarp(5, 0.5),
       "copy": Rotate(probability=0.0), "uniform": InjectNoise(UniformNoise(0.1))}
name = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
pipe = Pipeline(stages=(Rotate(probability=0.0), OPS[name[:-6]]), master_seed=1) if name.endswith("_chain") \
    else Pipeline(stages=(OPS[name],), master_seed=1)
x = device_walks(n, 1024, 5, torch.device("cuda"))
out = torch.empty((n, pipe.projected_length(1024)), dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    _engine.launch_device(pipe.stages, x, out, flags, 1)
torch.cuda.synchronize(); print("ok")
