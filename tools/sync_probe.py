import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench_inputs
from bench_inputs import device_walks
from paper_2601_03159_b200 import Pipeline, _engine
n = 100000
full = bench_inputs.pipeline(5)
x = device_walks(n, 1024, 5, torch.device("cuda"))
out = torch.empty((n, 1024), dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
def t(pipe):
    for _ in range(2):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 3
nopool = Pipeline(stages=full.stages[:16] + full.stages[17:], master_seed=5)
nouni = Pipeline(stages=full.stages[:7] + full.stages[8:], master_seed=5)
for se in (1, 2, 3, 4, 5, 6):
    os.environ["SA_SYNC_EVERY"] = str(se)
    print(f"sync {se}: full {t(full):7.3f}  no-pool {t(nopool):7.3f}  no-uniform {t(nouni):7.3f}", flush=True)
os.environ["SA_SYNC_EVERY"] = "4"
for seed in (5, 6, 7):
    p = Pipeline(stages=full.stages, master_seed=seed)
    print(f"seed {seed}: {t(p):7.3f}", flush=True)
