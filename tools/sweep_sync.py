"""Barrier placement policies for config 5."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench_inputs
from bench_inputs import device_walks
from paper_2601_03159_b200 import _engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
pipe = bench_inputs.pipeline(5)
x = device_walks(n, 1024, 5, torch.device("cuda"))
out = torch.empty((n, 1024), dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
ref = None
for pol, every, thr in [(0, 4, 20), (0, 3, 20), (1, 4, 20), (1, 3, 20), (1, 2, 20), (1, 4, 40), (1, 6, 40), (1, 8, 20), (1, 99, 20), (1, 99, 40), (0, 4, 20)]:
    os.environ.update(SA_SYNC_POLICY=str(pol), SA_SYNC_EVERY=str(every), SA_SYNC_COST_X10=str(thr))
    for _ in range(2):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    ref = out.clone() if ref is None else ref
    print(f"policy={pol} every={every} thr={thr / 10:.1f}: {ms:8.3f} ms  {n * 1024 / ms / 1e6:6.2f} Gpts/s same={torch.equal(ref, out)}", flush=True)
