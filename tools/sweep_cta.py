"""Config-5 kernel time vs CTA shape (SA_CTA_WARPS) and barrier cadence (SA_SYNC_EVERY)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench_inputs
from bench_inputs import device_walks
from paper_2601_03159_b200 import _engine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
N, L = bench_inputs.CONFIG_SHAPES[cfg]
pipe = bench_inputs.pipeline(cfg)
x = device_walks(n, L, 5, torch.device("cuda"))
out = torch.empty((n, pipe.projected_length(L)), dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
ref = None
for warps, sync, sched in [(0, 4, 1), (7, 4, 1), (4, 4, 1), (2, 4, 1), (0, 4, 1)]:
    os.environ['SA_SCHEDULE'] = str(sched)
    os.environ["SA_CTA_WARPS"] = str(warps)
    os.environ["SA_SYNC_EVERY"] = str(sync)
    for _ in range(2):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    if ref is None:
        ref = out.clone()
    same = torch.equal(ref, out)
    print(f"cfg{cfg} warps={warps or 'fit':>3} sync_every={sync} sched={sched}  {ms:8.3f} ms  {n * out.shape[1] / ms / 1e6:7.2f} Gpts/s  same={same}", flush=True)
