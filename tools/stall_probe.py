import sys, os, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bench_inputs
from paper_2601_03159_b200 import _engine
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
mode = sys.argv[1] if len(sys.argv) > 1 else "gc-on"
if mode == "gc-off":
    gc.disable()
worst = []
for i, n, L in bench_inputs.sweep_datasets():
    x = torch.from_numpy(bench_inputs.synthetic_walks(n, L, i)).cuda()
    pipe = bench_inputs.sweep_pipeline(L, i)
    out = torch.empty_like(x)
    low = _engine._lower(pipe.stages, 0, True)
    for _ in range(2): _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
    h1 = time.perf_counter()
    b.record(); torch.cuda.synchronize()
    worst.append((a.elapsed_time(b), (h1 - h0) * 1e3, i, n, L))
worst.sort(reverse=True)
print(mode, "total %.1f ms" % sum(w[0] for w in worst))
for g, h, i, n, L in worst[:4]:
    print(f"  gpu {g:8.3f} ms  host-enqueue {h:8.3f} ms  ds {i} n={n} L={L}")
