"""Config-5 stage ablation: time without stage j -> contribution of stage j."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench_inputs
from bench_inputs import device_walks
from paper_2601_03159_b200 import Pipeline, _engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
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
base = t(full)
print(f"full config5: {base:.3f} ms for {n} series")
rows = []
for j, s in enumerate(full.stages):
    import dataclasses
    st = list(full.stages)
    st[j] = dataclasses.replace(st[j], probability=0.0)  # same indices / streams / barrier grouping
    p = Pipeline(stages=tuple(st), master_seed=full.master_seed)
    d = base - t(p)
    rows.append((d, j, s.kind, repr(s)[:60]))
for d, j, k, r in sorted(rows, reverse=True):
    print(f"{d:7.3f} ms ({100 * d / base:5.1f}%)  stage {j:2d} {r}")
print(f"sum of contributions {sum(r[0] for r in rows):.3f} ms; residual (load/store/prepass) {base - sum(r[0] for r in rows):.3f} ms")
