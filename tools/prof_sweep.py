"""Launch one sweep dataset's pipeline a few times (ncu target): python tools/prof_sweep.py 73"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench_inputs
from paper_2601_03159_b200 import _engine
want = int(sys.argv[1])
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for i, n, L in bench_inputs.sweep_datasets():
    if i != want:
        continue
    x = torch.from_numpy(bench_inputs.synthetic_walks(n, L, i)).cuda()
    pipe = bench_inputs.sweep_pipeline(L, i)
    out = torch.empty_like(x)
    for _ in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    torch.cuda.synchronize()
    print("ok", n, L, [type(s).__name__ for s in pipe.stages])
