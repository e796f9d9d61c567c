import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import bench_inputs
from paper_2601_03159_b200 import _engine
def factors(n):
    f, d = [], 2
    while d * d <= n:
        while n % d == 0: f.append(d); n //= d
        d += 1
    if n > 1: f.append(n)
    return f
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
rows = []
for i, n, L in bench_inputs.sweep_datasets():
    x = torch.from_numpy(bench_inputs.synthetic_walks(n, L, i)).cuda()
    pipe = bench_inputs.sweep_pipeline(L, i)
    out = torch.empty_like(x)
    for _ in range(2): _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed); b.record(); torch.cuda.synchronize()
    rows.append((a.elapsed_time(b), i, n, L))
tot = sum(r[0] for r in rows)
print("total %.1f ms" % tot)
for ms, i, n, L in sorted(rows, reverse=True)[:15]:
    Lf = L // 2 if L % 2 == 0 else L
    print(f"{ms:8.3f} ms  ds {i:3d} n={n:6d} L={L:5d}  fft N={Lf} factors={factors(Lf)}  us/series={1e3*ms/n:.2f}")
print("median ms", np.median([r[0] for r in rows]))
if len(sys.argv) > 1:
    import json; json.dump(rows, open(sys.argv[1], "w"))
