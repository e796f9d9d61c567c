"""Config 3 (and other spectral-only chains) on the radix-16 vs radix-8 CTA
kernels: time + agreement + oracle check on a sample.
Usage: python tools/spec_ab.py [n] [L]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import bench_inputs as B
    from paper_2601_03159_b200 import FrequencyMask, Pipeline, RandomSinusoid, _engine

    n, L = int(sys.argv[2]), int(sys.argv[3])
    x = torch.from_numpy(B.ar2_input(n, L)).cuda()
    pipe = B.pipeline(3) if L == 2048 else Pipeline(stages=(FrequencyMask(max(1, L // 20)), RandomSinusoid(1.0)),
                                                    master_seed=2)
    out = torch.empty_like(x)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    low = _engine._lower(pipe.stages, 0, True)
    for _ in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(15):
        a.record()
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    np.save(sys.argv[4], out.cpu().numpy())
    print(f"{os.environ.get('SA_SPEC_R16', '1')}: median {np.median(ts):.4f} ms  flags {int(flags.item())}")
    sys.exit(0)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
outs = []
for v in ("0", "1", "0", "1"):
    f = f"/tmp/spec_ab_{v}.npy"
    subprocess.run([sys.executable, __file__, "--child", str(n), str(L), f], env=dict(os.environ, SA_SPEC_R16=v),
                   check=True)
    outs.append(f)
import numpy as np  # noqa: E402

sys.path.insert(0, ROOT)
o0, o1 = np.load(outs[0]), np.load(outs[1])
scale = max(1.0, float(np.abs(o0).max()))
print("max |r16 - r8| / scale:", float(np.abs(o0 - o1).max()) / scale)
import bench_inputs as B  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2601_03159_b200 import FrequencyMask, Pipeline, RandomSinusoid  # noqa: E402

pipe = B.pipeline(3) if L == 2048 else Pipeline(stages=(FrequencyMask(max(1, L // 20)), RandomSinusoid(1.0)),
                                                master_seed=2)
xs = B.ar2_input(n, L)[:256]
want = O.run_pipeline(pipe, xs)
print("max |r16 - oracle| / scale (256 rows):", float(np.abs(o1[:256] - want).max()) / scale)
