"""Where the drop-in call's time goes on the GPU box: Pipeline.run(Batch(numpy))
on config 5 (1e6 x 1024 f64), split into Batch validation, output first touch,
host copies and the device pipeline.  Usage: python tools/host_probe.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_inputs  # noqa: E402
from paper_2601_03159_b200 import Batch, pinned_empty  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
for f in ("enabled", "defrag"):
    try:
        print(f"THP {f}:", open(f"/sys/kernel/mm/transparent_hugepage/{f}").read().strip())
    except OSError:
        pass
print("cpus", os.cpu_count())


def t(label, fn, reps=4):
    fn()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        best = min(best, time.perf_counter() - t0)
    print(f"{label:60s} {best * 1e3:9.1f} ms  ({8 * n * 1024 / best / 1e9:6.1f} GB/s of one array)", flush=True)
    return r


pipe = bench_inputs.pipeline(5)
x = bench_inputs.device_walks(n, 1024, 5, torch.device("cuda")).cpu().numpy()
quick = os.environ.get("PROBE_QUICK")
t("Batch(x) (np.isfinite(x).all())", lambda: Batch(x))
if not quick:
    t("np.isfinite(x).all()", lambda: np.isfinite(x).all())
    t("np.empty + fill 0 (first touch)", lambda: np.empty_like(x).fill(0.0))
y = np.empty_like(x)
y.fill(0)
if not quick:
    t("np.copyto pre-touched (1 thread)", lambda: np.copyto(y, x))
b = Batch._from_device_checked(x)
t("Pipeline.run(b) fresh pageable out", lambda: pipe.run(b))
t("Pipeline.run(b, out=pretouched pageable)", lambda: pipe.run(b, out=y))
o = pinned_empty(x.shape)
t("Pipeline.run(b, out=pinned)", lambda: pipe.run(b, out=o))
t("Pipeline.run(Batch(x))", lambda: pipe.run(Batch(x)))
import subprocess
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
