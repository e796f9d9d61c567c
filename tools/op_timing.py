"""Per-operator kernel time on the device (p=1, one stage), us per series."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench_inputs import device_walks
from paper_2601_03159_b200 import *
from paper_2601_03159_b200 import _engine
n, L = int(sys.argv[1]) if len(sys.argv) > 1 else 50000, 1024
x = device_walks(n, L, 5, torch.device("cuda"))
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
ops = [("copy(rotate p0)", Rotate(probability=0.0)), ("rotate", Rotate()), ("reverse", Reverse()), ("scale", Scale(0.1)),
       ("jitter", Jitter(0.05)), ("uniform", InjectNoise(UniformNoise(0.1))), ("dropout", Dropout(0.05)),
       ("quantize", Quantize(16)), ("drift", Drift(0.5, 5)), ("spike", InjectNoise(SpikeNoise(5, 2.0))),
       ("slope", InjectNoise(SlopeTrendNoise(0.5))), ("permute4", PermuteSegments(4)), ("crop819", Crop(819)),
       ("resize1500", Resize(1500)), ("time_warp", TimeWarp(5, 0.5)), ("window_warp", WindowWarp(128, 4, 0.5)),
       ("pool4", Pool(4)), ("convolve7", Convolve("hann", 7)), ("speed_warp", SpeedWarp(3, 3.0)),
       ("freq_mask", FrequencyMask(51)), ("app", AmplitudePhasePerturb(0.1, 0.1)), ("sinusoid", RandomSinusoid(0.5))]
import bench_inputs
ops.append(("CONFIG5", bench_inputs.pipeline(5)))
for name, aug in ops:
    pipe = aug if isinstance(aug, Pipeline) else Pipeline(stages=(aug,), master_seed=1)
    Lo = pipe.projected_length(L)
    out = torch.empty((n, Lo), dtype=torch.float64, device="cuda")
    low = _engine._lower(pipe.stages, 0, True)
    for _ in range(2):
        _engine.launch_device(pipe.stages, x, out, flags, 1, lowered=low)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for i in range(3):
        _engine.launch_device(pipe.stages, x, out, flags, 1, lowered=low)
        ev[i + 1].record()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
    ms = sum(per) / 3
    if max(per) > 1.5 * min(per):
        print("   uneven launches:", ["%.3f" % v for v in per], flush=True)
    gbs = 8 * n * (L + Lo) / (ms / 1e3) / 1e9
    print(f"{name:18s} {ms:8.3f} ms  {ms * 1e3 / n * 148:8.2f} us/series/SM  {gbs:7.1f} GB/s", flush=True)
