"""A/B kernel timing of builds of the backend (tools/build_variant.sh):
python tools/ab_timing.py ab/libA.so ab/libB.so -- jitter app CONFIG5
Each build runs in a fresh process; builds alternate for `rounds` rounds and
each op's time is the median of 15 launches (ms)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    lib, names, n = sys.argv[2], sys.argv[3].split(","), int(sys.argv[4])
    from paper_2601_03159_b200 import _native
    _native.LIB_PATH = os.path.abspath(lib)
    import torch
    import bench_inputs
    from bench_inputs import device_walks
    from paper_2601_03159_b200 import _engine
    from paper_2601_03159_b200 import *  # noqa
    OPS = {"jitter": Jitter(0.05), "app": AmplitudePhasePerturb(0.1, 0.1), "spike": InjectNoise(SpikeNoise(5, 2.0)),
           "drift": Drift(0.5, 5), "time_warp": TimeWarp(5, 0.5), "speed_warp": SpeedWarp(3, 3.0),
           "fmask": FrequencyMask(51), "sinusoid": RandomSinusoid(0.5), "uniform": InjectNoise(UniformNoise(0.1)),
           "dropout": Dropout(0.05), "quantize": Quantize(16), "copy": Rotate(probability=0.0),
           "window_warp": WindowWarp(128, 4, 0.5), "convolve": Convolve("hann", 7), "pool": Pool(4),
           "scale": Scale(0.1), "rotate": Rotate(), "reverse": Reverse(), "permute": PermuteSegments(4),
           "gauss": InjectNoise(GaussianNoise(0.1)), "slope": InjectNoise(SlopeTrendNoise(0.5))}
    L = int(os.environ.get("AB_L", "1024"))
    x = device_walks(n, L, 5, torch.device("cuda"))
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = {}
    for name in names:
        if name == "CONFIG5P1":  # config 5's chain with every stage firing
            import dataclasses
            c5 = bench_inputs.pipeline(5)
            pipe = Pipeline(stages=tuple(dataclasses.replace(st, probability=1.0) for st in c5.stages), master_seed=5)
        elif name == "SWCONV":  # config 4's two working stages (no resize), any AB_L
            pipe = Pipeline(stages=(SpeedWarp(3, 3.0), Convolve("hann", 7)), master_seed=3)
        elif name == "CHAIN5":  # config 5's chain with length-scaled parameters, any AB_L
            pipe = bench_inputs.sweep_pipeline(L, 5)
        elif name.startswith("REP"):  # REP<k>_<op>: k copies of one op (composition experiments)
            kk, op = name[3:].split("_", 1)
            pipe = Pipeline(stages=tuple(OPS[op] for _ in range(int(kk))), master_seed=1)
        elif name.endswith("_chain"):  # the op inside a mixed chain (warp path, not a CTA kernel)
            pipe = Pipeline(stages=(Rotate(probability=0.0), OPS[name[:-6]]), master_seed=1)
        elif name.startswith("CONFIG"):
            pipe = bench_inputs.pipeline(int(name[6:]))
        else:
            pipe = Pipeline(stages=(OPS[name],), master_seed=1)
        out = torch.empty((n, pipe.projected_length(L)), dtype=torch.float64, device="cuda")
        low = _engine._lower(pipe.stages, 0, True)
        for _ in range(3):
            _engine.launch_device(pipe.stages, x, out, flags, 1, lowered=low)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(16)]
        ev[0].record()
        for i in range(15):
            _engine.launch_device(pipe.stages, x, out, flags, 1, lowered=low)
            ev[i + 1].record()
        torch.cuda.synchronize()
        per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(15))
        res[name] = per[7]
    print(json.dumps(res))
    sys.exit(0)

args = sys.argv[1:]
sep = args.index("--")
libs, names = args[:sep], args[sep + 1:]
n = int(os.environ.get("AB_N", "50000"))
rounds = int(os.environ.get("AB_ROUNDS", "2"))
acc = {l: {} for l in libs}
for _ in range(rounds):
    for l in libs:
        o = subprocess.run([sys.executable, __file__, "--child", l, ",".join(names), str(n)], capture_output=True,
                           text=True)
        if o.returncode:
            print(o.stderr[-2000:]); sys.exit(1)
        for k, v in json.loads(o.stdout.strip().splitlines()[-1]).items():
            acc[l].setdefault(k, []).append(v)
print("%-12s" % "op" + "".join("%18s" % os.path.basename(l) for l in libs))
for k in names:
    print("%-12s" % k + "".join("%18s" % ("%.3f" % min(acc[l][k])) for l in libs))
