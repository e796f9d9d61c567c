#!/usr/bin/env python
"""Benchmark of the fused B200 augmentation pipeline (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl b200|reference]
                    [--workload pipeline|sweep|transforms|dtw|datafiles]

One "step" = one pass of the whole augmentation chain over the batch of the
chosen BASELINE config (default: config 5, all 20 length-preserving augmenters
at p=0.5 on 1,000,000 x 1,024 float64 series, the configuration the metric
"pipeline at 1/2/4/8 B200" is quoted on).  With --gpus N the batch is sharded
by contiguous series ranges over N ranks, one process per GPU (torchrun's
RANK / WORLD_SIZE / LOCAL_RANK; without them bench.py launches the N ranks
itself); there is no data-path collective -- torch.distributed carries only
the barrier and the max-over-ranks of the timings -- and total work is fixed
as N grows ("strong" scaling).

value  = output points (all ranks) / max-over-ranks device time, inputs resident
         in HBM, CUDA events on the launching stream.
e2e    = same metric through the host-buffer C ABI call (sa_pipeline_run_host)
         from pinned host memory: H2D + kernels + D2H inside the timed region.
e2e_pageable = the drop-in user's call, Pipeline.run(Batch(numpy)) on ordinary
         (pageable) numpy arrays in and out.
roofline.achieved = algorithmic bytes 8*(n*L_in + n_out*L_out) per launch /
         mean kernel duration (per GPU); peak = MEASURED_PEAKS.json hbm_gbs.
cpu_baseline = the GENUINE reference (seriesaug from oracle/_ref, the
         BASELINE-only kinds as its plugins) on a bounded sample of the same
         workload: a process pool over all host cores running its per-sample
         loop, rank 0 at N=1; cpu_port = the C oracle (a restatement) likewise.
--impl reference times that reference CPU path alone (rank 0) on the same
         config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "augmented points/sec"
UNIT = "points/s"
LIB_PATH = os.path.join(ROOT, "paper_2601_03159_b200", "_lib", "libseriesaug_b200.so")

WORKLOADS = {
    1: "config1: AddNoise/Jitter(sigma=0.05) on 1,000 x 512 sum-of-sinusoids",
    2: "config2: Crop(819)->Drift->Quantize(16)->Dropout(0.05)->Pool(4)->Reverse (p=0.5) on 10,000 x 1,024 walks",
    3: "config3: rfft->FrequencyMask(102 = 10% of 1,025 bins)->random-phase sinusoid->irfft on 50,000 x 2,048 AR(2)",
    4: "config4: SpeedWarp(3, 3.0, cubic)->Resize(1500)->Convolve(hann,7) on 100,000 x 1,500 walk+sine",
    5: "config5: all 20 length-preserving augmenters at p=0.5 on 1,000,000 x 1,024 walks (8.2 GB)",
    "sweep": ("config5 sweep: the 20-augmenter chain (length-scaled parameters) over 100 synthetic datasets, "
              "series counts log-uniform in [20, 24,000], lengths log-uniform in [24, 2,900] (random walks)"),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _profile_json(name):
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def fp64_peak():
    """Measured FP64 FMA peak of the box (tools/micro/fp64_peak.cu), TFLOP/s."""
    d = _profile_json("r02_fp64_peak.json")
    return (float(d["fp64_fma_tflops"]), "measured (profiles/r02_fp64_peak.json)") if d else \
        (37.0, "nominal B200 FP64")


def fft_flops_per_series(cfg, L):
    """Algorithmic FP64 flops of the FFT-bearing configs:
    one rfft + irfft pair, 2 x 2.5 L log2 L per series (config 3)."""
    import math

    return 2 * 2.5 * L * math.log2(L) if cfg == 3 else None


def ncu_traffic(cfg):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/ncu_traffic.json, tools/ncu_record.py)."""
    t = _profile_json("ncu_traffic.json").get(cfg if isinstance(cfg, str) else f"config{cfg}")
    return t.get("value") if isinstance(t, dict) else t


def build_sha16() -> str | None:
    """Identity of the library under test (the ncu instruction counts carry
    the hash of the build they were captured on): the kernel sources and build
    recipe -- nvcc's output is not byte-reproducible, so hashing the .so would
    mark every rebuild of the same sources stale.  An alternative build named
    by SA_LIB_PATH (A/B runs) is identified by its bytes."""
    alt = os.environ.get("SA_LIB_PATH")
    h = hashlib.sha256()
    try:
        if alt:
            with open(alt, "rb") as fh:
                h.update(fh.read())
        else:
            src = os.path.join(ROOT, "paper_2601_03159_b200", "csrc")
            for name in sorted(os.listdir(src)):
                with open(os.path.join(src, name), "rb") as fh:
                    h.update(name.encode() + b"\0" + fh.read())
            with open(os.path.join(ROOT, "include", "seriesaug_b200.h"), "rb") as fh:
                h.update(fh.read())
        return h.hexdigest()[:16]
    except OSError:
        return None


def config_dict(cfg, N, L, L_out, world, pipe_cfg):
    """The line's `config`: identical for the device and the reference arm."""
    return {"workload": WORKLOADS[cfg], "n_series": N, "len_in": L, "len_out": L_out,
            "stages": [s["kind"] for s in pipe_cfg["stages"]], "master_seed": pipe_cfg["master_seed"],
            "parallelism": f"series-range shards x{world}, no collective",
            "l2": "inputs larger than L2 (no flush needed)" if 8 * N * L / world > 256e6 else
                  "input smaller than L2: repeated steps may hit L2"}


def reduce_timings(t, k: int, dev):
    """Max over ranks of t[:k] (times), sum of t[k:] (counts).  NCCL reduces
    device tensors only; the gloo test backend reduces host tensors."""
    import torch
    import torch.distributed as dist

    where = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    tm = t[:k].clone().to(where)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    lt = t[k:].clone().to(where)
    dist.all_reduce(lt, op=dist.ReduceOp.SUM)
    return torch.cat([tm, lt]).cpu()


# ------------------------------------------------------------------ CPU legs
def reference_cpu(pipe_cfg: dict, L: int, target_s: float, cores: int | None = None, steps: int = 1,
                  warmup: int = 1, first: int = 0):
    """The genuine reference on all host cores (oracle/ref_runner.py: one
    process per core, each running the reference's per-sample loop over its
    own contiguous block of series), sized so one pass takes ~target_s.
    Returns (points per pass, seconds per pass, cores, rows per core)."""
    from oracle import ref_runner as R

    pool = R.ProcessPool(cores)
    try:
        rows = 4
        pool.assign(R.config_tasks(pipe_cfg, L, rows, pool.cores, first=first))
        pool.run()  # first-call costs (lazy imports inside numpy / scipy)
        pts, dt = pool.run()
        rows = int(min(max(rows, rows * target_s / max(dt, 1e-6)), 200_000))
        pool.assign(R.config_tasks(pipe_cfg, L, rows, pool.cores, first=first))
        for _ in range(warmup):
            pool.run()
        runs = [pool.run() for _ in range(steps)]
    finally:
        pool.close()
    pts = runs[-1][0]
    return pts, sum(dt for _, dt in runs) / len(runs), pool.cores, rows


def reference_baseline(pipe_cfg: dict, L: int, label: str, target_s: float = 8.0) -> dict:
    pts, dt, cores, rows = reference_cpu(pipe_cfg, L, target_s)
    return {"value": pts / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{cores} x {rows} series of {label} through the unmodified reference "
                      f"(seriesaug, per-sample loop, one process per core): {pts} output points in {dt:.2f} s"}


def port_baseline(pipe_cfg: dict, L: int, label: str, target_s: float = 5.0):
    """The C oracle (oracle/sa_oracle.c, a restatement of the reference's
    algorithm) on all host threads, same workload: the strongest CPU
    implementation of the path at hand."""
    from oracle import oracle as O
    from oracle import ref_runner as R

    threads = os.cpu_count() or 1
    probe = R.walks(max(64, 8 * threads), L, 1)
    t0 = time.perf_counter()
    O.run_config(pipe_cfg, probe, threads=threads)
    per_row = (time.perf_counter() - t0) / probe.shape[0]
    n = int(min(max(256, target_s / max(per_row, 1e-9)), 200_000))
    x = R.walks(n, L, 2)
    t0 = time.perf_counter()
    out = O.run_config(pipe_cfg, x, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": out.size / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} series of {label} through the C oracle ({out.size} output points, {dt:.2f} s)"}


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference's CPU pipeline on this box's
    host cores, on the same workload, config and metric as the device arm."""
    import bench_inputs as B

    if rank != 0:
        return
    if args.workload == "sweep":
        return run_sweep_reference(args)
    cfg = args.config
    N, L = B.CONFIG_SHAPES[cfg]
    if args.n_series:
        N = args.n_series
    pipe_cfg = B.pipeline_config(cfg)
    L_out = L
    for s in pipe_cfg["stages"]:
        if s["kind"] == "crop" and s["probability"] == 1.0:
            L_out = s["params"]["size"]
    label = WORKLOADS[cfg].split(":")[0]
    pts, dt, cores, rows = reference_cpu(pipe_cfg, L, args.ref_step_s, steps=args.steps,
                                         warmup=max(1, min(args.warmup, 2)))
    v = pts / dt
    # the reference's other two modes, once each: its own
    # Pipeline.run serially and with parallel=True (its GIL-bound thread pool)
    from oracle import ref_runner as R

    modes = {"processes": {"value": v, "cores": cores}}
    for name, par in (("serial", False), ("threads", True)):
        n = max(8, int(v / cores * (2.0 if par else 1.0) / L))
        p2, d2 = R.time_pipeline(pipe_cfg, n, L, par)
        modes[name] = {"value": p2 / d2, "cores": 1 if not par else (os.cpu_count() or 1), "series": n}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded random walks; BASELINE config shapes)",
        "config": config_dict(cfg, N, L, L_out, world, pipe_cfg),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"per step: {cores} processes x {rows} series of {label} ({pts} output "
                                   f"points) through the unmodified reference, per-sample loop"},
        "reference_modes": modes,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ device arm
def run_b200(args, rank, world, local_rank, dist_ok):
    import ctypes

    import torch
    import torch.distributed as dist

    from bench_inputs import CONFIG_SHAPES, device_walks, host_input, pipeline_config
    from paper_2601_03159_b200 import Batch, Pipeline, _engine, _native
    from paper_2601_03159_b200.sharding import shard_range

    cfg = args.config
    dev_index = env_int("SA_BENCH_DEVICE", local_rank)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    _native.ensure_device(dev_index)
    N, L = CONFIG_SHAPES[cfg]
    if args.n_series:
        N = args.n_series
    pipe_cfg = pipeline_config(cfg)
    pipe = Pipeline.parse(pipe_cfg)
    L_out = pipe.projected_length(L)
    r0, r1 = shard_range(N, rank, world)
    n = r1 - r0
    if cfg == 5:
        x = device_walks(n, L, 5, dev, row0=r0)
    else:
        x = torch.from_numpy(host_input(cfg, n=N)[r0:r1]).to(dev)
    rows_out = n * pipe.row_factor()
    out = torch.empty((rows_out, L_out), dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    lowered = _engine._lower(pipe.stages, 0, True)
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, series_offset=r0,
                              stream=stream.cuda_stream, lowered=lowered)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    if int(flags.item()):
        raise RuntimeError(f"kernel flagged {int(flags.item())}")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    launches0 = _native.launch_count()
    barrier()
    torch.cuda.synchronize()
    with Clocks(dev_index) as clk:
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                ev[2 * k].record(stream)
                step()
                ev[2 * k + 1].record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = _native.launch_count() - launches0
    step_ms = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    if int(flags.item()):
        raise RuntimeError(f"kernel flagged {int(flags.item())}")
    if args.check_out:
        os.makedirs(args.check_out, exist_ok=True)
        np.save(os.path.join(args.check_out, f"rank{rank}_of{world}.npy"), out.cpu().numpy())

    # e2e: host-buffer C ABI from pinned memory (H2D + kernel + D2H timed)
    e2e_s = e2e_pg_s = None
    h2d = 8 * n * L
    d2h = 8 * rows_out * L_out
    if not args.no_e2e:
        hin = x.cpu().pin_memory()
        hout = torch.empty((rows_out, L_out), dtype=torch.float64).pin_memory()
        arr, aux = lowered

        def e2e_step():
            rc = _native.lib().sa_pipeline_run_host(
                arr, len(pipe.stages), aux.ctypes.data_as(ctypes.c_void_p), aux.size, pipe.master_seed, r0,
                hin.data_ptr(), n, L, hout.data_ptr(), L_out)
            _native.check(rc, "sa_pipeline_run_host")

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        e2e_s = (time.perf_counter() - t0) / args.steps
        barrier()
        if not torch.equal(hout[: min(64, rows_out)].to(dev), out[: min(64, rows_out)]):
            raise RuntimeError("e2e output differs from the device-resident output")
        del hin, hout
        # the drop-in user's call: Pipeline.run(Batch(numpy)) on pageable arrays
        # (rank shards: the same call on the rank's rows with its global offset)
        hx = x.cpu().numpy()
        k_pg = max(1, min(args.steps, 3))

        def pageable_step():
            if world == 1:
                return pipe.run(Batch(hx)).values
            return _engine.run_host(pipe.stages, hx, pipe.master_seed, series_offset=r0, len_out=L_out)

        for _ in range(3):  # steady state of repeated calls (page-locked output blocks cached)
            res = pageable_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_pg):
            res = pageable_step()
        e2e_pg_s = (time.perf_counter() - t0) / k_pg
        barrier()
        if not torch.equal(torch.from_numpy(res[: min(64, rows_out)]).to(dev), out[: min(64, rows_out)]):
            raise RuntimeError("pageable e2e output differs from the device-resident output")
        del res, hx

    t = torch.tensor([total_ms / args.steps, sum(step_ms) / len(step_ms), e2e_s or 0.0, e2e_pg_s or 0.0,
                      float(launches)], dtype=torch.float64)
    if world > 1:
        t = reduce_timings(t, 4, dev)
    ms_per_step, kern_ms, e2e_max, e2e_pg_max, launches_all = [float(v) for v in t.tolist()]
    if rank != 0:
        return
    pts = N * pipe.row_factor() * L_out
    value = pts / (ms_per_step / 1e3)
    peak, peak_src = measured_peak()
    bytes_launch = 8 * (n * L + rows_out * L_out)
    achieved = bytes_launch / (kern_ms / 1e3) / 1e9
    props = torch.cuda.get_device_properties(dev)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded random walks / BASELINE config distributions; no corpus available)",
        "config": config_dict(cfg, N, L, L_out, world, pipe_cfg),
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(cfg), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_launch, "kernel_ms": kern_ms,
                     "peak_north_star": 8000.0, "frac_north_star": achieved / 8000.0},
        "input_points_per_s": N * L / (ms_per_step / 1e3),
        "gpu_launches": int(launches_all),
        "clocks": clk.summary(),
        "device": {"name": torch.cuda.get_device_name(dev), "sms": props.multi_processor_count,
                   "numpy": np.__version__, "torch": torch.__version__, "build_sha16": build_sha16()},
    }
    ff = fft_flops_per_series(cfg, L)
    if ff:  # the FFT-bearing config's compute-side bound (FP64 FMA pipe)
        fpk, fsrc = fp64_peak()
        ach_f = ff * n / (kern_ms / 1e3) / 1e12
        line["fp64_roofline"] = {"achieved": ach_f, "peak": fpk, "unit": "TFLOP/s", "frac": ach_f / fpk,
                                 "peak_source": fsrc, "flops_per_series": ff,
                                 "note": "rfft + irfft = 2 x 2.5 L log2 L per series (SURVEY.md 8(d))"}
    # the kernel is issue bound (numpy-exact RNG and FP64 arithmetic per element):
    # warp-instructions per launch (ncu capture; valid only for the build it
    # was captured on) over the live kernel time, against 4 issue slots x SMs
    # x the sampled SM clock
    ins = _profile_json("ncu_instructions.json").get(f"config{cfg}")
    if isinstance(ins, dict) and N == CONFIG_SHAPES[cfg][0]:
        sm_mhz = line["clocks"].get("sm_mhz") or 1965.0
        peak_issue = 4.0 * props.multi_processor_count * sm_mhz * 1e6
        ach_issue = ins["instructions"] / world / (kern_ms / 1e3)
        line["issue_roofline"] = {"achieved": ach_issue, "peak": peak_issue, "unit": "warp-instructions/s",
                                  "frac": ach_issue / peak_issue,
                                  "instructions_per_launch": ins["instructions"] / world,
                                  "captured_build_sha16": ins.get("build_sha16"),
                                  "stale": ins.get("build_sha16") != build_sha16(),
                                  "source": "profiles/ncu_instructions.json (ncu smsp__inst_executed.sum)"}
    if e2e_s is not None:
        line["e2e"] = {"value": pts / e2e_max, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
                       "d2h_bytes_per_step": d2h * world,
                       "path": "sa_pipeline_run_host (C ABI) from page-locked host buffers"}
        line["e2e_pageable"] = {"value": pts / e2e_pg_max, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
                                "d2h_bytes_per_step": d2h * world, "steps": max(1, min(args.steps, 3)),
                                "path": "Pipeline.run(Batch(numpy)) on pageable numpy arrays (the drop-in call)"}
    if world == 1 and not args.no_cpu:
        label = WORKLOADS[cfg].split(":")[0]
        line["cpu_baseline"] = reference_baseline(pipe_cfg, L, label)
        line["cpu_port"] = port_baseline(pipe_cfg, L, label)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ sweep
def run_sweep(args, rank, world, local_rank, dist_ok):
    """BASELINE config 5's sweep: one step = the 20-augmenter chain over all
    100 datasets (one fused launch each), datasets dealt to ranks round-robin
    by size; inputs resident in HBM.  e2e = Pipeline.run(Batch(numpy)) per
    dataset (host numpy in and out, the drop-in call)."""
    import torch
    import torch.distributed as dist

    import bench_inputs as B
    from paper_2601_03159_b200 import Batch, _engine, _native

    dev_index = env_int("SA_BENCH_DEVICE", local_rank)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    _native.ensure_device(dev_index)
    ds = sorted(B.sweep_datasets(), key=lambda d: -d[1] * d[2])
    mine = ds[rank::world]
    work = []
    for i, n, L in mine:
        pipe = B.sweep_pipeline(L, i)
        hx = B.synthetic_walks(n, L, i)
        x = torch.from_numpy(hx).to(dev)
        out = torch.empty((n, L), dtype=torch.float64, device=dev)
        work.append((pipe, hx, x, out, _engine._lower(pipe.stages, 0, True)))
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    # The datasets are independent: small ones occupy a few SMs for the
    # latency of one row's chain, so they run on K side streams (largest
    # first, each to the least-loaded stream by points) and overlap.
    K = max(1, args.sweep_streams)
    side = [torch.cuda.Stream(device=dev) for _ in range(K)]
    # Datasets of less than one wave of rows are latency bound (one warp runs
    # a row's whole chain): they go first, longest rows first, so their
    # latency overlaps the large datasets instead of forming the step's tail.
    wave = torch.cuda.get_device_properties(dev).multi_processor_count * 12
    order = sorted(range(len(work)), key=lambda k: (work[k][2].shape[0] >= wave, -work[k][2].shape[1]
                                                    if work[k][2].shape[0] < wave else -work[k][2].numel()))
    if env_int("SA_SWEEP_ORDER", 1) == 0:
        order = list(range(len(work)))
    work = [work[k] for k in order]
    load = [0] * K
    assign = []
    for pipe, hx, x, out, low in work:
        q = load.index(min(load))
        load[q] += x.numel()
        assign.append(q)
    fork, joins = torch.cuda.Event(), [torch.cuda.Event() for _ in range(K)]

    def step():
        fork.record(stream)
        for q in range(K):
            side[q].wait_event(fork)
        for (pipe, hx, x, out, low), q in zip(work, assign):
            _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, stream=side[q].cuda_stream,
                                  lowered=low)
        for q in range(K):
            joins[q].record(side[q])
            stream.wait_event(joins[q])

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    assert int(flags.item()) == 0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    launches0 = _native.launch_count()
    if world > 1:
        dist.barrier()
    with Clocks(dev_index) as clk:
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for k in range(args.steps):
                step()
                ev[k + 1].record(stream)
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms = ev[0].elapsed_time(ev[-1]) / args.steps
    # e2e through the public call on host numpy arrays, with the reference's
    # own protocol per dataset (bench.py:65-81 _time_runs: the Batch is given,
    # one warm-up call, then `repeats` timed calls, median): summed medians
    k_e2e = max(3, min(args.steps, 5))
    e2e_s = 0.0
    for pipe, hx, x, out, low in (work if not args.no_e2e else []):
        b = Batch(hx)
        pipe.run(b)
        ts = []
        for _ in range(k_e2e):
            t0 = time.perf_counter()
            res = pipe.run(b).values
            ts.append(time.perf_counter() - t0)
        e2e_s += statistics.median(ts)
    pipe, hx, x, out, low = work[-1]
    if not args.no_e2e and not np.array_equal(res.view(np.uint64), out.cpu().numpy().view(np.uint64)):
        raise RuntimeError("sweep e2e output differs from the device-resident output")
    t = torch.tensor([ms, e2e_s, float(launches)], dtype=torch.float64)
    if world > 1:
        t = reduce_timings(t, 2, dev)
    ms, e2e_s, launches = [float(v) for v in t.tolist()]
    if rank != 0:
        return
    pts = sum(n * L for _, n, L in ds)
    peak, src = measured_peak()
    line = {
        "metric": METRIC, "value": pts / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random walks, seed = dataset id)",
        "config": dict(sweep_config_dict(ds, world), streams=K),
        "roofline": {"bound": "hbm", "achieved": 16 * pts / world / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": 16 * pts / world / (ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": src,
                     "note": "100 launches of 0.06-4 ms: mostly latency / tail bound, not HBM"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": None if args.no_e2e else {"value": pts / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * pts,
                                         "d2h_bytes_per_step": 8 * pts,
                "path": "Pipeline.run(batch) per dataset on pageable numpy input, the reference's _time_runs protocol "
                        "(warm-up + median of %d calls per dataset, summed)" % k_e2e},
        "device": {"name": torch.cuda.get_device_name(dev), "build_sha16": build_sha16()},
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = sweep_reference_baseline(ds, target_s=10.0)
    print(json.dumps(line), flush=True)


def sweep_config_dict(ds, world):
    return {"workload": WORKLOADS["sweep"], "datasets": len(ds), "points": sum(n * L for _, n, L in ds),
            "n_range": [min(d[1] for d in ds), max(d[1] for d in ds)],
            "len_range": [min(d[2] for d in ds), max(d[2] for d in ds)],
            "parallelism": f"datasets dealt to {world} rank(s), no collective; per rank on concurrent streams",
            "l2": "datasets of 4 KB - 0.5 GB; consecutive launches touch different data"}


def sweep_reference_baseline(ds, target_s: float) -> dict:
    """The genuine reference on every dataset of the sweep, a bounded sample
    of series per dataset (same fraction everywhere), all host cores: a pool
    task per (dataset, block of series)."""
    import bench_inputs as B
    from oracle import ref_runner as R

    cores = os.cpu_count() or 1
    pool = R.ProcessPool(cores)
    try:
        def tasks_for(frac):
            """Worker w gets slice w of every dataset's sampled series (the
            same number of series of each dataset per worker: balanced)."""
            per = [[] for _ in range(cores)]
            pts = 0
            for i, n, L in ds:
                rows = max(1, int(round(n * frac / cores)))
                cfgj = json.dumps(B.sweep_config(L, i), sort_keys=True)
                for w in range(cores):
                    per[w].append((cfgj, L, w * rows, rows, i * 1_000_003 + w))
                pts += cores * rows * L
            return per, pts

        def run(frac):
            tasks, pts = tasks_for(frac)
            pool.assign(tasks)
            pool.run()
            return pts, pool.run()[1]

        total = sum(n * L for _, n, L in ds)
        p, dt = run(0.001)
        frac = min(1.0, target_s * (p / dt) / total)
        p, dt = run(frac)
    finally:
        pool.close()
    return {"value": p / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{frac:.4f} of the series of every dataset (at least one per process) through the "
                      f"unmodified reference (per-sample loop, each of {cores} processes a slice of every "
                      f"dataset): {p} output points in {dt:.2f} s"}


def run_sweep_reference(args):
    import bench_inputs as B

    ds = sorted(B.sweep_datasets(), key=lambda d: -d[1] * d[2])
    base = sweep_reference_baseline(ds, target_s=args.ref_step_s * 4)
    v = base["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": env_int("WORLD_SIZE", 1),
        "steps": 1, "warmup": 1, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random walks, seed = dataset id)",
        "config": sweep_config_dict(ds, env_int("WORLD_SIZE", 1)), "cpu_baseline": base,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_suite(args):
    """Device-resident kernel throughput of configs 1-5 and of the config-5
    sweep (100 datasets) -- documentation numbers, not the driver's line."""
    import torch

    import bench_inputs
    from paper_2601_03159_b200 import _engine, _native

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    _native.ensure_device(0)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)

    def timed(pipe, x, reps=5):
        out = torch.empty((x.shape[0] * pipe.row_factor(), pipe.projected_length(x.shape[1])),
                          dtype=torch.float64, device=dev)
        low = _engine._lower(pipe.stages, 0, True)
        for _ in range(2):
            _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            _engine.launch_device(pipe.stages, x, out, flags, pipe.master_seed, lowered=low)
        b.record()
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
        return a.elapsed_time(b) / reps, out.numel()

    res = {}
    for cfg in (1, 2, 3, 4, 5):
        N, L = bench_inputs.CONFIG_SHAPES[cfg]
        x = bench_inputs.device_walks(N, L, 5, dev) if cfg == 5 else \
            torch.from_numpy(bench_inputs.host_input(cfg)).to(dev)
        ms, pts = timed(bench_inputs.pipeline(cfg), x)
        byt = 8 * (x.numel() + pts)
        res[f"config{cfg}"] = {"ms": ms, "gpts_s": pts / ms / 1e6, "hbm_gbs": byt / ms / 1e6,
                               "hbm_frac": byt / ms / 1e6 / measured_peak()[0]}
        ff = fft_flops_per_series(cfg, L)
        if ff:
            tf = ff * N / (ms / 1e3) / 1e12
            res[f"config{cfg}"].update(fp64_tflops=tf, fp64_frac=tf / fp64_peak()[0])
        if cfg in (1, 2):  # launch-bound sizes: the same chain replayed from a CUDA graph
            run = bench_inputs.pipeline(cfg).capture_device(x.contiguous())
            for _ in range(3):
                run.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                run.replay()
            b.record()
            torch.cuda.synchronize()
            run.check()
            gms = a.elapsed_time(b) / 20
            res[f"config{cfg}_graph"] = {"ms": gms, "gpts_s": pts / gms / 1e6, "hbm_gbs": byt / gms / 1e6,
                                         "hbm_frac": byt / gms / 1e6 / measured_peak()[0]}
        del x
    tot_ms, tot_pts = 0.0, 0
    for i, n, L in bench_inputs.sweep_datasets():
        x = torch.from_numpy(bench_inputs.synthetic_walks(n, L, i)).to(dev)
        ms, pts = timed(bench_inputs.sweep_pipeline(L, i), x, reps=3)
        tot_ms += ms
        tot_pts += pts
    res["sweep100"] = {"ms": tot_ms, "gpts_s": tot_pts / tot_ms / 1e6, "datasets": 100, "points": tot_pts}
    print(json.dumps(res), flush=True)




DS_SHAPE = (100_000, 1024)
DS_WORKLOAD = ("datafiles: TS dataset of 100,000 x 1,024 random walks (repr floats, 3 header lines, "
               "labels): parse_dataset + format_dataset, text resident in HBM")


def ds_text(n, L):
    """The synthetic dataset: random walks formatted by the device codec and
    checked against the oracle's formatting on a sample of rows."""
    import torch

    from bench_inputs import device_walks
    from paper_2601_03159_b200 import format_dataset_device
    from oracle import datafiles_oracle as O

    x = device_walks(n, L, 7, torch.device("cuda", 0))
    headers = ("@problemName walks", "@timeStamps false", "@data")
    labels = tuple(f"c{r % 5}" for r in range(n))
    data = format_dataset_device(x, "ts", headers, labels)
    head = "".join(h + "\n" for h in headers)
    sample = O.format_rows(x[:50].cpu().numpy(), "ts", headers, labels[:50])
    if not data.startswith(sample.encode()) or not data.startswith(head.encode()):
        raise RuntimeError("device formatting differs from the oracle")
    return x, data, headers, labels


def ds_cpu_baseline(data: bytes, n: int, target_rows: int = 3000):
    """The reference algorithm (oracle/datafiles_oracle.py: Python's float /
    repr, as the reference) on the first rows of the same file, one core."""
    from oracle import datafiles_oracle as O

    text = data.decode()
    cut = 0
    for _ in range(3 + target_rows):
        cut = text.index("\n", cut) + 1
    part = text[:cut]
    t0 = time.perf_counter()
    fmt, headers, labels, values = O.parse(part)
    t1 = time.perf_counter()
    O.format_rows(values, fmt, headers, labels)
    t2 = time.perf_counter()
    nbytes = len(part.encode())
    return {"value": 2 * nbytes / (t2 - t0), "unit": "B/s", "cores": 1, "kind": "port",
            "sample": f"first {target_rows} of {n} rows ({nbytes} bytes) parsed + formatted "
                      f"({t1 - t0:.2f} s + {t2 - t1:.2f} s)",
            "parse_bps": nbytes / (t1 - t0), "format_bps": nbytes / (t2 - t1)}


def run_side_reference(args, rank):
    """--impl reference for the transforms / dtw legs: the CPU path alone."""
    if rank != 0:
        return
    from bench_inputs import ar2_input, host_input

    if args.workload == "transforms":
        host = ar2_input(4000, TR_SHAPE[1])
        for _ in range(args.warmup):
            transforms_cpu(host, rows=500)
        base = [transforms_cpu(host) for _ in range(args.steps)]
        metric, unit, wl = "transformed points/s", "points/s", TR_WORKLOAD
    else:
        a = host_input(2, 32 * (os.cpu_count() or 1))
        b = a[:, ::-1].copy()
        for _ in range(args.warmup):
            dtw_cpu(a, b, pairs=8)
        base = [dtw_cpu(a, b) for _ in range(args.steps)]
        metric, unit, wl = "DTW cells/s", "cells/s", DTW_WORKLOAD
    v = sum(x["value"] for x in base) / len(base)
    print(json.dumps({
        "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "replicas",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": wl},
        "cpu_baseline": dict(base[-1], value=v),
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def run_datafiles_reference(args, rank):
    """The reference algorithm on the host (oracle port), bounded sample."""
    if rank != 0:
        return
    from oracle import datafiles_oracle as O

    n, L = DS_SHAPE
    rng = np.random.default_rng(7)
    rows = 2000
    x = np.cumsum(rng.normal(0, 1, (rows, L)), axis=1)
    headers = ("@problemName walks", "@timeStamps false", "@data")
    labels = tuple(f"c{r % 5}" for r in range(rows))
    text = O.format_rows(x, "ts", headers, labels)
    for _ in range(args.warmup):
        O.format_rows(O.parse(text)[3], "ts", headers, labels)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fmt, h, lab, v = O.parse(text)
        O.format_rows(v, fmt, h, lab)
    dt = (time.perf_counter() - t0) / args.steps
    nb = len(text.encode())
    val = 2 * nb / dt
    print(json.dumps({
        "impl": "reference", "metric": "dataset text bytes/s (parse + format)", "value": val, "unit": "B/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "replicas", "vs_baseline": None, "dtype": "f64+u8",
        "data": "synthetic (seeded random walks)",
        "config": {"workload": DS_WORKLOAD, "sample_series": rows, "len": L, "text_bytes": nb},
        "cpu_baseline": {"value": val, "unit": "B/s", "cores": 1, "kind": "port",
                         "sample": f"{rows} of {n} rows per step"},
        "e2e": {"value": val, "unit": "B/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def run_datafiles(args, rank, world, local_rank):
    """One step = parse the resident TS text into the batch + format the
    batch back into text (the two ends of `seriesaug augment`)."""
    import torch

    from paper_2601_03159_b200 import _native, format_dataset_device, parse_dataset_device
    from paper_2601_03159_b200.datafiles import _parse_device, format_dataset_to_device

    if rank != 0:
        return
    torch.cuda.set_device(0)
    _native.ensure_device(0)
    n, L = DS_SHAPE
    if args.n_series:
        n = args.n_series
    x, data, headers, labels = ds_text(n, L)
    nbytes = len(data)
    d_text = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    hv = memoryview(data)

    def step(pev=None, fev=None):
        dd = _parse_device(d_text, nbytes, hv, None, True, events=pev)
        out = format_dataset_to_device(dd.values, dd.format, dd.header_lines, dd.labels, events=fev)
        return dd, out

    for _ in range(args.warmup):
        dd, out = step()
    torch.cuda.synchronize()
    if not torch.equal(out, d_text) or not torch.equal(dd.values, x):
        raise RuntimeError("parse/format round trip differs")
    launches0 = _native.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    pev, fev = [], []
    torch.cuda.synchronize()
    with Clocks(local_rank) as clk:
        for k in range(args.steps):
            ev[2 * k].record()
            step(pev, fev)
            ev[2 * k + 1].record()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)) / args.steps
    p_ms = sum(a.elapsed_time(b) for a, b in pev) / len(pev)
    f_ms = sum(a.elapsed_time(b) for a, b in fev) / len(fev)
    # e2e through the public calls with host buffers: file bytes -> batch in
    # host memory; host batch -> file bytes
    # the public calls a user makes with host buffers: parse_dataset (text ->
    # DatasetFile with a numpy batch) and format_dataset (DatasetFile -> text)
    from paper_2601_03159_b200 import Batch, DatasetFile, format_dataset, parse_dataset

    text = data.decode()
    host_ds = DatasetFile(batch=Batch(x.cpu().numpy()), format="ts", header_lines=headers, labels=labels)
    format_dataset(host_ds)  # warm-up: staging buffer
    t0 = time.perf_counter()
    for _ in range(args.steps):
        got = parse_dataset(text)
        out_text = format_dataset(host_ds)
    e2e_s = (time.perf_counter() - t0) / args.steps
    if out_text != text or not np.array_equal(got.batch.values, host_ds.batch.values):
        raise RuntimeError("e2e round trip differs")
    peak, peak_src = measured_peak()
    vals_b = 8 * n * L
    # dominant kernels: rows_parse (text in, values out) and row_write
    # (values in, text out); each moves text + values bytes once
    ach_p = (nbytes + vals_b) / (p_ms / 1e3) / 1e9
    ach_f = (nbytes + vals_b) / (f_ms / 1e3) / 1e9
    dom = "rows_parse_kernel" if p_ms >= f_ms else "row_write_kernel"
    ach = ach_p if p_ms >= f_ms else ach_f
    line = {
        "metric": "dataset text bytes/s (parse + format)", "value": 2 * nbytes / (ms / 1e3), "unit": "B/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "replicas", "vs_baseline": None, "dtype": "f64+u8",
        "data": "synthetic (seeded random walks, device-formatted; oracle-checked sample)",
        "config": {"workload": DS_WORKLOAD, "n_series": n, "len": L, "text_bytes": nbytes,
                   "rows_parse_ms": p_ms, "row_write_ms": f_ms, "rows_parse_gbs": ach_p, "row_write_gbs": ach_f,
                   "l2": "text and batch larger than L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "peak_source": peak_src, "kernel": dom,
                     "algorithmic_bytes_per_launch": nbytes + vals_b},
        "e2e": {"value": 2 * nbytes / e2e_s, "unit": "B/s", "h2d_bytes_per_step": nbytes + vals_b,
                "d2h_bytes_per_step": nbytes + vals_b},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if not args.no_cpu:
        line["cpu_baseline"] = ds_cpu_baseline(data, n)
    print(json.dumps(line), flush=True)


TR_SHAPE = (50_000, 2048)
TR_WORKLOAD = ("transforms: fft_forward + fft_inverse + dct_forward + dct_inverse (orthonormal) on 50,000 x 2,048 "
               "AR(2) series (config 3 shape), device resident")


def _timed_steps(fn, steps, warmup, stream=None):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with Clocks(0) as clk:
        ev[0].record()
        for k in range(steps):
            fn()
            ev[k + 1].record()
        torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    return sum(per) / steps, clk.summary()


def run_transforms(args, rank):
    """One step = rfft + irfft + DCT-II + DCT-III of the whole batch
    (freqtransform.py:91-116) through the C ABI on resident buffers."""
    import ctypes

    import torch

    from bench_inputs import ar2_input
    from paper_2601_03159_b200 import Batch, _native, dct_forward, dct_inverse, fft_forward, fft_inverse

    if rank != 0:
        return
    torch.cuda.set_device(0)
    _native.ensure_device(0)
    n, L = TR_SHAPE
    if args.n_series:
        n = args.n_series
    host = ar2_input(n, L)
    x = torch.from_numpy(host).cuda()
    B = L // 2 + 1
    re = torch.empty((n, B), dtype=torch.float64, device="cuda")
    im = torch.empty_like(re)
    back = torch.empty_like(x)
    dc = torch.empty_like(x)
    idc = torch.empty_like(x)
    lib = _native.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    launches0 = _native.launch_count()

    def step():
        _native.check(lib.sa_fft_forward(x.data_ptr(), n, L, re.data_ptr(), im.data_ptr(), st))
        _native.check(lib.sa_fft_inverse(re.data_ptr(), im.data_ptr(), n, L, back.data_ptr(), st))
        _native.check(lib.sa_dct_forward(x.data_ptr(), n, L, dc.data_ptr(), st))
        _native.check(lib.sa_dct_inverse(dc.data_ptr(), n, L, idc.data_ptr(), st))

    ms, clocks = _timed_steps(step, args.steps, args.warmup)
    launches = (_native.launch_count() - launches0) // (args.steps + args.warmup) * args.steps
    err = max(float((back - x).abs().max()), float((idc - x).abs().max()))
    if err > 1e-8 * max(1.0, float(x.abs().max())):
        raise RuntimeError(f"transform round trip error {err}")
    pts = 4 * n * L
    byts = 8 * n * (L + 2 * B) * 2 + 8 * n * L * 4  # rfft/irfft: L + 2B each; dct/idct: 2L each
    # e2e through the public API (host Batch in, host arrays out)
    b = Batch(host)
    spec = fft_forward(b)  # warm-up: staging buffers
    fft_inverse(spec)
    dct_inverse(dct_forward(b))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        spec = fft_forward(b)
        fft_inverse(spec)
        dct_inverse(dct_forward(b))
    e2e_s = (time.perf_counter() - t0) / args.steps
    peak, src = measured_peak()
    ach = byts / (ms / 1e3) / 1e9
    line = {
        "metric": "transformed points/s", "value": pts / (ms / 1e3), "unit": "points/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "replicas", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded AR(2), BASELINE config 3 distribution)",
        "config": {"workload": TR_WORKLOAD, "n_series": n, "len": L, "round_trip_max_err": err,
                   "l2": "inputs larger than L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": ncu_traffic("transforms"), "peak_source": src, "algorithmic_bytes_per_step": byts,
                     "scope": "rfft_cta_kernel + irfft_cta_kernel + dct2_cta_kernel + dct3_cta_kernel (L = 2048: CTA-cooperative register FFT)"},
        "e2e": {"value": pts / e2e_s, "unit": "points/s", "h2d_bytes_per_step": 8 * n * L * 3 + 16 * n * B,
                "d2h_bytes_per_step": 8 * n * L * 3 + 16 * n * B},
        "gpu_launches": int(launches), "clocks": clocks,
    }
    if not args.no_cpu:
        line["cpu_baseline"] = transforms_cpu(host)
    print(json.dumps(line), flush=True)


def transforms_cpu(host, rows=4000):
    """The reference's own CPU path: numpy.fft.rfft/irfft and scipy.fft.dct/
    idct (freqtransform.py:93-116), one core as the reference calls them."""
    import scipy.fft

    x = host[:rows]
    L = x.shape[1]
    t0 = time.perf_counter()
    spec = np.fft.rfft(x, axis=1)
    np.fft.irfft(spec, n=L, axis=1)
    c = scipy.fft.dct(x, type=2, norm="ortho", axis=1)
    scipy.fft.idct(c, type=2, norm="ortho", axis=1)
    dt = time.perf_counter() - t0
    return {"value": 4 * x.size / dt, "unit": "points/s", "cores": 1, "kind": "reference",
            "sample": f"{rows} of {host.shape[0]} series through numpy/scipy pocketfft ({dt:.2f} s)"}


DTW_SHAPE = (10_000, 1024)
DTW_WORKLOAD = ("dtw: DTW distance of 10,000 (original, augmented) pairs of length 1,024 (config 2 walks vs their "
                "config-2-pipeline output at full length), one launch")


def run_dtw(args, rank):
    """One step = the DTW distance of every pair (the `quality` command's
    work, dtw.py:40-86) in one batched launch."""
    import ctypes

    import torch

    from bench_inputs import host_input
    from paper_2601_03159_b200 import (Batch, Drift, Jitter, Pipeline, Quantize, Reverse, _native,
                                       dtw_distances)

    if rank != 0:
        return
    torch.cuda.set_device(0)
    _native.ensure_device(0)
    n, L = DTW_SHAPE
    if args.n_series:
        n = args.n_series
    a_host = host_input(2, n)
    pipe = Pipeline(stages=(Jitter(0.1), Drift(0.5, 5, probability=0.5), Quantize(16, probability=0.5),
                            Reverse(probability=0.5)), master_seed=1)
    b_host = pipe.run(Batch(a_host)).values
    a, b = torch.from_numpy(a_host).cuda(), torch.from_numpy(b_host).cuda()
    dist = torch.empty(n, dtype=torch.float64, device="cuda")
    lib = _native.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    launches0 = _native.launch_count()

    def step():
        _native.check(lib.sa_dtw_batch(a.data_ptr(), b.data_ptr(), n, L, L, dist.data_ptr(), st))

    ms, clocks = _timed_steps(step, args.steps, args.warmup)
    launches = (_native.launch_count() - launches0) // (args.steps + args.warmup) * args.steps
    # spot check against the oracle (bitwise: one addition per cell)
    from oracle import oracle as O

    got = dist.cpu().numpy()
    for i in (0, n // 2, n - 1):
        if O.dtw(a_host[i], b_host[i])[0] != got[i]:
            raise RuntimeError("DTW distance differs from the oracle")
    cells = n * L * L
    ba, bb = Batch(a_host), Batch(b_host)
    dtw_distances(ba, bb)  # warm-up: staging buffers
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dtw_distances(ba, bb)
    e2e_s = (time.perf_counter() - t0) / args.steps
    peak, src = measured_peak()
    byts = 8 * n * 2 * L + 8 * n
    ach = byts / (ms / 1e3) / 1e9
    line = {
        "metric": "DTW cells/s", "value": cells / (ms / 1e3), "unit": "cells/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "replicas",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded walks and their augmented copies)",
        "config": {"workload": DTW_WORKLOAD, "pairs": n, "len_a": L, "len_b": L,
                   "l2": "inputs smaller than L2: compute bound, L2 residency irrelevant"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "peak_source": src, "algorithmic_bytes_per_step": byts,
                     "scope": "dtw_batch_kernel (an O(L^2) dynamic programme per pair: issue bound, not HBM)"},
        "e2e": {"value": cells / e2e_s, "unit": "cells/s", "h2d_bytes_per_step": 16 * n * L,
                "d2h_bytes_per_step": 8 * n},
        "gpu_launches": int(launches), "clocks": clocks,
    }
    if not args.no_cpu:
        line["cpu_baseline"] = dtw_cpu(a_host, b_host)
    print(json.dumps(line), flush=True)


def dtw_cpu(a, b, pairs=None):
    """The reference algorithm restated in C (oracle sao_dtw), all host
    threads over a sample of pairs."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    threads = os.cpu_count() or 1
    pairs = min(pairs or 32 * threads, a.shape[0])
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: O.dtw(a[i], b[i]), range(pairs)))
    dt = time.perf_counter() - t0
    cells = pairs * a.shape[1] * b.shape[1]
    return {"value": cells / dt, "unit": "cells/s", "cores": threads, "kind": "port",
            "sample": f"{pairs} pairs through the C oracle ({dt:.2f} s)"}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int) -> int:
    """No torchrun environment but --gpus N > 1: launch the N ranks here, one
    process per GPU, with the variables torchrun would set."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    return max(abs(p.wait()) for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-series", type=int, default=0, help="override the config's series count")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--suite", action="store_true", help="configs 1-5 + sweep, device-resident, one JSON")
    ap.add_argument("--workload", default="pipeline",
                    choices=["pipeline", "sweep", "datafiles", "transforms", "dtw"],
                    help="sweep: BASELINE config 5's 100-dataset sweep; datafiles / transforms / dtw: the "
                         "SURVEY.md §8(f) next rows")
    ap.add_argument("--check-out", default="", help="directory: each rank saves its output shard (tests)")
    ap.add_argument("--sweep-streams", type=int, default=4, help="sweep: concurrent streams per GPU")
    ap.add_argument("--ref-step-s", type=float, default=3.0,
                    help="reference arm: seconds of host-core work per timed step")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":  # rank 0 alone runs the CPU reference
            os.environ["WORLD_SIZE"] = str(args.gpus)
        else:
            sys.exit(spawn_ranks(args.gpus))
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.workload in ("transforms", "dtw"):
        if args.impl == "reference":
            run_side_reference(args, rank)
        elif args.workload == "transforms":
            run_transforms(args, rank)
        else:
            run_dtw(args, rank)
        return
    if args.workload == "datafiles":
        if args.impl == "reference":
            run_datafiles_reference(args, rank)
        else:
            run_datafiles(args, rank, world, local_rank)
        return
    if args.suite:
        run_suite(args)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = os.environ.get("SA_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dev = torch.device("cuda", env_int("SA_BENCH_DEVICE", local_rank))
            torch.cuda.set_device(dev)
            dist.init_process_group("nccl", device_id=dev)
        else:  # tests: several ranks sharing one GPU synchronise over gloo
            dist.init_process_group(backend)
    try:
        if args.workload == "sweep":
            run_sweep(args, rank, world, local_rank, True)
        else:
            run_b200(args, rank, world, local_rank, True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
