#!/bin/bash
# Full bench + reference arm + ncu evidence (run under gpurun).
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
lscpu > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch-list rc=$?"
CMD2="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD2 > gpurun_out/plain_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o gpurun_out/prof_bench $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
