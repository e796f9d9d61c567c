#!/bin/bash
# Round-2 final refresh: config-5 bench (+ reference arm), suite, sweep, launch list,
# ncu full capture (summary + traffic / instruction records tagged with the build hash)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
CMD2="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD2 > gpurun_out/plain_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/prof_bench $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_bench.ncu-rep gpurun_out/ncu_config5.txt "config5 bench kernel ($CMD2)" > /dev/null 2>&1; echo "summary rc=$?"
python tools/ncu_record.py gpurun_out/prof_bench.ncu-rep config5 > gpurun_out/ncu_record.txt 2>&1; echo "record rc=$?"
cp profiles/ncu_traffic.json profiles/ncu_instructions.json gpurun_out/
ncu -i gpurun_out/prof_bench.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/cfg5_final_src.csv 2>/dev/null; gzip -f gpurun_out/cfg5_final_src.csv
rm -f gpurun_out/prof_bench.ncu-rep
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --suite > gpurun_out/suite.json 2> gpurun_out/suite.err; echo "suite rc=$?"
timeout 900 python bench.py --workload sweep > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch-list rc=$?"
