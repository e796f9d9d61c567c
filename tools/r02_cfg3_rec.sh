#!/bin/bash
# config-3 table-twiddle A/B, parity, and an ncu record of the config-5 bench kernel for the issue roofline
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
{
AB_N=50000 AB_L=2048 timeout 300 python tools/ab_timing.py ab/libwt3.so ab/libwt4.so -- CONFIG3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
} > gpurun_out/c3.txt 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD2 > gpurun_out/plain_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/prof_bench $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> gpurun_out/c3.txt
python tools/ncu_record.py gpurun_out/prof_bench.ncu-rep config5 >> gpurun_out/c3.txt 2>&1
rm -f gpurun_out/prof_bench.ncu-rep
cat gpurun_out/c3.txt
