#!/bin/bash
# A/B timing of ab/lib*.so builds on the config chains (run under gpurun)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
libs="$@"
{
AB_N=50000 timeout 300 python tools/ab_timing.py $libs -- CONFIG5 CONFIG2 copy jitter app fmask_chain
AB_N=100000 AB_L=1500 timeout 300 python tools/ab_timing.py $libs -- CONFIG4
AB_N=50000 AB_L=2048 timeout 300 python tools/ab_timing.py $libs -- CONFIG3
} > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
