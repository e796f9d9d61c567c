#!/bin/bash
# A/B + source profiles for configs 3 and 4 (run under gpurun)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
{
AB_N=100000 AB_L=1500 timeout 300 python tools/ab_timing.py ab/libst.so ab/libwt1.so -- CONFIG4
AB_N=50000 timeout 300 python tools/ab_timing.py ab/libst.so ab/libwt1.so -- CONFIG5 speed_warp convolve
} > gpurun_out/ab2.txt 2>&1
CFG=3 N=50000 K=spectral_cta bash tools/prof_cfg_src.sh
CFG=4 N=100000 bash tools/prof_cfg_src.sh
cat gpurun_out/ab2.txt
