#!/bin/bash
# Source-level hot spots of the config-5 chain kernel (run on the GPU box).
cd "$(dirname "$0")/.."
P="python tools/prof_one.py --config 5 --n ${N:-100000}"
$P > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:chain_kernel -s 2 -c 1 -o gpurun_out/cfg5 $P > gpurun_out/cfg5_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/cfg5.ncu-rep gpurun_out/ncu_cfg5_src.txt cfg5 > /dev/null
ncu -i gpurun_out/cfg5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/cfg5_src.csv 2>/dev/null
python tools/src_hot.py gpurun_out/cfg5_src.csv 80 >> gpurun_out/ncu_cfg5_src.txt
gzip -f gpurun_out/cfg5_src.csv
rm -f gpurun_out/cfg5.ncu-rep
