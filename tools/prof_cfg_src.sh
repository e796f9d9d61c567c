#!/bin/bash
# Source-level hot spots of the chain kernel for a bench config: CFG=4 N=100000 bash tools/prof_cfg_src.sh
cd "$(dirname "$0")/.."
C=${CFG:-5}
P="python tools/prof_one.py --config $C --n ${N:-100000}"
$P > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"${K:-chain_kernel}" -s 2 -c 1 -o gpurun_out/cfg$C $P > gpurun_out/cfg${C}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/cfg$C.ncu-rep gpurun_out/ncu_cfg${C}_src.txt cfg$C > /dev/null
ncu -i gpurun_out/cfg$C.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/cfg${C}_src.csv 2>/dev/null
python tools/src_hot.py gpurun_out/cfg${C}_src.csv 50 >> gpurun_out/ncu_cfg${C}_src.txt
gzip -f gpurun_out/cfg${C}_src.csv
rm -f gpurun_out/cfg$C.ncu-rep
