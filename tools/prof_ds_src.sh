#!/bin/bash
# Source-level profile of the chain kernel on one sweep dataset: DS=65 bash tools/prof_ds_src.sh
cd "$(dirname "$0")/.."
D=${DS:-65}
P="python tools/prof_one.py --sweep-ds $D"
$P > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"${K:-chain_kernel}" -s 2 -c 1 -o gpurun_out/ds$D $P > gpurun_out/ds${D}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/ds$D.ncu-rep gpurun_out/ncu_ds${D}_src.txt ds$D > /dev/null
ncu -i gpurun_out/ds$D.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ds${D}_src.csv 2>/dev/null
python tools/src_hot.py gpurun_out/ds${D}_src.csv 50 >> gpurun_out/ncu_ds${D}_src.txt
gzip -f gpurun_out/ds${D}_src.csv
rm -f gpurun_out/ds$D.ncu-rep
