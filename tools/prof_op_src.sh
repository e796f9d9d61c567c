#!/bin/bash
# Source-level ncu of single-op chains: bash tools/prof_op_src.sh jitter app ...
cd "$(dirname "$0")/.."
for op in "$@"; do
  P="python tools/prof_op.py $op 50000"
  $P > /dev/null 2>&1 || { echo "plain run $op failed"; continue; }
  ncu --set full --import-source on --clock-control none -k regex:chain_kernel -s 2 -c 1 -o gpurun_out/op_$op $P > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/op_$op.ncu-rep gpurun_out/ncu_op_$op.txt $op > /dev/null
  ncu -i gpurun_out/op_$op.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/op_${op}_src.csv 2>/dev/null
  python tools/src_hot.py gpurun_out/op_${op}_src.csv 60 >> gpurun_out/ncu_op_$op.txt
  gzip -f gpurun_out/op_${op}_src.csv; rm -f gpurun_out/op_$op.ncu-rep
done
