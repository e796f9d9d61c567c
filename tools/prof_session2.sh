#!/bin/bash
# ncu --set full captures of the secondary kernels (one kernel each), run
# only after the same command exits 0 without ncu.
mkdir -p gpurun_out
run() {  # name, kernel regex, command...
  local name=$1 k=$2; shift 2
  timeout 300 "$@" > /dev/null 2>&1 || { echo "$name: plain run failed"; return; }
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$k" -s 2 -c 1 \
      -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1; echo "$name rc=$?"
}
run cfg3 chain_kernel python tools/prof_one.py --config 3 --n 50000
run dtw dtw_batch python bench.py --workload dtw --steps 1 --warmup 1 --no-cpu --n-series 4000
run dct dct_kernel python bench.py --workload transforms --steps 1 --warmup 1 --no-cpu --n-series 20000
run rfft rfft_kernel python bench.py --workload transforms --steps 1 --warmup 1 --no-cpu --n-series 20000
run rowsparse rows_parse python bench.py --workload datafiles --steps 1 --warmup 1 --no-cpu --n-series 20000
run rowwrite row_write python bench.py --workload datafiles --steps 1 --warmup 1 --no-cpu --n-series 20000
# summarise on the box (the reports are too large to bring back together)
for name in cfg3 dtw dct rfft rowsparse rowwrite; do
  [ -f gpurun_out/prof_$name.ncu-rep ] || continue
  python tools/ncu_summary.py gpurun_out/prof_$name.ncu-rep gpurun_out/r01_ncu_$name.txt "$name" > /dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$name.csv 2>/dev/null
  python tools/src_hot.py gpurun_out/src_$name.csv 25 >> gpurun_out/r01_ncu_$name.txt 2>&1
  rm -f gpurun_out/prof_$name.ncu-rep gpurun_out/src_$name.csv
done
ls gpurun_out/r01_ncu_*
