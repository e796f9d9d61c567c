#!/bin/bash
# ncu summaries of the CTA transform kernels (run on the GPU box after the bench exited 0)
cd "$(dirname "$0")/.."
B="python bench.py --workload transforms --steps 1 --warmup 3 --no-e2e --no-cpu"
$B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:_kernel --csv $B > gpurun_out/cta_launches.csv 2>/dev/null
for k in "^rfft_cta" irfft_cta dct2_cta dct3_cta; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/${k#^} $B > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/${k#^}.ncu-rep gpurun_out/ncu_${k#^}.txt ${k#^} > /dev/null
  ncu -i gpurun_out/${k#^}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${k#^}_src.csv 2>/dev/null
  python tools/src_hot.py gpurun_out/${k#^}_src.csv 25 >> gpurun_out/ncu_${k#^}.txt
  rm -f gpurun_out/${k#^}.ncu-rep gpurun_out/${k#^}_src.csv
done
# config 3's spectral-only chain kernel
python tools/prof_one.py --config 3 --n 50000 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:spectral_cta -s 2 -c 1 -o gpurun_out/spectral_cta python tools/prof_one.py --config 3 --n 50000 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/spectral_cta.ncu-rep gpurun_out/ncu_spectral_cta.txt spectral_cta > /dev/null
ncu -i gpurun_out/spectral_cta.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/spectral_cta_src.csv 2>/dev/null
python tools/src_hot.py gpurun_out/spectral_cta_src.csv 25 >> gpurun_out/ncu_spectral_cta.txt
rm -f gpurun_out/spectral_cta.ncu-rep gpurun_out/spectral_cta_src.csv
