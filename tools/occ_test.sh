export PYTHONUNBUFFERED=1
L=${L:-700}
{
for kv in "SA_WIDE=0 SA_CTA_WARPS=8" "SA_WIDE=0" "SA_WIDE=1"; do
  echo "L=$L $kv $(env $kv AB_L=$L AB_N=100000 AB_ROUNDS=2 timeout 300 python tools/ab_timing.py paper_2601_03159_b200/_lib/libseriesaug_b200.so -- SWCONV CHAIN5 | tail -2 | tr '\n' ' ')"
done
} > gpurun_out/occ_$L.txt 2>&1
cat gpurun_out/occ_$L.txt
