export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
{
for g in 1 2 4; do
  echo "== groups $g"
  SA_SYNC_GROUPS=$g AB_N=200000 timeout 300 python tools/ab_timing.py ab/libgrp.so -- CONFIG5 | tail -1
done
SA_SYNC_GROUPS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "config5 or golden_pipeline or baseline_config or exact_op" 2>&1 | tail -3
SA_SYNC_GROUPS=1 AB_N=100000 AB_L=1500 timeout 300 python tools/ab_timing.py ab/libst.so ab/libgrp.so -- CONFIG4 | tail -2
} > gpurun_out/grp.txt 2>&1
cat gpurun_out/grp.txt
