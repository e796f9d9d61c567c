export PYTHONUNBUFFERED=1
for kv in "X=1" "SA_SYNC_EVERY=2" "SA_SYNC_EVERY=3" "SA_SYNC_EVERY=5" "SA_SYNC_EVERY=6" "SA_SCHEDULE_BITS=14" "SA_SCHEDULE_BITS=18" "SA_ADAPTIVE_SYNC=0" "SA_SYNC_POLICY=1"; do
  echo "$kv $(env $kv AB_N=200000 AB_ROUNDS=1 timeout 300 python tools/ab_timing.py paper_2601_03159_b200/_lib/libseriesaug_b200.so -- CONFIG5 | tail -1)"
done
