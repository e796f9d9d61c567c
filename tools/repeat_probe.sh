#!/bin/bash
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clk.csv &
SMI=$!
for i in 1 2 3 4; do
  timeout 120 python tools/sweep_cta.py 5 50000 2>&1 | grep "sched=1"
done
kill $SMI
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/clk.csv')))[1:]
sm=[int(r[0].split()[0]) for r in rows if r and r[0].strip()[:1].isdigit()]
print("sm clock samples", len(sm), "min", min(sm), "max", max(sm))
print("reasons", sorted(set(r[4].strip() for r in rows if len(r)>4)))
PY
