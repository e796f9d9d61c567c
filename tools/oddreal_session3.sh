#!/bin/bash
export PYTHONUNBUFFERED=1
for sf in 3 5; do for al in 0 1; do
echo "== L=2369 STARVED_FIT=$sf ALIGN=$al"; SA_GLOBAL_ALIGN=$al SA_STARVED_FIT=$sf AB_N=17877 AB_L=2369 timeout 300 python tools/ab_timing.py ab/liboddreal3.so -- CHAIN5 app
done; done
for sf in 3 5; do
echo "== L=2600 STARVED_FIT=$sf"; SA_STARVED_FIT=$sf AB_N=20000 AB_L=2600 timeout 300 python tools/ab_timing.py ab/liboddreal3.so -- CHAIN5 app jitter time_warp
echo "== L=2900 STARVED_FIT=$sf"; SA_STARVED_FIT=$sf AB_N=20000 AB_L=2900 timeout 300 python tools/ab_timing.py ab/liboddreal3.so -- CHAIN5 app jitter time_warp
echo "== L=2300 STARVED_FIT=$sf"; SA_STARVED_FIT=$sf AB_N=20000 AB_L=2300 timeout 300 python tools/ab_timing.py ab/liboddreal3.so -- CHAIN5 app jitter time_warp
done
