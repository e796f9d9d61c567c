#!/bin/bash
# A/B of backend builds (ab/lib*.so, tools/build_variant.sh) on the configs, odd / prime lengths and the sweep
# usage (under gpurun): bash tools/oddreal_ab.sh ab/libA.so ab/libB.so
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
libs="$@"
AB_N=50000 python tools/ab_timing.py $libs -- CONFIG5 CONFIG2 jitter app fmask_chain
AB_N=100000 AB_L=1500 python tools/ab_timing.py $libs -- CONFIG4
AB_N=17877 AB_L=2369 python tools/ab_timing.py $libs -- CHAIN5 app
AB_N=10878 AB_L=2136 python tools/ab_timing.py $libs -- CHAIN5 app
AB_N=16461 AB_L=541 python tools/ab_timing.py $libs -- CHAIN5 app
AB_N=12249 AB_L=440 python tools/ab_timing.py $libs -- CHAIN5 app
AB_N=15921 AB_L=219 python tools/ab_timing.py $libs -- CHAIN5 app
AB_N=13349 AB_L=56 python tools/ab_timing.py $libs -- CHAIN5
for lib in $libs; do
  SA_LIB_PATH=$PWD/$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'config5 ms', d['ms_per_step'])"
  SA_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload sweep --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'sweep ms', d['ms_per_step'], 'Gpts/s', d['value']/1e9)"
done
