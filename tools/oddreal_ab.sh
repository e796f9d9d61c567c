#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
AB_N=50000 python tools/ab_timing.py ab/libbase.so ab/liboddreal4.so ab/liboddreal8.so -- CONFIG5 CONFIG2 jitter app fmask_chain
AB_N=17877 AB_L=2369 python tools/ab_timing.py ab/liboddreal4.so ab/liboddreal8.so -- CHAIN5 app
AB_N=5571 AB_L=909 python tools/ab_timing.py ab/liboddreal4.so ab/liboddreal8.so -- CHAIN5 app
for lib in ab/libbase.so ab/liboddreal8.so; do
  SA_LIB_PATH=$PWD/$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'config5 ms', d['ms_per_step'])"
  SA_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload sweep --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'sweep ms', d['ms_per_step'], 'Gpts/s', d['value']/1e9)"
done
