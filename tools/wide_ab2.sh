export PYTHONUNBUFFERED=1
{
for w in 0 1; do SA_WIDE=$w timeout 300 python bench.py --workload sweep --no-e2e --no-cpu --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wide',$w,d['ms_per_step'],d['value']/1e9)"; done
AB_N=10000 timeout 300 python tools/ab_timing.py ab/libfin.so ab/libwide.so -- CONFIG2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
} > gpurun_out/wide2.txt 2>&1
cat gpurun_out/wide2.txt
