export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
{
AB_N=50000 AB_L=2048 timeout 300 python tools/ab_timing.py ab/libst.so ab/libwt2.so -- CONFIG3
AB_N=100000 AB_L=1500 timeout 300 python tools/ab_timing.py ab/libst.so ab/libwt2.so -- CONFIG4
for o in 0 1; do SA_SWEEP_ORDER=$o timeout 300 python bench.py --workload sweep --no-e2e --no-cpu --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('order',$o,d['ms_per_step'],d['value']/1e9)"; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
} > gpurun_out/t.txt 2>&1
cat gpurun_out/t.txt
