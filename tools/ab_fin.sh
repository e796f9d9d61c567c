export PYTHONUNBUFFERED=1
{
AB_N=200000 AB_ROUNDS=2 timeout 300 python tools/ab_timing.py ab/libnofin.so ab/libfin.so -- CONFIG5 CONFIG2 jitter drift quantize
AB_N=100000 AB_L=1500 AB_ROUNDS=2 timeout 300 python tools/ab_timing.py ab/libnofin.so ab/libfin.so -- CONFIG4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
} > gpurun_out/fin.txt 2>&1
cat gpurun_out/fin.txt
