export PYTHONUNBUFFERED=1
{
AB_N=100000 AB_L=1500 timeout 300 python tools/ab_timing.py ab/libwt2.so ab/libwt3.so -- CONFIG4
AB_N=50000 timeout 300 python tools/ab_timing.py ab/libwt2.so ab/libwt3.so -- CONFIG5 speed_warp
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
} > gpurun_out/t2.txt 2>&1
cat gpurun_out/t2.txt
