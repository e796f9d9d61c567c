export PYTHONUNBUFFERED=1
{
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config or exact_op or golden_pipeline or nonfinite" 2>&1 | tail -2
AB_N=100000 AB_L=1500 AB_ROUNDS=3 timeout 300 python tools/ab_timing.py ab/libgat3.so ab/libgat4.so -- CONFIG4 speed_warp convolve
} > gpurun_out/gather.txt 2>&1
cat gpurun_out/gather.txt
