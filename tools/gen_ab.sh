export PYTHONUNBUFFERED=1
D=73,74,10,59,33,31,27,81,92,6
{
SA_LIB_PATH=ab/libgen4.so python tools/ds_time.py $D BASE=1
SA_LIB_PATH=ab/libgen8.so python tools/ds_time.py $D BASE=1
python -m pytest tests/test_gpu_parity.py -q -x -k "sweep or spectral or fft or bluestein or long" 2>&1 | tail -2
} > gpurun_out/gen.txt 2>&1
cat gpurun_out/gen.txt
