export PYTHONUNBUFFERED=1
D=65,77,97,90,89,38,11,64,92,6
{
SA_LIB_PATH=ab/libwide768.so python tools/ds_time.py $D BASE=1 SA_WIDE_MAXL=128 SA_WIDE_MAXL=600
SA_LIB_PATH=ab/libwide512.so python tools/ds_time.py $D SA_WIDE_MAXL=128 SA_WIDE_MAXL=600
} > gpurun_out/wide.txt 2>&1
cat gpurun_out/wide.txt
