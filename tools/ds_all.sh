export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/ds_time.py $(python -c "print(','.join(str(i) for i in range(100)))") > gpurun_out/ds_all.txt 2>&1
echo done
