#!/bin/bash
# quick GPU validation + timing pass (run under gpurun)
export PYTHONUNBUFFERED=1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 250 python tools/op_timing.py 50000 2>&1 | tail -30
