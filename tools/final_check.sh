#!/bin/bash
# Full GPU suite + smoke + config-4 ncu summary of the gather CTA kernel (run under gpurun)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CFG=4 N=100000 K=gather_cta bash tools/prof_cfg_src.sh; echo "prof rc=$?"
