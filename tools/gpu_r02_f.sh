#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ffu.py -q -rA -s > gpurun_out/r02f_ffu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02f_ffu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r02f_smoke.log
