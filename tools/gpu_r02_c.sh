#!/bin/bash
# locking: C3 fallback trace, C4 trace, bench, GPU parity (fullsize + parity files)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c3 8 > gpurun_out/r02c_c3_moves.txt 2> gpurun_out/r02c_c3_trace.txt
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c4 2 > gpurun_out/r02c_c4_moves.txt 2> gpurun_out/r02c_c4_trace.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
timeout 2400 python -m pytest tests -m gpu -q -rA -s -x --durations=15 > gpurun_out/r02c_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02c_pytest_gpu.log
