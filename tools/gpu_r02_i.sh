#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CTM_ISO_DEBUG=1 timeout 300 python tools/prof_solve.py 2 > gpurun_out/r02i_solve.txt 2>&1
for pw in 1 2 4 8; do
  CTM_ISO_GPOW=$pw timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r02i_bench_gpow$pw.json 2>/dev/null
done
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c3 8 > gpurun_out/r02i_c3_moves.txt 2> gpurun_out/r02i_c3_trace.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "main_ts or side_ts or reduced_env_with or c4_dl" > gpurun_out/r02i_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02i_pytest.log
