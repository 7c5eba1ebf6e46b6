#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c3 8 > gpurun_out/r02d_c3_moves.txt 2> gpurun_out/r02d_c3_trace.txt
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c4 3 > gpurun_out/r02d_c4_moves.txt 2> gpurun_out/r02d_c4_trace.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
