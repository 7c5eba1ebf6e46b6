#!/bin/bash
# bench with R24b (main TS basis stage two) vs CTM_TS_MAIN_SVD=1, and the C3 fallback trace
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_bench_b.json 2> gpurun_out/r02_bench_b.err
CTM_TS_MAIN_SVD=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_bench_b_svd2.json 2>> gpurun_out/r02_bench_b.err
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c3 6 > gpurun_out/r02_c3_fallbacks.txt 2> gpurun_out/r02_c3_fallbacks_trace.txt
CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c4 1 > gpurun_out/r02_c4_trace_moves.txt 2> gpurun_out/r02_c4_trace.txt
