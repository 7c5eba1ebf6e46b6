#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
timeout 2400 python tools/trotter_timing.py > gpurun_out/r02k_trotter.jsonl 2> gpurun_out/r02k_trotter.err
