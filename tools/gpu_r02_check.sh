#!/bin/bash
# Round-2 GPU check: full GPU suite (incl. the full-size parity tests), smoke, default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA -s --durations=30 > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r02_smoke.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo "bench exit $?" >> gpurun_out/r02_bench.err
