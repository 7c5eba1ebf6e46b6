#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "absorb_truncate or entrywise or reduced_env" > gpurun_out/r02e_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02e_pytest.log
