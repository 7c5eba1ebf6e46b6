#!/bin/bash
# chol look-ahead with a branch-free rsqrt + lean plain epilogue: micro-bench, parity subset, A/B bench
cd "$(dirname "$0")/.."
O=gpurun_out/q
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik && timeout 120 $O/bik 160 > $O/bik160.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "absorb or reduced_env or side_isometry or entrywise or iterations" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do
  CTM_LIB_PATH=$PWD/ab/libctm_r02base.so timeout 600 python bench.py --no-cpu-baseline > $O/bench_base_$r.json 2> $O/bench_base_$r.err; echo "bench base $r rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_new_$r.json 2> $O/bench_new_$r.err; echo "bench new $r rc=$?" >> $O/rc.txt
done
