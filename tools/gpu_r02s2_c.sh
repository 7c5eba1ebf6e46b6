#!/bin/bash
# Jacobi shapes II, chol_kernel ncu source capture, full GPU suite, bench
cd "$(dirname "$0")/.."
O=gpurun_out/s2c
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_jacobi_cfg.cu -o $O/bjc && timeout 180 $O/bjc > $O/jacobi_cfg.jsonl 2>&1; echo "jac rc=$?" >> $O/rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik && timeout 60 $O/bik 160 > $O/bik160.txt 2>&1; echo "bik rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:chol_kernel -s 3 -c 1 -o $O/chol_full -f $O/bik 160 > $O/ncu_chol.log 2>&1; echo "ncu chol rc=$?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 1800 python -m pytest tests -m gpu -x -q -rA --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
