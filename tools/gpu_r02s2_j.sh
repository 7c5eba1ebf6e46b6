#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s2j
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik && for n in 32 64 128 160; do timeout 60 $O/bik $n 2>&1 | grep '"chol"'; done > $O/chol.jsonl 2>&1; echo "bik rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not shadowed" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "prev=tools/ab_old/libctm_dmmatrail.so,new=" --procs 4 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
