#!/bin/bash
# Cholesky smem-block change (kernel + move), deferred split-K combine, A/B against the previous build
cd "$(dirname "$0")/.."
O=gpurun_out/s2d
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik && (timeout 60 $O/bik 160; timeout 60 $O/bik 128; timeout 60 $O/bik 232) > $O/bik_new.txt 2>&1; echo "bik rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not shadowed" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 2000 python tools/ab_move.py --libs "prev=tools/ab_old/libctm_prev.so,oldchol=tools/ab_old/libctm_oldchol.so,new=,nodefer=@CTM_ISO_NODEFER=1" --procs 4 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
