#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s2h
mkdir -p $O
for f in NONE CTM_CHOL_DFMA_TRAIL; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -D$f -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik_$f && for n in 32 64 128 160; do timeout 60 $O/bik_$f $n 2>&1 | grep '"chol"\|trsm' | sed "s/^{/{\"build\":\"$f\",/"; done >> $O/chol.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not shadowed" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "prev=tools/ab_old/libctm_oldchol.so,new=" --procs 4 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
