#!/bin/bash
# Jacobi cluster shapes (kernel + move A/B), Cholesky phase cycles, quick parity
cd "$(dirname "$0")/.."
O=gpurun_out/s2b
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_jacobi_cfg.cu -o $O/bjc && timeout 180 $O/bjc > $O/jacobi_cfg.jsonl 2>&1; echo "jac rc=$?" >> $O/rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCTM_CHOL_PROF -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik_prof && (timeout 60 $O/bik_prof 160; timeout 60 $O/bik_prof 128) > $O/chol_prof.txt 2>&1; echo "chol rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not shadowed" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "old=@CTM_ISO_JAC_OLD=1,new=" --procs 4 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
