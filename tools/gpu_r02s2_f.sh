#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s2f
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/bench_chol_diag.cu -o $O/bcd && timeout 60 $O/bcd > $O/chol_diag.jsonl 2>&1; echo "bcd rc=$?" >> $O/rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik && for n in 32 64 128 160; do timeout 60 $O/bik $n 2>&1 | grep '"chol"'; done > $O/chol_n_noinline.txt 2>&1; echo "bik rc=$?" >> $O/rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCTM_CHOL_SKIP_W4 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik4 && for n in 32 64 128 160; do timeout 60 $O/bik4 $n 2>&1 | grep '"chol"'; done > $O/chol_n_noinline_skipw4.txt 2>&1; echo "bik4 rc=$?" >> $O/rc.txt
