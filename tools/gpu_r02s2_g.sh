#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s2g
mkdir -p $O
for f in NONE XDIAG XTRAIL XPANEL; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCTM_CHOL_$f -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o $O/bik_$f && for n in 32 64 96 128 160; do timeout 60 $O/bik_$f $n 2>&1 | grep '"chol"' | sed "s/^{/{\"build\":\"$f\",/"; done >> $O/chol_phases.jsonl 2>&1
done
echo done >> $O/rc.txt
