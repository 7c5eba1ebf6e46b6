#!/bin/bash
# Round-2 session 3: ncu --set full of the solver's fgemm (G-form filter degree and the transposed M^T Y product) and of the Jacobi cluster kernel inside a bench step
cd "$(dirname "$0")/.."
O=gpurun_out/s3m
mkdir -p $O
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:fgemm -s 60 -c 3 -o $O/prof_fgemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_fgemm.log 2>&1; echo "ncu fgemm rc=$?" >> $O/rc.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:jacobi_cluster -s 3 -c 1 -o $O/prof_jacobi python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_jacobi.log 2>&1; echo "ncu jacobi rc=$?" >> $O/rc.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:trsm_rows -s 20 -c 1 -o $O/prof_trsm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_trsm.log 2>&1; echo "ncu trsm rc=$?" >> $O/rc.txt
