#!/bin/bash
# persistent tc_gemm A/B + quick parity + Jacobi cluster-shape study
cd "$(dirname "$0")/.."
O=gpurun_out/s2a
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_jacobi_cfg.cu -o $O/bjc && timeout 120 $O/bjc > $O/jacobi_cfg.jsonl 2>&1; echo "jac rc=$?" >> $O/rc.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "absorb or entrywise or injected or reduced_env or norm_2x2 or directional" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for arm in pers nopers pers2 nopers2; do
  if [[ $arm == nopers* ]]; then export CTM_TC_NOPERS=1; else unset CTM_TC_NOPERS; fi
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_$arm.json 2> $O/bench_$arm.err; echo "bench $arm rc=$?" >> $O/rc.txt
done
unset CTM_TC_NOPERS
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_pers.csv python tools/prof_move.py c4 inject > $O/ncu1.log 2>&1; echo "ncu pers rc=$?" >> $O/rc.txt
CTM_TC_NOPERS=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_nopers.csv python tools/prof_move.py c4 inject > $O/ncu2.log 2>&1; echo "ncu nopers rc=$?" >> $O/rc.txt
