#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CTM_ISO_DEBUG=1 timeout 300 python tools/prof_solve.py 3 > gpurun_out/r02g_solve.txt 2>&1
CTM_PROF_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r02g_solve_launches.csv python tools/prof_solve.py 2 > gpurun_out/r02g_ncu.log 2>&1
