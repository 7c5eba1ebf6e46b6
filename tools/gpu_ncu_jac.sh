#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
./tools/bench_iso_kernels 160 > gpurun_out/r02_bik160.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_cluster -c 1 -o gpurun_out/r02_jac160 ./tools/bench_iso_kernels 160 > gpurun_out/r02_ncu_jac.log 2>&1
