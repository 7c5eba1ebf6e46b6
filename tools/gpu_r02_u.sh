#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/u
mkdir -p $O
for r in 1 2; do
CTM_LIB_PATH=$PWD/ab/libctm_r02base.so timeout 600 python tools/trace_move.py c4 > $O/trace_base_$r.txt 2>&1
timeout 600 python tools/trace_move.py c4 > $O/trace_new_$r.txt 2>&1
done
