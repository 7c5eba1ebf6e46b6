#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s2i
mkdir -p $O
timeout 600 python tools/trace_move.py c4 > $O/trace_c4.txt 2>&1; echo "trace rc=$?" >> $O/rc.txt
cp gpurun_out/r02_trace.jsonl $O/trace_c4.jsonl 2>/dev/null
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu0.log 2>&1; echo "ncu bench rc=$?" >> $O/rc.txt
