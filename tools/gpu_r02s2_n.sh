#!/bin/bash
# TMA coordinates per CTA + launch threshold; full GPU suite with the re-tuned solver; per-step ncu; bench
cd "$(dirname "$0")/.."
O=gpurun_out/s2n
mkdir -p $O
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_tma.csv python tools/prof_move.py c4 inject > $O/ncu1.log 2>&1; echo "ncu tma rc=$?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_tma.json 2> $O/bench_tma.err; echo "bench tma rc=$?" >> $O/rc.txt
CTM_TC_TMA=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_notma.json 2> $O/bench_notma.err; echo "bench notma rc=$?" >> $O/rc.txt
timeout 2700 python -m pytest tests -m gpu -q -rA --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
