#!/bin/bash
# TMA-staged tc_gemm (parity, per-step ncu, bench) + new solver defaults (C3/C4/C5 A/B against the old ones)
cd "$(dirname "$0")/.."
O=gpurun_out/s2m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not shadowed" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_tma.csv python tools/prof_move.py c4 inject > $O/ncu1.log 2>&1; echo "ncu tma rc=$?" >> $O/rc.txt
CTM_TC_TMA=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_notma.csv python tools/prof_move.py c4 inject > $O/ncu2.log 2>&1; echo "ncu notma rc=$?" >> $O/rc.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_tma.json 2> $O/bench_tma.err; echo "bench tma rc=$?" >> $O/rc.txt
CTM_TC_TMA=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_notma.json 2> $O/bench_notma.err; echo "bench notma rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "new=,notma=@CTM_TC_TMA=0,old=@CTM_ISO_SAFE1=2.0@CTM_ISO_SAFE=1.25@CTM_ISO_TAIL=6" --procs 3 --moves 12 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "new=,old=@CTM_ISO_SAFE1=2.0@CTM_ISO_SAFE=1.25@CTM_ISO_TAIL=6" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 900 python tools/ab_move.py --config c3 --libs "new=,old=@CTM_ISO_SAFE1=2.0@CTM_ISO_SAFE=1.25@CTM_ISO_TAIL=6" --procs 2 --moves 12 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
