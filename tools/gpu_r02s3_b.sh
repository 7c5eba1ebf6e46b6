#!/bin/bash
# Round-2 session 3: ncu launch list (names, grids, block sizes) of one bench step; knob A/B at C4
cd "$(dirname "$0")/.."
O=gpurun_out/s3b
mkdir -p $O
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu0.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "base=,sw0=@CTM_ISO_SWEEPS1=0,pw2=@CTM_ISO_POWER=2,pw3=@CTM_ISO_POWER=3,sw0pw2=@CTM_ISO_SWEEPS1=0@CTM_ISO_POWER=2" --procs 3 --moves 10 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
