#!/bin/bash
# per-launch times of the C4 contraction-only move: base library vs current
cd "$(dirname "$0")/.."
O=gpurun_out/p
mkdir -p $O
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
true
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/inject_new.csv python tools/prof_move.py c4 inject > $O/ncu_new.log 2>&1; echo "new rc=$?" >> $O/rc.txt
