#!/bin/bash
# per-launch device times of one contraction-only C4 move (ncu launch list)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r02_launches_inject${TAG}.csv python tools/prof_move.py c4 inject > gpurun_out/r02_launches_inject.log 2>&1
