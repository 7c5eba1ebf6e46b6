#!/bin/bash
# fragment double buffering: parity of the FB configs, per-step times per forced config
cd "$(dirname "$0")/.."
O=gpurun_out/y
mkdir -p $O
for c in 3 4 5; do
  CTM_TC_CFG=$c timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "absorb or reduced_env or entrywise" > $O/pytest_cfg$c.log 2>&1; echo "pytest cfg$c rc=$?" >> $O/rc.txt
done
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
for c in 0 3 4 5; do
  CTM_TC_CFG=$c timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/inject_cfg$c.csv python tools/prof_move.py c4 inject > $O/ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?" >> $O/rc.txt
done
