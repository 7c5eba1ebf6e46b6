#!/bin/bash
# separable k-offsets in tc_gemm: parity, per-step launch list, A/B of the full move
cd "$(dirname "$0")/.."
O=gpurun_out/x
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/inject_sep.csv python tools/prof_move.py c4 inject > $O/ncu1.log 2>&1; echo "ncu sep rc=$?" >> $O/rc.txt
CTM_TC_NOSEP=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/inject_nosep.csv python tools/prof_move.py c4 inject > $O/ncu2.log 2>&1; echo "ncu nosep rc=$?" >> $O/rc.txt
timeout 1800 python tools/ab_move.py --libs "base=ab/libctm_r02base.so,sep=,nosep=@CTM_TC_NOSEP=1" --procs 3 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
