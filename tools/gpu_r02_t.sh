#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/t4
mkdir -p $O
timeout 2400 python tools/ab_move.py --libs "base=ab/libctm_r02base.so,cand1=ab/libctm_cand1.so,new=,newslab=@CTM_TC_SPLIT=slab" --procs 4 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
