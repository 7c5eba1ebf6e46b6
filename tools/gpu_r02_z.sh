#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/z2
mkdir -p $O
timeout 2400 python tools/ab_move.py --libs "sep=ab/libctm_sep_nofb.so,fball=ab/libctm_fb_all.so,fb01=" --procs 4 --moves 15 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
