#!/bin/bash
# Round-2 session 3: fgemm BK = 32 variants A/B; c4_dl fallback trace
cd "$(dirname "$0")/.."
O=gpurun_out/s3g
mkdir -p $O
L="st4=ab/libctm_st4.so,st6=ab/libctm_st6.so,st4bk32=ab/libctm_st4_bk32.so,st3bk32=ab/libctm_st3_bk32.so,st6bk32=ab/libctm_st6_bk32.so"
timeout 1500 python tools/ab_move.py --libs "$L" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
CTM_ISO_DEBUG=1 timeout 600 python tools/warm_moves.py c4_dl 6 iterate > /dev/null 2> $O/c4dl_debug.txt; echo "c4_dl debug rc=$?" >> $O/rc.txt
