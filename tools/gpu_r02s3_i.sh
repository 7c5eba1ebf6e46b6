#!/bin/bash
# Round-2 session 3: fgemm BM = 64 variants A/B against the adopted BK 32 / 3 stages / BM 32
cd "$(dirname "$0")/.."
O=gpurun_out/s3i
mkdir -p $O
L="st3bk32=ab/libctm_st3_bk32.so,st3bk32bm64=ab/libctm_st3_bk32_bm64.so,st2bk32bm64=ab/libctm_st2_bk32_bm64.so,st4bk16bm64=ab/libctm_st4_bk16_bm64.so"
timeout 1500 python tools/ab_move.py --libs "$L" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
