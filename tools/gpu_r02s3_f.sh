#!/bin/bash
# Round-2 session 3: warm start with back-off; fgemm pipeline depth A/B (4 / 6 / 8 stages)
cd "$(dirname "$0")/.."
O=gpurun_out/s3f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tma.py tests/test_gpu_fullsize.py -q -x -s -k "tma or c2-20-True or golden or warm_start" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "st4=ab/libctm_st4.so,st6=ab/libctm_st6.so,st8=ab/libctm_st8.so" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "st4=ab/libctm_st4.so,st6=ab/libctm_st6.so,st8=ab/libctm_st8.so" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "st4=ab/libctm_st4.so,st6=ab/libctm_st6.so,st8=ab/libctm_st8.so" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
timeout 600 python tools/warm_moves.py c4 12 > $O/warm_c4.jsonl 2> $O/warm_c4.err; echo "warm c4 rc=$?" >> $O/rc.txt
timeout 600 python tools/warm_moves.py c4_dl 20 iterate > $O/warm_c4dl_iter.jsonl 2> $O/warm_c4dl.err; echo "warm c4_dl rc=$?" >> $O/rc.txt
