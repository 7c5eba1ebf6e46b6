#!/bin/bash
# Round-2 session 3: fgemm BK 32 / 64 variants A/B (all with the stagnation rule fix); c4_dl fallbacks after the fix
cd "$(dirname "$0")/.."
O=gpurun_out/s3h
mkdir -p $O
timeout 600 python tools/warm_moves.py c4_dl 20 iterate > $O/c4dl_iter.jsonl 2> $O/c4dl.err; echo "c4_dl rc=$?" >> $O/rc.txt
L="st4bk16=ab/libctm_st4_bk16.so,st3bk32=ab/libctm_st3_bk32.so,st2bk32=ab/libctm_st2_bk32.so,st2bk64=ab/libctm_st2_bk64.so,st3bk64=ab/libctm_st3_bk64.so"
timeout 1500 python tools/ab_move.py --libs "$L" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c2 --libs "$L" --procs 2 --moves 10 > $O/ab_c2.jsonl 2> $O/ab_c2.err; echo "ab c2 rc=$?" >> $O/rc.txt
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "golden or c3-20-False or side_isometry_projectors or main_ts or side_ts" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
