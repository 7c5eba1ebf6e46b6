#!/bin/bash
# Round-2 session 3: fgemm with warp-level split-K (every warp the whole 32 x 32 tile over a quarter of the k-steps)
cd "$(dirname "$0")/.."
O=gpurun_out/s3n
mkdir -p $O
CTM_LIB_PATH=ab/libctm_ws.so timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "golden or side_isometry_projectors or main_ts or side_ts or iterations_gauge" > $O/pytest_ws.log 2>&1; echo "pytest ws rc=$?" >> $O/rc.txt
L="base=,ws=ab/libctm_ws.so,ws_st3bk64=ab/libctm_ws_st3_bk64.so,ws_st2bk64=ab/libctm_ws_st2_bk64.so,ws_st4bk32=ab/libctm_ws_st4_bk32.so"
timeout 1500 python tools/ab_move.py --libs "$L" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
